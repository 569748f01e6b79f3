"""Build libb200conv.so in-tree with nvcc for sm_100a (no JIT cache, no torch
extension machinery): one object per .cu compiled in parallel, linked with the
static CUDA runtime so the library loads without a GPU (the driver is resolved
at first CUDA call)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libb200conv.so")
SOURCES = ["abi.cu", "conv_single.cu", "conv_multi_simt.cu", "conv_multi_tc.cu", "conv_multi_gemm.cu", "workspace.cu"]
HEADERS = ["kernels.h", "ptx.cuh", "latency_model.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-I", os.path.join(ROOT, "include")]


DIAG_LIB = os.path.join(PKG, "libb200conv_diag.so")


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "b200conv.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, diag: bool = False, defines=(), out: str = "") -> str:
    """Build the product library; diag=True builds libb200conv_diag.so instead
    (-DB200CONV_DIAG: timeline stamps and work-skipping switches for the
    tools/ timeline scripts; never loaded by the product path).  defines/out:
    an A/B variant (-D flags) written to `out` (tools/, B200CONV_LIB_PATH)."""
    lib = out or (DIAG_LIB if diag else LIB)
    if not force and not out and not _stale(lib):
        return lib
    objdir = os.path.join(PKG, "build_diag" if diag else "build") if not out else "/tmp/b200ab_" + os.path.basename(lib) + ".objs"
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *(["-DB200CONV_DIAG"] if diag else []), *[f"-D{d}" for d in defines], "-Xptxas", "-v", "-c",
               os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj, r.stderr

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
           "-o", tmp, *[o for o, _ in results]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python -m paper_2212_00404_b200.build [--force] [-v] [--diag] [--out PATH -DNAME=V ...]
    a = sys.argv[1:]
    out = a[a.index("--out") + 1] if "--out" in a else ""
    print(build(force="--force" in a, verbose="-v" in a, diag="--diag" in a,
                defines=[x[2:] for x in a if x.startswith("-D")], out=out))
