"""Thin Python binding of libb200conv.so (include/b200conv.h).

Argument marshalling only: every step of the convolution runs in the CUDA
kernels behind the C ABI.  PyTorch provides device memory and streams.  There
is no CPU or eager fallback: if the library is missing or the device is not a
B200 the calls raise.

Names follow the ABI: ``conv_single``, ``conv_multi``, ``conv_single_ex``,
``conv_multi_ex``, ``conv_single_host``, ``conv_multi_host``, plus the
allocating conveniences ``single(I, F)`` and ``multi(I, F, precision)``, which
consume and produce exactly the tensors ``torch.nn.functional.conv2d(I[None],
F)[0]`` does (NCHW/OIHW, N = 1, valid, stride 1 — PAPER.md Eq. 1).
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libb200conv.so")

CONV_FP32, CONV_TF32, CONV_BF16 = 0, 1, 2
PRECISIONS = {"fp32": CONV_FP32, "tf32": CONV_TF32, "bf16": CONV_BF16}
STATUS = {0: "CONV_OK", 1: "CONV_E_SHAPE", 2: "CONV_E_NULL", 3: "CONV_E_ALIGN",
          4: "CONV_E_PRECISION", 5: "CONV_E_DEVICE", 6: "CONV_E_LAUNCH"}
EXPORTS = ["conv_single", "conv_multi", "conv_single_ex", "conv_multi_ex", "conv_single_host",
           "conv_multi_host", "conv_single_host_async", "conv_multi_host_async", "conv_multi_batched_ex",
           "conv_plan_multi_batched", "conv_single_pad_ex", "conv_multi_pad_ex",
           "conv_single_strided_ex", "conv_multi_strided_ex", "conv_plan_multi_strided", "conv_plan_single", "conv_plan_multi", "conv_status_string",
           "conv_version", "conv_latency_model", "conv_multi_allgather_ex"]


class ConvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class ConvPlan(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in
                ("kernel", "grid_x", "grid_y", "grid_z", "block_x", "cluster_x", "tile_m",
                 "tile_n", "smem_bytes", "tma_f", "launches", "chunk_k")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_lock = threading.Lock()
_lib = None


def load(path: str | None = None) -> ctypes.CDLL:
    """Load the C-ABI library (raises if it was not built — no fallback).
    B200CONV_LIB_PATH selects another build of it (A/B measurements)."""
    global _lib
    path = path or os.environ.get("B200CONV_LIB_PATH") or LIB_PATH
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(f"{path} missing: build it with `python -m paper_2212_00404_b200.build`"
                                   " (no CPU fallback exists)")
            lib = ctypes.CDLL(path)
            P, I32 = ctypes.c_void_p, ctypes.c_int
            lib.conv_single.argtypes = [P, I32, I32, P, I32, I32, P]
            lib.conv_multi.argtypes = [P, I32, I32, I32, P, I32, I32, P]
            lib.conv_single_ex.argtypes = [P, I32, I32, P, I32, I32, P, P]
            lib.conv_multi_ex.argtypes = [P, I32, I32, I32, P, I32, I32, P, I32, P]
            lib.conv_single_host.argtypes = [P, I32, I32, P, I32, I32, P, P]
            lib.conv_multi_host.argtypes = [P, I32, I32, I32, P, I32, I32, P, I32, P]
            lib.conv_single_host_async.argtypes = [P, I32, I32, P, I32, I32, P, P]
            lib.conv_multi_host_async.argtypes = [P, I32, I32, I32, P, I32, I32, P, I32, P]
            lib.conv_plan_single.argtypes = [I32, I32, I32, I32, ctypes.POINTER(ConvPlan)]
            lib.conv_plan_multi.argtypes = [I32, I32, I32, I32, I32, I32, ctypes.POINTER(ConvPlan)]
            lib.conv_multi_batched_ex.argtypes = [P, I32, I32, I32, I32, P, I32, I32, P, I32, P]
            lib.conv_single_pad_ex.argtypes = [P, I32, I32, P, I32, I32, I32, P, P]
            lib.conv_multi_pad_ex.argtypes = [P, I32, I32, I32, I32, P, I32, I32, I32, P, I32, P]
            lib.conv_plan_multi_batched.argtypes = [I32, I32, I32, I32, I32, I32, I32, ctypes.POINTER(ConvPlan)]
            lib.conv_single_strided_ex.argtypes = [P, I32, I32, P, I32, I32, I32, I32, P, P]
            lib.conv_multi_strided_ex.argtypes = [P, I32, I32, I32, I32, P, I32, I32, I32, I32, P, I32, P]
            lib.conv_plan_multi_strided.argtypes = [I32, I32, I32, I32, I32, I32, I32, I32, I32,
                                                    ctypes.POINTER(ConvPlan)]
            lib.conv_status_string.argtypes = [I32]
            lib.conv_status_string.restype = ctypes.c_char_p
            lib.conv_version.argtypes = []
            lib.conv_latency_model.argtypes = [I32, ctypes.POINTER(ctypes.c_double)]
            lib.conv_multi_allgather_ex.argtypes = [P, I32, I32, I32, P, I32, I32, I32, I32,
                                                    ctypes.POINTER(ctypes.c_void_p), I32, P, I32, P]
            lib.conv_diag_nop.argtypes = [P]
            lib.conv_diag_nop.restype = I32
            for n in EXPORTS:
                if n != "conv_status_string":
                    getattr(lib, n).restype = I32
            _lib = lib
    return _lib


def _check(status: int):
    if status != 0:
        raise ConvError(status, load().conv_status_string(status).decode())


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _prec(p) -> int:
    return PRECISIONS[p] if isinstance(p, str) else int(p)


# ---------------------------------------------------------------- raw ABI names
def conv_single(I, Wx, Wy, F, K, M, O):
    _check(load().conv_single(_ptr(I), Wx, Wy, _ptr(F), K, M, _ptr(O)))


def conv_multi(I, C, Wx, Wy, F, K, M, O):
    _check(load().conv_multi(_ptr(I), C, Wx, Wy, _ptr(F), K, M, _ptr(O)))


def conv_single_ex(I, Wx, Wy, F, K, M, O, stream=None):
    _check(load().conv_single_ex(_ptr(I), Wx, Wy, _ptr(F), K, M, _ptr(O), _stream(stream)))


def conv_multi_ex(I, C, Wx, Wy, F, K, M, O, precision="fp32", stream=None):
    _check(load().conv_multi_ex(_ptr(I), C, Wx, Wy, _ptr(F), K, M, _ptr(O), _prec(precision),
                                _stream(stream)))


def conv_single_host(I, Wx, Wy, F, K, M, O, stream=None):
    _check(load().conv_single_host(_ptr(I), Wx, Wy, _ptr(F), K, M, _ptr(O), _stream(stream)))


def conv_single_host_async(I, Wx, Wy, F, K, M, O, stream=None):
    """As conv_single_host without the final stream synchronisation (pinned buffers)."""
    _check(load().conv_single_host_async(_ptr(I), Wx, Wy, _ptr(F), K, M, _ptr(O), _stream(stream)))


def conv_multi_host_async(I, C, Wx, Wy, F, K, M, O, precision="fp32", stream=None):
    """As conv_multi_host without the final stream synchronisation (pinned buffers)."""
    _check(load().conv_multi_host_async(_ptr(I), C, Wx, Wy, _ptr(F), K, M, _ptr(O), _prec(precision),
                                        _stream(stream)))


def conv_multi_host(I, C, Wx, Wy, F, K, M, O, precision="fp32", stream=None):
    _check(load().conv_multi_host(_ptr(I), C, Wx, Wy, _ptr(F), K, M, _ptr(O), _prec(precision),
                                  _stream(stream)))


def plan_single(Wx, Wy, K, M) -> dict:
    p = ConvPlan()
    _check(load().conv_plan_single(Wx, Wy, K, M, ctypes.byref(p)))
    return p.as_dict()


def conv_multi_batched_ex(I, N, C, Wx, Wy, F, K, M, O, precision="fp32", stream=None):
    _check(load().conv_multi_batched_ex(_ptr(I), N, C, Wx, Wy, _ptr(F), K, M, _ptr(O), _prec(precision),
                                        _stream(stream)))


def conv_single_pad_ex(I, Wx, Wy, F, K, M, pad, O, stream=None):
    _check(load().conv_single_pad_ex(_ptr(I), Wx, Wy, _ptr(F), K, M, pad, _ptr(O), _stream(stream)))


def conv_multi_pad_ex(I, N, C, Wx, Wy, F, K, M, pad, O, precision="fp32", stream=None):
    _check(load().conv_multi_pad_ex(_ptr(I), N, C, Wx, Wy, _ptr(F), K, M, pad, _ptr(O), _prec(precision),
                                    _stream(stream)))


def plan_multi_batched(N, C, Wx, Wy, K, M, precision="fp32") -> dict:
    p = ConvPlan()
    _check(load().conv_plan_multi_batched(N, C, Wx, Wy, K, M, _prec(precision), ctypes.byref(p)))
    return p.as_dict()


def plan_multi(C, Wx, Wy, K, M, precision="fp32") -> dict:
    p = ConvPlan()
    _check(load().conv_plan_multi(C, Wx, Wy, K, M, _prec(precision), ctypes.byref(p)))
    return p.as_dict()


def conv_multi_allgather_ex(I, C, Wx, Wy, F, K, M, m0, M_total, O_peers, O_mc=None, precision="fp32",
                            stream=None):
    """NEXT-2: this rank's filters m0..m0+M-1 straight into every O in O_peers
    (device pointers or tensors [M_total][Ho][Wo]); O_mc: multicast address."""
    arr = (ctypes.c_void_p * len(O_peers))(*[_ptr(o) for o in O_peers])
    _check(load().conv_multi_allgather_ex(_ptr(I), C, Wx, Wy, _ptr(F), K, M, m0, M_total, arr, len(O_peers),
                                          _ptr(O_mc), _prec(precision), _stream(stream)))


def latency_model(profile: str = "b200") -> dict:
    """The paper's latency-hiding model (§2.2) for "b200" (this
    device) or "gtx1080ti" (the paper's Table 1)."""
    out = (ctypes.c_double * 5)()
    _check(load().conv_latency_model({"b200": 0, "gtx1080ti": 1}[profile], out))
    return dict(zip(("n_fma", "volume", "threads_per_sm", "v_s", "bytes_per_clk"), list(out)))


def diag_nop(stream=None):
    """One empty kernel with the hot path's launch attributes (launch floor)."""
    _check(load().conv_diag_nop(_stream(stream)))


def version() -> int:
    return load().conv_version()


# ---------------------------------------------------------------- conveniences
# Every convenience validates its tensors before any pointer reaches the ABI:
# the C entry points only see raw pointers and sizes, so a wrong dtype, shape,
# device or stride here would become an out-of-bounds access there.
def _want_dtype(precision):
    return torch.bfloat16 if _prec(precision) == CONV_BF16 else torch.float32


def _check_inputs(I, F, precision, i_dims, f_dims, cuda=True):
    where = "CUDA" if cuda else "CPU"
    want = _want_dtype(precision)
    for name, t, nd in (("I", I, i_dims), ("F", F, f_dims)):
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{name} must be a torch.Tensor")
        if t.is_cuda != cuda:
            raise ValueError(f"{name} must be a {where} tensor")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if t.dim() != nd:
            raise ValueError(f"{name} must have {nd} dimensions, got shape {tuple(t.shape)}")
        if t.dtype != want:
            raise ValueError(f"precision {precision} expects {want} {name}, got {t.dtype}")
    if cuda and I.device != F.device:
        raise ValueError("I and F must be on the same device")
    if F.shape[-1] != F.shape[-2]:
        raise ValueError(f"F must hold square K x K filters, got {tuple(F.shape)}")
    if f_dims == 4 and F.shape[1] != I.shape[-3]:
        raise ValueError(f"channel mismatch: I has {I.shape[-3]} channels, F {F.shape[1]}")


def _output(out, shape, like, cuda=True):
    if out is None:
        return torch.empty(shape, device=like.device if cuda else "cpu", dtype=torch.float32)
    if not isinstance(out, torch.Tensor) or out.dtype != torch.float32 or tuple(out.shape) != tuple(shape):
        raise ValueError(f"out must be a float32 tensor of shape {tuple(shape)}")
    if out.is_cuda != cuda or (cuda and out.device != like.device) or not out.is_contiguous():
        raise ValueError("out must be contiguous and on the inputs' device")
    return out


def _out_hw(Wy, Wx, K, pad=0, stride=1):
    Ho, Wo = (Wy + 2 * pad - K) // stride + 1, (Wx + 2 * pad - K) // stride + 1
    if K < 1 or Ho < 1 or Wo < 1 or pad < 0 or stride < 1:
        raise ValueError(f"K={K} does not fit the {Wy}x{Wx} map (pad {pad}, stride {stride})")
    return Ho, Wo


def single(I: torch.Tensor, F: torch.Tensor, out: torch.Tensor | None = None, stream=None):
    """Eq. 2: I[Wy][Wx] f32, F[M][K][K] f32 -> O[M][Ho][Wo] f32 (kernel KS)."""
    _check_inputs(I, F, "fp32", 2, 3)
    Wy, Wx = I.shape
    M, K, _ = F.shape
    O = _output(out, (M, *_out_hw(Wy, Wx, K)), I)
    conv_single_ex(I, Wx, Wy, F, K, M, O, stream)
    return O


def multi(I: torch.Tensor, F: torch.Tensor, precision="fp32", out: torch.Tensor | None = None,
          stream=None):
    """Eq. 1: I[C][Wy][Wx], F[M][C][K][K] -> O[M][Ho][Wo] f32.

    precision "fp32" (KM-SIMT), "tf32" (KM-TC) take float32 I, F; "bf16"
    (KM-TC) takes bfloat16 I, F."""
    _check_inputs(I, F, precision, 3, 4)
    C, Wy, Wx = I.shape
    M, _, K, _ = F.shape
    O = _output(out, (M, *_out_hw(Wy, Wx, K)), I)
    conv_multi_ex(I, C, Wx, Wy, F, K, M, O, precision, stream)
    return O


def multi_batched(I: torch.Tensor, F: torch.Tensor, precision="fp32", out: torch.Tensor | None = None,
                  stream=None):
    """Eq. 1 on a batch: I[N][C][Wy][Wx], F[M][C][K][K] -> O[N][M][Ho][Wo] f32
    (= torch.nn.functional.conv2d(I, F) without padding, stride 1)."""
    _check_inputs(I, F, precision, 4, 4)
    N, C, Wy, Wx = I.shape
    M, _, K, _ = F.shape
    O = _output(out, (N, M, *_out_hw(Wy, Wx, K)), I)
    conv_multi_batched_ex(I, N, C, Wx, Wy, F, K, M, O, precision, stream)
    return O


def conv_single_strided_ex(I, Wx, Wy, F, K, M, pad, stride, O, stream=None):
    _check(load().conv_single_strided_ex(_ptr(I), Wx, Wy, _ptr(F), K, M, pad, stride, _ptr(O), _stream(stream)))


def conv_multi_strided_ex(I, N, C, Wx, Wy, F, K, M, pad, stride, O, precision="fp32", stream=None):
    _check(load().conv_multi_strided_ex(_ptr(I), N, C, Wx, Wy, _ptr(F), K, M, pad, stride, _ptr(O),
                                        _prec(precision), _stream(stream)))


def plan_multi_strided(C, Wx, Wy, K, M, pad, stride, precision="fp32", N=1) -> dict:
    p = ConvPlan()
    _check(load().conv_plan_multi_strided(N, C, Wx, Wy, K, M, pad, stride, _prec(precision), ctypes.byref(p)))
    return p.as_dict()


def multi_strided(I: torch.Tensor, F: torch.Tensor, stride: int, pad: int = 0, precision="fp32",
                  out: torch.Tensor | None = None, stream=None):
    """Strided, zero-padded Eq. 1: I[N][C][Wy][Wx] -> O[N][M][Ho][Wo],
    Ho = (Wy+2p-K)//s+1 (= torch.nn.functional.conv2d(I, F, stride=s, padding=p))."""
    _check_inputs(I, F, precision, 4, 4)
    N, C, Wy, Wx = I.shape
    M, _, K, _ = F.shape
    O = _output(out, (N, M, *_out_hw(Wy, Wx, K, pad, stride)), I)
    conv_multi_strided_ex(I, N, C, Wx, Wy, F, K, M, pad, stride, O, precision, stream)
    return O


def single_strided(I: torch.Tensor, F: torch.Tensor, stride: int, pad: int = 0,
                   out: torch.Tensor | None = None, stream=None):
    """Strided, zero-padded Eq. 2 (C = 1, FP32): I[Wy][Wx], F[M][K][K] -> O[M][Ho][Wo]."""
    _check_inputs(I, F, "fp32", 2, 3)
    Wy, Wx = I.shape
    M, K, _ = F.shape
    O = _output(out, (M, *_out_hw(Wy, Wx, K, pad, stride)), I)
    conv_single_strided_ex(I, Wx, Wy, F, K, M, pad, stride, O, stream)
    return O


def multi_padded(I: torch.Tensor, F: torch.Tensor, pad: int, precision="fp32", out: torch.Tensor | None = None,
                 stream=None):
    """Zero-padded Eq. 1: I[N][C][Wy][Wx] -> O[N][M][Wy+2p-K+1][Wx+2p-K+1]
    (= torch.nn.functional.conv2d(I, F, padding=pad))."""
    _check_inputs(I, F, precision, 4, 4)
    N, C, Wy, Wx = I.shape
    M, _, K, _ = F.shape
    O = _output(out, (N, M, *_out_hw(Wy, Wx, K, pad)), I)
    conv_multi_pad_ex(I, N, C, Wx, Wy, F, K, M, pad, O, precision, stream)
    return O


def single_padded(I: torch.Tensor, F: torch.Tensor, pad: int, out: torch.Tensor | None = None, stream=None):
    """Zero-padded Eq. 2: I[Wy][Wx], F[M][K][K] -> O[M][Wy+2p-K+1][Wx+2p-K+1]."""
    _check_inputs(I, F, "fp32", 2, 3)
    Wy, Wx = I.shape
    M, K, _ = F.shape
    O = _output(out, (M, *_out_hw(Wy, Wx, K, pad)), I)
    conv_single_pad_ex(I, Wx, Wy, F, K, M, pad, O, stream)
    return O


def multi_host(I: torch.Tensor, F: torch.Tensor, precision="fp32", out: torch.Tensor | None = None,
               stream=None):
    """End-to-end on host tensors through conv_multi_host (H2D, kernel, D2H, sync)."""
    _check_inputs(I, F, precision, 3, 4, cuda=False)
    C, Wy, Wx = I.shape
    M, _, K, _ = F.shape
    O = _output(out, (M, *_out_hw(Wy, Wx, K)), I, cuda=False)
    conv_multi_host(I, C, Wx, Wy, F, K, M, O, precision, stream)
    return O


def single_host(I: torch.Tensor, F: torch.Tensor, out: torch.Tensor | None = None, stream=None):
    """End-to-end on host tensors through conv_single_host (H2D, kernel, D2H, sync)."""
    _check_inputs(I, F, "fp32", 2, 3, cuda=False)
    Wy, Wx = I.shape
    M, K, _ = F.shape
    O = _output(out, (M, *_out_hw(Wy, Wx, K)), I, cuda=False)
    conv_single_host(I, Wx, Wy, F, K, M, O, stream)
    return O
