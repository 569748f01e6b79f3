"""KM-TC/G GEMM per-CTA timeline (diag build, B200CONV_GM_DBG=1) of one layer
launched back to back.  usage: gm_timeline.py <label-substring> [...]"""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
from paper_2212_00404_b200 import conv
from paper_2212_00404_b200 import build as _b
conv.load(_b.build(diag=True))
dev = torch.device("cuda", 0)
lib = conv.load()
for want in sys.argv[1:]:
    for c in bench.suite_calls(1, 0):
        if want not in c["label"] or c["kind"] != "multi" or c["prec"] == "fp32":
            continue
        dt = torch.bfloat16 if c["prec"] == "bf16" else torch.float32
        I = torch.from_numpy(synth.uniform01(synth.SEED_I, (c["C"], c["Wy"], c["Wx"]))).to(dev, dt)
        Fs = [torch.from_numpy(synth.uniform_pm1(synth.SEED_F + j, (c["M"], c["C"], c["K"], c["K"]))).to(dev, dt)
              for j in range(4)]
        Os = [torch.empty((c["M"], c["Ho"], c["Wo"]), device=dev) for _ in range(4)]
        call = lambda j: conv.conv_multi_ex(I, c["C"], c["Wx"], c["Wy"], Fs[j % 4], c["K"], c["M"], Os[j % 4], c["prec"])
        for j in range(4): call(j)
        torch.cuda.synchronize()
        os.environ["B200CONV_GM_DBG"] = os.environ.get("DBG", "1")
        for j in range(4): call(j)
        torch.cuda.synchronize()
        os.environ.pop("B200CONV_GM_DBG")
        p = conv.plan_multi(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], c["prec"])
        if p["kernel"] != 3:
            print(c["label"], "is not on KM-TC/G", p)
            continue
        G = p["grid_x"] * p["grid_y"] * p["grid_z"]
        buf = (ctypes.c_ulonglong * 16384)()
        lib.conv_diag_gm_cta_stamps(buf)
        allb = np.array(list(buf), dtype=np.uint64)
        tu = allb[:8192].reshape(1024, 8)[:min(G, 1024)]
        lp = allb[8192:].reshape(1024, 8)[:min(G, 1024)].astype(np.int64)
        end = (tu[:, 6] >> np.uint64(8)) | (tu[:, 0] & ~np.uint64((1 << 56) - 1))
        t = tu.astype(np.int64)
        t[:, 6] = end.astype(np.int64)
        t[:, 5] = np.where(t[:, 5] == 0, t[:, 4], t[:, 5])
        r = (t - t[:, 0].min()) / 1e3
        print(f"== {c['label']} plan {p} CTAs {G} (percentiles 0/50/90/100 of us since the first CTA start)")
        for k, name in [(0, "start"), (1, "pdl-wait"), (2, "stage0 full"), (3, "mma done"), (4, "partial stored"),
                        (5, "cluster sync"), (7, "slices loaded"), (6, "end")]:
            v = r[:, k]
            print(f"  {name:14s} " + " ".join(f"{np.percentile(v, q):7.2f}" for q in (0, 50, 90, 100)))
        d = np.diff(lp, axis=1)
        print("  store-loop clock64 deltas per iteration (median over CTAs):", np.median(d, axis=0))
