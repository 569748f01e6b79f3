"""KM-SIMT per-CTA timeline (B200CONV_SIMT_DBG=1) for bench layers launched back
to back.  usage: simt_timeline.py <label-substring> [...]"""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
from paper_2212_00404_b200 import conv
from paper_2212_00404_b200 import build as _b
conv.load(_b.build(diag=True))       # the -DB200CONV_DIAG library (stamps / DBG switches)
dev = torch.device("cuda", 0)
lib = conv.load()
for want in sys.argv[1:]:
    for c in bench.suite_calls(1, 0):
        if want not in c["label"] or c["prec"] != "fp32" or c["kind"] != "multi":
            continue
        I = torch.from_numpy(synth.uniform01(synth.SEED_I, (c["C"], c["Wy"], c["Wx"]))).to(dev)
        F = torch.from_numpy(synth.uniform_pm1(synth.SEED_F + c["cfg_index"], (c["M"], c["C"], c["K"], c["K"]))).to(dev)
        Os = [torch.empty((c["M"], c["Ho"], c["Wo"]), device=dev) for _ in range(6)]
        call = lambda O: conv.conv_multi_ex(I, c["C"], c["Wx"], c["Wy"], F, c["K"], c["M"], O, "fp32")
        for O in Os: call(O)
        torch.cuda.synchronize()
        os.environ["B200CONV_SIMT_DBG"] = "1"
        for O in Os: call(O)
        torch.cuda.synchronize()
        os.environ["B200CONV_SIMT_DBG"] = "0"
        p = conv.plan_multi(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], "fp32")
        G = p["grid_x"] * p["grid_y"] * p["grid_z"]
        buf = (ctypes.c_ulonglong * 5120)()
        lib.conv_diag_simt_stamps(buf)
        tu = np.array(list(buf), dtype=np.uint64).reshape(1024, 5)[:min(G, 1024)]
        tu[:, 4] >>= np.uint64(8)
        tu[:, 4] |= tu[:, 0] & ~np.uint64((1 << 56) - 1)
        t = tu.astype(np.int64)
        r = (t - t[:, 0].min()) / 1e3
        print(f"== {c['label']} plan {p} CTAs {G} (pctl 0/50/90/100, us)")
        for k, name in enumerate(["start", "pdl-wait", "chunk0", "loop done", "end"]):
            print(f"  {name:10s}", " ".join(f"{v:6.2f}" for v in np.percentile(r[:, k], [0, 50, 90, 100])))
        S = p["grid_x"]
        for sp in range(S):
            rs = r[np.arange(len(r)) % S == sp]
            print(f"  split {sp}: start {np.percentile(rs[:, 0], 50):6.2f}  chunk0 {np.percentile(rs[:, 2], 50):6.2f}  "
                  f"loop done p0/50/100 " + " ".join(f"{v:6.2f}" for v in np.percentile(rs[:, 3], [0, 50, 100])))
