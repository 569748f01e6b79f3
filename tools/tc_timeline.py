"""KM-TC per-CTA timeline (B200CONV_TC_DBG=256) for layers launched back to
back.  usage: tc_timeline.py <label-substring> [...]  (bench layer labels)"""
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
        if want not in c["label"] or c["kind"] != "multi" or c["prec"] == "fp32":
            continue
        dt = torch.bfloat16 if c["prec"] == "bf16" else torch.float32
        I = torch.from_numpy(synth.uniform01(synth.SEED_I, (c["C"], c["Wy"], c["Wx"]))).to(dev, dt)
        F = torch.from_numpy(synth.uniform_pm1(synth.SEED_F + c["cfg_index"], (c["M"], c["C"], c["K"], c["K"]))).to(dev, dt)
        Os = [torch.empty((c["M"], c["Ho"], c["Wo"]), device=dev) for _ in range(6)]
        call = lambda O: conv.conv_multi_ex(I, c["C"], c["Wx"], c["Wy"], F, c["K"], c["M"], O, c["prec"])
        os.environ["B200CONV_TC_DBG"] = "0"
        for O in Os: call(O)
        torch.cuda.synchronize()
        os.environ["B200CONV_TC_DBG"] = str(256 + int(os.environ.get("EXTRA_DBG", "0")))
        for O in Os: call(O)
        torch.cuda.synchronize()
        os.environ["B200CONV_TC_DBG"] = "0"
        p = conv.plan_multi(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], c["prec"])
        G = p["grid_x"] * p["grid_y"] * p["grid_z"]
        buf = (ctypes.c_ulonglong * 8192)()
        lib.conv_diag_tc_cta_stamps(buf)
        tu = np.array(list(buf), dtype=np.uint64).reshape(1024, 8)[:min(G, 1024)]
        tu[:, 5] >>= np.uint64(8)
        tu[:, 5] |= tu[:, 0] & ~np.uint64((1 << 56) - 1)
        t = tu.astype(np.int64)
        t[:, 6] = np.where(t[:, 6] == 0, t[:, 4], t[:, 6])
        t[:, 7] = np.where(t[:, 7] == 0, t[:, 6], t[:, 7])
        r = (t - t[:, 0].min()) / 1e3
        print(f"== {c['label']} plan {p} CTAs {G} (pctl 0/50/90/100, us)")
        for k, name in [(0, "start"), (1, "pdl-wait"), (2, "kb0 ready"), (3, "mma done"), (4, "epilogue"), (6, "clustersync"), (7, "slices in"), (5, "end")]:
            print(f"  {name:10s}", " ".join(f"{v:6.2f}" for v in np.percentile(r[:, k], [0, 50, 90, 100])))
        break
