"""Run one bench layer (by label substring) a few times with rotating buffers
(for ncu captures).  usage: run_layer.py <label-substring> [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
from paper_2212_00404_b200 import conv

want = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dev = torch.device("cuda", 0)
for c in bench.suite_calls(1, 0):
    if want not in c["label"]:
        continue
    dt = torch.bfloat16 if c["prec"] == "bf16" else torch.float32
    I = torch.from_numpy(synth.uniform01(synth.SEED_I, (c["C"], c["Wy"], c["Wx"]))).to(dev, dt)
    F = torch.from_numpy(synth.uniform_pm1(synth.SEED_F + c["cfg_index"], (c["M"], c["C"], c["K"], c["K"]))).to(dev, dt)
    if c["kind"] == "single":
        I, F = I[0].contiguous(), F[:, 0].contiguous()
    Os = [torch.empty((c["M"], c["Ho"], c["Wo"]), device=dev) for _ in range(reps)]
    for O in Os:
        if c["kind"] == "single":
            conv.conv_single_ex(I, c["Wx"], c["Wy"], F, c["K"], c["M"], O)
        else:
            conv.conv_multi_ex(I, c["C"], c["Wx"], c["Wy"], F, c["K"], c["M"], O, c["prec"])
    torch.cuda.synchronize()
    print(c["label"], conv.plan_single(c["Wx"], c["Wy"], c["K"], c["M"]) if c["kind"] == "single"
          else conv.plan_multi(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], c["prec"]))
