"""Run one KS layer `reps` times on rotating outputs (for ncu DRAM-byte
sequences with --cache-control none).  usage: ks_seq.py W K M [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2212_00404_b200 import conv

W, K, M = (int(a) for a in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 12
dev = torch.device("cuda", 0)
I = torch.from_numpy(synth.uniform01(1, (W, W))).to(dev)
F = torch.from_numpy(synth.uniform_pm1(2, (M, K, K))).to(dev)
Os = [torch.empty((M, W - K + 1, W - K + 1), device=dev) for _ in range(reps)]
for O in Os:
    conv.conv_single_ex(I, W, W, F, K, M, O)
torch.cuda.synchronize()
