"""Run the batched 28x28x256 layer a few times (for ncu captures).
usage: run_batched.py <N> <prec> [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2212_00404_b200 import conv
N, prec = int(sys.argv[1]), sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dev = torch.device("cuda", 0)
dt = torch.bfloat16 if prec == "bf16" else torch.float32
C, W, K, M = 256, 28, 3, 256
I = torch.from_numpy(synth.uniform01(synth.SEED_I + N, (N, C, W, W))).to(dev, dt)
F = torch.from_numpy(synth.uniform_pm1(synth.SEED_F + N, (M, C, K, K))).to(dev, dt)
O = torch.empty((N, M, W - K + 1, W - K + 1), device=dev)
for _ in range(reps):
    conv.conv_multi_batched_ex(I, N, C, W, W, F, K, M, O, prec)
torch.cuda.synchronize()
print(conv.plan_multi_batched(N, C, W, W, K, M, prec))
