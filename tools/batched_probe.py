"""Batched tensor-core throughput on the 28x28x256 layer (and friends) vs N."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2212_00404_b200 import conv
dev = torch.device("cuda")
s = torch.cuda.Stream()
PEAK = {"tf32": 1610.1 / 2, "bf16": 1610.1}
for (C, W, K, M) in [(256, 28, 3, 256), (128, 28, 3, 128), (96, 27, 5, 256)]:
    for prec in ("tf32", "bf16"):
        for N in (1, 8, 32, 64):
            dt = torch.bfloat16 if prec == "bf16" else torch.float32
            I = torch.rand(N, C, W, W, device=dev).to(dt)
            F = (torch.rand(M, C, K, K, device=dev) * 2 - 1).to(dt)
            Ho = W - K + 1
            nb = 3
            Os = [torch.empty(N, M, Ho, Ho, device=dev) for _ in range(nb)]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                for j in range(3): conv.conv_multi_batched_ex(I, N, C, W, W, F, K, M, Os[j % nb], prec, s.cuda_stream)
                s.synchronize()
                g.capture_begin()
                for j in range(10): conv.conv_multi_batched_ex(I, N, C, W, W, F, K, M, Os[j % nb], prec, s.cuda_stream)
                g.capture_end()
                g.replay(); s.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s); g.replay(); e1.record(s); s.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / 10
            fl = 2.0 * N * M * C * K * K * Ho * Ho
            tf = fl / us / 1e6
            print(f"{C}x{W}x{W} K{K} M{M} {prec} N={N:3d}: {us:8.2f} us  {tf:7.1f} TFLOP/s  {100 * tf / PEAK[prec]:5.1f}% of tensor peak  plan S={conv.plan_multi_batched(N, C, W, W, K, M, prec)['grid_x']}", flush=True)
