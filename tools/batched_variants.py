"""Batched layer time under env variants: batched_variants.py "ENV=v&..;.." N C W K M prec"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_00404_b200 import conv
if os.environ.get("B200CONV_LIB_PATH"):           # A/B against another build of the library
    conv.load(os.environ["B200CONV_LIB_PATH"])
dev = torch.device("cuda"); s = torch.cuda.Stream()
variants = sys.argv[1].split(";")
N, C, W, K, M = (int(v) for v in sys.argv[2:7]); prec = sys.argv[7]
dt = torch.bfloat16 if prec == "bf16" else torch.float32
I = torch.rand(N, C, W, W, device=dev).to(dt); F = (torch.rand(M, C, K, K, device=dev) * 2 - 1).to(dt)
Ho = W - K + 1
Os = [torch.empty(N, M, Ho, Ho, device=dev) for _ in range(3)]
out = []
for v in variants:
    env = dict(kv.split("=", 1) for kv in v.split("&") if kv)
    old = {k: os.environ.get(k) for k in env}; os.environ.update(env)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for j in range(3): conv.conv_multi_batched_ex(I, N, C, W, W, F, K, M, Os[j % 3], prec, s.cuda_stream)
        s.synchronize(); g.capture_begin()
        for j in range(10): conv.conv_multi_batched_ex(I, N, C, W, W, F, K, M, Os[j % 3], prec, s.cuda_stream)
        g.capture_end(); g.replay(); s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); g.replay(); e1.record(s); s.synchronize()
    for k, o in old.items():
        if o is None: os.environ.pop(k)
        else: os.environ[k] = o
    us = e0.elapsed_time(e1) * 1e3 / 10
    tf = 2.0 * N * M * C * K * K * Ho * Ho / us / 1e6
    out.append(f"{v or 'base'}: {us:7.1f} us {tf:6.1f} TF/s")
print(f"N={N} C={C} W={W} K={K} M={M} {prec}: " + " | ".join(out))
