"""Probe HBM write bandwidth with rotating buffers (torch fill / copy vs our KS)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_00404_b200 import conv
import synth
dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
def timeit(fn, reps=16):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for i in range(3): fn(i)
        s.synchronize()
        g.capture_begin()
        for i in range(reps): fn(i)
        g.capture_end()
        g.replay(); s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); g.replay(); e1.record(s)
    s.synchronize()
    return 1e3 * e0.elapsed_time(e1) / reps
out = {}
n = 256 * 224 * 224
for nb in (1, 8):
    bufs = [torch.empty(n, device=dev) for _ in range(nb)]
    src = [torch.empty(n, device=dev).normal_() for _ in range(nb)]
    out[f"fill_rot{nb}_us"] = timeit(lambda i: bufs[i % nb].fill_(1.0))
    out[f"copy_rot{nb}_us"] = timeit(lambda i: bufs[i % nb].copy_(src[i % nb]))
    out[f"zero_rot{nb}_us"] = timeit(lambda i: bufs[i % nb].zero_())
for K in (1, 3, 5, 7):
    I = torch.from_numpy(synth.uniform01(1, (224, 224))).to(dev)
    F = torch.from_numpy(synth.uniform_pm1(2, (256, K, K))).to(dev)
    Ho = 225 - K
    for nb in (1, 8):
        Os = [torch.empty((256, Ho, Ho), device=dev) for _ in range(nb)]
        out[f"ks_k{K}_m256_rot{nb}_us"] = timeit(lambda i: conv.conv_single_ex(I, 224, 224, F, K, 256, Os[i % nb], s.cuda_stream))
    out[f"plan_k{K}"] = conv.plan_single(224, 224, K, 256)
print(json.dumps(out, indent=0))
