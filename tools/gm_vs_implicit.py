"""KM-TC/G (im2col + GEMM) vs the implicit KM-TC kernel on the configs[4]
shape at the per-rank filter counts of 1/2/4/8 GPUs and on the layers the
planner sends to KM-TC/G (B200CONV_GM=2 forces the GEMM, =0 the implicit
kernel).  12 launches back to back per graph, rotating F/O, best of 5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2212_00404_b200 import conv

dev = torch.device("cuda", 0)
s = torch.cuda.Stream()


def timeit(fn, reps=12):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        s.synchronize()
        g.capture_begin()
        for i in range(reps):
            fn(i)
        g.capture_end()
        g.replay()
        s.synchronize()
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s); g.replay(); b.record(s); s.synchronize()
            best = min(best, 1e3 * a.elapsed_time(b) / reps)
    return best


for (C, W, K, M) in [(512, 14, 3, 4096), (512, 14, 3, 2048), (512, 14, 3, 1024), (512, 14, 3, 512),
                     (512, 7, 3, 512), (256, 14, 3, 256)]:
    for prec in ("tf32", "bf16"):
        dt = torch.bfloat16 if prec == "bf16" else torch.float32
        I = torch.from_numpy(synth.uniform01(1, (C, W, W))).to(dev, dt)
        Fs = [torch.from_numpy(synth.uniform_pm1(2 + j, (M, C, K, K))).to(dev, dt) for j in range(4)]
        Os = [torch.empty((M, W - K + 1, W - K + 1), device=dev) for _ in range(4)]
        out = []
        for mode in ("", "2", "0"):
            if mode:
                os.environ["B200CONV_GM"] = mode
            else:
                os.environ.pop("B200CONV_GM", None)
            p = conv.plan_multi(C, W, W, K, M, prec)
            us = timeit(lambda j: conv.conv_multi_ex(I, C, W, W, Fs[j % 4], K, M, Os[j % 4], prec, s.cuda_stream))
            out.append(f"{'plan' if not mode else ('gemm' if mode == '2' else 'implicit')} k{p['kernel']} "
                       f"S{p['cluster_x']} {us:7.2f}")
        os.environ.pop("B200CONV_GM", None)
        print(f"C{C} W{W} M{M} {prec}: " + " | ".join(out), flush=True)
