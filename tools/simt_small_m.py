"""KM-SIMT forced configurations on the configs[4] shard of M filters:
usage: simt_small_m.py M "tile,S,ws[/NST];..." """
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2212_00404_b200 import conv
dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
M = int(sys.argv[1])
C, W, K = 512, 14, 3
I = torch.from_numpy(synth.uniform01(synth.SEED_I, (C, W, W))).to(dev)
Fs = [torch.from_numpy(synth.uniform_pm1(synth.SEED_F, (M, C, K, K))).to(dev) for _ in range(4)]
Os = [torch.empty((M, 12, 12), device=dev) for _ in range(4)]


def timeit(fn, reps=20):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for i in range(3): fn(i)
        s.synchronize()
        g.capture_begin()
        for i in range(reps): fn(i)
        g.capture_end()
        g.replay(); s.synchronize()
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); g.replay(); e1.record(s); s.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


out = []
for v in [""] + sys.argv[2].split(";"):
    force, _, nst = v.partition("/")          # "tile,S,ws[/NST]"
    for k, x in (("B200CONV_SIMT_FORCE", force), ("B200CONV_SIMT_NST", nst)):
        if x:
            os.environ[k] = x
        else:
            os.environ.pop(k, None)
    p = conv.plan_multi(C, W, W, K, M, "fp32")
    us = timeit(lambda j: conv.conv_multi_ex(I, C, W, W, Fs[j % 4], K, M, Os[j % 4], "fp32", s.cuda_stream))
    out.append(f"{v or 'planner'}[{p['tile_m']}x{p['tile_n']} S{p['grid_x']} L{p['launches']}]: {us:.2f}")
print(f"M={M}: " + " | ".join(out))
