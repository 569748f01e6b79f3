"""Back-to-back (CUDA graph, 12 launches, rotating O) time of KS layers under
environment variants.  usage: ks_variants.py "ENV=v,ENV2=w;..." W K M [W K M ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2212_00404_b200 import conv
if os.environ.get("B200CONV_LIB_PATH"):           # A/B against another build of the library
    conv.load(os.environ["B200CONV_LIB_PATH"])
dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
variants = [v for v in sys.argv[1].split(";")]
args = [int(a) for a in sys.argv[2:]]

def timeit(fn, reps=12):
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

for i in range(0, len(args), 3):
    W, K, M = args[i:i + 3]
    I = torch.from_numpy(synth.uniform01(1, (W, W))).to(dev)
    F = torch.from_numpy(synth.uniform_pm1(2, (M, K, K))).to(dev)
    nb = max(2, min(12, int(3 * 126e6 // (4 * M * (W - K + 1) ** 2)) + 1))
    Os = [torch.empty((M, W - K + 1, W - K + 1), device=dev) for _ in range(nb)]
    out = []
    for v in variants:
        env = dict(kv.split("=") for kv in v.split(",") if kv)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        us = timeit(lambda j: conv.conv_single_ex(I, W, W, F, K, M, Os[j % nb], s.cuda_stream))
        for k, o in old.items():
            if o is None: os.environ.pop(k)
            else: os.environ[k] = o
        out.append(f"{v or 'base'}: {us:6.2f}")
    print(f"{W}x{W} K{K} M{M} G={conv.plan_single(W, W, K, M)['grid_x']}: " + " | ".join(out), flush=True)
