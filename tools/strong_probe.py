"""Per-rank cost of the filter-sharded configs[4] step on one GPU: the
3-precision step (FP32 -> TF32 -> BF16, one PDL-chained CUDA graph, rotating
F/O sets larger than L2) at M = 4096 / G for G = 1, 2, 4, 8, and each
precision's call alone.  usage: strong_probe.py [G ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2212_00404_b200 import conv

dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
c = synth.SHARD_SWEEP
C, W, K = c["C"], c["Wx"], c["K"]
Ho = W - K + 1
I32 = torch.from_numpy(synth.uniform01(synth.SEED_I, (C, W, W))).to(dev)


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


for G in [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]:
    M = c["M"] // G
    F32 = torch.from_numpy(synth.uniform_pm1(synth.SEED_F + 104, (M, C, K, K))).to(dev)
    bufs = {}
    for p in ("fp32", "tf32", "bf16"):
        dt = torch.bfloat16 if p == "bf16" else torch.float32
        per = F32.numel() * (2 if p == "bf16" else 4)
        nb = max(2, min(8, int(3 * 126e6 // per) + 1))
        bufs[p] = (I32.to(dt), [F32.to(dt).clone() for _ in range(nb)],
                   [torch.empty((M, Ho, Ho), device=dev) for _ in range(nb)])

    def call(p, j):
        I, Fs, Os = bufs[p]
        conv.conv_multi_ex(I, C, W, W, Fs[j % len(Fs)], K, M, Os[j % len(Os)], p, s.cuda_stream)

    one = {p: timeit(lambda j, p=p: call(p, j)) for p in bufs}
    step = timeit(lambda j: [call(p, j) for p in bufs])
    if os.environ.get("ORDERS"):
        import itertools
        for order in itertools.permutations(bufs):
            print(f"  order {'>'.join(order)}: {timeit(lambda j: [call(p, j) for p in order]):7.2f} us", flush=True)
    print(f"G={G} M={M}: step {step:7.2f} us | " + " | ".join(f"{p} {one[p]:7.2f}" for p in one) +
          f" | plans " + " ".join(str(conv.plan_multi(C, W, W, K, M, p)["kernel"]) for p in bufs), flush=True)
