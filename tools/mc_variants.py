"""Back-to-back (CUDA graph, 12 launches, rotating O) time of multi-channel
bench layers under environment variants.
usage: mc_variants.py "ENV=v&ENV2=w;..." <label-substring> [...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
from paper_2212_00404_b200 import conv
if os.environ.get("B200CONV_LIB_PATH"):           # A/B against another build of the library
    conv.load(os.environ["B200CONV_LIB_PATH"])
dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
variants = sys.argv[1].split(";")


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


for want in sys.argv[2:]:
    for c in bench.suite_calls(1, 0):
        if want not in c["label"] or c["kind"] != "multi":
            continue
        dt = torch.bfloat16 if c["prec"] == "bf16" else torch.float32
        I = torch.from_numpy(synth.uniform01(synth.SEED_I, (c["C"], c["Wy"], c["Wx"]))).to(dev, dt)
        Fs = [torch.from_numpy(synth.uniform_pm1(synth.SEED_F + c["cfg_index"], (c["M"], c["C"], c["K"], c["K"]))).to(dev, dt)]
        nb = max(2, min(12, int(3 * 126e6 // (Fs[0].numel() * Fs[0].element_size() + 4 * c["M"] * c["Ho"] * c["Wo"])) + 1))
        Fs += [Fs[0].clone() for _ in range(nb - 1)]
        Os = [torch.empty((c["M"], c["Ho"], c["Wo"]), device=dev) for _ in range(nb)]
        out = []
        for v in variants:
            env = dict(kv.split("=", 1) for kv in v.split("&") if kv)
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            us = timeit(lambda j: conv.conv_multi_ex(I, c["C"], c["Wx"], c["Wy"], Fs[j % nb], c["K"], c["M"],
                                                     Os[j % nb], c["prec"], s.cuda_stream))
            for k, o in old.items():
                if o is None: os.environ.pop(k)
                else: os.environ[k] = o
            out.append(f"{v or 'base'}: {us:6.2f}")
        print(f"{c['label']}: " + " | ".join(out), flush=True)
