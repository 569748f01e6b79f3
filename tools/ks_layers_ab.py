"""KS per-layer A/B: back-to-back graph timing of single-channel layers for two
library builds (B200CONV_LIB_PATH), interleaved.  usage: ks_layers_ab.py libA libB [label-substrings...]"""
import os, subprocess, sys, json
labels = sys.argv[3:] or ["single_224x224_k3", "single_224x224_k1_m256", "single_224x224_k5_m256",
                          "single_56x56_k3_m256", "single_28x28_k3_m256", "single_14x14_k3_m256"]
code = r'''
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, bench, synth
from paper_2212_00404_b200 import conv
dev = torch.device("cuda", 0); s = torch.cuda.Stream()
out = {}
for c in bench.suite_calls(1, 0):
    if c["kind"] != "single" or not any(l in c["label"] for l in json.loads(sys.argv[1])): continue
    I = torch.from_numpy(synth.uniform01(1, (c["Wy"], c["Wx"]))).to(dev)
    F = torch.from_numpy(synth.uniform_pm1(2, (c["M"], c["K"], c["K"]))).to(dev)
    Os = [torch.empty((c["M"], c["Ho"], c["Wo"]), device=dev) for _ in range(8)]
    fn = lambda j: conv.conv_single_ex(I, c["Wx"], c["Wy"], F, c["K"], c["M"], Os[j % 8], s.cuda_stream)
    for j in range(3): fn(j)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        g.capture_begin()
        for j in range(16): fn(j)
        g.capture_end()
        g.replay(); s.synchronize()
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s); g.replay(); b.record(s); s.synchronize()
            best = min(best, 1e3 * a.elapsed_time(b) / 16)
    out[c["label"]] = round(best, 2)
print(json.dumps(out))
'''
res = {}
for rnd in range(2):
    for lib in sys.argv[1:3]:
        env = dict(os.environ, B200CONV_LIB_PATH=os.path.abspath(lib))
        r = subprocess.run([sys.executable, "-c", code, json.dumps(labels)], env=env, capture_output=True, text=True)
        d = json.loads(r.stdout.strip().splitlines()[-1])
        for k, v in d.items():
            res.setdefault(k, {}).setdefault(lib, []).append(v)
for k, v in res.items():
    print(f"{k:34s} " + "  ".join(f"{os.path.basename(l)}: {min(t):7.2f}" for l, t in v.items()))
