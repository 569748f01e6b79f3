import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, synth
from paper_2212_00404_b200 import conv
dev = torch.device("cuda", 0)
pk = bench.peaks()
calls = [c for c in bench.suite() if c["label"] in ("single_224x224_k1_m256:fp32", "single_224x224_k3_m256:fp32", "target_28x28_c256_m256_k3:fp32", "target_28x28_c256_m256_k3:tf32")]
for c in calls:
    dt = torch.bfloat16 if c["prec"] == "bf16" else torch.float32
    I = torch.from_numpy(synth.uniform01(synth.SEED_I, (c["C"], c["Wy"], c["Wx"]))).to(dev, dt)
    F = torch.from_numpy(synth.uniform_pm1(synth.SEED_F + c["cfg_index"], (c["M"], c["C"], c["K"], c["K"]))).to(dev, dt)
    if c["kind"] == "single":
        I, F = I[0].contiguous(), F[:, 0].contiguous()
    c["I"], c["F"] = I, F
    c["O"] = torch.empty((c["M"], c["Ho"], c["Wo"]), device=dev)
stream = torch.cuda.Stream()
sh = stream.cuda_stream
def launch(c):
    if c["kind"] == "single":
        conv.conv_single_ex(c["I"], c["Wx"], c["Wy"], c["F"], c["K"], c["M"], c["O"], sh)
    else:
        conv.conv_multi_ex(c["I"], c["C"], c["Wx"], c["Wy"], c["F"], c["K"], c["M"], c["O"], c["prec"], sh)
def capture(fn):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        stream.synchronize(); g.capture_begin(); fn(); g.capture_end()
    return g
res = {}
for rep in range(3):
    r = bench._layer_b2b(calls, launch, capture, stream, dev, pk)
    res[f"b2b_{rep}"] = {k: v["us"] for k, v in r.items()}
# no rotation
def norot(c, reps=12):
    g = capture(lambda: [launch(c) for _ in range(reps)])
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        stream.synchronize(); e0.record(stream); g.replay(); e1.record(stream)
    stream.synchronize()
    return 1e3 * e0.elapsed_time(e1) / reps
res["norot"] = {c["label"]: norot(c) for c in calls}
print(json.dumps(res, indent=0))
