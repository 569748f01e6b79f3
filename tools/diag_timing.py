"""Diagnostic: graph step time with/without event nodes, per-call back-to-back times."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
from paper_2212_00404_b200 import conv

dev = torch.device("cuda", 0)
calls = bench.suite()
for c in calls:
    dt = torch.bfloat16 if c["prec"] == "bf16" else torch.float32
    I = torch.from_numpy(synth.uniform01(synth.SEED_I, (c["C"], c["Wy"], c["Wx"]))).to(dev, dt)
    F = torch.from_numpy(synth.uniform_pm1(synth.SEED_F + c["cfg_index"], (c["M"], c["C"], c["K"], c["K"]))).to(dev, dt)
    if c["kind"] == "single":
        I, F = I[0].contiguous(), F[:, 0].contiguous()
    c["I"], c["F"] = I, F
    c["O"] = torch.empty((c["M"], c["Ho"], c["Wo"]), device=dev)
s = torch.cuda.Stream()
sh = s.cuda_stream
def launch(c):
    if c["kind"] == "single":
        conv.conv_single_ex(c["I"], c["Wx"], c["Wy"], c["F"], c["K"], c["M"], c["O"], sh)
    else:
        conv.conv_multi_ex(c["I"], c["C"], c["Wx"], c["Wy"], c["F"], c["K"], c["M"], c["O"], c["prec"], sh)
with torch.cuda.stream(s):
    for c in calls: launch(c)
s.synchronize()
def graph_of(fn):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        g.capture_begin(); fn(); g.capture_end()
    return g
def time_graph(g, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        g.replay(); s.synchronize()
        e0.record(s)
        for _ in range(reps): g.replay()
        e1.record(s)
    s.synchronize()
    return e0.elapsed_time(e1) / reps
out = {}
g = graph_of(lambda: [launch(c) for c in calls])
out["step_ms_no_events"] = time_graph(g, 50)
# direct (non-graph) step
with torch.cuda.stream(s):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        for c in calls: launch(c)
    e1.record(s)
s.synchronize()
out["step_ms_direct"] = e0.elapsed_time(e1) / 10
# per-call: graph of 20 back-to-back launches
per = {}
for c in calls:
    gg = graph_of(lambda: [launch(c) for _ in range(20)])
    per[c["label"]] = round(1e3 * time_graph(gg, 5) / 20, 3)
out["per_call_us_b2b"] = per
out["sum_per_call_ms"] = sum(per.values()) / 1e3
# empty kernel floor via torch (tiny kernel)
x = torch.zeros(1, device=dev)
gg = graph_of(lambda: [x.add_(1) for _ in range(100)])
out["tiny_torch_kernel_us"] = 1e3 * time_graph(gg, 10) / 100
print(json.dumps(out))
