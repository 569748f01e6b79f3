"""Host-side enqueue cost of the async host entry points and the device *_ex calls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, bench, synth
from paper_2212_00404_b200 import conv
dev = torch.device("cuda")
calls = bench.suite()
host, devb = [], []
for c in calls:
    dt = torch.bfloat16 if c["prec"] == "bf16" else torch.float32
    I = torch.from_numpy(synth.uniform01(1, (c["C"], c["Wy"], c["Wx"]))).to(dt)
    F = torch.from_numpy(synth.uniform_pm1(2, (c["M"], c["C"], c["K"], c["K"]))).to(dt)
    if c["kind"] == "single":
        I, F = I[0].contiguous(), F[:, 0].contiguous()
    O = torch.empty((c["M"], c["Ho"], c["Wo"]))
    host.append((I.pin_memory(), F.pin_memory(), O.pin_memory()))
    devb.append((I.to(dev), F.to(dev), O.to(dev)))
s = [torch.cuda.Stream(), torch.cuda.Stream()]
def step_host():
    for i, (c, (Ih, Fh, Oh)) in enumerate(zip(calls, host)):
        sh = s[i & 1].cuda_stream
        if c["kind"] == "single": conv.conv_single_host_async(Ih, c["Wx"], c["Wy"], Fh, c["K"], c["M"], Oh, sh)
        else: conv.conv_multi_host_async(Ih, c["C"], c["Wx"], c["Wy"], Fh, c["K"], c["M"], Oh, c["prec"], sh)
def step_dev():
    for i, (c, (Id, Fd, Od)) in enumerate(zip(calls, devb)):
        sh = s[0].cuda_stream
        if c["kind"] == "single": conv.conv_single_ex(Id, c["Wx"], c["Wy"], Fd, c["K"], c["M"], Od, sh)
        else: conv.conv_multi_ex(Id, c["C"], c["Wx"], c["Wy"], Fd, c["K"], c["M"], Od, c["prec"], sh)
for fn, name in ((step_host, "host_async"), (step_dev, "device _ex")):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter(); fn(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"{name}: enqueue {1e3 * (t1 - t0):.2f} ms for {len(calls)} calls ({1e6 * (t1 - t0) / len(calls):.1f} us/call), total {1e3 * (t2 - t0):.2f} ms")
