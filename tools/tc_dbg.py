import os, sys, json, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
res = {}
for dbg in (0, 64, 15, 79):
    out = subprocess.run([sys.executable, "-c", f"""
import os, sys
sys.path.insert(0, '{os.path.dirname(os.path.dirname(os.path.abspath(__file__)))}')
os.environ['B200CONV_TC_DBG'] = '{dbg}'
import torch, bench, synth
from paper_2212_00404_b200 import conv
from paper_2212_00404_b200 import build as _b
conv.load(_b.build(diag=True))       # the -DB200CONV_DIAG library (stamps / DBG switches)
dev = torch.device('cuda', 0)
r = {{}}
for c in bench.suite_calls(1, 0):
    if c['kind'] != 'multi' or c['prec'] == 'fp32': continue
    if not any(n in c['name'] for n in ('sweep', 'target', 'resnet_7')): continue
    dt = torch.bfloat16 if c['prec'] == 'bf16' else torch.float32
    I = torch.from_numpy(synth.uniform01(1, (c['C'], c['Wy'], c['Wx']))).to(dev, dt)
    F = torch.from_numpy(synth.uniform_pm1(2, (c['M'], c['C'], c['K'], c['K']))).to(dev, dt)
    Os = [torch.empty((c['M'], c['Ho'], c['Wo']), device=dev) for _ in range(4)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(3): conv.conv_multi_ex(I, c['C'], c['Wx'], c['Wy'], F, c['K'], c['M'], Os[i%4], c['prec'], s.cuda_stream)
        g = torch.cuda.CUDAGraph(); s.synchronize(); g.capture_begin()
        for i in range(12): conv.conv_multi_ex(I, c['C'], c['Wx'], c['Wy'], F, c['K'], c['M'], Os[i%4], c['prec'], s.cuda_stream)
        g.capture_end(); g.replay(); s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); g.replay(); e1.record(s)
    s.synchronize()
    r[c['label']] = round(1e3 * e0.elapsed_time(e1) / 12, 2)
print(r)
"""], capture_output=True, text=True)
    res[dbg] = out.stdout.strip() or out.stderr[-500:]
for k, v in res.items(): print(k, v)
