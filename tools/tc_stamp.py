import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np, synth
from paper_2212_00404_b200 import conv
from paper_2212_00404_b200 import build as _b
conv.load(_b.build(diag=True))       # the -DB200CONV_DIAG library (stamps / DBG switches)
dbg = sys.argv[1]
os.environ['B200CONV_TC_DBG'] = dbg
dev = torch.device('cuda', 0)
LAYERS = [tuple(int(v) if v.isdigit() else v for v in a.split(',')) for a in sys.argv[2:]] or [(512, 14, 3, 4096, 'tf32'), (256, 28, 3, 256, 'tf32')]
for (C, W, K, M, prec) in LAYERS:
    dt = torch.bfloat16 if prec == 'bf16' else torch.float32
    I = torch.from_numpy(synth.uniform01(1, (C, W, W))).to(dev, dt)
    F = torch.from_numpy(synth.uniform_pm1(2, (M, C, K, K))).to(dev, dt)
    O = torch.zeros((M, W - K + 1, W - K + 1), device=dev)
    for _ in range(3):
        conv.conv_multi_ex(I, C, W, W, F, K, M, O, prec)
    torch.cuda.synchronize()
    import ctypes
    buf = (ctypes.c_ulonglong * 1024)()
    conv.load().conv_diag_stamps(buf)
    t = np.array(list(buf), dtype=np.int64)
    n = int((t[:256] > 0).sum())
    P, G, Mm = t[:n], t[256:256 + n], t[512:512 + n]
    t0 = P[0]
    print(f"== C{C} W{W} M{M} {prec} dbg={dbg} iters={n}")
    print("P (cyc):", np.round((P - t0) / 1.0, 0)[:16].tolist(), "... last", round((P[-1] - t0) / 1.0, 0))
    print("G (cyc):", np.round((G - t0) / 1.0, 0)[:16].tolist(), "... last", round((G[-1] - t0) / 1.0, 0))
    print("M (cyc):", np.round((Mm - t0) / 1.0, 0)[:16].tolist(), "... last", round((Mm[-1] - t0) / 1.0, 0))
    A, B = t[768:768 + 16], t[896:896 + 16]
    print("loop top (cyc):", np.round((A - t0) / 1.0, 0).tolist())
    print("after wait(cyc):", np.round((B - t0) / 1.0, 0).tolist())
