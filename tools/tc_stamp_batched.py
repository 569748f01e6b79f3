"""Per-k-block clock64 stamps of CTA (0,0,0) of the batched KM-TC kernel
(B200CONV_TC_DBG=128): producer issue P, gather warp 0 arrive G, MMA issue M.
usage: tc_stamp_batched.py N prec  (env STAMP_DBG adds B200CONV_TC_DBG bits, default 128)"""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2212_00404_b200 import conv
from paper_2212_00404_b200 import build as _b
conv.load(_b.build(diag=True))       # the -DB200CONV_DIAG library (stamps / DBG switches)
N, prec = int(sys.argv[1]), sys.argv[2]
os.environ["B200CONV_TC_DBG"] = os.environ.get("STAMP_DBG", "128")
dev = torch.device("cuda", 0)
dt = torch.bfloat16 if prec == "bf16" else torch.float32
C, W, K, M = 256, 28, 3, 256
I = torch.from_numpy(synth.uniform01(7, (N, C, W, W))).to(dev, dt)
F = torch.from_numpy(synth.uniform_pm1(8, (M, C, K, K))).to(dev, dt)
O = torch.empty((N, M, W - 2, W - 2), device=dev)
for _ in range(3): conv.conv_multi_batched_ex(I, N, C, W, W, F, K, M, O, prec)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 1024)()
conv.load().conv_diag_stamps(buf)
t = np.array(list(buf), dtype=np.int64)
n = min(72 if prec == "tf32" else 36, 128)
P, G, Mm = t[:n], t[256:256 + n], t[512:512 + n]
t0 = P[0]
print(f"N={N} {prec} iters={n} total {Mm[n-1]-t0} cyc")
print("dM  (MMA issue intervals):", np.diff(Mm)[:40].tolist())
print("M-G (MMA issue after gather arrive):", (Mm - G)[:40].tolist())
print("G-P (producer issue -> gather arrive):", (G - P)[:40].tolist())
print("P-M[i-NS] (producer issue after MMA i-NS issue), NS = 6:", (P[6:] - Mm[:-6])[:30].tolist())
