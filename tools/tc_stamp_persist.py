"""Per-ring-iteration clock64 stamps of CTA 0 of the persistent KM-TC kernel
(diagnostic build): P producer past `empty`, G0 gather warp 0 past `pfull`
(patch landed), G1 its `full` arrive, M MMA issuer past `full`.
usage: tc_stamp_persist.py N prec"""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2212_00404_b200 import conv
from paper_2212_00404_b200 import build as _b
conv.load(_b.build(diag=True))
N, prec = int(sys.argv[1]), sys.argv[2]
dev = torch.device("cuda", 0)
dt = torch.bfloat16 if prec == "bf16" else torch.float32
C, W, K, M = 256, 28, 3, 256
I = torch.rand(N, C, W, W, device=dev).to(dt)
F = (torch.rand(M, C, K, K, device=dev) * 2 - 1).to(dt)
O = torch.empty((N, M, W - 2, W - 2), device=dev)
for _ in range(3): conv.conv_multi_batched_ex(I, N, C, W, W, F, K, M, O, prec)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 1024)()
conv.load().conv_diag_stamps(buf)
t = np.array(list(buf), dtype=np.int64).reshape(4, 256)
P, G0, G1, Mm = t
n = 120
t0 = P[0]
print(f"N={N} {prec}: iterations 0..{n-1}, cycles from the first producer issue")
print("M[i] - M[i-1] (MMA issue interval):", np.diff(Mm[:n]).tolist())
print("G0 - P (patch TMA latency):", (G0 - P)[:n].tolist())
print("G1 - G0 (gather build):", (G1 - G0)[:n].tolist())
print("M - G1 (MMA issue after gather arrive; B wait or MMA queue):", (Mm - G1)[:n].tolist())
for ns in (5, 6):
    print(f"P[i] - M[i-{ns}] (producer wake after the MMA that frees the stage was issued):", (P[ns:n] - Mm[:n - ns]).tolist())
