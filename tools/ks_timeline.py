"""KS per-CTA timeline (B200CONV_KS_DBG=1 globaltimer stamps) for chosen layers,
launched back to back.  usage: ks_timeline.py <Wx> <K> <M> [...]
(B200CONV_TL_C=3: run the C = 3 multi-channel variant, KS-C3, instead)"""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2212_00404_b200 import conv
from paper_2212_00404_b200 import build as _b
conv.load(_b.build(diag=True))       # the -DB200CONV_DIAG library (stamps / DBG switches)
dev = torch.device("cuda", 0)
args = [int(a) for a in sys.argv[1:]]
lib = conv.load()
for i in range(0, len(args), 3):
    W, K, M = args[i:i + 3]
    C3 = os.environ.get("B200CONV_TL_C") == "3"
    I = torch.from_numpy(synth.uniform01(1, (3, W, W) if C3 else (W, W))).to(dev)
    F = torch.from_numpy(synth.uniform_pm1(2, (M, 3, K, K) if C3 else (M, K, K))).to(dev)
    Os = [torch.empty((M, W - K + 1, W - K + 1), device=dev) for _ in range(8)]
    os.environ["B200CONV_KS_DBG"] = "0"
    for O in Os: (conv.conv_multi_ex(I, 3, W, W, F, K, M, O) if C3 else conv.conv_single_ex(I, W, W, F, K, M, O))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for O in Os: (conv.conv_multi_ex(I, 3, W, W, F, K, M, O) if C3 else conv.conv_single_ex(I, W, W, F, K, M, O))
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / len(Os)
    os.environ["B200CONV_KS_DBG"] = "1"
    for O in Os: (conv.conv_multi_ex(I, 3, W, W, F, K, M, O) if C3 else conv.conv_single_ex(I, W, W, F, K, M, O))
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 4096)()
    lib.conv_diag_ks_stamps(buf)
    G = (conv.plan_multi(3, W, W, K, M) if C3 else conv.plan_single(W, W, K, M))["grid_x"]
    tu = np.array(list(buf), dtype=np.uint64).reshape(1024, 4)[:min(G, 1024)]
    smid = (tu[:, 3] & np.uint64(255)).astype(np.int64)
    tu[:, 3] >>= np.uint64(8)
    tu[:, 3] |= tu[:, 0] & ~np.uint64((1 << 56) - 1)     # restore the top bits
    t = tu.astype(np.int64)
    t0 = t[:, 0].min()
    r = (t - t0) / 1e3
    q = lambda c: " ".join(f"{v:6.2f}" for v in np.percentile(r[:, c], [0, 50, 90, 100]))
    print(f"== {W}x{W} K{K} M{M}: {G} CTAs, eager b2b {us:.2f} us/launch (pctl 0/50/90/100, us)")
    print("  start    ", q(0)); print("  pdl-wait ", q(1)); print("  staged   ", q(2)); print("  done     ", q(3))
    dur = r[:, 3] - r[:, 2]
    print("  busy     ", " ".join(f"{v:6.2f}" for v in np.percentile(dur, [0, 50, 90, 100])))
    per_sm = {}
    for sm, d, e in zip(smid, dur, r[:, 3]):
        per_sm.setdefault(int(sm), []).append((round(float(d), 2), round(float(e), 2)))
    ks = sorted(per_sm, key=lambda k: -max(e for _, e in per_sm[k]))
    print("  latest SMs:", [(k, per_sm[k]) for k in ks[:6]])
    print("  earliest SMs:", [(k, per_sm[k]) for k in ks[-4:]])
    cnt = np.bincount([len(v) for v in per_sm.values()])
    print("  CTAs per SM histogram:", cnt.tolist(), "SMs used", len(per_sm))
    os.environ["B200CONV_KS_DBG"] = "2"
    for O in Os: (conv.conv_multi_ex(I, 3, W, W, F, K, M, O) if C3 else conv.conv_single_ex(I, W, W, F, K, M, O))
    torch.cuda.synchronize()
    fb = (ctypes.c_ulonglong * 16)()
    lib.conv_diag_ks_fine(fb)
    f = np.array(list(fb)[:4], dtype=np.int64)
    print("  CTA0 warp0 unit0: taps %.3f us, compute %.3f us, stores %.3f us" % ((f[1] - f[0]) / 1e3, (f[2] - f[1]) / 1e3, (f[3] - f[2]) / 1e3))
