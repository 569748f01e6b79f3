"""Small invocations of every kernel of the library, for compute-sanitizer
(tools/sanitize.sh): KS, KS-C3, KM-SIMT (cluster and workspace splits, batch,
stride), KM-TC (implicit: split-K over L2 / DSMEM, persistent batch), KM-TC/G
(im2col + GEMM, strided), the pad / pad-rows / split-K reduce kernels.  Each
result is compared with torch's CPU float64 conv2d (loose bound: the point here
is the sanitizer's verdict, parity lives in tests/)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as Fn

import synth
from paper_2212_00404_b200 import conv

dev = torch.device("cuda", 0)
fails = 0


def check(name, O, I, F, pad=0, stride=1):
    global fails
    ref = Fn.conv2d(I.double().cpu(), F.double().cpu(), padding=pad, stride=stride)
    err = float((O.double().cpu() - ref).abs().max() / (ref.abs().max() + 1e-30))
    ok = err < 2e-2
    fails += not ok
    print(f"{'ok ' if ok else 'BAD'} {name:48s} rel err {err:.2e}", flush=True)


def t(a):
    return torch.from_numpy(a).to(dev)


def multi(C, W, K, M, prec, env=None, N=None, pad=0, stride=1, name=""):
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        dt = torch.bfloat16 if prec == "bf16" else torch.float32
        n = N or 1
        I = t(synth.uniform01(3, (n, C, W, W))).to(dt)
        F = t(synth.uniform_pm1(4, (M, C, K, K))).to(dt)
        if N is None and pad == 0 and stride == 1:
            O = conv.multi(I[0].contiguous(), F, prec)[None]
        elif stride == 1 and pad == 0:
            O = conv.multi_batched(I, F, prec)
        elif stride == 1:
            O = conv.multi_padded(I, F, pad, prec)
        else:
            O = conv.multi_strided(I, F, stride, pad, prec)
        torch.cuda.synchronize()
        check(f"{name} C{C} W{W} K{K} M{M} N{n} p{pad} s{stride} {prec}", O, I.float(), F.float(), pad, stride)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


# KS (single channel): K = 1 / 3 / 5 / 7, small-map and band variants
for W, K, M in [(32, 3, 4), (20, 1, 8), (40, 3, 16), (17, 5, 8), (30, 7, 4), (9, 3, 5)]:
    I, F = t(synth.uniform01(1, (W, W))), t(synth.uniform_pm1(2, (M, K, K)))
    check(f"KS W{W} K{K} M{M}", conv.single(I, F)[None], I[None, None], F[:, None])
I, F = t(synth.uniform01(1, (21, 21))), t(synth.uniform_pm1(2, (6, 3, 3)))
check("KS padded p1", conv.single_padded(I, F, 1)[None], I[None, None].float(), F[:, None], 1)
check("KS strided s2 p1", conv.single_strided(I, F, 2, 1)[None], I[None, None], F[:, None], 1, 2)
# KS-L (line-aligned flat chunks), forced on small maps of several alignment periods
os.environ["B200CONV_KS_FLAT"] = "1"
for W, H, M in [(30, 30, 12), (12, 9, 7), (58, 20, 20)]:
    I, F = t(synth.uniform01(1, (H, W))), t(synth.uniform_pm1(2, (M, 3, 3)))
    check(f"KS-L W{W}x{H} M{M}", conv.single(I, F)[None], I[None, None], F[:, None])
os.environ.pop("B200CONV_KS_FLAT")
# KS-C3 stems
for prec in ("fp32", "tf32", "bf16"):
    multi(3, 40, 3, 16, prec, name="KS-C3")
# KM-SIMT: every split mode
multi(32, 14, 3, 48, "fp32", {"B200CONV_SIMT_FORCE": "0,1,0"}, name="KM-SIMT nosplit")
multi(32, 14, 3, 48, "fp32", {"B200CONV_SIMT_FORCE": "3,4,0"}, name="KM-SIMT cluster")
multi(32, 14, 3, 48, "fp32", {"B200CONV_SIMT_FORCE": "7,5,1"}, name="KM-SIMT workspace")
multi(64, 14, 3, 256, "fp32", {"B200CONV_SIMT_FORCE": "3,4,1"}, name="KM-SIMT 256x48 fixed-36 workspace")
multi(13, 11, 3, 21, "fp32", name="KM-SIMT odd (cp.async F)")
multi(16, 12, 3, 40, "fp32", N=3, name="KM-SIMT batch")
multi(16, 15, 3, 24, "fp32", N=2, pad=1, stride=2, name="KM-SIMT strided")
# KM-TC implicit and KM-TC/G
for prec in ("tf32", "bf16"):
    multi(64, 14, 3, 96, prec, {"B200CONV_GM": "0"}, name="KM-TC implicit")
    multi(64, 14, 3, 96, prec, {"B200CONV_GM": "0", "B200CONV_TC_SPLIT": "3"}, name="KM-TC split L2")
    multi(64, 14, 3, 96, prec, {"B200CONV_GM": "0", "B200CONV_TC_SPLIT": "3", "B200CONV_TC_DSMEM": "1"},
          name="KM-TC split DSMEM")
    multi(64, 28, 3, 64, prec, N=40, name="KM-TC persistent batch")
    multi(32, 28, 3, 256, prec, N=26, name="KM-TC persistent batch BN=256")
    multi(64, 7, 3, 256, prec, {"B200CONV_GM": "2"}, name="KM-TC/G")
    multi(64, 7, 3, 256, prec, {"B200CONV_GM": "2", "B200CONV_GM_SPLIT": "3"}, name="KM-TC/G split")
    multi(64, 7, 3, 256, prec, {"B200CONV_GM": "2", "B200CONV_GM_SPLIT": "3", "B200CONV_GM_DSMEM": "1"},
          name="KM-TC/G split DSMEM")
    multi(64, 14, 3, 512, prec, {"B200CONV_GM": "2", "B200CONV_GM_SPLIT": "4"}, name="KM-TC/G 144-px split")
    multi(3, 20, 3, 16, prec, N=2, pad=1, stride=2, name="KM-TC/G strided (pad rows)")
    multi(32, 9, 3, 40, prec, N=2, pad=1, name="KM-TC padded")
print("FAILS", fails)
sys.exit(1 if fails else 0)
