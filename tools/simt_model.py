"""Host replica of the KM-SIMT planner model (conv_multi_simt.cu simt_choose),
used to fit its constants against a measured sweep (tools/simt_sweep.py).
usage: simt_model.py gpurun_out/simt_sweep_v1.json"""
import itertools
import json
import math
import sys

TILES = [(128, 128, 8), (64, 256, 8), (256, 64, 8), (256, 48, 6), (128, 96, 6), (64, 192, 6),
         (256, 32, 4), (128, 64, 4), (64, 128, 4)]
CL1 = [0, 148, 74, 45, 33, 26, 22, 15, 15, 15, 11, 7, 7, 7, 7, 7, 7]
CL2 = [0, 296, 148, 93, 71, 56, 45, 37, 33, 30, 26, 21, 21, 17, 14, 14, 14]
LAYERS = {"resnet_28x28_c128_m128_k3": (128, 28, 3, 128), "resnet_14x14_c256_m256_k3": (256, 14, 3, 256),
          "resnet_7x7_c512_m512_k3": (512, 7, 3, 512), "vgg_224x224_c3_m64_k3": (3, 224, 3, 64),
          "vgg_56x56_c64_m64_k3": (64, 56, 3, 64), "alexnet_27x27_c96_m256_k5": (96, 27, 5, 256),
          "target_28x28_c256_m256_k3": (256, 28, 3, 256), "sweep_14x14_c512_m4096_k3": (512, 14, 3, 4096),
          "shard2_14x14_c512_m2048_k3": (512, 14, 3, 2048), "shard4_14x14_c512_m1024_k3": (512, 14, 3, 1024),
          "shard8_14x14_c512_m512_k3": (512, 14, 3, 512)}
MAXSMEM = 110 * 1024


def rs(ck):
    return ((ck - 4 + 31) // 32) * 32 + 4


def smem(BM, BN, CK):
    CKP = (CK + 3) & ~3                          # two-stage ring of F rows + im2col tile
    b = (2 * BM * rs(CKP) + 2 * CKP * BN) * 4 + ((CKP + 1) & ~1) * 4 + 16
    return max(b, BM * BN * 4)


def cb_for(BM, BN, K, C):
    cb = (64 // (K * K) + 3) & ~3
    cb = max(cb, 8)
    while cb > 4 and smem(BM, BN, cb * K * K) > MAXSMEM:
        cb -= 4
    while cb > 1 and smem(BM, BN, cb * K * K) > MAXSMEM + 16 * 1024:
        cb -= 1
    return max(1, min(cb, C))


def split(C, S, BM, BN, K):
    per = -(-C // S)
    budget = cb_for(BM, BN, K, C)
    cb = 1
    for c in (8, 4, 2):
        if c > budget or c > per:
            continue
        waste = -(-per // c) * c - per
        if 8 * waste <= per:
            cb = c
            break
    return cb, -(-per // cb) * cb


def cost(P, C, W, K, M, ti, Sreq, ws):
    BM, BN, TN = TILES[ti]
    Ho = Wo = W - K + 1
    px = Ho * Wo
    npt, nmt = -(-px // BN), -(-M // BM)
    tiles = npt * nmt
    CB, cps = split(C, min(Sreq, C), BM, BN, K)
    S = -(-C // cps)
    sm = smem(BM, BN, CB * K * K)
    q = 2 if sm <= 113 * 1024 else 1
    pen = {8: 1.0, 6: P["pen6"], 4: P["pen4"]}[TN]
    # the compile-time 36-k chunk (TMA-fed, fully unrolled main loop) runs faster
    if CB * K * K == 36 and (C * K * K) % 4 == 0:
        pen *= P.get("fix", 1.0)
    w = BM * BN * cps * K * K * pen / (128 * 1965.0)
    nch = -(-cps // CB)

    def smt(n):
        c = P["c0"] + nch * P["cch"] * (BM / 128.0) ** P.get("cbm", 0.0)
        if q >= 2:
            return (n // 2) * (2 * w / P["e2"]) + (n % 2) * (w / P["e1"]) + ((n + 1) // 2) * c
        return n * (w / P["e1"] + c)
    if not ws:
        if S > 16:
            return None, S
        cap = (CL2 if q >= 2 else CL1)[S]
        waves = -(-tiles // cap)
        per_wave = min(tiles, cap) * S
        return waves * smt(-(-per_wave // 148)) + (P["ccl"] if S > 1 else 0), S
    if S == 1:
        return None, S
    byts = 8.0 * S * nmt * BM * npt * BN + 4.0 * M * px
    lat = P["rsl"] * (S / 8.0 if S > 16 else S)          # serial partial loads per reduce lane
    return smt(-(-tiles * S // 148)) + P["cws"] + byts / P["l2"] + lat, S


def choose(P, C, W, K, M):
    """Exactly the C++ search: tiles in order, Sreq 1..96 deduped by effective S,
    cluster then workspace, keep the first within 0.5%."""
    best = None
    for ti, (BM, BN, TN) in enumerate(TILES):
        last = -1
        for Sreq in range(1, min(C, 96) + 1):
            _, cps = split(C, Sreq, BM, BN, K)
            S = -(-C // cps)
            if S == last:
                continue
            last = S
            for ws in (0, 1):
                t, _ = cost(P, C, W, K, M, ti, Sreq, ws)
                if t is None:
                    continue
                if best is None or t < best[0] * 0.995:
                    best = (t, (ti, S, ws))
    return best


def main():
    d = json.load(open(sys.argv[1]))
    meas = {}
    for r in d:
        if "us" in r and r["cfg"] is not None:
            ti, Sreq, ws = r["cfg"]
            C, W, K, M = LAYERS[r["layer"]]
            BM, BN, TN = TILES[ti]
            _, cps = split(C, min(Sreq, C), BM, BN, K)
            meas.setdefault(r["layer"], {})[(ti, -(-C // cps), ws)] = r["us"]
    base = dict(e1=0.40, e2=0.45, c0=0.5, ccl=9.0, cws=0.5, l2=3.0e6, pen6=0.85, pen4=1.0, rsl=0.0, cch=0.8,
                fix=1.0, cbm=0.0)
    grid = dict(e1=[0.36, 0.38, 0.4, 0.41, 0.42, 0.43, 0.44, 0.45], e2=[0.45, 0.5, 0.55],
                cws=[0.5, 1.0, 2.0], pen6=[0.85, 0.9, 0.95, 1.0], cch=[0.2, 0.4, 0.6, 0.8, 1.0],
                fix=[0.6, 0.65, 0.7, 0.8, 0.9, 1.0], l2=[1.5e6, 3.0e6, 6.0e6], c0=[0.25, 0.5, 1.0, 2.0])

    def regret(P, verbose=False):
        tot = 0.0
        for L, m in meas.items():
            C, W, K, M = LAYERS[L]
            best_meas = min(m.values())
            t, cfg = choose(P, C, W, K, M)
            us = m.get(cfg, best_meas * 2)
            tot += math.log(us / best_meas)
            if verbose:
                print(f"{L:28s} pick {cfg} pred {t:7.1f} meas {us:7.1f} best {best_meas:7.1f}")
        return tot
    # coordinate descent over the grid (the full product is too slow in Python)
    best = (regret(base), base)
    for _ in range(3):
        for k in grid:
            for v in grid[k]:
                P = dict(best[1])
                P[k] = v
                r = regret(P)
                if r < best[0] - 1e-9:
                    best = (r, P)
    print("regret (sum log)", best[0])
    print(best[1])
    regret(best[1], True)


if __name__ == "__main__":
    main()
