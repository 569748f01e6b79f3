"""KS-L plan checks that need no GPU (`-m "not gpu"`): for every shape the
planner accepts (the forced path, B200CONV_KS_FLAT=1), the shared memory it
requests covers what ks_flat_kernel stages (conv_single.cu, KS-L): the units
(filter group g, 64-float chunk c) dealt evenly over the warps of one wave of
2 CTAs per SM; a CTA spanning one or two groups stages the input rows of its
chunk ranges as two blocks (block B after block A's extent, 16-B aligned), a
CTA spanning three or more stages the whole map; every valid output pixel's
3-row window lies in its block.  This is the host planner checked against the
kernel's indexing, restated from the kernel's comments."""
import random

from paper_2212_00404_b200 import conv

SMS = 148          # num_sms() without a device


def head(g, P, HW):
    """First 128-B-aligned flat index of the planes of filter group g."""
    return (32 - ((g % P) * (HW & 31)) % 32) % 32


def rows(h, c0, c1, HW, Wo, Wy):
    p_lo, p_hi = max(0, h + 64 * (c0 - 1)), min(HW - 1, h + 64 * c1 - 1)
    lo = p_lo // Wo
    return lo, max(lo, min(Wy, p_hi // Wo + 3))


def staged_floats_ok(Wx, Wy, M, R, smem_bytes):
    Wo, Ho = Wx - 2, Wy - 2
    HW = Ho * Wo
    g, b = 32, HW & 31
    while b:
        g, b = b, g % b
    P = 32 // g
    NG = -(-M // (R * P)) * P
    nch = 1 + -(-HW // 64)
    U = NG * nch
    G = min(-(-U // 8), (2 if R == 8 else 3) * SMS)
    NW = G * 8
    ub, ur = U // NW, U % NW
    have = smem_bytes // 4
    for cta in range(G):
        cw = cta * 8
        u0, u1 = cw * ub + min(cw, ur), (cw + 8) * ub + min(cw + 8, ur)
        if u0 >= u1:
            continue
        gA, gB = u0 // nch, (u1 - 1) // nch
        if gB > gA + 1:
            rA, rB = (0, Wy), (0, 0)
        else:
            cA0, cA1 = u0 - gA * nch, (u1 - gA * nch if gB == gA else nch)
            rA = rows(head(gA, P, HW), cA0, cA1, HW, Wo, Wy)
            rB = rows(head(gB, P, HW), 0, u1 - gB * nch, HW, Wo, Wy) if gB != gA else (0, 0)
            # every valid pixel's window rows inside its block
            for gg, c0, c1, (lo, hi) in [(gA, cA0, cA1, rA)] + ([(gB, 0, u1 - gB * nch, rB)] if gB != gA else []):
                h = head(gg, P, HW)
                for c in range(c0, c1):
                    for lane in (0, 31):
                        p = h + 64 * (c - 1) + 2 * lane
                        if 0 <= p < HW and not (lo <= p // Wo and p // Wo + 3 <= hi):
                            return False
        for pad in range(4):
            off_b = (pad + (rA[1] - rA[0]) * Wx + 3 + 4) & ~3
            need = max(off_b + pad + (rB[1] - rB[0]) * Wx + 4, pad + 3 * Wx + 4)
            if gB == gA + 1:
                need = max(need, off_b + pad + 3 * Wx + 4)
            if need > have:
                return False
    return True


def test_ksl_plans_cover_the_staged_rows(monkeypatch):
    monkeypatch.setenv("B200CONV_KS_FLAT", "1")
    rng = random.Random(5)
    shapes = [(224, 224, 256), (224, 224, 1024), (14, 14, 32), (10, 10, 4), (12, 9, 7), (66, 130, 9)]
    shapes += [(rng.randrange(4, 260, 2), rng.randrange(3, 240), rng.choice([1, 7, 32, 100, 256, 512]))
               for _ in range(120)]
    checked = 0
    for Wx, Wy, M in shapes:
        p = conv.plan_single(Wx, Wy, 3, M)
        if p["tile_n"] != -2:
            continue
        checked += 1
        assert p["grid_x"] <= 2 * SMS and p["smem_bytes"] <= 110 * 1024
        assert staged_floats_ok(Wx, Wy, M, p["tile_m"], p["smem_bytes"]), (Wx, Wy, M, p)
    assert checked > 60


def test_ksl_default_planner_scope(monkeypatch):
    monkeypatch.delenv("B200CONV_KS_FLAT", raising=False)
    assert conv.plan_single(224, 224, 3, 256)["tile_n"] == -2     # 888-B rows, large map, many filters
    assert conv.plan_single(226, 226, 3, 256)["tile_n"] > 0       # 896-B rows: whole lines
    assert conv.plan_single(224, 224, 3, 64)["tile_n"] > 0        # few filters: row-block kernel
    assert conv.plan_single(58, 58, 3, 256)["tile_n"] > 0         # small map: row-block kernel
    monkeypatch.setenv("B200CONV_KS_FLAT", "0")
    assert conv.plan_single(224, 224, 3, 256)["tile_n"] > 0
