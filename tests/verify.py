#!/usr/bin/env python
"""verify — run one convolution through the C ABI on the GPU and check it
against the fp64 oracle (SURVEY §8(b) "Verify CLI"; exit codes after SPEC.md
S:417 "0 success, 2 infeasible plan, 3 verification failure, 1 usage error").

Test infrastructure (it lives under tests/ because it calls oracle/):

    python tests/verify.py --mode multi --wx 14 --wy 14 --c 64 --k 3 --m 64 --precision tf32
    python tests/verify.py --mode single --wx 224 --wy 224 --k 3 --m 32 --seed 7

Inputs are synth.py's seeded recipe (I ~ U[0,1), F ~ U[-1,1)); the check is
north_star's per-output |O - O_oracle| <= tau * sum|I*F| (tau 1e-5 FP32,
2e-3 TF32, 1e-2 BF16); outputs beyond --max-full are compared on a seeded
sample of --samples indices (oracle.conv_multi_sampled, same arithmetic).
Prints one line: PASS/FAIL, max err/A, the plan.
"""
from __future__ import annotations

import argparse
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

TAU = {"fp32": 1e-5, "tf32": 2e-3, "bf16": 1e-2}
EXIT_OK, EXIT_USAGE, EXIT_INFEASIBLE, EXIT_FAIL = 0, 1, 2, 3


def parse(argv):
    ap = argparse.ArgumentParser(prog="verify", description=__doc__.split("\n\n")[0])
    ap.add_argument("--mode", choices=["single", "multi"], required=True)
    ap.add_argument("--wx", type=int, required=True)
    ap.add_argument("--wy", type=int, required=True)
    ap.add_argument("--c", type=int, default=1)
    ap.add_argument("--k", type=int, required=True)
    ap.add_argument("--m", type=int, required=True)
    ap.add_argument("--precision", choices=list(TAU), default="fp32")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--samples", type=int, default=20000)
    ap.add_argument("--max-full", type=int, default=4_000_000)
    return ap.parse_args(argv)


def main(argv=None) -> int:
    try:
        a = parse(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_USAGE
    if a.mode == "single" and (a.c != 1 or a.precision != "fp32"):
        print("usage: --mode single is C = 1, FP32", file=sys.stderr)
        return EXIT_USAGE
    if min(a.wx, a.wy, a.c, a.k, a.m) < 1 or a.k > min(a.wx, a.wy):
        print(f"infeasible: K={a.k} > min(Wx={a.wx}, Wy={a.wy}) or a dimension < 1 (S:104)")
        return EXIT_INFEASIBLE
    import numpy as np
    import torch

    import oracle
    import synth
    from paper_2212_00404_b200 import conv

    I = synth.uniform01(synth.SEED_I + a.seed, (a.c, a.wy, a.wx))
    F = synth.uniform_pm1(synth.SEED_F + a.seed, (a.m, a.c, a.k, a.k))
    dt = torch.bfloat16 if a.precision == "bf16" else torch.float32
    Id, Fd = torch.from_numpy(I).cuda().to(dt), torch.from_numpy(F).cuda().to(dt)
    try:
        if a.mode == "single":
            O = conv.single(Id[0].contiguous(), Fd[:, 0].contiguous())
            plan = conv.plan_single(a.wx, a.wy, a.k, a.m)
        else:
            O = conv.multi(Id, Fd, a.precision)
            plan = conv.plan_multi(a.c, a.wx, a.wy, a.k, a.m, a.precision)
    except conv.ConvError as e:
        print(f"infeasible: {e}")
        return EXIT_INFEASIBLE if e.status == 1 else EXIT_FAIL
    Og = O.cpu().numpy().astype(np.float64).ravel()
    n = Og.size
    if n <= a.max_full:
        Oo, A = oracle.conv_multi(I, F)
        Oo, A, Og_s = Oo.ravel(), A.ravel(), Og
    else:
        rng = np.random.default_rng(a.seed)
        idx = np.unique(np.concatenate([rng.integers(0, n, a.samples), np.arange(256), np.arange(n - 256, n)]))
        Oo, A = oracle.conv_multi_sampled(I, F, idx)
        Og_s = Og[idx]
    err = np.abs(Og_s - Oo)
    ok = bool(np.all(err <= TAU[a.precision] * A) and np.all(Og_s[A == 0] == 0))
    rel = float((err / np.where(A > 0, A, 1)).max()) if err.size else 0.0
    kname = {0: "KS", 1: "KM-SIMT", 2: "KM-TC", 3: "KM-TC/G", 4: "KS-C3"}.get(plan["kernel"], "?")
    print(f"{'PASS' if ok else 'FAIL'}: max err/A {rel:.3g} (tau {TAU[a.precision]:g}), "
          f"{err.size} outputs checked, kernel {kname}, plan {plan}")
    return EXIT_OK if ok else EXIT_FAIL


if __name__ == "__main__":
    sys.exit(main())
