"""NEXT-4 A/B: the paper's latency-model planner (B200CONV_PLANNER=paper) vs
the fitted thresholds (=fitted) on every single-channel sweep layer whose
decision differs, plus the multi-channel FP32 layers (KM-SIMT ring depth).
Each layer: 12 launches back to back in a CUDA graph with rotating outputs,
best of 5 replays, the two planners interleaved 3 times; median reported.
usage: planner_ab.py > profiles/planner_ab_<tag>.txt"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
from paper_2212_00404_b200 import conv

dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
n_fma = conv.latency_model("b200")["n_fma"]


def timeit(fn, reps=12):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        s.synchronize()
        g.capture_begin()
        for i in range(reps):
            fn(i)
        g.capture_end()
        g.replay()
        s.synchronize()
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s); g.replay(); b.record(s); s.synchronize()
            best = min(best, 1e3 * a.elapsed_time(b) / reps)
    return best


print(f"# N_FMA (B200) = {n_fma:.0f} FMAs per SM; paper rule: method 2 (1-row KS blocks) when "
      f"M*Ho*Wo*K^2/148 < N_FMA")
print(f"{'layer':36s} {'FMA/SM':>9s} {'method':>6s} {'paper us':>9s} {'fitted us':>9s}  plan(paper) / plan(fitted)")
tot = {"paper": 0.0, "fitted": 0.0}
for c in bench.suite_calls(1, 0):
    if c["prec"] != "fp32":
        continue
    single = c["kind"] == "single"
    if single:
        if c["K"] < 3:
            continue
        paper_small = c["M"] * c["Ho"] * c["Wo"] * c["K"] ** 2 / 148 < n_fma
        fitted_small = c["Ho"] <= (32 if c["K"] == 3 else 16)
        if paper_small == fitted_small:
            continue
    I = torch.from_numpy(synth.uniform01(synth.SEED_I, (c["C"], c["Wy"], c["Wx"]))).to(dev)
    F = torch.from_numpy(synth.uniform_pm1(synth.SEED_F, (c["M"], c["C"], c["K"], c["K"]))).to(dev)
    if single:
        I, F = I[0].contiguous(), F[:, 0].contiguous()
    Os = [torch.empty((c["M"], c["Ho"], c["Wo"]), device=dev) for _ in range(6)]
    res, plans = {"paper": [], "fitted": []}, {}
    for _ in range(3):
        for mode in ("paper", "fitted"):
            os.environ["B200CONV_PLANNER"] = mode
            if single:
                fn = lambda j: conv.conv_single_ex(I, c["Wx"], c["Wy"], F, c["K"], c["M"], Os[j % 6], s.cuda_stream)
                plans[mode] = conv.plan_single(c["Wx"], c["Wy"], c["K"], c["M"])
            else:
                fn = lambda j: conv.conv_multi_ex(I, c["C"], c["Wx"], c["Wy"], F, c["K"], c["M"], Os[j % 6], "fp32",
                                                  s.cuda_stream)
                plans[mode] = conv.plan_multi(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], "fp32")
            res[mode].append(timeit(fn))
    fma = c["flop"] / 2 / 148
    mp, mf = statistics.median(res["paper"]), statistics.median(res["fitted"])
    tot["paper"] += mp
    tot["fitted"] += mf
    pp, pf = plans["paper"], plans["fitted"]
    print(f"{c['label']:36s} {fma:9.0f} {1 if fma >= n_fma else 2:6d} {mp:9.2f} {mf:9.2f}  "
          f"{pp['grid_x']}x{pp['tile_n']} / {pf['grid_x']}x{pf['tile_n']}", flush=True)
os.environ.pop("B200CONV_PLANNER", None)
print(f"# total: paper {tot['paper']:.2f} us, fitted {tot['fitted']:.2f} us")
