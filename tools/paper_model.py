"""The paper's latency-hiding model (§2.2) re-derived for
B200, applied to every bench layer (analysis only: the
library's planners are the measured models in the kernels).

Paper: N_FMA = latency x N_cores x 2 (the "x2" is the FMA counted
as two operations, reading Q15) and V_s = (bytes/clock) x latency:
a CTA set that executes >= N_FMA FMAs per SM per data set hides the global
latency by prefetching (method 1); otherwise the data in flight must reach
V_s (method 2).  B200 constants: 148 SMs x 128 FP32 lanes, HBM 6554 GB/s
(MEASURED_PEAKS.json) at 1965 MHz, DRAM latency 577 cycles (B300_MICROARCH.md,
MLP = 1), 227 KB shared memory per CTA, 2048 threads per SM.

usage: python tools/paper_model.py   (CPU only; prints a table)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench

LAT, SMS, LANES, CLK = 577, 148, 128, 1.965e9
pk = bench.peaks()
BPC = pk["hbm_gbs"] * 1e9 / CLK                       # bytes per clock, chip
N_FMA = LAT * LANES                                   # FMAs per SM to cover one latency (1 FMA / lane / clk)
V_S = BPC * LAT                                       # bytes in flight, chip
print(f"B200: N_FMA = {N_FMA:,} FMAs per SM per data set (paper's x2 convention: {2 * N_FMA:,});"
      f" V_s = {V_S / 1e6:.2f} MB in flight = {V_S / SMS / 1024:.1f} KB per SM"
      f" = {V_S / SMS / 16:.0f} 16-B loads per SM ({V_S / SMS / 4:.0f} 4-B loads > 2048 threads:"
      f" the paper's one-word-per-thread rule cannot cover HBM latency on B200 — 16-B vectors / TMA bulk copies do)")
rows = []
for c in bench.suite_calls(1, 0):
    fma = c["flop"] / 2
    per_sm = fma / SMS
    method = "1 (prefetch / compute)" if per_sm >= N_FMA else "2 (bandwidth / latency)"
    rows.append((c["label"], fma, per_sm / N_FMA, method, bench.roof(c, c["prec"], "KS" if c["kind"] == "single" else "KM", pk, SMS)[0]))
print(f"{'layer':38s} {'FMA':>12s} {'FMA/SM / N_FMA':>15s}  paper's method           roofline bound")
for r in rows:
    if r[0].startswith("single") and not r[0].startswith(("single_224", "single_56x56_k7")):
        continue
    print(f"{r[0]:38s} {r[1]:12.3e} {r[2]:15.2f}  {r[3]:24s} {r[4]}")
n1 = sum(1 for r in rows if r[3].startswith("1"))
print(f"\n{n1} of {len(rows)} calls of the step have >= N_FMA FMAs per SM (method 1); the rest are latency/bandwidth bound")
