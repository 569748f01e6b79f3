"""Turn the round's ncu captures into committed summaries under profiles/:
   launches_<r>.csv  -> profiles/launches_<r>.csv (per-launch time + DRAM bytes, labelled)
                     -> profiles/traffic.json (DRAM bytes per launch per kernel group)
   full_*.ncu-rep    -> profiles/ncu_full_<name>_<r>.txt (key metrics)"""
import csv, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import summary, KEYS

r = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = os.path.join(ROOT, "gpurun_out", f"launches_{r}.csv")
rows = list(csv.reader(open(src)))
hdr = [i for i, x in enumerate(rows) if x and x[0] == "ID"][0]
H = rows[hdr]
ki, mi, vi, ui = H.index("Kernel Name"), H.index("Metric Name"), H.index("Metric Value"), H.index("Metric Unit")
idi = H.index("ID")
per = {}
for x in rows[hdr + 1:]:
    if len(x) <= vi:
        continue
    d = per.setdefault(int(x[idi]), {"kernel": x[ki]})
    v = float(x[vi].replace(",", ""))
    u = x[ui]
    if x[mi] == "gpu__time_duration.sum":
        d["us"] = v / 1e3 if u in ("ns", "nsecond") else (v if u in ("us", "usecond") else v * 1e3)
    elif x[mi].startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}.get(u, 1)
        d[x[mi]] = v * scale
calls = bench.suite()
pk = bench.peaks()
from paper_2212_00404_b200 import conv
# one call of the hot path is plan["launches"] kernels (KM-SIMT workspace split:
# main + reduce; KM-TC/G: im2col + GEMM): fold them into one row per call
launches = sorted(per.items())
merged, pos = [], 0
for c in calls:
    pl = (conv.plan_single(c["Wx"], c["Wy"], c["K"], c["M"]) if c["kind"] == "single"
          else conv.plan_multi(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], c["prec"]))
    parts = [d for _, d in launches[pos:pos + pl["launches"]]]
    pos += pl["launches"]
    m = {"kernel": " + ".join(d["kernel"].split("(")[0][:40] for d in parts)}
    for key in ("us", "dram__bytes_read.sum", "dram__bytes_write.sum"):
        m[key] = sum(d.get(key, 0) for d in parts)
    merged.append((len(merged), m))
out_rows, groups = [], {}
for (i, d), c in zip(merged, calls):
    b = bench.roof_for(c, pk)[0]
    key = f"{c['kernel']}/{b}"
    traffic = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    out_rows.append([c["label"], key, d["kernel"][:90], round(d.get("us", 0), 3), int(traffic),
                     int(c["bytes_alg"])])
    g = groups.setdefault(key, {"us": 0.0, "traffic": 0.0, "alg": 0.0, "n": 0})
    g["us"] += d.get("us", 0); g["traffic"] += traffic; g["alg"] += c["bytes_alg"]; g["n"] += 1
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", f"launches_{r}.csv"), "w", newline="") as fh:
    w = csv.writer(fh)
    w.writerow(["layer", "group", "kernel", "ncu_us_cold", "dram_bytes", "alg_bytes"])
    w.writerows(out_rows)
tot = sum(g["us"] for g in groups.values())
traffic = {k: int(g["traffic"] / g["n"]) for k, g in groups.items()}
json.dump(traffic, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
# the bench's live per-group shares (profiles/bench_<r>.json), side by side
live = {}
bj = os.path.join(ROOT, "profiles", f"bench_{r}.json")
if os.path.exists(bj):
    live = {k: v["share"] for k, v in json.load(open(bj)).get("kernels", {}).items()}
big = [k for k, g in groups.items() if g["us"] / g["n"] >= 8.0]          # launches well above the launch floor
tot_big = sum(groups[k]["us"] for k in big)
live_big = sum(live.get(k, 0.0) for k in big)
with open(os.path.join(ROOT, "profiles", f"launch_shares_{r}.txt"), "w") as fh:
    fh.write(f"# ncu launch list of one bench step ({len(out_rows)} launches), cold-cache + serialised\n")
    fh.write("# 'live' = the bench's share of the PDL-chained step (bench_<r>.json).  ncu serialises\n"
             "# launches and flushes caches, so tiny launches (KS on 7-56 px maps: ~2 us live) cost\n"
             "# 5-7 us each here; among groups averaging >= 8 us per ncu launch the shares are\n"
             "# compared renormalised over those groups ('ncu big' vs 'live big').\n")
    fh.write(f"# {'group':24s} {'launches':>8s} {'ncu us':>10s} {'share':>7s} {'live':>7s} {'ncu big':>8s} {'live big':>8s}"
             f" {'dram/launch':>12s} {'alg/launch':>12s}\n")
    for k, g in sorted(groups.items(), key=lambda kv: -kv[1]["us"]):
        lv = live.get(k)
        nb = f"{g['us'] / tot_big:8.3f}" if k in big and tot_big else f"{'':8s}"
        lb = f"{lv / live_big:8.3f}" if k in big and lv is not None and live_big else f"{'':8s}"
        fh.write(f"  {k:24s} {g['n']:8d} {g['us']:10.1f} {g['us'] / tot:7.3f} "
                 f"{(f'{lv:7.3f}' if lv is not None else ' ' * 7)} {nb} {lb} "
                 f"{g['traffic'] / g['n']:12.0f} {g['alg'] / g['n']:12.0f}\n")
print(open(os.path.join(ROOT, "profiles", f"launch_shares_{r}.txt")).read())
for f in sorted(os.listdir(os.path.join(ROOT, "gpurun_out"))):
    if f.startswith("full_") and f.endswith(f"_{r}.ncu-rep"):
        name, s = summary(os.path.join(ROOT, "gpurun_out", f))
        extra = subprocess.run(["ncu", "-i", os.path.join(ROOT, "gpurun_out", f), "--page", "raw", "--csv"],
                               capture_output=True, text=True).stdout
        rr = list(csv.reader(extra.splitlines()))
        want = ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
        raw = {}
        if len(rr) > 2:
            for i, n in enumerate(rr[0]):
                if n in want:
                    raw[n] = f"{rr[2][i]} {rr[1][i]}"
        out = os.path.join(ROOT, "profiles", f"ncu_{f[:-8]}.txt")
        with open(out, "w") as fh:
            fh.write(f"{name}\n")
            for k in KEYS:
                if k in s:
                    fh.write(f"  {k:40s} {s[k]}\n")
            for k, v in raw.items():
                fh.write(f"  {k:40s} {v}\n")
        print(open(out).read())
