"""Write profiles/ncu_<name>_<tag>.txt summaries (details page key lines + the
raw pipe / DRAM metrics) for every gpurun_out/full_*_<tag>.ncu-rep, and fold
the per-launch DRAM bytes into profiles/traffic.json (keys configs4/<kernel>/n1).
usage: ncu_round_summary.py <tag>"""
import csv, glob, io, json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summary, KEYS

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size"]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {n: (v[i] + (" " + u[i] if u[i] else "")) for i, n in enumerate(h)
            if n in RAW or ("pipe_tensor" in n and n.endswith(".avg.pct_of_peak_sustained_active"))}


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def to_bytes(s):
    val, unit = s.split()
    return float(val) * SCALE[unit]


tag = sys.argv[1]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tr_path = os.path.join(root, "profiles", "traffic.json")
traffic = json.load(open(tr_path)) if os.path.exists(tr_path) else {}
KMAP = {"simt": "KM-SIMT", "tcg_tf32": "KM-TC/G-tf32", "tcg_bf16": "KM-TC/G-bf16"}
for p in sorted(glob.glob(os.path.join(root, "gpurun_out", f"full_*_{tag}.ncu-rep"))):
    name = os.path.basename(p)[len("full_"):-len(f"_{tag}.ncu-rep")]
    kname, s = summary(p)
    r = raw(p)
    lines = [kname[:160]] + [f"  {k:38s} {s[k]}" for k in KEYS if k in s] + [f"  {k} {v}" for k, v in sorted(r.items())]
    with open(os.path.join(root, "profiles", f"ncu_full_{name}_{tag}.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    if name in KMAP:
        try:
            traffic[f"configs4/{KMAP[name]}/n1"] = int(to_bytes(r["dram__bytes_read.sum"]) +
                                                       to_bytes(r["dram__bytes_write.sum"]))
        except (KeyError, ValueError):
            pass
    print("\n".join(lines))
json.dump(traffic, open(tr_path, "w"), indent=1)
