"""Summarise an .ncu-rep (details page) into key lines."""
import csv, io, subprocess, sys
KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Waves Per SM", "One or More Eligible", "Warp Cycles Per Issued Instruction",
        "Issued Instructions", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Mem Busy", "Max Bandwidth", "Mem Pipes Busy"]
def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ki = hdr.index("Kernel Name"); si = hdr.index("Section Name"); mi = hdr.index("Metric Name")
    ui = hdr.index("Metric Unit"); vi = hdr.index("Metric Value")
    seen = {}
    for r in rows[1:]:
        if len(r) <= vi: continue
        if r[mi] in KEYS and r[mi] not in seen:
            seen[r[mi]] = f"{r[vi]} {r[ui]}"
    name = rows[1][ki] if len(rows) > 1 else "?"
    return name, seen
if __name__ == "__main__":
    for p in sys.argv[1:]:
        name, s = summary(p)
        print(f"== {p}\n   {name[:110]}")
        for k in KEYS:
            if k in s: print(f"   {k:38s} {s[k]}")
