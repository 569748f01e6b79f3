"""Top SASS instructions by executed count / stall samples from an ncu source page csv."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia = hdr.index("Address"); isrc = hdr.index("Source"); ie = hdr.index("Instructions Executed")
ist = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ie] or 0), int(r[ist] or 0), r[ia], r[isrc]))
    except (ValueError, IndexError):
        pass
tot_e = sum(d[0] for d in data); tot_s = sum(d[1] for d in data)
print("total executed", tot_e, "stall samples", tot_s)
key = 1 if len(sys.argv) > 2 and sys.argv[2] == "stall" else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
for d in sorted(data, key=lambda d: -d[key])[:n]:
    print(f"{d[0]:10d} {d[1]:6d}  {d[2]}  {d[3][:90]}")
