"""Stall-sample totals by reason and by basic-block execution count from an
ncu source page csv (ncu -i X --page source --csv --print-source sass).
usage: ncu_stalls.py <csv> [main_loop_exec_count]"""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ie = h.index("Instructions Executed")
cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
tot = defaultdict(int)
blk = defaultdict(lambda: [0, 0, 0])
for r in rows[2:]:
    try:
        e = int(r[ie] or 0)
    except (ValueError, IndexError):
        continue
    s = 0
    for i in cols:
        v = int(r[i] or 0)
        tot[h[i]] += v
        s += v
    blk[e][0] += 1; blk[e][1] += e; blk[e][2] += s
T = sum(tot.values())
for k in sorted(tot, key=lambda k: -tot[k]):
    if tot[k]:
        print(f"{k:28s} {tot[k]:6d} {tot[k] / T:6.3f}")
print("\nblocks by stall samples (exec count per instr, #instr, executed, samples)")
for e, (n, ex, s) in sorted(blk.items(), key=lambda x: -x[1][2])[:12]:
    print(f"{e:9d} {n:5d} {ex:11d} {s:6d} {s / T:6.3f}")
