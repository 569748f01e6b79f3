"""Executed warp-instructions grouped by SASS opcode from an ncu source page csv
(ncu -i X --page source --csv --print-source sass)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
isrc = hdr.index("Source"); ie = hdr.index("Instructions Executed")
cnt = collections.Counter()
for r in rows[2:]:
    try:
        n = int(r[ie] or 0)
    except (ValueError, IndexError):
        continue
    s = r[isrc].strip()
    if s.startswith("@"):
        s = s.split(None, 1)[1] if " " in s else s
    op = s.split()[0] if s else "?"
    cnt[op.split(".")[0]] += n
tot = sum(cnt.values())
print("total", tot)
for op, n in cnt.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{op:12s} {n:10d} {n / tot:6.3f}")
