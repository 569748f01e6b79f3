"""Compare per-layer times of two bench report markdowns: cmp_reports.py A.md B.md [prefix]"""
import sys
def rows(f):
    d = {}
    for l in open(f):
        p = [x.strip() for x in l.split('|')]
        if len(p) > 6 and ':' in p[1] and not p[1].startswith('layer'):
            try:
                d[p[1]] = (float(p[2]), p[5])
            except ValueError:
                pass
    return d
a, b = rows(sys.argv[1]), rows(sys.argv[2])
pre = sys.argv[3] if len(sys.argv) > 3 else ""
ta = tb = 0.0
for k in a:
    if k.startswith(pre) and k in b:
        ta += a[k][0]; tb += b[k][0]
        print(f"{k:36s} {a[k][0]:8.2f} -> {b[k][0]:8.2f}  ({a[k][0] / b[k][0]:.2f}x)  frac {b[k][1]}")
print(f"total {ta:.1f} -> {tb:.1f} us")
