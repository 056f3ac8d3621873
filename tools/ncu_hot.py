"""Top stall instructions of one kernel from `ncu --page source --csv --print-source sass` output (tools only)."""
import csv
import sys


def iv(s):
    try:
        return int(s)
    except ValueError:
        return 0


r = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = r[1]
rows = [x for x in r[2:] if len(x) >= len(h)]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_")]
tot = sum(iv(x[si]) for x in rows)
print("total samples", tot)
agg = {}
for x in rows:
    for i in stall_cols:
        agg[h[i]] = agg.get(h[i], 0) + iv(x[i])
print(sorted(((v, k) for k, v in agg.items() if v), reverse=True)[:8])
for k, x in enumerate(rows):
    x.append(k)
for x in sorted(rows, key=lambda x: -iv(x[si]))[:n]:
    st = sorted([(iv(x[i]), h[i][6:]) for i in stall_cols if iv(x[i])], reverse=True)[:3]
    print(f"{iv(x[si]):6d} #{x[-1]:<5} {x[1].strip()[:64]:<64} {st}")
