"""Top SASS instructions by warp-stall samples from `ncu -i X --page source --csv`."""
import csv
import sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ci = h.index("Warp Stall Sampling (All Samples)")
data = rows[2:]
tot = sum(int(r[ci] or 0) for r in data)
idx = sorted(range(len(data)), key=lambda i: -int(data[i][ci] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]
cols = [c for c in ("stall_long_sb", "stall_barrier", "stall_wait", "stall_lg", "stall_short_sb", "stall_mio") if c in h]
print("total samples", tot)
for i in sorted(idx):
    r = data[i]
    extra = " ".join(f"{c[6:]}={r[h.index(c)]}" for c in cols if r[h.index(c)] not in ("0", ""))
    print(f"{i:5d} {100*int(r[ci])/tot:5.1f}% {r[1].strip()[:60]:60s} {extra}")
