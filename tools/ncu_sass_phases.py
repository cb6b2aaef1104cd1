"""Split a kernel's SASS (ncu --page source --csv --print-source sass) at BAR.SYNC / WARPSYNC and
report stall samples and executed instructions per segment.  usage: ncu_sass_phases.py sass.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Address" in r)
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
S, X, SRC = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def I(v):
    try:
        return int(float(v))
    except ValueError:
        return 0


T = sum(I(r[S]) for r in data) or 1
E = sum(I(r[X]) for r in data) or 1
seg, start = [], 0
mark = ("BAR.SYNC", "WARPSYNC")
for i, r in enumerate(data):
    if any(m in r[SRC] for m in mark) or i == len(data) - 1:
        seg.append((start, i))
        start = i + 1
print(f"{'seg':>9} {'stall':>6} {'inst':>6}  top reasons / end instruction")
for a, b in seg:
    st = sum(I(data[k][S]) for k in range(a, b + 1))
    ex = sum(I(data[k][X]) for k in range(a, b + 1))
    if st / T < 0.01 and ex / E < 0.01:
        continue
    rs = {c: sum(I(data[k][hdr.index(c)]) for k in range(a, b + 1)) for c in cols}
    top = sorted(rs.items(), key=lambda kv: -kv[1])[:3]
    print(f"{a:4d}-{b:4d} {st / T:6.3f} {ex / E:6.3f}  " + " ".join(f"{c[6:]}={v / T:.3f}" for c, v in top)
          + f"  | {data[b][SRC].strip()[:40]}")
