"""Top SASS instructions by warp-stall samples (with their dominant stall reasons) from
`ncu --page source --csv --print-source sass`.  usage: python tools/ncu_sass_top.py sass.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hi = next(i for i, r in enumerate(rows) if "Address" in r)
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]


def I(r, k):
    try:
        return int(float(r[hdr.index(k)]))
    except ValueError:
        return 0


S = "Warp Stall Sampling (All Samples)"
T = sum(I(r, S) for r in data) or 1
E = sum(I(r, "Instructions Executed") for r in data) or 1
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {c: sum(I(r, c) for r in data) for c in cols}
print("stall mix:", {c[6:]: round(v / T, 3) for c, v in sorted(tot.items(), key=lambda kv: -kv[1])[:8]})
print(f"samples {T} instructions {E}")
for i in sorted(range(len(data)), key=lambda i: -I(data[i], S))[:top]:
    r = data[i]
    why = sorted(((I(r, c), c[6:]) for c in cols), reverse=True)[:2]
    print(f"{i:5d} {I(r, S) / T:6.3f} {r[hdr.index('Source')][:56]:56s} {why}")
