"""Per-source-line stall / instruction shares from `ncu --page source --csv --print-source cuda,sass`.

usage: python tools/ncu_lines.py mixed.csv [top]
"""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    out, fname, hdr = [], None, None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and len(r) == len(hdr) and r[0]:
            def I(k):
                try:
                    return int(float(r[k]))
                except ValueError:
                    return 0
            out.append((fname, r[0], I(4), I(7), r[1].strip()))
    T = sum(o[2] for o in out) or 1
    E = sum(o[3] for o in out) or 1
    print(f"stall samples {T}  instructions {E}")
    for f, ln, s, e, src in sorted(out, key=lambda o: -o[2])[:top]:
        print(f"{f}:{ln:>4} stall {s / T:6.3f} inst {e / E:6.3f}  {src[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
