"""Rank SASS lines of an `ncu --page source --csv --print-source sass` export by a column.
  python tools/ncu_src_top.py src.csv ["L1 Wavefronts Shared"] [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
col = sys.argv[2] if len(sys.argv) > 2 else "L1 Wavefronts Shared"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
hdr = rows[1]
ci = hdr.index(col)
si = hdr.index("Source")
ii = hdr.index("Instructions Executed")
ideal = hdr.index("L1 Wavefronts Shared Ideal") if "L1 Wavefronts Shared Ideal" in hdr else None
samp = hdr.index("Warp Stall Sampling (All Samples)")


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


body = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(num(r[ci]) for r in body)
print(f"total {col}: {tot:.4g}")
for r in sorted(body, key=lambda r: -num(r[ci]))[:n]:
    extra = f" ideal {num(r[ideal]):.3g}" if ideal is not None else ""
    print(f"{num(r[ci]):12.4g} ({100 * num(r[ci]) / max(tot, 1):5.1f}%) inst {num(r[ii]):10.4g}{extra} samp {r[samp]:>6s}  {r[0]} {r[si][:80]}")
