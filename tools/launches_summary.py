"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
kn, val, unit = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[start + 1:]:
    if len(r) <= val:
        continue
    name = r[kn].replace("void ", "").replace("bcts::<unnamed>::", "").replace("bcts::", "")
    name = name.split("(")[0].strip()
    agg[name][0] += 1
    agg[name][1] += float(r[val].replace(",", "")) * scale.get(r[unit], 1.0)
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':58s} {'launches':>8s} {'total us':>10s} {'share':>6s}")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n[:58]:58s} {c:8d} {t:10.1f} {100 * t / tot:5.1f}%")
