"""Summarise an `ncu --metrics ... --csv` log: one line per launch (kernel, grid, metrics)."""
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
idx = {h: i for i, h in enumerate(hdr)}
cur = None
for r in rows[1:]:
    if len(r) < len(hdr):
        continue
    key = (r[idx["ID"]], r[idx["Kernel Name"]].split("(")[0][-28:], r[idx["Grid Size"]])
    if key != cur:
        print()
        print(key, end=" ")
        cur = key
    name = r[idx["Metric Name"]].replace("smsp__average_warps_issue_stalled_", "stall_")
    name = name.replace("_per_issue_active.ratio", "").replace(".avg.pct_of_peak_sustained_active", "%")
    print(name[:40], r[idx["Metric Value"]], end=" | ")
print()
