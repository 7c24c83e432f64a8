"""Print the headline numbers and per-kernel-class times of bench.py JSON lines (file args)."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        if not line.startswith('{'):
            continue
        d = json.loads(line)
        if "ms_per_step" not in d:
            print(d)
            continue
        r = d.get("roofline") or {}
        print(f"{d['config'].get('workload', '')[:40]} ms/step {d['ms_per_step']:.4f} value {d['value']:.4g} "
              f"frac {r.get('frac', 0):.3f} e2e {d.get('e2e', {}).get('ms_per_step', 0):.4f} clocks {d.get('clocks')}")
        for k, v in (d.get("kernels") or {}).items():
            print(f"   {k:14s} {v['ms_per_launch'] * v['launches_per_step']:.4f} ms  {v.get('achieved', 0):.1f} {v.get('unit', '')}")
