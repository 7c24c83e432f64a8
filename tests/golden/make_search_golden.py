"""Freeze whole-search oracle results at the BASELINE sizes of C3, C4 and C5 (calls only oracle/).

The complete recursive-DFS oracle (oracle/bcts_oracle.c, Eq. 1 P:53-55 / Alg. 1, Eq. 3/5
P:205-213) is run on the same seeded inputs the GPU tests feed the CUDA path:

  C5   : the single root, full depth-4 tree (104,976 leaves), BCTS on
  C5S  : the same with spread Q-hat weights (synth.inputs head_scale = 64; tests only)
  C3   : all 64 roots, depth 3
  C3S  : 16 roots, depth 3, spread weights
  C4   : a 16-root subset (every 64th of the 1024 roots), depth 5 (7,776 leaves per root)
  C4d2 : all 1024 C4 roots at depth 2 (action agreement over many roots)
  C4Sd2: the same with spread weights

Nothing here comes from the CUDA path. Outputs are the oracle's fp64 reference mode (bf16-emulating
nets, R17). Run: python tests/golden/make_search_golden.py [case ...]
  -> tests/golden/search_golden.json (cases are merged into the existing file)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import Oracle  # noqa: E402
from synth.inputs import config  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "search_golden.json")

# name: (config, root indices (None = all of config.n_roots), depth)
CASES = {
    "C5": ("C5", None, 4),
    "C5S": ("C5S", None, 4),
    "C3": ("C3", None, 3),
    "C3S": ("C3S", list(range(16)), 3),
    "C4": ("C4", list(range(0, 1024, 64)), 5),
    "C4d2": ("C4", None, 2),
    "C4Sd2": ("C4S", None, 2),
}


def run_case(name, threads):
    cname, idx, d = CASES[name]
    cfg = config(cname)
    roots = cfg.roots()
    if idx is not None:
        roots = roots[idx]
    else:
        idx = list(range(cfg.n_roots))
    o = Oracle.from_config(cfg)
    gamma32 = float(np.float32(cfg.gamma))   # the C ABI takes gamma as float (R3)
    t = time.time()
    r = o.search(roots, d, gamma32, cfg.beta, 1, mode=0, threads=threads)
    dt = time.time() - t
    print(f"{name}: {len(idx)} roots, d={d}: {dt:.1f} s on {threads} threads", flush=True)
    return {"config": cname, "roots": idx, "depth": d, "gamma": gamma32, "beta": cfg.beta, "correction": 1,
            "head_scale": cfg.extra.get("head_scale", 1.0), "oracle_seconds": dt, "threads": threads,
            "actions": r["actions"].tolist(), "root_q": r["root_q"].tolist(),
            "vanilla_q": r["vanilla_q"].tolist(), "terms": r["terms"].tolist(),
            "best_leaf": r["best_leaf"].tolist()}


def main():
    names = sys.argv[1:] or list(CASES)
    threads = os.cpu_count() or 1
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data["_source"] = ("oracle/ only (complete recursive DFS, fp64 reference mode): "
                       "tests/golden/make_search_golden.py; inputs from synth/ (seeded)")
    for n in names:
        data[n] = run_case(n, threads)
        json.dump(data, open(OUT, "w"), indent=0)
    print("ok")


if __name__ == "__main__":
    main()
