"""Timing of the early-pruned search (NEXT-4; R30-R33) next to the unpruned one.

One JSON line per case: ms per search (CUDA events on the handle's stream, L2 flushed before each
timed call, W warm-up calls), survivors per level, leaves scored, and the per-kernel-class split
from the handle's profiler (a separate profiled repeat). Not the headline bench: bench.py is.

  python tools/bench_prune.py [--steps 10] [--warmup 3] > profiles/r01_bench_prune.jsonl
"""
import argparse
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = [
    # (config, roots, depth, rule, first_level, beam, bounds)
    ("C5", 1, 4, "none", 0, 0, None),
    ("C5", 1, 4, "beam", 3, 64, None),
    ("C5", 1, 4, "beam", 2, 16, None),
    ("C5", 1, 4, "bound", 1, 0, (-1.0, 1.0, -10.0, 10.0)),
    ("C5", 1, 5, "beam", 3, 64, None),
    ("C5", 1, 6, "beam", 3, 32, None),
    ("C4", 1024, 5, "none", 0, 0, None),
    ("C4", 1024, 5, "beam", 2, 4, None),
    ("C2", 256, 4, "none", 0, 0, None),
    ("C2", 256, 4, "beam", 1, 2, None),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2107_01715_b200 as P
    from synth.inputs import config
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    handles = {}
    for cname, n, d, rule, first, beam, bounds in CASES:
        cfg = dataclasses.replace(config(cname), n_roots=n)
        if cname not in handles:
            handles[cname] = P.Handle.from_config(cfg)
        h = handles[cname]
        roots = torch.from_numpy(cfg.roots().view(np.uint8).reshape(n, -1).copy()).to(dev)
        code = {"none": None, "beam": P.PRUNE_BEAM, "bound": P.PRUNE_BOUND}[rule]
        b = bounds or (0.0, 0.0, 0.0, 0.0)

        def call():
            if code is None:
                return h.search(roots, n, d, cfg.gamma, cfg.beta, 1, extra=True)
            return h.search_pruned(roots, n, d, cfg.gamma, code, first, beam, *b, beta=cfg.beta, correction=1)

        for _ in range(args.warmup):
            out = call()
        torch.cuda.synchronize()
        ms = []
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = call()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        h.profile(True)
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            call()
        torch.cuda.synchronize()
        prof = h.profile_read()
        h.profile(False)
        tot = sum(v["ms"] for v in prof.values()) or 1.0
        surv = [int(x) for x in out["survivors"]] if "survivors" in out else [n * cfg.A ** k for k in range(d + 1)]
        line = {"config": cname, "roots": n, "depth": d, "A": cfg.A, "rule": rule, "first_level": first,
                "beam": beam, "bounds": bounds, "ms_per_search": float(np.median(ms)), "ms_min": float(min(ms)),
                "decisions_per_s": n / (float(np.median(ms)) / 1e3), "survivors": surv,
                "leaves_scored": out["stats"]["leaves"], "unpruned_leaves": n * cfg.A ** d,
                "kernel_share": {k: round(v["ms"] / tot, 4) for k, v in prof.items()},
                "prune_ms_per_search": prof.get("prune", {}).get("ms", 0.0) / args.steps,
                "actions_head": out["actions"][:4].cpu().tolist()}
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
