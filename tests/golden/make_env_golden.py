"""Freeze env golden vectors (calls only oracle/): sha256 of the record after each
step of a fixed action sequence from seeded roots, plus the rewards.

Run: python tests/golden/make_env_golden.py  -> tests/golden/env_golden.json
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import Oracle  # noqa: E402
from synth.inputs import config  # noqa: E402

out = {"_source": "frozen once from oracle/ by tests/golden/make_env_golden.py (ENV_SPEC, DESIGN.md §3)"}
for name, n in (("C2", 4), ("C3", 2)):
    cfg = config(name)
    o = Oracle.from_config(cfg)
    roots = cfg.roots(n)
    seqs = []
    for r in range(n):
        rec = roots[r]
        acts = [(7 * k + 3 * r) % cfg.A for k in range(6)]
        digests, rewards = [], []
        for a in acts:
            rec, rew = o.step(rec, a)
            digests.append(hashlib.sha256(rec.tobytes()).hexdigest())
            rewards.append(rew)
        seqs.append({"root": r, "actions": acts, "sha256": digests, "rewards": rewards})
    out[name] = {"seed": cfg.seed, "A": cfg.A, "sequences": seqs}
json.dump(out, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "env_golden.json"), "w"), indent=1)
print("ok")
