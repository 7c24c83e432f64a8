"""Split one search step into its two phases and time each on the device (CUDA events, L2
flushed before every step): the shard phase (level expansion, leaf net, backup) and the
finalize phase (prologue net pass over [roots | level-1 children], Eq. 3/5).

  python tools/time_phases.py [--config C5] [--depth 4] [--roots 1] [--iters 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2107_01715_b200 as P  # noqa: E402
from synth.inputs import config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--depth", type=int, default=0)
ap.add_argument("--roots", type=int, default=0)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--world", type=int, default=1, help="time rank 0's share of a world-size-W partition")
ap.add_argument("--profile", action="store_true", help="also print the per-kernel-class breakdown")
a = ap.parse_args()
cfg = config(a.config)
n = a.roots or cfg.n_roots
d = a.depth or cfg.depth
h = P.Handle.from_config(cfg)
dev = torch.device("cuda", 0)
roots = torch.from_numpy(cfg.roots(n).view(np.uint8).copy()).to(dev)
keys = torch.empty(n * cfg.A, dtype=torch.int64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
L = n * cfg.A ** d
b, e = P.shard_range(n, d, cfg.A, 0, a.world)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
tot = np.zeros(2)
for it in range(a.iters + 3):
    flush.fill_(it & 0xFF)
    torch.cuda.synchronize()
    ev[0].record()
    h.keys_init(keys)
    h.search_shard(roots, n, d, cfg.gamma, b, e, keys)
    ev[1].record()
    h.finalize(roots, n, d, cfg.gamma, cfg.beta, 1, keys, extra=False)
    ev[2].record()
    torch.cuda.synchronize()
    if it >= 3:
        tot += [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])]
tot /= a.iters
if a.profile:   # per kernel class (event pairs on the handle's stream), one more pass of iters
    h.profile(True)
    for it in range(a.iters):
        h.keys_init(keys)
        h.search_shard(roots, n, d, cfg.gamma, b, e, keys)
        h.finalize(roots, n, d, cfg.gamma, cfg.beta, 1, keys, extra=False)
    torch.cuda.synchronize()
    for k, v in sorted(h.profile_read().items(), key=lambda kv: -kv[1]["ms"]):
        print(f"  {k:14s} {v['ms'] / a.iters * 1e3:8.1f} us/step  {v['launches'] / a.iters:5.1f} launches/step")
    h.profile(False)
print(f"{a.config} n={n} d={d} rank 0 of {a.world} (leaves [{b}, {e})): shard {tot[0]:.3f} ms, finalize (prologue + Eq. 3/5) {tot[1]:.3f} ms, "
      f"total {tot.sum():.3f} ms")
