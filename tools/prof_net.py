"""Small driver for ncu: evaluate the leaf Q-net on one sub-batch of leaf states.

  python tools/prof_net.py [--config C5] [--n 2048] [--iters 3] [--simt]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2107_01715_b200 as P  # noqa: E402
from synth.inputs import atari_roots, config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--simt", action="store_true")
a = ap.parse_args()
cfg = config(a.config)
h = P.Handle.from_config(cfg, flags=P.F_SIMT_NET if a.simt else 0)
recs = torch.from_numpy(atari_roots(a.n, 1).copy()).cuda()
for _ in range(a.iters):
    q = h.q_rows(recs, a.n)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(a.iters):
    q = h.q_rows(recs, a.n)
e.record()
torch.cuda.synchronize()
print(f"q_rows n={a.n}: {s.elapsed_time(e) / a.iters:.3f} ms per call; q[0,:4]={q[0, :4].tolist()}")
