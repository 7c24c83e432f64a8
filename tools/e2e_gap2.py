"""Isolated vs back-to-back C5 searches (device events): where does the ~0.27 ms an isolated search
costs beyond the pipelined step go? python tools/e2e_gap2.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2107_01715_b200 as P  # noqa: E402
from synth.inputs import config  # noqa: E402

cfg = config("C5")
h = P.Handle.from_config(cfg)
roots = cfg.roots(1)
dr = torch.from_numpy(roots.view(np.uint8).copy()).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()


def ev():
    return torch.cuda.Event(enable_timing=True)


for _ in range(5):
    h.search(dr, 1, 4, cfg.gamma, cfg.beta, 1)
torch.cuda.synchronize()
s, e = ev(), ev()
s.record(st)
for _ in range(20):
    h.search(dr, 1, 4, cfg.gamma, cfg.beta, 1)
e.record(st)
torch.cuda.synchronize()
print(f"back to back: {s.elapsed_time(e) / 20:.3f} ms per search")
for mode in ("sync", "sync+flush", "busy-before", "flush+busy-before"):
    ts = []
    for i in range(10):
        if "flush" in mode:
            flush.fill_(i & 0xFF)
        torch.cuda.synchronize()
        if "busy" in mode:
            torch.cuda._sleep(2_000_000)   # ~1 ms of a spinning kernel: the search is queued behind it
        s, e = ev(), ev()
        s.record(st)
        h.search(dr, 1, 4, cfg.gamma, cfg.beta, 1)
        e.record(st)
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    print(f"{mode}: {np.median(ts):.3f} ms")
h.profile(True)
for i in range(3):
    flush.fill_(i & 0xFF)
    torch.cuda.synchronize()
    h.search(dr, 1, 4, cfg.gamma, cfg.beta, 1)
torch.cuda.synchronize()
for k, v in h.profile_read().items():
    print(k, round(v["ms"] / 3, 4), v["launches"] / 3)
