"""Where the end-to-end time of bcts_search_host goes (C5): device-timed search (events around the
graph-replayed bcts_search_ex) vs wall-clock bcts_search_host, with and without an L2 flush and a
synchronize in front. Usage: python tools/e2e_gap.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2107_01715_b200 as P  # noqa: E402
from synth.inputs import config  # noqa: E402

cfg = config("C5")
h = P.Handle.from_config(cfg)
roots = cfg.roots(1)
dr = torch.from_numpy(roots.view(np.uint8).copy()).cuda()
pin = torch.from_numpy(roots.view(np.uint8).reshape(1, -1).copy()).pin_memory()
act = torch.zeros(1, dtype=torch.int32).pin_memory()
q = torch.zeros(1, cfg.A, dtype=torch.float32).pin_memory()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    h.search(dr, 1, 4, cfg.gamma, cfg.beta, 1)
    h.search_host(pin, 1, 4, cfg.gamma, cfg.beta, 1, act, q)
torch.cuda.synchronize()
dev, host_f, host_nf, host_b2b = [], [], [], []
for i in range(20):
    flush.fill_(i & 0xFF)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(torch.cuda.current_stream())
    h.search(dr, 1, 4, cfg.gamma, cfg.beta, 1)
    e.record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    dev.append(s.elapsed_time(e))
    flush.fill_(i & 0xFF)
    torch.cuda.synchronize()
    t = time.perf_counter()
    h.search_host(pin, 1, 4, cfg.gamma, cfg.beta, 1, act, q)
    host_f.append((time.perf_counter() - t) * 1e3)
    torch.cuda.synchronize()
    t = time.perf_counter()
    h.search_host(pin, 1, 4, cfg.gamma, cfg.beta, 1, act, q)
    host_nf.append((time.perf_counter() - t) * 1e3)
t = time.perf_counter()
for i in range(20):
    h.search_host(pin, 1, 4, cfg.gamma, cfg.beta, 1, act, q)
host_b2b = (time.perf_counter() - t) * 1e3 / 20
med = lambda x: float(np.median(x))  # noqa: E731
print(f"device (events, search_ex graph): {med(dev):.3f} ms; search_host after flush: {med(host_f):.3f} ms; "
      f"search_host, warm L2: {med(host_nf):.3f} ms; back to back: {host_b2b:.3f} ms")
