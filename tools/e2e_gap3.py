"""Where the end-to-end (bcts_search_host) time goes beyond the device-timed step (C5).

  (a) wall of bcts_search_host after an L2 flush + synchronize (bench.py's e2e loop)
  (b) the same isolated search through device pointers: wall and device events around it
  (c) wall of an empty graph launch + synchronize (fixed host overhead)
python tools/e2e_gap3.py"""
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
dact = torch.empty(1, dtype=torch.int32, device="cuda")
dq = torch.empty(1, cfg.A, dtype=torch.float32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
N = 20

for i in range(5):
    h.search_host(pin, 1, 4, cfg.gamma, cfg.beta, 1, act, q)
    h.search(dr, 1, 4, cfg.gamma, cfg.beta, 1, out={"actions": dact, "root_q": dq})
torch.cuda.synchronize()

wa = []
for i in range(N):
    flush.fill_(i & 0xFF)
    torch.cuda.synchronize()
    t = time.perf_counter()
    h.search_host(pin, 1, 4, cfg.gamma, cfg.beta, 1, act, q)
    wa.append(time.perf_counter() - t)
print(f"(a) search_host wall: median {np.median(wa) * 1e3:.3f} ms, mean {np.mean(wa) * 1e3:.3f}")

wb, eb = [], []
for i in range(N):
    flush.fill_(i & 0xFF)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    s.record()
    h.search(dr, 1, 4, cfg.gamma, cfg.beta, 1, out={"actions": dact, "root_q": dq})
    e.record()
    e.synchronize()
    wb.append(time.perf_counter() - t)
    eb.append(s.elapsed_time(e))
print(f"(b) search (device ptrs) wall: median {np.median(wb) * 1e3:.3f} ms; events {np.median(eb):.3f} ms")

wb2, eb2 = [], []
for i in range(N):
    flush.fill_(i & 0xFF)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    h.search(dr, 1, 4, cfg.gamma, cfg.beta, 1, out={"actions": dact, "root_q": dq})
    e.record()
    torch.cuda.synchronize()
    eb2.append(s.elapsed_time(e))
print(f"(b2) flush queued right before (no host gap): events {np.median(eb2):.3f} ms")

x = torch.zeros(1, device="cuda")
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    with torch.cuda.graph(g, stream=st):
        x.add_(1)
torch.cuda.synchronize()
wc = []
for i in range(N):
    torch.cuda.synchronize()
    t = time.perf_counter()
    g.replay()
    torch.cuda.synchronize()
    wc.append(time.perf_counter() - t)
print(f"(c) empty graph launch + sync wall: median {np.median(wc) * 1e6:.1f} us")

wd = []
for i in range(N):
    flush.fill_(i & 0xFF)
    torch.cuda.synchronize()
    t = time.perf_counter()
    torch.cuda._sleep(1_000_000)
    torch.cuda.synchronize()
    wd.append(time.perf_counter() - t)
print(f"(d) ~1M-cycle sleep kernel wall: median {np.median(wd) * 1e3:.3f} ms")
