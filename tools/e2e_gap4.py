"""bench.py's end-to-end loop, instrumented: per call the wall time of bcts_search_host and the device span
from an event recorded on the (default) stream just before the call to one recorded just after it returns.
python tools/e2e_gap4.py [steps]"""
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
n, A = 1, cfg.A
pin = torch.from_numpy(cfg.roots(1).view(np.uint8).reshape(1, -1).copy()).pin_memory()
act = torch.empty(n, dtype=torch.int32).pin_memory()
q = torch.empty(n, A, dtype=torch.float32).pin_memory()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
walls, devs = [], []
for i in range(5 + steps):
    flush.fill_(i & 0xFF)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    h.search_host(pin, n, cfg.depth, cfg.gamma, cfg.beta, 1, act, q)
    dt = time.perf_counter() - t0
    e1.record()
    torch.cuda.synchronize()
    if i >= 5:
        walls.append(dt * 1e3)
        devs.append(e0.elapsed_time(e1))
walls, devs = np.array(walls), np.array(devs)
print(f"wall  ms: mean {walls.mean():.4f} median {np.median(walls):.4f} min {walls.min():.4f} max {walls.max():.4f}")
print(f"event ms: mean {devs.mean():.4f} median {np.median(devs):.4f} min {devs.min():.4f} max {devs.max():.4f}")
print("wall - event per call (us):", np.round((walls - devs) * 1e3, 1).tolist())
