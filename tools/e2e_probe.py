"""Wall-clock of consecutive bcts_search_host calls (C5): the first is eager (+ graph capture),
later calls replay the graph. Usage: python tools/e2e_probe.py [steps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2107_01715_b200 as P
from synth.inputs import config
cfg = config("C5")
h = P.Handle.from_config(cfg)
roots = cfg.roots(1)
pin = torch.from_numpy(roots.view(np.uint8).reshape(1, -1).copy()).pin_memory()
act = torch.zeros(1, dtype=torch.int32).pin_memory()
q = torch.zeros(1, cfg.A, dtype=torch.float32).pin_memory()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    flush.fill_(i & 0xFF)
    torch.cuda.synchronize()
    t = time.perf_counter()
    h.search_host(pin, 1, 4, cfg.gamma, cfg.beta, 1, act, q)
    print(f"call {i}: {(time.perf_counter() - t) * 1e3:.3f} ms, action {int(act[0])}")
