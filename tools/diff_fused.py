"""Fused-leaf conv1 (k_conv1_sib) vs materialised leaves (standard conv1): same search, compare."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2107_01715_b200 as P
from synth.inputs import config
for name, n, d in [("C3", 3, 2), ("C5", 1, 2), ("C5", 1, 3)]:
    cfg = config(name)
    ha = P.Handle.from_config(cfg)
    hb = P.Handle.from_config(cfg, flags=P.F_MATERIALIZE_LEAVES)
    roots = torch.from_numpy(cfg.roots(n).view(np.uint8).reshape(n, -1).copy()).cuda()
    a = ha.search(roots, n, d, cfg.gamma, 1.0, 0, extra=True)
    b = hb.search(roots, n, d, cfg.gamma, 1.0, 0, extra=True)
    torch.cuda.synchronize()
    va, vb = a["vanilla_q"].cpu().numpy(), b["vanilla_q"].cpu().numpy()
    print(name, n, d, "max |fused - materialised| / scale:", (np.abs(va - vb).max(1) / np.abs(vb).max(1)).max(),
          "best_leaf equal:", (a["best_leaf"].cpu().numpy() == b["best_leaf"].cpu().numpy()).mean())
