"""Measure the BCTS_F_TF32 path against the fp64 oracle (R34): level-state errors of the
tf32 DNN forward model and root-Q / action errors of whole searches (DNN and INT_HASH MLP2 configs).
  python tools/tf32_check.py"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2107_01715_b200 as P  # noqa: E402
from oracle import Oracle  # noqa: E402
from synth.inputs import config  # noqa: E402
from tests.helpers import action_agreement, rel_err  # noqa: E402

DEV = torch.device("cuda", 0)
TH = os.cpu_count() or 1


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).copy()).to(DEV)


def cfgs(name):
    if name == "D3":
        return dataclasses.replace(config("D10"), name="D3", A=3, seed=23, wseed=123)
    return config(name)


for name, n, levels in (("D10", 4, 3), ("D3", 3, 4), ("D2", 4, 7)):
    cfg = cfgs(name)
    h = P.Handle.from_config(cfg, flags=P.F_TF32)
    o = Oracle.from_config(cfg)
    roots = cfg.roots(n)
    g = float(np.float32(cfg.gamma))
    for level in range(1, levels + 1):
        st, cum = h.expand(dev(roots), n, level, np.float32(cfg.gamma))
        st, cum = st.cpu().numpy(), cum.cpu().numpy()
        per = cfg.A ** level
        idx = range(n * per) if n * per <= 300 else np.random.default_rng(level).choice(n * per, 300, replace=False)
        es, er = 0.0, 0.0
        for j in idx:
            r, i = divmod(int(j), per)
            rec, R = o.node(roots[r], level, i, g, mode=0)
            x = np.frombuffer(rec.tobytes(), dtype=np.float32)
            y = st[j].view(np.float32)
            es = max(es, float(np.abs(y - x).max() / max(np.abs(x).max(), 1e-6)))
            er = max(er, abs(float(cum[j]) - R) / max(abs(R), 1e-3))
        print(f"{name} level {level}: max state err / max|state| {es:.2e}, max R err {er:.2e}", flush=True)
    h.close()

for name, n, d in (("D2", 64, 8), ("D10", 16, 4), ("D3", 7, 5), ("C2", 64, 4)):
    cfg = cfgs(name)
    h = P.Handle.from_config(cfg, flags=P.F_TF32)
    o = Oracle.from_config(cfg)
    roots = cfg.roots(n)
    gamma = float(np.float32(cfg.gamma))
    out = h.search(dev(roots), n, d, cfg.gamma, 1.0, 1, extra=True)
    torch.cuda.synchronize()
    g = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in out.items()}
    r = o.search(roots, d, gamma, 1.0, 1, mode=0, threads=TH)
    eq, ev = rel_err(g["root_q"], r["root_q"]).max(), rel_err(g["vanilla_q"], r["vanilla_q"]).max()
    frac, exact, near = action_agreement(g["actions"], r["root_q"], 1e-2)
    print(f"{name} n={n} d={d}: root_q rel err {eq:.2e}, vanilla_q {ev:.2e}; actions {frac:.4f} "
          f"(exact {exact}, near {near}); identical actions {(g['actions'] == r['actions']).mean():.4f}", flush=True)
    h.close()
