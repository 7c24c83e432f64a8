"""GPU parity at the BASELINE sizes of C3, C4 and C5 against COMPLETE oracle searches.

The expected values are `tests/golden/search_golden.json`, written by `tests/golden/make_search_golden.py`,
which calls only `oracle/` (the recursive-DFS oracle in its fp64 reference mode: Eq. 1, Alg. 1
P:310-327 with the return rule P:324, Eq. 3, Eq. 5) on the same seeded inputs
(`synth/`). Cases:

  C5    the headline: 1 root, A = 18, d = 4, the full 104,976-leaf tree, BCTS on
  C5S   the same with "spread" Q-hat weights (synth head_scale = 64: output layers x64, tests only)
  C3    all 64 roots at d = 3 (Nature net)
  C3S   16 roots at d = 3 with spread weights
  C4    a 16-root subset (every 64th root) at d = 5
  C4d2  all 1024 C4 roots at d = 2 (action agreement over many roots)
  C4Sd2 the same with spread weights

Comparison rules (R18/R19): root Q (corrected) and vanilla Q within RTOL = 1e-3 of
max_a |oracle q| per root, 5e-3 for the spread variants (the north star's ceiling is 2e-2); pi_o exact or a near-tie of the oracle's
Q-hat(s0, .); delta_o, delta_e, B within 4e-3 of the root's Q scale (B = sqrt(ln A)(...) amplifies the
delta errors by < 4); actions accepted under the near-tie rule, >= 99.9 % (north star); where the GPU's best
leaf differs from the oracle's, the oracle's own total at the GPU's leaf must lie within RTOL of the
oracle's segment max (several leaves are correct there: the argmax set of Eq. 1). Random-init Q-hat is
nearly flat across leaves, so the spread variants are the discriminating cases: they additionally
require most best leaves to agree exactly.
"""
import json
import os

import numpy as np
import pytest

from tests.helpers import action_agreement, rel_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2107_01715_b200 as P  # noqa: E402
from oracle import Oracle  # noqa: E402
from synth.inputs import config  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "search_golden.json")
DEV = torch.device("cuda", 0)
RTOL = 1e-3          # random-init weights (Q-hat nearly flat): observed <= 2e-5 on C5 (round 1)
RTOL_SPREAD = 5e-3   # spread weights: bf16 RNE flips of hidden activations (R17: same rounding points, fp32
                     # vs fp64 accumulation order) are no longer masked by the bias; observed 1.3e-3 on C3S
TERMS_TOL = 4e-3
MAX_LEAF_CHECKS = 192

_data = json.load(open(GOLDEN))
CASES = sorted(k for k in _data if not k.startswith("_"))
_handles = {}


def _handle(cname):
    if cname not in _handles:
        _handles[cname] = P.Handle.from_config(config(cname))
    return _handles[cname]


@pytest.mark.parametrize("case", CASES)
def test_full_size_vs_complete_oracle(case):
    gd = _data[case]
    cfg = config(gd["config"])
    assert abs(cfg.extra.get("head_scale", 1.0) - gd["head_scale"]) == 0
    roots = cfg.roots()[np.array(gd["roots"])]
    n, d, A = roots.shape[0], gd["depth"], cfg.A
    h = _handle(gd["config"])
    rd = torch.from_numpy(np.ascontiguousarray(roots).view(np.uint8).copy()).to(DEV)
    out = h.search(rd, n, d, cfg.gamma, gd["beta"], gd["correction"], extra=True)
    torch.cuda.synchronize()
    g = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in out.items()}
    o_q = np.array(gd["root_q"])
    o_v = np.array(gd["vanilla_q"])
    o_t = np.array(gd["terms"])
    o_a = np.array(gd["actions"])
    o_bl = np.array(gd["best_leaf"])
    assert g["stats"]["leaves"] == n * A ** d
    RT = RTOL if gd["head_scale"] == 1.0 else RTOL_SPREAD

    # pi_o (lowest argmax of Q-hat(s0, .)): identical, or -- where the oracle's root row has a near-tie
    # (R19) -- another member of the argmax set; such a root's corrected Q follows its own pi_o (Eq. 3
    # penalises every a != pi_o), so its root Q is compared through vanilla Q only
    scale = np.maximum(np.abs(o_q).max(axis=1), 1e-6)
    o = None
    pio_g, pio_o = g["terms"][:, 0].astype(np.int64), o_t[:, 0].astype(np.int64)
    bad = np.nonzero(pio_g != pio_o)[0]
    if len(bad):
        o = Oracle.from_config(cfg)
        for r in bad:
            q0 = o.qrow(roots[r])
            assert q0.max() - q0[pio_g[r]] <= 2 * RT * max(np.abs(q0).max(), 1e-6), (case, r)
    same = pio_g == pio_o
    assert len(bad) <= max(1, n // 1000), len(bad)

    err_q, err_v = rel_err(g["root_q"][same], o_q[same]), rel_err(g["vanilla_q"], o_v)
    frac, exact, near = action_agreement(g["actions"][same], o_q[same], RT)
    bl_same = float((g["best_leaf"] == o_bl).mean())
    print(f"{case}: n={n} d={d}: max rel err root_q {err_q.max():.2e}, vanilla_q {err_v.max():.2e}; "
          f"actions {frac:.4f} (exact {exact}, near-ties {near}, oracle action == GPU action "
          f"{int((g['actions'] == o_a).sum())}/{n}); pi_o identical {int(same.sum())}/{n} (others near-ties); "
          f"best leaf identical {bl_same:.4f}")
    assert err_q.max() <= RT and err_v.max() <= RT
    assert frac >= 0.999

    # BCTS terms delta_o, delta_e, B where pi_o agrees
    terr = np.abs(g["terms"][same, 1:] - o_t[same, 1:]) / scale[same, None]
    print(f"{case}: max terms err / Q scale {terr.max() if terr.size else 0:.2e}")
    assert (terr <= TERMS_TOL * RT / RTOL).all()

    # best leaves: where they differ, the GPU's leaf must be one of the (near-)maximisers of its segment
    lpr = A ** d
    diff = np.argwhere(g["best_leaf"] != o_bl)
    for r, a in diff:
        leaf = int(g["best_leaf"][r, a])
        assert a * (lpr // A) <= leaf < (a + 1) * (lpr // A), (case, r, a)
    if len(diff):
        o = o or Oracle.from_config(cfg)
        rng = np.random.default_rng(0)
        pick = diff if len(diff) <= MAX_LEAF_CHECKS else diff[rng.choice(len(diff), MAX_LEAF_CHECKS, replace=False)]
        for r, a in pick:
            tot = o.leaf_total(roots[r], d, int(g["best_leaf"][r, a]), gd["gamma"], mode=0)
            assert o_v[r, a] - tot <= RT * scale[r], (case, r, a, tot, o_v[r, a])
            assert tot <= o_v[r, a] + 1e-12 * scale[r]
    if gd["head_scale"] != 1.0:
        assert bl_same >= 0.99, bl_same   # observed 0.9992-1.0
    torch.cuda.empty_cache()
