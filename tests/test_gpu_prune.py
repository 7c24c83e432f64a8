"""GPU parity of the early-pruned search (NEXT-4; R30-R33) through the C-ABI.

  * fp32 envs/nets (TABULAR, INT_HASH + MLP2, DNN + MLP2): bit-exact vs oracle_search_pruned in
    the fp32-mirror mode -- same survivors per level, vanilla_q, best_leaf, actions;
  * BOUND rule: GPU pruned == GPU unpruned bit for bit (soundness, R31), also on the bf16 Rainbow
    net with q in the C51 support;
  * BEAM rule on bf16 conv nets (R33): exact survivor counts, wide beam == unpruned, narrow beam's
    vanilla_q <= the unpruned one, best leaf's oracle total within the bf16 search tolerance.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2107_01715_b200 as P  # noqa: E402
from oracle import Oracle  # noqa: E402
from synth.inputs import ENV_TABULAR, NET_TABLE, Tabular, config, tabular_roots  # noqa: E402
from tests.test_gpu_parity import RTOL_BF16_SEARCH, dev, handle, run  # noqa: E402

KEYS = ("vanilla_q", "best_leaf", "actions", "root_q", "terms")


def prun(h, roots_np, d, gamma, rule, first=1, beam=1, bounds=(0.0, 0.0, 0.0, 0.0), beta=1.0, corr=1):
    n = roots_np.shape[0]
    out = h.search_pruned(dev(roots_np), n, d, gamma, rule, first, beam, *bounds, beta=beta, correction=corr)
    torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in out.items()}


def check_vs_oracle(g, m, n, A):
    np.testing.assert_array_equal(g["survivors"], m["survivors"])
    np.testing.assert_array_equal(g["vanilla_q"], m["vanilla_q"].astype(np.float32))
    np.testing.assert_array_equal(g["best_leaf"], m["best_leaf"])
    np.testing.assert_array_equal(g["actions"], m["actions"])


def random_mdp(rng, nS, A):
    nxt = rng.integers(0, nS, size=nS * A).astype(np.int32)
    rew = rng.integers(-5, 6, size=nS * A).astype(float)
    q = (rng.normal(size=nS * A) * 0.2).astype(np.float32).astype(float)
    return Tabular(A, nxt, rew, q)


@pytest.mark.parametrize("rule", [P.PRUNE_BOUND, P.PRUNE_BEAM])
def test_tabular_random_mdps_vs_oracle(rule):
    rng = np.random.default_rng(40 + rule)
    gamma = float(np.float32(0.9))
    pruned = 0
    for i in range(12):
        A, d = int(rng.integers(2, 5)), int(rng.integers(2, 6))
        t = random_mdp(rng, int(rng.integers(4, 40)), A)
        h = P.Handle(ENV_TABULAR, A, NET_TABLE, tab=t)
        o = Oracle(ENV_TABULAR, A, NET_TABLE, tab=t)
        roots = tabular_roots(rng.integers(0, t.nS, size=int(rng.integers(1, 6))))
        n = roots.shape[0]
        b = (float(t.reward.min()), float(t.reward.max()), float(t.q.min()), float(t.q.max()))
        for first in range(1, d):
            beam = int(rng.integers(1, 4))
            g = prun(h, roots, d, gamma, rule, first, beam, b)
            m = o.search_pruned(roots, d, gamma, rule, first, beam, *b, beta=1.0, correction=1, mode=1)
            check_vs_oracle(g, m, n, A)
            pruned += int(g["survivors"][d] < n * A ** d)
            if rule == P.PRUNE_BOUND:   # soundness: identical to the unpruned GPU search
                u = run(h, roots, d, gamma, 1.0, 1)
                for k in KEYS:
                    np.testing.assert_array_equal(g[k], u[k])
        h.close()
    assert pruned > 3


@pytest.mark.parametrize("cname,n,d", [("C2", 16, 4), ("D10", 8, 3), ("D2", 8, 6)])
@pytest.mark.parametrize("first,beam", [(1, 1), (1, 3), (2, 2)])
def test_beam_fp32_nets_vs_oracle(cname, n, d, first, beam):
    cfg = config(cname)
    h = handle(cname)
    o = Oracle.from_config(cfg)
    roots = cfg.roots(n)
    gamma = float(np.float32(cfg.gamma))
    g = prun(h, roots, d, cfg.gamma, P.PRUNE_BEAM, first, beam)
    m = o.search_pruned(roots, d, gamma, P.PRUNE_BEAM, first, beam, beta=1.0, correction=1, mode=1)
    check_vs_oracle(g, m, n, cfg.A)


def test_bound_rule_rainbow_equals_unpruned():
    """C51 support bounds Q-hat exactly (q in [v_min, v_max]); Atari-shaped rewards in [-1, 1]."""
    cfg = config("C5")
    h = handle("C5")
    roots = cfg.roots(1)
    for d, first in ((3, 1), (3, 2), (2, 1)):
        g = prun(h, roots, d, cfg.gamma, P.PRUNE_BOUND, first, 0, (-1.0, 1.0, -10.0, 10.0))
        u = run(h, roots, d, cfg.gamma, 1.0, 1)
        for k in KEYS:
            np.testing.assert_array_equal(g[k], u[k])


@pytest.mark.parametrize("cname,n,d,beam", [("C5", 1, 3, 4), ("C4", 2, 4, 5), ("C3", 2, 3, 7)])
def test_beam_conv_nets_properties(cname, n, d, beam):
    cfg = config(cname)
    h = handle(cname)
    o = Oracle.from_config(cfg)
    roots = cfg.roots(n)
    A = cfg.A
    u = run(h, roots, d, cfg.gamma, 1.0, 0)
    g = prun(h, roots, d, cfg.gamma, P.PRUNE_BEAM, 1, beam, corr=0)
    exp = [n, n * A] + [n * A * min(beam, A)] + [n * A * min(beam, min(beam, A) * A)] * (d - 3)
    exp = exp[:d] + [exp[d - 1] * A]
    assert list(g["survivors"]) == exp
    assert (g["vanilla_q"] <= u["vanilla_q"]).all()
    scale = np.maximum(np.abs(u["vanilla_q"]).max(axis=1, keepdims=True), 1e-6)
    gamma = float(np.float32(cfg.gamma))
    for r in range(n):
        for a in range(A):
            t = o.leaf_total(roots[r], d, int(g["best_leaf"][r, a]), gamma, mode=0)
            assert abs(g["vanilla_q"][r, a] - t) <= RTOL_BF16_SEARCH * scale[r, 0], (r, a)
    # a beam as wide as every group is the unpruned search
    w = prun(h, roots, d, cfg.gamma, P.PRUNE_BEAM, 1, A ** (d - 1), corr=0)
    for k in KEYS:
        np.testing.assert_array_equal(w[k], u[k])


def test_beam_fused_vs_materialized_leaves():
    cfg = config("C5")
    roots = cfg.roots(1)
    a = prun(handle("C5"), roots, 3, cfg.gamma, P.PRUNE_BEAM, 2, 3, corr=0)
    b = prun(handle("C5", flags=P.F_MATERIALIZE_LEAVES), roots, 3, cfg.gamma, P.PRUNE_BEAM, 2, 3, corr=0)
    np.testing.assert_array_equal(a["survivors"], b["survivors"])
    scale = np.abs(b["vanilla_q"]).max()
    assert (np.abs(a["vanilla_q"] - b["vanilla_q"]) <= 1e-4 * scale).all()


def test_root_chunking_bit_identical():
    """A workspace budget that forces several root chunks gives the same bits (keys are global)."""
    cfg = config("C2")
    roots = cfg.roots(48)
    a = prun(handle("C2"), roots, 4, cfg.gamma, P.PRUNE_BEAM, 1, 2)
    small = P.Handle.from_config(cfg, workspace_bytes_max=(8 << 20) + (200 << 10))
    b = prun(small, roots, 4, cfg.gamma, P.PRUNE_BEAM, 1, 2)
    assert b["stats"]["chunks"] > 1
    for k in KEYS + ("survivors",):
        np.testing.assert_array_equal(a[k], b[k])
    small.close()


def test_prune_rejects_bad_arguments():
    cfg = config("C2")
    h = handle("C2")
    roots = dev(cfg.roots(2))
    bad = [dict(rule=P.PRUNE_BEAM, beam=0), dict(rule=7), dict(rule=P.PRUNE_BOUND, r_lo=1.0, r_hi=0.0),
           dict(rule=P.PRUNE_BOUND, q_lo=float("nan"))]
    for kw in bad:
        with pytest.raises(P.BctsError) as e:
            h.search_pruned(roots, 2, 3, 0.99, **kw)
        assert "INVALID_ARG" in str(e.value)
    with pytest.raises(P.BctsError):
        h.search_pruned(roots, 2, 0, 0.99, P.PRUNE_BEAM, 1, 1)
