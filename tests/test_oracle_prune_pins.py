"""Pins of the oracle's early-pruned search (NEXT-4, "future work"; R30-R33).

What fixes the answers here, independent of oracle_search_pruned itself:
  * soundness of the BOUND rule (R31): with valid reward / value bounds no pruned node can hold
    its group's best leaf, so the result equals the unpruned DFS (oracle_search) exactly;
  * a beam at least as wide as every group, or no rule, is the unpruned search;
  * brute force on tiny tabular MDPs: every action path enumerated in Python, the rule applied
    to explicit path sets (structurally unlike the C level lists).
"""
import numpy as np
import pytest

from oracle import Oracle
from synth.inputs import ENV_TABULAR, NET_TABLE, Tabular, config, tabular_roots

KEYS = ("actions", "root_q", "vanilla_q", "terms", "best_leaf")


def tab_oracle(t):
    return Oracle(ENV_TABULAR, t.A, NET_TABLE, tab=t)


def random_mdp(rng, nS, A, r_scale=5, q_scale=0.1):
    nxt = rng.integers(0, nS, size=nS * A).astype(np.int32)
    rew = rng.integers(-r_scale, r_scale + 1, size=nS * A).astype(float)
    q = rng.normal(size=nS * A) * q_scale
    return Tabular(A, nxt, rew, q)


def disc(gamma, d):
    g = [1.0]
    for _ in range(d):
        g.append(g[-1] * gamma)
    return g


def brute(t, s0, d, gamma, rule, first=1, beam=1, bounds=None):
    """Python brute force (mode 0): paths as tuples, rolled out from the root each time."""
    A, g = t.A, disc(gamma, d)

    def roll(path):
        s, R = s0, 0.0
        for k, a in enumerate(path):
            R = R + g[k] * t.reward[s * A + a]
            s = int(t.next[s * A + a])
        return s, R

    def idx(path):
        f = 0
        for a in path:
            f = f * A + a
        return f

    alive = [()]
    surv = [1]
    for k in range(1, d):
        level = [p + (a,) for p in alive for a in range(A)]
        if rule and k >= first:
            kept = []
            for a0 in range(A):
                grp = [p for p in level if p[0] == a0]
                if rule == 1:
                    r_lo, r_hi, q_lo, q_hi = bounds
                    L = U = S = 0.0
                    ra, qa = max(abs(r_lo), abs(r_hi)), max(abs(q_lo), abs(q_hi))
                    for j in range(k, d):
                        L, U, S = L + g[j] * r_lo, U + g[j] * r_hi, S + g[j] * ra
                    L, U, S = L + g[d] * q_lo, U + g[d] * q_hi, S + g[d] * qa
                    Rs = [roll(p)[1] for p in grp]
                    best = max((R + L) - np.ldexp(abs(R) + S, -16) for R in Rs)
                    kept += [p for p, R in zip(grp, Rs) if not ((R + U) + np.ldexp(abs(R) + S, -16) < best)]
                else:
                    def est(p):
                        s, R = roll(p)
                        return R + g[k] * t.q[s * A:(s + 1) * A].max()
                    kept += sorted(grp, key=lambda p: (-est(p), idx(p)))[:beam]
            level = sorted(kept, key=idx)
        alive = level
        surv.append(len(alive))
    van = np.full(A, -np.inf)
    bl = np.zeros(A, np.int64)
    for p in alive:
        for a in range(A):
            s, R = roll(p + (a,))
            tot = R + g[d] * t.q[s * A:(s + 1) * A].max()
            f = idx(p + (a,))
            if tot > van[p[0] if p else a]:
                van[p[0] if p else a] = tot
                bl[p[0] if p else a] = f
    surv.append(len(alive) * A)
    return van, bl, surv


def full_counts(n, A, d):
    return [n * A ** k for k in range(d + 1)]


def test_no_rule_and_wide_beam_equal_dfs():
    rng = np.random.default_rng(30)
    for i in range(30):
        A, d = int(rng.integers(2, 5)), int(rng.integers(1, 5))
        t = random_mdp(rng, int(rng.integers(3, 40)), A)
        o = tab_oracle(t)
        roots = tabular_roots(rng.integers(0, t.nS, size=3))
        for mode in (0, 1):
            ref = o.search(roots, d, 0.9, 1.0, 1, mode=mode)
            for rule, beam in ((0, 1), (2, A ** max(d - 1, 0))):
                r = o.search_pruned(roots, d, 0.9, rule, 1, beam, beta=1.0, correction=1, mode=mode)
                for k in KEYS:
                    np.testing.assert_array_equal(r[k], ref[k])
                assert list(r["survivors"]) == full_counts(3, A, d)


def test_bound_rule_is_sound_and_prunes():
    """R31: valid bounds -> exactly the unpruned result; reward spread >> value spread -> pruning."""
    rng = np.random.default_rng(31)
    pruned_some = 0
    for i in range(40):
        A, d = int(rng.integers(2, 5)), int(rng.integers(2, 6))
        t = random_mdp(rng, int(rng.integers(3, 40)), A)
        o = tab_oracle(t)
        roots = tabular_roots(rng.integers(0, t.nS, size=2))
        b = (t.reward.min(), t.reward.max(), t.q.min(), t.q.max())
        for mode in (0, 1):
            ref = o.search(roots, d, 0.9, 1.0, 1, mode=mode)
            for first in (1, d - 1):
                r = o.search_pruned(roots, d, 0.9, 1, first, 0, *b, beta=1.0, correction=1, mode=mode)
                for k in KEYS:
                    np.testing.assert_array_equal(r[k], ref[k])
                full = full_counts(2, A, d)
                assert all(s <= f for s, f in zip(r["survivors"], full))
                pruned_some += int(r["survivors"][d] < full[d])
    assert pruned_some > 20


def test_bound_rule_loose_bounds_prune_nothing():
    rng = np.random.default_rng(32)
    t = random_mdp(rng, 20, 3)
    o = tab_oracle(t)
    r = o.search_pruned(tabular_roots([0, 5]), 4, 0.9, 1, 1, 0, -100.0, 100.0, -100.0, 100.0)
    assert list(r["survivors"]) == full_counts(2, 3, 4)


@pytest.mark.parametrize("rule", [1, 2])
def test_pruned_matches_python_brute_force(rule):
    rng = np.random.default_rng(33 + rule)
    for i in range(25):
        A, d = int(rng.integers(2, 4)), int(rng.integers(2, 5))
        t = random_mdp(rng, int(rng.integers(3, 30)), A, r_scale=int(rng.integers(0, 4)), q_scale=1.0)
        o = tab_oracle(t)
        s0 = int(rng.integers(0, t.nS))
        first = int(rng.integers(1, d))
        beam = int(rng.integers(1, 4))
        bounds = (t.reward.min(), t.reward.max(), t.q.min(), t.q.max())
        van, bl, surv = brute(t, s0, d, 0.9, rule, first, beam, bounds)
        r = o.search_pruned(tabular_roots([s0]), d, 0.9, rule, first, beam, *bounds, beta=0.0, correction=0)
        np.testing.assert_array_equal(r["vanilla_q"][0], van)
        np.testing.assert_array_equal(r["best_leaf"][0], bl)
        assert list(r["survivors"]) == surv
        assert r["actions"][0] == int(np.argmax(van))


def test_beam_one_is_greedy_by_estimate_chain():
    """beam=1 from level 1 on the C1 chain with exact Q* (R32): the depth-k estimate R + g^k max Q*
    equals Q*(s0, a0) along the optimal continuation, so each root action keeps its optimal path
    and the pruned vanilla values are the exact d-step values Q*(s0, a) (Eq. 1 with Q-hat = Q*)."""
    from synth.inputs import chain_c1
    t = chain_c1(exact=True)
    o = tab_oracle(t)
    for d in (2, 3, 4):
        for s0 in range(5):
            ref = o.search(tabular_roots([s0]), d, 0.9, 0.0, 0)
            r = o.search_pruned(tabular_roots([s0]), d, 0.9, 2, 1, 1, beta=0.0, correction=0)
            np.testing.assert_allclose(r["vanilla_q"], ref["vanilla_q"], atol=1e-12)
            np.testing.assert_allclose(r["vanilla_q"][0], t.q[s0 * 2:(s0 + 1) * 2], atol=1e-12)
            assert list(r["survivors"][1:d]) == [2] * (d - 1)


@pytest.mark.parametrize("cname,d,n", [("C2", 3, 3), ("D10", 3, 2)])
def test_hash_and_dnn_envs_wide_and_narrow_beam(cname, d, n):
    cfg = config(cname)
    o = Oracle.from_config(cfg)
    roots = cfg.roots(n)
    ref = o.search(roots, d, cfg.gamma, 1.0, 1, mode=1)
    r = o.search_pruned(roots, d, cfg.gamma, 2, 1, cfg.A ** (d - 1), mode=1)
    for k in KEYS:
        np.testing.assert_array_equal(r[k], ref[k])
    # BEAM narrower than the groups keeps exactly min(beam, group) nodes per group and level
    # (level 1: groups of one node; deeper: groups of 1*A or 2*A nodes, 2 kept)
    r2 = o.search_pruned(roots, d, cfg.gamma, 2, 1, 2, mode=1)
    exp = [n, n * cfg.A] + [n * cfg.A * 2] * (d - 2) + [n * cfg.A * 2 * cfg.A]
    assert list(r2["survivors"]) == exp
    assert all(r2["vanilla_q"].ravel() <= ref["vanilla_q"].ravel())


def test_rejects_bad_arguments():
    o = tab_oracle(random_mdp(np.random.default_rng(0), 5, 2))
    with pytest.raises(ValueError):
        o.search_pruned(tabular_roots([0]), 3, 0.9, 2, 1, 0)        # beam < 1
    with pytest.raises(ValueError):
        o.search_pruned(tabular_roots([0]), 3, 0.9, 1, 1, 0, 1.0, 0.0, 0.0, 1.0)   # r_lo > r_hi
    with pytest.raises(ValueError):
        o.search_pruned(tabular_roots([0]), 0, 0.9, 0)              # depth 0
