"""Pins of the CPU oracle against what PAPER.md and mathematics fix (not against itself).

Every test names the passage it instantiates. These run without a GPU.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import Oracle, bf16_round, penalty_eq5, bias_gap_eq4
from synth.inputs import (ENV_ATARI_HASH, ENV_INT_HASH, ENV_TABULAR, NET_TABLE, Tabular, chain_c1,
                          config, tabular_roots, worked_w1, worked_w2, atari_roots, int_roots,
                          make_weights, NET_NATURE_BF16, NET_RAINBOW_BF16)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
ROOT0 = tabular_roots([0])


def tab_oracle(t):
    return Oracle(ENV_TABULAR, t.A, NET_TABLE, tab=t)


def random_mdp(rng, nS, A, reward_ints=False):
    nxt = rng.integers(0, nS, size=nS * A)
    rew = rng.integers(-2, 3, size=nS * A).astype(float) if reward_ints else rng.normal(size=nS * A)
    q = rng.normal(size=nS * A)
    return Tabular(A, nxt.astype(np.int32), rew, q)


# ------------------------------------------------------------ worked examples
@pytest.mark.parametrize("name", ["W1", "W2"])
def test_worked_examples(name):
    g = GOLD[name]
    o = tab_oracle(worked_w1() if name == "W1" else worked_w2())
    for mode in (0, 1):
        for beta, key in ((1.0, "bcts_beta1"), (4.0, "bcts_beta4")):
            r = o.search(ROOT0, g["d"], g["gamma"], beta, 1, mode=mode)
            np.testing.assert_allclose(r["vanilla_q"][0], g["vanilla"], rtol=0, atol=1e-12)
            np.testing.assert_allclose(r["terms"][0, 1:], [g["delta_o"], g["delta_e"], g["B"]], atol=5e-7)
            np.testing.assert_allclose(r["root_q"][0], g[key], atol=5e-7)
            assert r["actions"][0] == g[key + "_action"]
        van = o.search(ROOT0, g["d"], g["gamma"], 1.0, 0, mode=mode)
        assert van["actions"][0] == g["vanilla_action"]
    # flip threshold beta* = (max_{a!=pi_o} q_a - q_pi_o) / (gamma^d B)  (SURVEY §8c "Correction + action")
    bs = g["beta_star"]
    assert o.search(ROOT0, g["d"], g["gamma"], bs - 1e-5, 1)["actions"][0] == 1
    assert o.search(ROOT0, g["d"], g["gamma"], bs + 1e-5, 1)["actions"][0] == 0


def test_w2_leaf_totals_and_reward_shift():
    g = GOLD["W2"]
    t = worked_w2()
    o = tab_oracle(t)
    tot = []
    for i in range(4):
        rec, R = o.node(ROOT0, 2, i, g["gamma"])
        q = o.qrow(rec)
        tot.append(R + g["gamma"] ** 2 * q.max())
    np.testing.assert_allclose(tot, g["leaf_totals"], atol=0)
    r = o.search(ROOT0, 2, g["gamma"], 0.0, 0)
    assert r["best_leaf"][0, 1] == g["best_leaf"]
    # all rewards +1 -> vanilla [2.75, 3.5] (S:240 reward shift c(1+gamma) at d=2)
    t2 = Tabular(t.A, t.next, t.reward + 1.0, t.q)
    np.testing.assert_allclose(tab_oracle(t2).search(ROOT0, 2, 0.5, 0, 0)["vanilla_q"][0],
                               g["vanilla_reward_plus1"], atol=0)


def test_c1_chain_table():
    g = GOLD["C1"]
    o = tab_oracle(chain_c1())
    for row in g["rows"]:
        for mode in (0, 1):
            v = o.search(ROOT0, row["d"], g["gamma"], 1.0, 0, mode=mode)
            b = o.search(ROOT0, row["d"], g["gamma"], 1.0, 1, mode=mode)
            atol = 1e-12 if mode == 0 else 1e-6
            np.testing.assert_allclose(v["root_q"][0], row["vanilla"], atol=atol)
            assert v["actions"][0] == row["vanilla_action"]
            np.testing.assert_allclose(b["root_q"][0], row["bcts"], atol=max(atol, 5e-7))
            assert b["actions"][0] == row["bcts_action"]
            if row["d"] >= 1:
                np.testing.assert_allclose(b["terms"][0, 3], row["B"], atol=5e-7)
                np.testing.assert_allclose(b["terms"][0, 1:3], [0.0, 0.2], atol=1e-6)
    # d=3 leaf totals, leaf i = base-2 digits (a0 a1 a2)  (Alg. 1 replication order, R1)
    tot = []
    for i in range(8):
        rec, R = o.node(ROOT0, 3, i, 0.9)
        tot.append(R + 0.9 ** 3 * o.qrow(rec).max())
    np.testing.assert_allclose(tot, g["d3_leaf_totals"], atol=1e-12)


def value_iteration(t: Tabular, gamma, iters=2000):
    """Q* by value iteration -- a different algorithm from tree search."""
    q = np.zeros(t.nS * t.A)
    for _ in range(iters):
        v = q.reshape(t.nS, t.A).max(1)
        q = t.reward + gamma * v[t.next]
    return q


def test_exact_q_invariant_chain():
    """Exact Q* at the leaves => Q-hat_d = Q* for every d (Bellman optimality)."""
    t = chain_c1(exact=True)
    qstar = value_iteration(t, 0.9)
    np.testing.assert_allclose(qstar, t.q, atol=1e-12)   # the fixture table *is* Q*
    o = tab_oracle(t)
    for d in range(0, 7):
        r = o.search(ROOT0, d, 0.9, 1.0, 1)
        np.testing.assert_allclose(r["vanilla_q"][0], GOLD["C1"]["qstar_root"], atol=1e-12)
        np.testing.assert_allclose(r["root_q"][0], GOLD["C1"]["qstar_root"], atol=1e-12)  # delta=0 -> B=0


def test_exact_q_invariant_random_mdps():
    rng = np.random.default_rng(11)
    for _ in range(10):
        nS, A, gamma = int(rng.integers(3, 20)), int(rng.integers(2, 5)), 0.8
        t = random_mdp(rng, nS, A)
        t = Tabular(A, t.next, t.reward, value_iteration(t, gamma))
        o = tab_oracle(t)
        roots = tabular_roots(rng.integers(0, nS, size=3))
        for d in (1, 2, 3, 4):
            r = o.search(roots, d, gamma, 1.0, 1)
            np.testing.assert_allclose(r["vanilla_q"], t.q.reshape(nS, A)[roots], atol=1e-9)
            np.testing.assert_allclose(r["terms"][:, 1:3], 0, atol=1e-9)  # delta ~ 0


# ------------------------------------------------------------ SPEC examples
def test_spec_s207_return_rule():
    """A=2,d=2, leaf totals [1,3,7,2] -> flat argmax 2 -> root action floor(2/2)=1."""
    gamma = 0.5
    nxt = [[1, 2], [3, 4], [5, 6]] + [[k, k] for k in range(3, 7)]
    rew = np.zeros((7, 2))
    q = np.zeros((7, 2))
    for i, tot in enumerate(GOLD["SPEC"]["S207"]["leaf_totals"]):
        q[3 + i] = [tot / gamma ** 2, 0.0]
    o = tab_oracle(Tabular(2, np.array(nxt, np.int32).ravel(), rew.ravel(), q.ravel()))
    r = o.search(ROOT0, 2, gamma, 0.0, 0)
    assert r["actions"][0] == 1
    assert r["best_leaf"][0, 1] == 2
    np.testing.assert_allclose(r["vanilla_q"][0], [3, 7])


def test_spec_s208_all_zero():
    rng = np.random.default_rng(0)
    t = random_mdp(rng, 9, 3)
    t = Tabular(3, t.next, np.zeros_like(t.reward), np.zeros_like(t.q))
    r = tab_oracle(t).search(tabular_roots([0, 4]), 3, 0.9, 1.0, 1)
    assert (r["root_q"] == 0).all() and (r["actions"] == 0).all()


def test_spec_s224_depth1_closed_form_and_s226_leaf_shift():
    rng = np.random.default_rng(1)
    for _ in range(5):
        t = random_mdp(rng, 12, 3)
        o = tab_oracle(t)
        roots = tabular_roots(np.arange(12))
        r = o.search(roots, 1, 0.7, 0.0, 0)
        Q = t.q.reshape(12, 3)
        exp = t.reward.reshape(12, 3) + 0.7 * Q[t.next.reshape(12, 3)].max(-1)
        np.testing.assert_allclose(r["vanilla_q"], exp, atol=1e-12)
        for d in (1, 2, 3):
            base = o.search(roots, d, 0.7, 0.0, 0)["vanilla_q"]
            sh = tab_oracle(Tabular(3, t.next, t.reward, t.q + 2.5)).search(roots, d, 0.7, 0.0, 0)["vanilla_q"]
            np.testing.assert_allclose(sh - base, 0.7 ** d * 2.5, atol=1e-12)


def test_spec_s240_reward_shift():
    rng = np.random.default_rng(2)
    t = random_mdp(rng, 15, 4)
    roots = tabular_roots(np.arange(15))
    for d in (1, 2, 3, 4):
        a = tab_oracle(t).search(roots, d, 0.9, 0.0, 0)
        b = tab_oracle(Tabular(4, t.next, t.reward + 1.5, t.q)).search(roots, d, 0.9, 0.0, 0)
        np.testing.assert_allclose(b["vanilla_q"] - a["vanilla_q"], 1.5 * (1 - 0.9 ** d) / (1 - 0.9), atol=1e-12)
        assert (a["actions"] == b["actions"]).all()


def test_spec_s159_bellman_stats():
    """A=2, delta=[1,3], pi_o=0 -> (delta_o, delta_e) = (1,3)."""
    t = Tabular(2, np.array([1, 2, 1, 1, 2, 2], np.int32), np.array([1.0, 3.0, 0, 0, 0, 0]),
                np.zeros(6))
    r = tab_oracle(t).search(ROOT0, 1, 0.5, 1.0, 1)
    assert r["terms"][0, 0] == 0
    np.testing.assert_allclose(r["terms"][0, 1:3], [1.0, 3.0], atol=0)


def test_spec_s348_correction_arithmetic():
    """root_q [5, 5.4], pi_o=0, penalty 0.5 -> [5, 4.9], action 0 (Eq. 3)."""
    g = 0.5
    # d=1: vanilla_q[a] = r_a + g*max Q(s1^a); q0=[6,0] -> pi_o=0; leaves Q rows give vanilla [5, 5.4]
    t = Tabular(2, np.array([1, 2, 1, 1, 2, 2], np.int32), np.array([5.0, 5.4, 0, 0, 0, 0]),
                np.array([6.0, 0.0, 0, 0, 0, 0]))
    o = tab_oracle(t)
    base = o.search(ROOT0, 1, g, 1.0, 1)
    B = base["terms"][0, 3]
    beta = 0.5 / (g * B)
    r = o.search(ROOT0, 1, g, beta, 1)
    np.testing.assert_allclose(r["vanilla_q"][0], [5.0, 5.4], atol=1e-12)
    np.testing.assert_allclose(r["root_q"][0], [5.0, 4.9], atol=1e-12)
    assert r["actions"][0] == 0


# ------------------------------------------------------------ Eq. 4 / Eq. 5
def test_eq5_closed_forms():
    # delta_e=2, delta_o=0, A=e, d=1 -> 2 - 2/sqrt(8) = 1.2928932...  (A=e is not an int:
    # evaluate with A such that log A = 1 through the equal-delta identity instead)
    assert abs((2.0 - 2.0 / math.sqrt(8)) - GOLD["SPEC"]["S325"]["B"]) < 1e-6
    for A in (2, 3, 6, 18):
        for d in (1, 2, 3, 4, 5):
            # d=1, delta_o=0: B = sqrt(ln A)*de - de/sqrt(8)
            if d == 1:
                assert abs(penalty_eq5(2.0, 0.0, A, 1) - (2 * math.sqrt(math.log(A)) - 2 / math.sqrt(8))) < 1e-12
            # S:324 equal deltas: sqrt(ln A) * delta * (sqrt(d) - sqrt(d-1))
            assert abs(penalty_eq5(0.7, 0.7, A, d) - math.sqrt(math.log(A)) * 0.7 * (math.sqrt(d) - math.sqrt(d - 1))) < 1e-12


def test_eq5_equals_eq4_under_sigma_delta_over_sqrt2():
    """Eq. 5 is Eq. 4 with sigma = delta/sqrt(2) substituted (Prop. 1)."""
    rng = np.random.default_rng(3)
    for _ in range(2000):
        de, do = rng.uniform(0, 5, size=2)
        A, d = int(rng.integers(2, 20)), int(rng.integers(1, 9))
        assert abs(penalty_eq5(de, do, A, d) - bias_gap_eq4(do / math.sqrt(2), de / math.sqrt(2), A, d)) < 1e-12


def test_beta_zero_and_correction_off_are_vanilla():
    rng = np.random.default_rng(4)
    t = random_mdp(rng, 20, 3)
    o = tab_oracle(t)
    roots = tabular_roots(np.arange(20))
    for d in (1, 2, 3):
        v = o.search(roots, d, 0.9, 1.0, 0)
        b0 = o.search(roots, d, 0.9, 0.0, 1)
        assert (v["root_q"] == v["vanilla_q"]).all()
        assert (b0["root_q"] == v["vanilla_q"]).all() and (b0["actions"] == v["actions"]).all()
        b = o.search(roots, d, 0.9, 1.0, 1)
        # pi_o's value is never changed (Eq. 3 first case)
        pio = b["terms"][:, 0].astype(int)
        np.testing.assert_array_equal(b["root_q"][np.arange(20), pio], v["vanilla_q"][np.arange(20), pio])


def test_depth0_is_greedy():
    """d=0 is the base agent itself: root Q = Q-hat(s0,.), action = first argmax."""
    rng = np.random.default_rng(5)
    t = random_mdp(rng, 10, 4)
    r = tab_oracle(t).search(tabular_roots(np.arange(10)), 0, 0.9, 1.0, 1)
    Q = t.q.reshape(10, 4)
    np.testing.assert_array_equal(r["root_q"], Q)
    np.testing.assert_array_equal(r["actions"], Q.argmax(1))


# ------------------------------------------------------------ brute force == DFS
def test_bruteforce_equals_dfs_random_mdps():
    """SPEC acceptance 1: over random deterministic MDPs, d in [1,5]."""
    rng = np.random.default_rng(6)
    for i in range(50):
        A = int(rng.integers(2, 5))
        nS = int(rng.integers(2, 50))
        t = random_mdp(rng, nS, A, reward_ints=bool(i % 2))
        o = tab_oracle(t)
        roots = tabular_roots(rng.integers(0, nS, size=2))
        d = int(rng.integers(1, 6))
        for mode in (0, 1):
            a = o.search(roots, d, 0.9, 1.0, 1, mode=mode)
            b = o.search(roots, d, 0.9, 1.0, 1, mode=mode, brute=True)
            for k in ("actions", "root_q", "vanilla_q", "terms", "best_leaf"):
                np.testing.assert_array_equal(a[k], b[k])


@pytest.mark.parametrize("cname,d,n", [("C2", 3, 4), ("C3", 1, 1)])
def test_bruteforce_equals_dfs_hash_envs(cname, d, n):
    cfg = config(cname)
    o = Oracle.from_config(cfg)
    roots = cfg.roots(n)
    a = o.search(roots, d, cfg.gamma, 1.0, 1, mode=1, threads=4)
    b = o.search(roots, d, cfg.gamma, 1.0, 1, mode=1, brute=True)
    for k in ("actions", "root_q", "vanilla_q", "best_leaf"):
        np.testing.assert_array_equal(a[k], b[k])


def test_mirror_mode_close_to_fp64():
    cfg = config("C2")
    o = Oracle.from_config(cfg)
    roots = cfg.roots(8)
    a = o.search(roots, 3, cfg.gamma, 1.0, 1, mode=0)
    b = o.search(roots, 3, cfg.gamma, 1.0, 1, mode=1)
    scale = np.maximum(np.abs(a["root_q"]).max(1, keepdims=True), 1e-6)
    assert (np.abs(a["root_q"] - b["root_q"]) <= 1e-5 * scale).all()


# ------------------------------------------------------------ env + nets
def test_tabular_chain_transitions():
    o = tab_oracle(chain_c1())
    rec, r = o.step(tabular_roots([2]), 1)
    assert rec.view(np.int32)[0] == 3 and r == 0.0
    for a in (0, 1):
        rec, r = o.step(tabular_roots([4]), a)
        assert rec.view(np.int32)[0] == 4 and r == 0.0        # absorbing terminal S:52


def test_atari_step_frame_shift_and_rewards():
    """Frame stacking: child frames 0..2 are parent frames 1..3; reward P(+-1)=1/8."""
    cfg = config("C3")
    o = Oracle.from_config(cfg)
    root = atari_roots(1, 77)[0]
    rewards = []
    for a in range(18):
        child, r = o.step(root, a)
        pw = root[16:].view(np.uint32)
        cw = child[16:].view(np.uint32)
        np.testing.assert_array_equal(cw & 0x00FFFFFF, pw >> 8)
        assert child[:8].tobytes() != root[:8].tobytes()
        rewards.append(r)
        again, r2 = o.step(root, a)
        assert again.tobytes() == child.tobytes() and r2 == r          # determinism
    # statistics over many steps
    keys = []
    rec = root
    cnt = {-1.0: 0, 0.0: 0, 1.0: 0}
    for i in range(400):
        rec, r = o.step(rec, i % 18)
        cnt[r] += 1
        keys.append(rec[:8].tobytes())
    assert len(set(keys)) == 400
    assert 25 <= cnt[1.0] <= 80 and 25 <= cnt[-1.0] <= 80


def test_int_hash_step_properties():
    cfg = config("C2")
    o = Oracle.from_config(cfg)
    rec = int_roots(1, 9)[0]
    cnt = {-1.0: 0, 0.0: 0, 1.0: 0}
    for i in range(800):
        nxt, r = o.step(rec, i % 4)
        assert nxt.tobytes() != rec.tobytes()
        cnt[r] += 1
        rec = nxt
    assert 140 <= cnt[1.0] <= 260 and 140 <= cnt[-1.0] <= 260   # P(+-1) = 1/4 each


def test_bf16_round_matches_torch():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(7)
    x = np.concatenate([rng.normal(size=3000) * 10.0 ** rng.integers(-6, 6, size=3000),
                        np.float32(np.array([1.0, 1.00390625, 1.005859375, 1.0078125, -3.3e-3]))]).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    got = np.array([bf16_round(float(v)) for v in x])
    np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("net", [NET_NATURE_BF16, NET_RAINBOW_BF16])
def test_conv_net_matches_torch_functional(net):
    """Oracle conv/linear stack vs torch.nn.functional.conv2d/linear in float64 (library routine)."""
    torch = pytest.importorskip("torch")
    F = torch.nn.functional
    A = 6
    blob, w = make_weights(net, A, 1234)
    o = Oracle(ENV_ATARI_HASH, A, net, weights=blob)
    rec = atari_roots(2, 99)

    def bf(t):
        return t.to(torch.float32).to(torch.bfloat16).to(torch.float64)

    def W(name):
        return torch.from_numpy(w[name].astype(np.float64))

    for i in range(2):
        words = rec[i, 16:].view(np.uint32).reshape(84, 84)
        x = np.stack([(words >> (8 * c)) & 0xFF for c in range(4)]).astype(np.float64)[None]
        x = torch.from_numpy(x)
        h = bf(F.relu(F.conv2d(x, bf(W("conv1.w")), W("conv1.b"), stride=4)))
        h = bf(F.relu(F.conv2d(h, bf(W("conv2.w")), W("conv2.b"), stride=2)))
        h = bf(F.relu(F.conv2d(h, bf(W("conv3.w")), W("conv3.b"), stride=1))).reshape(1, -1)
        if net == NET_NATURE_BF16:
            h = bf(F.relu(F.linear(h, bf(W("fc1.w")), W("fc1.b"))))
            q = F.linear(h, bf(W("fc2.w")), W("fc2.b"))[0]
        else:
            hv = bf(F.relu(F.linear(h, bf(W("fc_h_v.w")), W("fc_h_v.b"))))
            ha = bf(F.relu(F.linear(h, bf(W("fc_h_a.w")), W("fc_h_a.b"))))
            v = F.linear(hv, bf(W("fc_z_v.w")), W("fc_z_v.b")).reshape(1, 51)
            adv = F.linear(ha, bf(W("fc_z_a.w")), W("fc_z_a.b")).reshape(A, 51)
            p = torch.softmax(v + adv - adv.mean(0, keepdim=True), dim=1)
            q = (p * torch.linspace(-10, 10, 51, dtype=torch.float64)).sum(1)
        got = o.qrow(rec[i])
        scale = float(q.abs().max())
        assert np.abs(got - q.numpy()).max() <= 2e-3 * scale + 1e-7, (got, q)
        if net == NET_RAINBOW_BF16:
            assert (got >= -10).all() and (got <= 10).all()


def test_node_replay_consistent_with_steps():
    cfg = config("C3")
    o = Oracle.from_config(cfg)
    root = cfg.roots(1)[0]
    A = cfg.A
    idx = 5 * A + 11                      # a0=5, a1=11
    c1, r1 = o.step(root, 5)
    c2, r2 = o.step(c1, 11)
    rec, R = o.node(root, 2, idx, cfg.gamma)
    assert rec.tobytes() == c2.tobytes()
    assert R == r1 + cfg.gamma * r2


def test_env_golden_vectors_frozen():
    """The oracle's env step must not drift from the frozen golden vectors."""
    import hashlib
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "env_golden.json")))
    for name in ("C2", "C3"):
        cfg = config(name)
        o = Oracle.from_config(cfg)
        roots = cfg.roots(len(gold[name]["sequences"]))
        for s in gold[name]["sequences"]:
            rec = roots[s["root"]]
            for a, h, rw in zip(s["actions"], s["sha256"], s["rewards"]):
                rec, r = o.step(rec, a)
                assert hashlib.sha256(rec.tobytes()).hexdigest() == h and r == rw


# ------------------------------------------------------------ NEXT-2: Lemma 2 exact biases
def test_inv_norm_cdf_vs_scipy_and_roundtrip():
    """Phi^-1 (App. A.1) against scipy.stats.norm.ppf and Phi(Phi^-1(p)) = p via math.erfc."""
    from scipy.stats import norm
    from oracle import inv_norm_cdf
    rng = np.random.default_rng(8)
    ps = np.concatenate([rng.uniform(1e-12, 1 - 1e-12, 2000), [0.5, 0.975, 1e-10, 1 - 1e-10, 0.02425, 0.97575]])
    for p in ps:
        z = inv_norm_cdf(p)
        assert abs(z - norm.ppf(p)) <= 1e-9 * max(1.0, abs(z))
        assert abs(0.5 * math.erfc(-z / math.sqrt(2)) - p) <= 1e-12 * max(p, 1e-3)
    assert abs(inv_norm_cdf(0.975) - 1.959964) < 1e-6          # S:279 example
    assert inv_norm_cdf(0.5) == 0.0 or abs(inv_norm_cdf(0.5)) < 1e-15


def test_lemma2_special_cases_and_ordering():
    """B_o = 0 at d=1; B_e = 0 at d=1, A=2; 0 <= B_o < B_e for sigma_o < sigma_e (Lemma 2)."""
    from oracle import B_n, bias_exact
    assert B_n(1) == 0.0
    for A in (2, 3, 4, 6, 18):
        assert bias_exact(1.0, 0.0, A, 1) == 0.0                   # B_o(d=1) = 0 -> gap = -B_o = 0 at sigma_e = 0
    assert bias_exact(0.3, 2.0, 2, 1) == 0.0                       # both single-element maxima at d=1, A=2
    for A in (2, 3, 4, 18):
        for d in range(1, 9):
            n_o, n_e = A ** (d - 1), A ** d - A ** (d - 1)
            bo, be = 0.7 * B_n(n_o), 1.3 * B_n(n_e)
            assert 0.0 <= bo < be or (A == 2 and d == 1)
    # B(n) is increasing (it is composed of two increasing functions)
    vals = [B_n(n) for n in (2, 3, 10, 100, 1e4, 1e6)]
    assert all(x < y for x, y in zip(vals, vals[1:]))


def test_lemma2_vs_library_formula_and_eq4_gap():
    """Exact gap via scipy's ppf in the App. A.2 formula; the Eq. 4 approximation's relative error at
    A=3, sigma_o=1, sigma_e=4 (App. A.6 setup) shrinks with d (+113%, +24%, +13%, +8%)."""
    from scipy.stats import norm
    from oracle import bias_exact, bias_gap_eq4
    gem = 0.5772156649015329

    def Bn(n):
        return 0.0 if n == 1 else gem * norm.ppf(1 - 1 / (math.e * n)) + (1 - gem) * norm.ppf(1 - 1 / n)

    for A in (2, 3, 18):
        for d in (1, 2, 3, 4, 5):
            ref = 4.0 * Bn(A ** d - A ** (d - 1)) - 1.0 * Bn(A ** (d - 1))
            assert abs(bias_exact(1.0, 4.0, A, d) - ref) <= 1e-9 * max(1.0, abs(ref))
    errs = [bias_gap_eq4(1, 4, 3, d) / bias_exact(1, 4, 3, d) - 1 for d in range(1, 7)]
    np.testing.assert_allclose(errs[:4], [1.13, 0.24, 0.13, 0.08], atol=0.01)
    assert all(a > b > 0 for a, b in zip(errs, errs[1:]))


def test_exact_bias_worked_examples():
    """W1: exact gap 0 (d=1, A=2); W2: 0.3675 -> BCTS-exact keeps vanilla's choice."""
    o = tab_oracle(worked_w1())
    r = o.search(ROOT0, 1, 0.5, 1.0, 2)
    assert r["terms"][0, 3] == 0.0
    np.testing.assert_array_equal(r["root_q"], r["vanilla_q"])
    o2 = tab_oracle(worked_w2())
    r2 = o2.search(ROOT0, 2, 0.5, 1.0, 2)
    assert abs(r2["terms"][0, 3] - 0.3675225) < 1e-6
    np.testing.assert_allclose(r2["root_q"][0], [1.25, 2.0 - 0.25 * 0.3675225285], atol=1e-9)


# ------------------------------------------------------------ NEXT-1: random-DNN forward model
def _dnn_torch(cfg):
    """The paper's DNN forward model as a stock torch.nn stack in fp64: three hidden
    layers of width 100 over [state(100); onehot(a)], ReLU, linear head 101 = (next state, reward)."""
    import torch
    from synth.inputs import make_env_weights, env_weight_specs
    blob = make_env_weights(cfg).astype(np.float64)
    specs = env_weight_specs(cfg.A)
    off, ts = 0, []
    for _, shape, _ in specs:
        n = int(np.prod(shape))
        ts.append(torch.from_numpy(blob[off:off + n].reshape(shape)))
        off += n
    layers = []
    for L in range(4):
        lin = torch.nn.Linear(ts[2 * L].shape[1], ts[2 * L].shape[0]).double()
        with torch.no_grad():
            lin.weight.copy_(ts[2 * L])
            lin.bias.copy_(ts[2 * L + 1])
        layers += [lin, torch.nn.ReLU()] if L < 3 else [lin]
    return torch.nn.Sequential(*layers)


@pytest.mark.parametrize("cname", ["D2", "D10"])
def test_dnn_step_matches_torch_sequential(cname):
    import torch
    cfg = config(cname)
    o = Oracle.from_config(cfg)
    net = _dnn_torch(cfg)
    roots = cfg.roots(5)
    for r in range(5):
        for a in range(cfg.A):
            x = torch.cat([torch.from_numpy(roots[r].astype(np.float64)),
                           torch.nn.functional.one_hot(torch.tensor(a), cfg.A).double()])
            ref = net(x).detach().numpy()
            rec, rew = o.step(roots[r], a)                  # fp32 mirror
            np.testing.assert_allclose(rec.view(np.float32), ref[:100], rtol=0, atol=2e-6)
            assert abs(rew - ref[100]) <= 2e-6
            rec0, R0 = o.node(roots[r], 1, a, cfg.gamma, mode=0)   # fp64 chain, state rounded to fp32
            np.testing.assert_allclose(rec0.view(np.float32), ref[:100].astype(np.float32), rtol=1e-6, atol=1e-7)
            assert abs(R0 - ref[100]) <= 1e-12


def test_dnn_mlp_leaf_value_matches_torch():
    """Leaf value Q-hat on the DNN env: MLP2 100-256-A over the raw fp32 state features (R27)."""
    import torch
    cfg = config("D10")
    o = Oracle.from_config(cfg)
    _, v = cfg.weights()
    s = cfg.roots(3)
    x = torch.from_numpy(s.astype(np.float64))
    h = torch.relu(x @ torch.from_numpy(v["l1.w"].astype(np.float64)).T + torch.from_numpy(v["l1.b"].astype(np.float64)))
    q = (h @ torch.from_numpy(v["l2.w"].astype(np.float64)).T + torch.from_numpy(v["l2.b"].astype(np.float64))).numpy()
    for r in range(3):
        np.testing.assert_allclose(o.qrow(s[r], mode=0), q[r], rtol=0, atol=1e-12)
        np.testing.assert_allclose(o.qrow(s[r], mode=1), q[r], rtol=0, atol=5e-6)


@pytest.mark.parametrize("cname,d", [("D2", 5), ("D10", 2)])
def test_dnn_bruteforce_equals_dfs_and_mirror_close(cname, d):
    cfg = config(cname)
    o = Oracle.from_config(cfg)
    roots = cfg.roots(3)
    for mode in (0, 1):
        a = o.search(roots, d, cfg.gamma, 1.0, 1, mode=mode, threads=4)
        b = o.search(roots, d, cfg.gamma, 1.0, 1, mode=mode, brute=True)
        for k in ("actions", "root_q", "vanilla_q", "best_leaf"):
            np.testing.assert_array_equal(a[k], b[k])
    f64 = o.search(roots, d, cfg.gamma, 1.0, 1, mode=0)
    f32 = o.search(roots, d, cfg.gamma, 1.0, 1, mode=1)
    assert np.abs(f64["vanilla_q"] - f32["vanilla_q"]).max() < 1e-4


def test_int_hash_mlp2_leaf_value_matches_torch():
    """C2 leaf value: MLP2 64-256-4 over x_j = (byte j of the 64-byte INT_HASH state) / 256 (SURVEY §8d,
    little-endian bytes of the 16 u32 words), pinned to torch.nn.functional.linear in float64 (a library
    routine). Covers roots and level-2 states so the feature map is exercised on stepped states too."""
    import torch
    F = torch.nn.functional
    cfg = config("C2")
    o = Oracle.from_config(cfg)
    _, v = cfg.weights()
    W = {k: torch.from_numpy(x.astype(np.float64)) for k, x in v.items()}
    states = list(cfg.roots(4))
    for i in (0, 5, 15):
        rec, _ = o.node(cfg.roots(1)[0], 2, i, float(np.float32(cfg.gamma)), mode=1)
        states.append(rec.view(np.uint32))
    for s in states:
        x = torch.from_numpy(np.ascontiguousarray(s).view(np.uint8).astype(np.float64)) / 256.0
        q = F.linear(F.relu(F.linear(x, W["l1.w"], W["l1.b"])), W["l2.w"], W["l2.b"]).numpy()
        np.testing.assert_allclose(o.qrow(s, mode=0), q, rtol=0, atol=1e-12)
        np.testing.assert_allclose(o.qrow(s, mode=1), q, rtol=0, atol=5e-6)


# ------------------------------------------------ hash env steps pinned to published hash vectors
# ENV_SPEC builds both synthetic envs from two standard mixers. They are pinned here to
# values published with the mixers themselves, so the env steps below are checked against a reference
# that is not the oracle's code: splitmix64 (Steele, Lea & Flood 2014 / Vigna's SplitMix64) from seed
# 1234567 yields 6457827717110365317, 3203168211198807973, 9817491932198370423, 4593380528125082431,
# 16408922859458223821; MurmurHash3's fmix32 maps 0 -> 0 and 1 -> 0x514E28B7.
_M64 = (1 << 64) - 1


def _splitmix64_finalizer(z):
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & _M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _fmix32(h):
    h ^= h >> 16
    h = (h * 0x85EBCA6B) & 0xFFFFFFFF
    h ^= h >> 13
    h = (h * 0xC2B2AE35) & 0xFFFFFFFF
    return h ^ (h >> 16)


def test_mixers_match_published_vectors():
    s, out = 1234567, []
    for _ in range(5):
        s = (s + 0x9E3779B97F4A7C15) & _M64
        out.append(_splitmix64_finalizer(s))
    assert out == [6457827717110365317, 3203168211198807973, 9817491932198370423, 4593380528125082431,
                   16408922859458223821]
    assert _fmix32(0) == 0 and _fmix32(1) == 0x514E28B7


def test_atari_hash_step_is_the_env_spec_over_splitmix64():
    """ATARI_HASH step (ENV_SPEC, frame stack P:355) with the pinned splitmix64: k' = mix64(key ^
    0x9E3779B97F4A7C15 (a + 1)); pixel p: new top byte = old top byte ^ byte p % 8 of mix64(k' + p / 8),
    the other three frames shift down; r = +1 / -1 / 0 from k' >> 61 = 7 / 0 / else."""
    cfg = config("C3")
    o = Oracle.from_config(cfg)
    roots = atari_roots(3, 4242)
    for rec in roots:
        key = int(rec[:8].view(np.uint64)[0])
        words = rec[16:].view(np.uint32).astype(np.uint64)
        for a in (0, 7, 17):
            child, r = o.step(rec, a)
            k2 = _splitmix64_finalizer(key ^ ((0x9E3779B97F4A7C15 * (a + 1)) & _M64))
            assert int(child[:8].view(np.uint64)[0]) == k2
            assert r == (1.0 if k2 >> 61 == 7 else -1.0 if k2 >> 61 == 0 else 0.0)
            noise = np.array([(_splitmix64_finalizer((k2 + p // 8) & _M64) >> (8 * (p % 8))) & 0xFF
                              for p in range(words.size)], dtype=np.uint64)
            want = (words >> np.uint64(8)) | (((words >> np.uint64(24)) ^ noise) << np.uint64(24))
            np.testing.assert_array_equal(child[16:].view(np.uint32), want.astype(np.uint32))


def test_int_hash_step_is_the_env_spec_over_fmix32():
    """INT_HASH step (ENV_SPEC) with the pinned fmix32: s'[w] = fmix32(s[w] ^ rotl(s[w + 1 mod 16], 13) ^
    0x9E3779B9 (a + 1) ^ 0x85EBCA6B w); r = +1 / -1 / 0 from s'[0] >> 30 = 3 / 0 / else."""
    cfg = config("C2")
    o = Oracle.from_config(cfg)
    for rec in int_roots(4, 4343):
        s = [int(x) for x in rec.view(np.uint32)]
        for a in range(4):
            child, r = o.step(rec, a)
            want = []
            for w in range(16):
                nx = s[(w + 1) % 16]
                rot = ((nx << 13) | (nx >> 19)) & 0xFFFFFFFF
                v = s[w] ^ rot ^ ((0x9E3779B9 * (a + 1)) & 0xFFFFFFFF) ^ ((0x85EBCA6B * w) & 0xFFFFFFFF)
                want.append(_fmix32(v))
            assert [int(x) for x in child.view(np.uint32)] == want
            t = want[0] >> 30
            assert r == (1.0 if t == 3 else -1.0 if t == 0 else 0.0)
