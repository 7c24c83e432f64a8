"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, element by element.

Tolerances (BASELINE.json north_star; DESIGN.md §2 R18/R19):
  * tree indexing, env states, rewards, actions on fp32 paths: bit-exact;
  * root Q on fp32 paths (C1, C2): within 1e-5 relative of the fp64 oracle;
  * bf16 tensor-core leaf path (C3-C5): within 2e-2 relative on root Q, >= 99.9%
    action agreement under the near-tie rule.
"""
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
from synth.inputs import (ENV_ATARI_HASH, NET_NATURE_BF16, NET_RAINBOW_BF16, Config, chain_c1,  # noqa: E402
                          config, make_weights, tabular_roots, worked_w1, worked_w2, atari_roots)

THREADS = os.cpu_count() or 1
DEV = torch.device("cuda", 0)
RTOL_F32, RTOL_BF16 = 1e-5, 2e-2
RTOL_BF16_SEARCH = 1e-3   # root Q of whole searches: observed <= 2e-5 (bf16 RNE flips); a broken trunk shows ~2e-3+ because random-init Q is flat across leaves


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).copy()).to(DEV)


def run(h, roots_np, d, gamma, beta=1.0, corr=1):
    n = roots_np.shape[0]
    out = h.search(dev(roots_np), n, d, gamma, beta, corr, extra=True)
    torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in out.items()}


_handles = {}


def handle(name, **kw):
    cfg = config(name) if isinstance(name, str) else name
    key = (cfg.name, cfg.A, cfg.net, tuple(sorted(kw.items())))
    if key not in _handles:
        _handles[key] = P.Handle.from_config(cfg, **kw)
    return _handles[key]


# ------------------------------------------------------------------ fp32 paths
@pytest.mark.parametrize("tabname", ["C1", "W1", "W2"])
def test_tabular_all_depths(tabname):
    tab = {"C1": chain_c1(), "W1": worked_w1(), "W2": worked_w2()}[tabname]
    gamma = 0.9 if tabname == "C1" else 0.5
    h = P.Handle(P.ENV_TABULAR, 2, P.NET_TABLE, tab=tab)
    o = Oracle(1, 2, 1, tab=tab)
    roots = tabular_roots([0])
    for d in range(0, 6):
        for corr in (0, 1):
            for beta in (0.0, 1.0, 4.0):
                g = run(h, roots, d, np.float32(gamma), beta, corr)
                m = o.search(roots, d, float(np.float32(gamma)), beta, corr, mode=1)
                r = o.search(roots, d, float(np.float32(gamma)), beta, corr, mode=0)
                np.testing.assert_array_equal(g["vanilla_q"], m["vanilla_q"].astype(np.float32))
                np.testing.assert_array_equal(g["actions"], r["actions"])
                assert rel_err(g["root_q"], r["root_q"]).max() <= RTOL_F32
                if d >= 1:
                    np.testing.assert_array_equal(g["best_leaf"], m["best_leaf"])
                if corr or d == 0:
                    assert g["terms"][0, 0] == r["terms"][0, 0]
                    np.testing.assert_allclose(g["terms"][0, 1:], r["terms"][0, 1:], rtol=1e-5, atol=1e-6)
    h.close()


def test_c1_headline_flip():
    """C1: vanilla d=3 picks 0 with [0.8019, 0.729]; BCTS picks 1 with [0.6432006, 0.729]."""
    h = P.Handle(P.ENV_TABULAR, 2, P.NET_TABLE, tab=chain_c1())
    v = run(h, tabular_roots([0]), 3, 0.9, 1.0, 0)
    b = run(h, tabular_roots([0]), 3, 0.9, 1.0, 1)
    assert v["actions"][0] == 0 and b["actions"][0] == 1
    np.testing.assert_allclose(v["root_q"][0], [0.8019, 0.729], atol=2e-6)
    np.testing.assert_allclose(b["root_q"][0], [0.6432006, 0.729], atol=2e-6)


@pytest.mark.parametrize("cname,n,levels", [("C1", 1, 4), ("C2", 3, 3), ("C3", 2, 2)])
def test_level_states_bit_exact(cname, n, levels):
    """Every node of every level: state record and cumulative reward bit-exact (Alg. 1)."""
    cfg = config(cname)
    tab = chain_c1() if cname == "C1" else None
    h = handle(cname) if tab is None else P.Handle.from_config(cfg, tab=tab)
    o = Oracle.from_config(cfg, tab=tab)
    roots = cfg.roots(n)
    for level in range(levels + 1):
        st, cum = h.expand(dev(roots), n, level, np.float32(cfg.gamma))
        st, cum = st.cpu().numpy(), cum.cpu().numpy()
        per = cfg.A ** level
        for r in range(n):
            for i in range(per):
                rec, R = o.node(roots[r], level, i, float(np.float32(cfg.gamma)), mode=1)
                assert st[r * per + i].tobytes() == rec.tobytes(), (level, r, i)
                assert cum[r * per + i] == np.float32(R), (level, r, i)


@pytest.mark.parametrize("corr", [0, 1])
def test_c2_full_config(corr):
    """C2 at its BASELINE size: 256 roots, A=4, d=4, MLP2 fp32 -- bit-exact vs the fp32 mirror."""
    cfg = config("C2")
    h = handle("C2")
    o = Oracle.from_config(cfg)
    roots = cfg.roots()
    gamma = float(np.float32(cfg.gamma))
    g = run(h, roots, cfg.depth, cfg.gamma, cfg.beta, corr)
    m = o.search(roots, cfg.depth, gamma, cfg.beta, corr, mode=1, threads=THREADS)
    r = o.search(roots, cfg.depth, gamma, cfg.beta, corr, mode=0, threads=THREADS)
    np.testing.assert_array_equal(g["vanilla_q"], m["vanilla_q"].astype(np.float32))
    np.testing.assert_array_equal(g["best_leaf"], m["best_leaf"])
    np.testing.assert_array_equal(g["actions"], m["actions"])
    np.testing.assert_array_equal(g["actions"], r["actions"])
    assert rel_err(g["root_q"], r["root_q"]).max() <= RTOL_F32
    if corr:
        np.testing.assert_array_equal(g["terms"][:, 0], r["terms"][:, 0])
        assert (np.abs(g["terms"][:, 1:] - r["terms"][:, 1:]) <= 1e-5 * np.maximum(1, np.abs(r["terms"][:, 1:]))).all()
    st = g["stats"]
    assert st["leaves"] == 256 * 4 ** 4


# ------------------------------------------------------------------ bf16 paths
def bf16_compare(g, r, what):
    err = rel_err(g["root_q"], r["root_q"])
    verr = rel_err(g["vanilla_q"], r["vanilla_q"])
    frac, exact, near = action_agreement(g["actions"], r["root_q"], RTOL_BF16)
    print(f"{what}: max rel err root_q {err.max():.2e} vanilla {verr.max():.2e}; actions {frac:.4f} "
          f"(exact {exact}, near-ties {near})")
    assert err.max() <= RTOL_BF16_SEARCH and verr.max() <= RTOL_BF16_SEARCH
    assert frac >= 0.999


@pytest.mark.parametrize("cname,n,d", [("C3", 3, 2), ("C4", 3, 3), ("C5", 2, 2), ("C3", 1, 1)])
def test_conv_nets_small_trees(cname, n, d):
    cfg = config(cname)
    h = handle(cname)
    o = Oracle.from_config(cfg)
    roots = cfg.roots(n)
    for corr in (0, 1):
        g = run(h, roots, d, cfg.gamma, cfg.beta, corr)
        r = o.search(roots, d, float(np.float32(cfg.gamma)), cfg.beta, corr, mode=0, threads=THREADS)
        bf16_compare(g, r, f"{cname} n={n} d={d} corr={corr}")
        if corr:
            np.testing.assert_array_equal(g["terms"][:, 0], r["terms"][:, 0])


@pytest.mark.parametrize("net,A,n,d", [(NET_RAINBOW_BF16, 7, 2, 2), (NET_RAINBOW_BF16, 2, 3, 3),
                                        (NET_RAINBOW_BF16, 33, 1, 1), (NET_NATURE_BF16, 5, 2, 2),
                                        (NET_RAINBOW_BF16, 64, 1, 2), (NET_NATURE_BF16, 64, 2, 1)])
def test_conv_nets_unusual_action_counts(net, A, n, d):
    """Action counts that are not multiples of the head's 4-action chunks or of the expansion's
    CTA split (A = 7, 5), the minimum A = 2, A > 32 (two lanes per action in the finalize warp) and the
    maximum A = 64 (the fused head's 16 action chunks), against the oracle."""
    cfg = Config(f"A{A}", ENV_ATARI_HASH, net, A, d, n, 0.99, 1.0, seed=40 + A, wseed=140 + A)
    h = handle(cfg)
    o = Oracle.from_config(cfg)
    roots = cfg.roots()
    for corr in (0, 1):
        g = run(h, roots, d, cfg.gamma, cfg.beta, corr)
        r = o.search(roots, d, float(np.float32(cfg.gamma)), cfg.beta, corr, mode=0, threads=THREADS)
        bf16_compare(g, r, f"{cfg.name} net={net} n={n} d={d} corr={corr}")
        if corr:
            np.testing.assert_array_equal(g["terms"][:, 0], r["terms"][:, 0])


@pytest.mark.parametrize("cname", ["C3", "C5"])
def test_q_rows_vs_oracle(cname):
    """Leaf value net, full rows: GPU bf16 tensor-core net vs the bf16-emulating fp64 oracle."""
    cfg = config(cname)
    h = handle(cname)
    o = Oracle.from_config(cfg)
    recs = atari_roots(16, 4242)
    q = h.q_rows(dev(recs), 16).cpu().numpy()
    ref = np.stack([o.qrow(recs[i]) for i in range(16)])
    err = rel_err(q, ref)
    print(f"{cname} q_rows max rel err {err.max():.2e}")
    assert err.max() <= RTOL_BF16 / 4


def test_simt_and_tensor_core_nets_agree():
    """The SIMT reference layer and the tcgen05 layer compute the same net (tolerance of bf16 RNE flips)."""
    cfg = config("C5")
    a = handle("C5")
    b = handle("C5", flags=P.F_SIMT_NET)
    recs = atari_roots(64, 77)
    qa = a.q_rows(dev(recs), 64).cpu().numpy()
    qb = b.q_rows(dev(recs), 64).cpu().numpy()
    assert rel_err(qa, qb).max() <= 1e-2


# ------------------------------------------------------------------ full-size configs (sampled)
def sampled_full_size(cname, n_check_roots, n_samples, seed):
    cfg = config(cname)
    h = handle(cname)
    o = Oracle.from_config(cfg)
    roots = cfg.roots()
    gamma32 = float(np.float32(cfg.gamma))
    g = run(h, roots, cfg.depth, cfg.gamma, cfg.beta, 1)
    A, d = cfg.A, cfg.depth
    lpr = A ** d
    rng = np.random.default_rng(seed)
    check = sorted(set([0, cfg.n_roots - 1] + list(rng.integers(0, cfg.n_roots, size=max(0, n_check_roots - 2)))))
    # BCTS terms at full size
    t, q0 = o.terms(roots[check], d, gamma32)
    np.testing.assert_array_equal(g["terms"][check, 0], t[:, 0])
    assert (np.abs(g["terms"][check, 1:] - t[:, 1:]) <= RTOL_BF16 * np.maximum(np.abs(t[:, 1:]), 1e-3)).all()
    for ci, r in enumerate(check):
        # the GPU's best leaf per root action, replayed by the oracle, reproduces vanilla_q
        for a in range(A):
            leaf = int(g["best_leaf"][r, a])
            assert a * lpr // A <= leaf < (a + 1) * lpr // A
            rec, R = o.node(roots[r], d, leaf, gamma32)
            tot = R + gamma32 ** d * o.qrow(rec).max()
            scale = max(np.abs(g["vanilla_q"][r]).max(), 1e-6)
            assert abs(tot - g["vanilla_q"][r, a]) <= RTOL_BF16 * scale, (r, a)
        # sampled leaves: states bit-exact (path replay) and never above the segment max
        st, cum = h.expand(dev(roots[r:r + 1]), 1, d, np.float32(cfg.gamma))
        leaves = sorted(set([0, lpr - 1, lpr // A, lpr // A - 1] + list(rng.integers(0, lpr, size=n_samples))))
        idx = torch.tensor(leaves, device=DEV)
        sub = st[idx].contiguous()
        qsub = h.q_rows(sub, len(leaves)).cpu().numpy()
        sub, cumsub = sub.cpu().numpy(), cum[idx].cpu().numpy()
        del st, cum
        for j, leaf in enumerate(leaves):
            rec, R = o.node(roots[r], d, leaf, gamma32, mode=1)
            assert sub[j].tobytes() == rec.tobytes(), (r, leaf)
            assert cumsub[j] == np.float32(R)
            qo = o.qrow(rec)
            assert rel_err(qsub[j:j + 1], qo[None]).max() <= RTOL_BF16 / 4
            tot = R + gamma32 ** d * qo.max()
            a0 = leaf // (lpr // A)
            assert tot <= g["vanilla_q"][r, a0] + RTOL_BF16 * max(np.abs(g["vanilla_q"][r]).max(), 1e-6)
        # corrected Q = vanilla - beta*g_d*B for a != pi_o (Eq. 3), with the oracle's B
        pio = int(t[ci, 0])
        pen = cfg.beta * np.float32(gamma32 ** d) * t[ci, 3]
        exp = g["vanilla_q"][r] - np.where(np.arange(A) == pio, 0.0, pen)
        assert rel_err(g["root_q"][r][None], exp[None]).max() <= RTOL_BF16
    torch.cuda.empty_cache()
    return g


def test_c5_full_size_sampled():
    g = sampled_full_size("C5", 1, 48, 5)
    assert g["stats"]["leaves"] == 18 ** 4


def test_c3_full_size_sampled():
    sampled_full_size("C3", 3, 16, 3)


@pytest.mark.slow
def test_c4_full_size_sampled():
    sampled_full_size("C4", 3, 12, 4)


# ------------------------------------------------------------------ invariants / edge cases
def test_chunking_and_ragged_bit_identical():
    """Any chunk size gives bit-identical outputs (max over packed keys is exact, §6)."""
    cfg = config("C2")
    roots = cfg.roots(37)                      # ragged root count
    base = run(handle("C2"), roots, 3, cfg.gamma, 1.0, 1)
    small = P.Handle.from_config(cfg, workspace_bytes_max=(1 << 20) + 40 * 1000)
    g = run(small, roots, 3, cfg.gamma, 1.0, 1)
    assert g["stats"]["chunks"] > 3
    for k in ("actions", "root_q", "vanilla_q", "terms", "best_leaf"):
        np.testing.assert_array_equal(g[k], base[k])
    c5 = Config("C5s", ENV_ATARI_HASH, NET_RAINBOW_BF16, 18, 3, 2, 0.99, 1.0, seed=5, wseed=105)
    r5 = c5.roots()
    a = run(handle(c5), r5, 3, 0.99)
    b = run(handle(c5, workspace_bytes_max=8 << 20), r5, 3, 0.99)
    assert b["stats"]["chunks"] > 1
    for k in ("actions", "root_q", "vanilla_q", "best_leaf"):
        np.testing.assert_array_equal(a[k], b[k])


@pytest.mark.parametrize("cname,n,d", [("C2", 5, 3), ("C5", 1, 3)])
def test_virtual_shards_bit_identical(cname, n, d):
    """Multi-GPU partition emulated on one GPU: each shard's keys computed separately,
    combined by elementwise max (the all-reduce), then finalize == single search."""
    cfg = config(cname)
    h = handle(cname)
    roots = cfg.roots(n)
    rd = dev(roots)
    ref = run(h, roots, d, cfg.gamma, 1.0, 1)
    for W in (2, 3, 8):
        keys = []
        for rank in range(W):
            b, e = P.shard_range(n, d, cfg.A, rank, W)
            k = torch.empty(n * cfg.A, dtype=torch.int64, device=DEV)
            h.keys_init(k)
            h.search_shard(rd, n, d, cfg.gamma, b, e, k)
            keys.append(k)
        red = keys[0]
        for k in keys[1:]:
            red = torch.maximum(red, k)
        out = h.finalize(rd, n, d, cfg.gamma, 1.0, 1, red)
        torch.cuda.synchronize()
        for key in ("actions", "root_q", "vanilla_q", "terms", "best_leaf"):
            np.testing.assert_array_equal(out[key].cpu().numpy(), ref[key])


def test_invariants_beta0_depth0():
    cfg = config("C5")
    h = handle("C5")
    roots = atari_roots(3, 11)
    v = run(h, roots, 2, cfg.gamma, 1.0, 0)
    b0 = run(h, roots, 2, cfg.gamma, 0.0, 1)
    np.testing.assert_array_equal(b0["root_q"], v["vanilla_q"])     # beta = 0 -> vanilla bit for bit
    np.testing.assert_array_equal(b0["actions"], v["actions"])
    z = run(h, roots, 0, cfg.gamma, 1.0, 1)                          # d = 0 -> greedy on Q_hat(s0, .)
    q = h.q_rows(dev(roots), 3).cpu().numpy()
    np.testing.assert_array_equal(z["root_q"], q)
    np.testing.assert_array_equal(z["actions"], q.argmax(1))


def test_errors_leave_outputs_untouched():
    h = handle("C2")
    roots = dev(config("C2").roots(2))
    act = torch.full((2,), -7, dtype=torch.int32, device=DEV)
    q = torch.full((2, 4), 3.5, dtype=torch.float32, device=DEV)
    for args, status in [((roots, 2, 3, 5), 1),          # A mismatch
                         ((roots, 2, -1, 4), 1),         # depth < 0
                         ((roots, 2, 13, 4), 1)]:        # depth too large
        r, n, d, A = args
        s = P.lib().bcts_search(h._h, P.bcts._p(r), n, d, A, 0.99, 1.0, 1, P.bcts._p(act), P.bcts._p(q))
        assert s == status
    for gamma in (0.0, 1.0, float("nan")):
        assert P.lib().bcts_search(h._h, P.bcts._p(roots), 2, 2, 4, gamma, 1.0, 1, P.bcts._p(act), P.bcts._p(q)) == 1
    assert P.lib().bcts_search(h._h, P.bcts._p(roots), 2, 2, 4, 0.9, -1.0, 1, P.bcts._p(act), P.bcts._p(q)) == 1
    assert P.lib().bcts_search(h._h, P.bcts._p(roots), 2, 2, 4, 0.9, 1.0, 3, P.bcts._p(act), P.bcts._p(q)) == 1
    assert P.lib().bcts_search(h._h, P.bcts._p(roots), 0, 2, 4, 0.9, 1.0, 1, None, None) == 0
    torch.cuda.synchronize()
    assert (act.cpu() == -7).all() and (q.cpu() == 3.5).all()
    bad = dev(tabular_roots([7]))
    ht = P.Handle(P.ENV_TABULAR, 2, P.NET_TABLE, tab=chain_c1())
    a1 = torch.zeros(1, dtype=torch.int32, device=DEV)
    q1 = torch.zeros(1, 2, dtype=torch.float32, device=DEV)
    assert P.lib().bcts_search(ht._h, P.bcts._p(bad), 1, 2, 2, 0.9, 1.0, 1, P.bcts._p(a1), P.bcts._p(q1)) == 1


def test_e2e_host_matches_device():
    cfg = config("C5")
    h = handle("C5")
    roots = atari_roots(2, 19)
    g = run(h, roots, 2, cfg.gamma, 1.0, 1)
    pin = torch.from_numpy(roots.copy()).pin_memory()
    act = torch.zeros(2, dtype=torch.int32).pin_memory()
    q = torch.zeros(2, cfg.A, dtype=torch.float32).pin_memory()
    h.search_host(pin, 2, 2, cfg.gamma, 1.0, 1, act, q)
    np.testing.assert_array_equal(act.numpy(), g["actions"])
    np.testing.assert_array_equal(q.numpy(), g["root_q"])


def test_e2e_graph_replay_reads_new_inputs():
    """bcts_search_host replays a CUDA graph captured after its first call with the same page-locked
    buffers: every replay must copy the buffer's CURRENT roots in and the new outputs out."""
    cfg = config("C5")
    h = P.Handle.from_config(cfg)
    pin = torch.zeros(2, P.RECORD_BYTES[P.ENV_ATARI_HASH], dtype=torch.uint8).pin_memory()
    act = torch.zeros(2, dtype=torch.int32).pin_memory()
    q = torch.zeros(2, cfg.A, dtype=torch.float32).pin_memory()
    for seed in (21, 22, 23, 24):   # call 1 eager (+ capture), calls 2-4 graph replays
        roots = atari_roots(2, seed)
        g = run(h, roots, 3, cfg.gamma, 1.0, 1)
        pin.copy_(torch.from_numpy(roots.view(np.uint8).reshape(2, -1)))
        h.search_host(pin, 2, 3, cfg.gamma, 1.0, 1, act, q)
        np.testing.assert_array_equal(act.numpy(), g["actions"])
        np.testing.assert_array_equal(q.numpy(), g["root_q"])
    h.close()


@pytest.mark.parametrize("cname,n,d", [("C2", 16, 3), ("C5", 2, 2)])
def test_exact_bias_correction(cname, n, d):
    """correction_on = 2: Lemma 2's exact gap (App. A.2) instead of Eq. 5 -- GPU (normcdfinv) vs oracle."""
    cfg = config(cname)
    h = handle(cname)
    o = Oracle.from_config(cfg)
    roots = cfg.roots(n)
    g = run(h, roots, d, cfg.gamma, 1.0, 2)
    r = o.search(roots, d, float(np.float32(cfg.gamma)), 1.0, 2, mode=0, threads=THREADS)
    tol = RTOL_F32 if cname == "C2" else RTOL_BF16
    assert rel_err(g["root_q"], r["root_q"]).max() <= tol
    np.testing.assert_array_equal(g["terms"][:, 0], r["terms"][:, 0])
    assert (np.abs(g["terms"][:, 3] - r["terms"][:, 3]) <= tol * np.maximum(1.0, np.abs(r["terms"][:, 3]))).all()
    frac, _, _ = action_agreement(g["actions"], r["root_q"], tol)
    assert frac == 1.0


# ------------------------------------------------- NEXT-1: random-DNN forward model
def dnn_cfg(name):
    """D2 / D10 (synth CONFIGS) and D3: A = 3, so 64-child tiles split sibling groups."""
    import dataclasses
    if name == "D3":
        return dataclasses.replace(config("D10"), name="D3", A=3, seed=23, wseed=123)
    return config(name)


@pytest.mark.parametrize("cname,n,levels", [("D2", 5, 7), ("D3", 3, 4), ("D10", 2, 2)])
def test_dnn_level_states_bit_exact(cname, n, levels):
    """k_expand_dnn: every node's 100 fp32 state values and R bit-exact vs the oracle's fp32 mirror
    (ragged 64-child tiles, sibling groups split across tiles for A = 3)."""
    cfg = dnn_cfg(cname)
    h = handle(cfg)
    o = Oracle.from_config(cfg)
    roots = cfg.roots(n)
    g = float(np.float32(cfg.gamma))
    for level in range(levels + 1):
        st, cum = h.expand(dev(roots), n, level, np.float32(cfg.gamma))
        st, cum = st.cpu().numpy(), cum.cpu().numpy()
        per = cfg.A ** level
        idx = range(n * per) if n * per <= 700 else np.random.default_rng(level).choice(n * per, 700, replace=False)
        for j in idx:
            r, i = divmod(int(j), per)
            rec, R = o.node(roots[r], level, i, g, mode=1)
            assert st[j].tobytes() == rec.tobytes(), (level, r, i)
            assert cum[j] == np.float32(R), (level, r, i)


@pytest.mark.parametrize("cname,n,d", [("D2", 64, 8), ("D3", 7, 5), ("D10", 16, 4), ("D10", 3, 1)])
@pytest.mark.parametrize("corr", [0, 1, 2])
def test_dnn_search_vs_oracle(cname, n, d, corr):
    """Search on the DNN forward model + MLP2 100-256-A leaf net, fp32: vanilla Q and best leaf
    bit-exact vs the fp32 mirror; root Q within 1e-5 of the fp64 oracle; actions equal."""
    cfg = dnn_cfg(cname)
    h = handle(cfg)
    o = Oracle.from_config(cfg)
    roots = cfg.roots(n)
    gamma = float(np.float32(cfg.gamma))
    gr = run(h, roots, d, cfg.gamma, 1.0, corr)
    m = o.search(roots, d, gamma, 1.0, corr, mode=1, threads=THREADS)
    r = o.search(roots, d, gamma, 1.0, corr, mode=0, threads=THREADS)
    np.testing.assert_array_equal(gr["vanilla_q"], m["vanilla_q"].astype(np.float32))
    np.testing.assert_array_equal(gr["best_leaf"], m["best_leaf"])
    assert rel_err(gr["root_q"], r["root_q"]).max() <= RTOL_F32
    frac, _, _ = action_agreement(gr["actions"], r["root_q"], RTOL_F32)
    assert frac == 1.0
    assert gr["stats"]["leaves"] == n * cfg.A ** d


# ------------------------------------------------- NEXT-3: propagated-value (PV) target
@pytest.mark.parametrize("cname,n,d", [("C2", 16, 3), ("D10", 4, 3), ("C5", 1, 2)])
def test_pv_targets_replay(cname, n, d):
    """App. B.3 (R29): target = Eq. 1 value of the executed action; the returned path starts with
    that action, and replaying it through the oracle's forward model reaches exactly that value."""
    cfg = dnn_cfg(cname) if cname.startswith("D") else config(cname)
    h = handle(cfg)
    o = Oracle.from_config(cfg)
    roots = cfg.roots(n)
    gamma = float(np.float32(cfg.gamma))
    out = h.search(dev(roots), n, d, cfg.gamma, 1.0, 1, extra=True)
    tgt, path = h.pv_targets(out["actions"], out["vanilla_q"], out["best_leaf"], n, d)
    torch.cuda.synchronize()
    tgt, path = tgt.cpu().numpy(), path.cpu().numpy()
    act = out["actions"].cpu().numpy()
    van = out["vanilla_q"].cpu().numpy()
    np.testing.assert_array_equal(path[:, 0], act)
    np.testing.assert_array_equal(tgt, van[np.arange(n), act])
    bf16 = cfg.net in (3, 4)
    for r in range(n):
        leaf = 0
        for t in range(d):
            leaf = leaf * cfg.A + int(path[r, t])
        if bf16:   # bf16 net: the replayed leaf's fp64-oracle total within the bf16 tolerance
            tot = o.leaf_total(roots[r], d, leaf, gamma, mode=0)
            assert abs(tot - tgt[r]) <= RTOL_BF16 * max(abs(tot), 1e-6)
        else:      # fp32 paths: bit-exact vs the fp32 mirror's R_d + gamma^d max Q of that leaf
            assert np.float32(o.leaf_total(roots[r], d, leaf, gamma, mode=1)) == tgt[r], r


def test_pv_targets_bad_action_and_args():
    h = handle("C2")
    n, d = 2, 2
    act = torch.tensor([1, 7], dtype=torch.int32, device=DEV)
    van = torch.zeros(n * 4, dtype=torch.float32, device=DEV)
    bl = torch.tensor([0, 5, 0, 0, 0, 0, 0, 0], dtype=torch.int64, device=DEV)
    tgt, path = h.pv_targets(act, van, bl, n, d)
    torch.cuda.synchronize()
    assert np.isnan(tgt[1].item()) and (path[1].cpu().numpy() == -1).all()
    np.testing.assert_array_equal(path[0].cpu().numpy(), [1, 1])
    with pytest.raises(P.BctsError):
        h.pv_targets(act, van, bl, n, 0)


# ------------------------------------------------- fused leaf level vs materialised leaves
@pytest.mark.parametrize("cname,n,d", [("C5", 1, 3), ("C4", 3, 4)])
def test_head_backup_bit_identical(cname, n, d):
    """The backup folded into the Rainbow head's epilogue (Alg. 1: warp max + atomicMax on
    packed (total, leaf) keys) equals the separate k_segmax pass bit for bit: both fold the same
    leaf totals and the max over packed keys is exact and order-independent (R4)."""
    cfg = config(cname)
    roots = cfg.roots(n)
    a = run(handle(cname), roots, d, cfg.gamma, 1.0, 1)
    b = run(handle(cname, flags=P.F_SEPARATE_BACKUP), roots, d, cfg.gamma, 1.0, 1)
    for k in ("actions", "root_q", "vanilla_q", "terms", "best_leaf"):
        np.testing.assert_array_equal(a[k], b[k])
    assert a["stats"]["kernel_launches"] < b["stats"]["kernel_launches"]


@pytest.mark.parametrize("A", [5, 7, 33])
def test_rainbow_head_chunk_tails(A):
    """k_zhead packs z_a in chunks of 4 actions x 51 rows (N = 208); the last chunk holds 1 (A = 5, 33 -> N = 64)
    or 3 (A = 7 -> N = 160) actions. Whole depth-2 searches vs the oracle (bf16 search tolerance, actions under
    the near-tie rule), spread head weights so the check discriminates."""
    cfg = Config(f"R{A}", ENV_ATARI_HASH, NET_RAINBOW_BF16, A, 2, 2, 0.99, 1.0, seed=50 + A, wseed=150 + A,
                 extra={"head_scale": 64.0})
    roots = cfg.roots()
    h = P.Handle.from_config(cfg)   # not cached: each conv-net handle binds ~7 GB of net scratch
    try:
        g = run(h, roots, 2, cfg.gamma, 1.0, 1)
    finally:
        h.close()
    r = Oracle.from_config(cfg).search(roots, 2, float(np.float32(cfg.gamma)), 1.0, 1, mode=0, threads=THREADS)
    assert rel_err(g["root_q"], r["root_q"]).max() <= RTOL_BF16_SEARCH
    assert rel_err(g["vanilla_q"], r["vanilla_q"]).max() <= RTOL_BF16_SEARCH
    assert action_agreement(g["actions"], r["root_q"], RTOL_BF16_SEARCH)[0] >= 0.999


@pytest.mark.parametrize("A,n,d", [(40, 2, 2), (2, 5, 3), (3, 7, 3)])
def test_fused_leaves_action_counts(A, n, d):
    """A = 40 (> 32): k_conv1_sib reads the child keys of actions 32..39 from the second per-parent lane
    table (each lane hashes actions l and l + 32 once per parent); A = 2, 3: a parent switch every 2-3
    children in every role's loop. Fused vs materialised leaves (the materialised path hashes every child
    in k_expand_atari) and the whole search vs the oracle."""
    cfg = Config(f"A{A}", ENV_ATARI_HASH, NET_NATURE_BF16, A, d, n, 0.99, 1.0, seed=40 + A, wseed=140 + A)
    roots = cfg.roots()
    ha, hb = P.Handle.from_config(cfg), P.Handle.from_config(cfg, flags=P.F_MATERIALIZE_LEAVES)   # not cached
    try:
        a = run(ha, roots, d, cfg.gamma, 1.0, 1)
        b = run(hb, roots, d, cfg.gamma, 1.0, 1)
    finally:
        ha.close()
        hb.close()
    # the two paths round act1 to bf16 after different fp32 sums (R17/R18): ~1e-5 absolute, which is above
    # 1e-4 relative for a root whose |Q| is ~0.02 (no reward on its paths), so R18's search tolerance
    scale = np.abs(b["vanilla_q"]).max(axis=1, keepdims=True)
    assert (np.abs(a["vanilla_q"] - b["vanilla_q"]) <= RTOL_BF16_SEARCH * scale).all()
    assert (a["best_leaf"] == b["best_leaf"]).mean() >= 0.9
    r = Oracle.from_config(cfg).search(roots, d, float(np.float32(cfg.gamma)), 1.0, 1, mode=0, threads=THREADS)
    assert rel_err(a["root_q"], r["root_q"]).max() <= RTOL_BF16_SEARCH
    assert action_agreement(a["actions"], r["root_q"], RTOL_BF16_SEARCH)[0] >= 0.999


@pytest.mark.parametrize("cname,n,d", [("C3", 3, 2), ("C5", 1, 2), ("C5", 1, 3), ("C4", 2, 3)])
def test_fused_leaves_match_materialized(cname, n, d):
    """k_conv1_sib (leaf expansion fused into conv1, sibling-factorised, fp16 operands with exact
    2^14-scaled weights) vs BCTS_F_MATERIALIZE_LEAVES (leaf states stored, standard conv1): the same
    bf16 net on the same leaves, so results agree up to fp32 accumulation order / bf16 RNE flips.
    Strict on purpose: random-init Q values are nearly flat across leaves, so a relative-to-max|Q|
    tolerance alone cannot tell a broken trunk from rounding (best-leaf agreement can)."""
    cfg = config(cname)
    ha = handle(cname)
    hb = handle(cname, flags=P.F_MATERIALIZE_LEAVES)
    roots = cfg.roots(n)
    a = run(ha, roots, d, cfg.gamma, 1.0, 0)
    b = run(hb, roots, d, cfg.gamma, 1.0, 0)
    scale = np.abs(b["vanilla_q"]).max(axis=1, keepdims=True)
    assert (np.abs(a["vanilla_q"] - b["vanilla_q"]) <= 1e-4 * scale).all()
    assert (a["best_leaf"] == b["best_leaf"]).mean() >= 0.9
