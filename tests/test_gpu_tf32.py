"""NEXT-1 on the tensor cores (BCTS_F_TF32, tf32_tc.cu) against the fp64 oracle (R34).

The flag runs the random-DNN forward model (R27) and the MLP2 net as tcgen05 kind::tf32
GEMMs: every operand is rounded to tf32 (unit roundoff u = 2^-11 ~ 4.9e-4) and accumulated in fp32 in
the MMA's order, so the path is not bit-exact with the fp32 default; it is held to tolerances derived
from u (R34) against the oracle's fp64 mode (mode=0: the same equations in double):
  * level states: max |s_gpu - s_oracle| <= STATE_TOL * max |s_oracle| per node (one rounding of each
    layer's inputs and weights per layer; the relative error does not grow with depth because the
    random layers are contractive -- observed <= 4.0e-4 at every level of D2 / D3 / D10);
  * cumulative reward R: |R_gpu - R_oracle| <= R_TOL * max(|R_oracle|, 1e-3) (observed <= 6.1e-3:
    R is a sum of small rewards, so its relative error is larger at shallow levels);
  * searches: root Q and vanilla Q within RTOL_TF32 of max_a |oracle q| (R18; observed <= 3.0e-3),
    actions under the near-tie rule (R19) >= 99.9 %.
"""
import dataclasses
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

DEV = torch.device("cuda", 0)
THREADS = os.cpu_count() or 1
STATE_TOL = 2e-3
R_TOL = 2e-2
RTOL_TF32 = 1e-2


def cfg_of(name):
    if name == "D3":   # A = 3: 128-child tiles split sibling groups
        return dataclasses.replace(config("D10"), name="D3", A=3, seed=23, wseed=123)
    return config(name)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).copy()).to(DEV)


_handles = {}


def handle(cfg, flags):
    key = (cfg.name, cfg.A, flags)
    if key not in _handles:
        _handles[key] = P.Handle.from_config(cfg, flags=flags)
    return _handles[key]


@pytest.mark.parametrize("cname,n,levels", [("D2", 4, 7), ("D3", 3, 4), ("D10", 4, 3)])
def test_tf32_level_states_vs_fp64_oracle(cname, n, levels):
    cfg = cfg_of(cname)
    h = handle(cfg, P.F_TF32)
    o = Oracle.from_config(cfg)
    roots = cfg.roots(n)
    g = float(np.float32(cfg.gamma))
    for level in range(1, levels + 1):
        st, cum = h.expand(dev(roots), n, level, np.float32(cfg.gamma))
        st, cum = st.cpu().numpy(), cum.cpu().numpy()
        per = cfg.A ** level
        idx = range(n * per) if n * per <= 400 else np.random.default_rng(level).choice(n * per, 400, replace=False)
        es = er = 0.0
        for j in idx:
            r, i = divmod(int(j), per)
            rec, R = o.node(roots[r], level, i, g, mode=0)
            x = np.frombuffer(rec.tobytes(), dtype=np.float32)
            y = st[j].view(np.float32)
            es = max(es, float(np.abs(y - x).max() / max(np.abs(x).max(), 1e-6)))
            er = max(er, abs(float(cum[j]) - R) / max(abs(R), 1e-3))
        print(f"{cname} level {level}: state err {es:.2e}, R err {er:.2e}")
        assert es <= STATE_TOL and er <= R_TOL, (level, es, er)


@pytest.mark.parametrize("cname,n,d,corr", [("D2", 64, 8, 1), ("D10", 16, 4, 0), ("D10", 16, 4, 1), ("D10", 16, 4, 2),
                                            ("D3", 7, 5, 1), ("C2", 64, 4, 1), ("C2", 5, 3, 1)])
def test_tf32_search_vs_fp64_oracle(cname, n, d, corr):
    cfg = cfg_of(cname)
    h = handle(cfg, P.F_TF32)
    o = Oracle.from_config(cfg)
    roots = cfg.roots(n)
    gamma = float(np.float32(cfg.gamma))
    out = h.search(dev(roots), n, d, cfg.gamma, 1.0, corr, extra=True)
    torch.cuda.synchronize()
    g = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in out.items()}
    r = o.search(roots, d, gamma, 1.0, corr, mode=0, threads=THREADS)
    eq, ev = rel_err(g["root_q"], r["root_q"]).max(), rel_err(g["vanilla_q"], r["vanilla_q"]).max()
    frac, exact, near = action_agreement(g["actions"], r["root_q"], RTOL_TF32)
    print(f"{cname} n={n} d={d} corr={corr}: root_q {eq:.2e}, vanilla_q {ev:.2e}, actions {frac:.4f} "
          f"(exact {exact}, near-ties {near})")
    assert eq <= RTOL_TF32 and ev <= RTOL_TF32
    assert frac >= 0.999
    assert g["stats"]["leaves"] == n * cfg.A ** d


def test_tf32_is_opt_in():
    """Without the flag the DNN path stays the bit-exact fp32 one (the flag changes results)."""
    cfg = cfg_of("D10")
    roots = cfg.roots(3)
    a = handle(cfg, 0).search(dev(roots), 3, 2, cfg.gamma, 1.0, 1, extra=True)
    b = handle(cfg, P.F_TF32).search(dev(roots), 3, 2, cfg.gamma, 1.0, 1, extra=True)
    torch.cuda.synchronize()
    m = Oracle.from_config(cfg).search(roots, 2, float(np.float32(cfg.gamma)), 1.0, 1, mode=1, threads=THREADS)
    np.testing.assert_array_equal(a["vanilla_q"].cpu().numpy(), m["vanilla_q"].astype(np.float32))
    assert not np.array_equal(b["vanilla_q"].cpu().numpy(), m["vanilla_q"].astype(np.float32))


def _host(out):
    return {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in out.items()}


@pytest.mark.parametrize("cname,n,d,ws", [("D10", 5, 4, 4 << 20), ("C2", 37, 4, (1 << 20) + 40 * 1000)])
def test_tf32_chunking_and_shards_bit_identical(cname, n, d, ws):
    """The tf32 path is deterministic per node (a tile's row sums do not depend on the other rows of the
    tile), so chunked searches (small workspace) and virtual multi-GPU shards (max over packed keys) give
    the unchunked search bit for bit, as on the fp32 path."""
    cfg = cfg_of(cname)
    roots = cfg.roots(n)
    rd = dev(roots)
    ref = _host(handle(cfg, P.F_TF32).search(rd, n, d, cfg.gamma, 1.0, 1, extra=True))
    small = P.Handle.from_config(cfg, flags=P.F_TF32, workspace_bytes_max=ws)
    ch = _host(small.search(rd, n, d, cfg.gamma, 1.0, 1, extra=True))
    assert ch["stats"]["chunks"] > 1
    h = handle(cfg, P.F_TF32)
    keys = []
    for rank in range(3):
        b, e = P.shard_range(n, d, cfg.A, rank, 3)
        k = torch.empty(n * cfg.A, dtype=torch.int64, device=DEV)
        h.keys_init(k)
        h.search_shard(rd, n, d, cfg.gamma, b, e, k)
        keys.append(k)
    red = torch.maximum(torch.maximum(keys[0], keys[1]), keys[2])
    sh = _host(h.finalize(rd, n, d, cfg.gamma, 1.0, 1, red))
    for key in ("actions", "root_q", "vanilla_q", "best_leaf"):
        np.testing.assert_array_equal(ch[key], ref[key])
        np.testing.assert_array_equal(sh[key], ref[key])
    small.close()


def test_tf32_pruned_bound_equals_unpruned():
    """NEXT-4 on the tf32 path: the exact BOUND rule (R31) prunes only subtrees that cannot hold a group's
    max, so the pruned search equals the unpruned tf32 search bit for bit."""
    cfg = cfg_of("D10")
    roots = cfg.roots(6)
    h = handle(cfg, P.F_TF32)
    ref = _host(h.search(dev(roots), 6, 4, cfg.gamma, 1.0, 1, extra=True))
    out = _host(h.search_pruned(dev(roots), 6, 4, cfg.gamma, 1, 2, 1, -5.0, 5.0, -50.0, 50.0, beta=1.0,
                                correction=1))
    for key in ("actions", "root_q", "vanilla_q", "best_leaf"):
        np.testing.assert_array_equal(out[key], ref[key])


def test_max_action_count_mlp_fp32_and_tf32():
    """A = 64 (the ABI's maximum; 4 N = 16 chunks of layer 2 in k_mlp_tc) on the INT_HASH env with the
    MLP2 net: the fp32 default bit-exact vs the oracle's fp32 mirror, the tf32 path within R34's
    tolerance of the fp64 oracle."""
    from synth.inputs import Config, ENV_INT_HASH, NET_MLP2_F32
    cfg = Config("I64", ENV_INT_HASH, NET_MLP2_F32, 64, 2, 12, 0.99, 1.0, seed=64, wseed=164)
    roots = cfg.roots()
    o = Oracle.from_config(cfg)
    g32 = float(np.float32(cfg.gamma))
    a = _host(handle(cfg, 0).search(dev(roots), 12, 2, cfg.gamma, 1.0, 1, extra=True))
    m = o.search(roots, 2, g32, 1.0, 1, mode=1, threads=THREADS)
    np.testing.assert_array_equal(a["vanilla_q"], m["vanilla_q"].astype(np.float32))
    np.testing.assert_array_equal(a["actions"], m["actions"])
    b = _host(handle(cfg, P.F_TF32).search(dev(roots), 12, 2, cfg.gamma, 1.0, 1, extra=True))
    r = o.search(roots, 2, g32, 1.0, 1, mode=0, threads=THREADS)
    assert rel_err(b["root_q"], r["root_q"]).max() <= RTOL_TF32
    assert action_agreement(b["actions"], r["root_q"], RTOL_TF32)[0] >= 0.999


def test_tf32_deep_tree_error_does_not_grow():
    """D2 at depth 12 (48 tf32 layer applications on the deepest paths, one cooperative launch for the 12
    levels): root Q stays within the same R34 tolerance of the fp64 oracle as at depth 8."""
    cfg = cfg_of("D2")
    roots = cfg.roots(8)
    out = _host(handle(cfg, P.F_TF32).search(dev(roots), 8, 12, cfg.gamma, 1.0, 1, extra=True))
    r = Oracle.from_config(cfg).search(roots, 12, float(np.float32(cfg.gamma)), 1.0, 1, mode=0, threads=THREADS)
    eq = rel_err(out["root_q"], r["root_q"]).max()
    print(f"D2 d=12: root_q rel err {eq:.2e}")
    assert eq <= RTOL_TF32
    assert action_agreement(out["actions"], r["root_q"], RTOL_TF32)[0] >= 0.999


@pytest.mark.parametrize("H,A", [(48, 5), (16, 3), (208, 7)])
def test_tf32_mlp_hidden_widths(H, A):
    """k_mlp_tc splits the hidden units between two epilogue halves at hs = ceil16(H / 2): H = 48 (halves of
    32 + 16), H = 16 (half 1 empty), H = 208 (112 + 96). INT_HASH + MLP2 with mlp_hidden = H: the tf32 path
    within R34's tolerance of the fp64 oracle, the fp32 default bit-exact vs the oracle's fp32 mirror."""
    from synth.inputs import ENV_INT_HASH, NET_MLP2_F32, int_roots, make_weights
    w = make_weights(NET_MLP2_F32, A, 300 + H, mlp_in=64, mlp_hidden=H)[0]
    roots = int_roots(9, 40 + H)
    o = Oracle(ENV_INT_HASH, A, NET_MLP2_F32, weights=w, mlp_in=64, mlp_hidden=H)
    g32 = float(np.float32(0.97))
    ht = P.Handle(ENV_INT_HASH, A, NET_MLP2_F32, weights=w, mlp_in=64, mlp_hidden=H, flags=P.F_TF32)
    hf = P.Handle(ENV_INT_HASH, A, NET_MLP2_F32, weights=w, mlp_in=64, mlp_hidden=H)
    try:
        b = _host(ht.search(dev(roots), 9, 3, 0.97, 1.0, 1, extra=True))
        a = _host(hf.search(dev(roots), 9, 3, 0.97, 1.0, 1, extra=True))
    finally:
        ht.close()
        hf.close()
    m = o.search(roots, 3, g32, 1.0, 1, mode=1, threads=THREADS)
    np.testing.assert_array_equal(a["vanilla_q"], m["vanilla_q"].astype(np.float32))
    r = o.search(roots, 3, g32, 1.0, 1, mode=0, threads=THREADS)
    eq = rel_err(b["root_q"], r["root_q"]).max()
    print(f"H={H} A={A}: tf32 root_q rel err {eq:.2e}")
    assert eq <= RTOL_TF32
    assert action_agreement(b["actions"], r["root_q"], RTOL_TF32)[0] >= 0.999
