"""GPU tests of the C-ABI boundary: the library-owned NCCL collective, caller-owned
workspace, CUDA-graph replay of the device-pointer path, per-phase stats, and invariants of the
internal variants (prologue fold on/off, host-composed sharding) -- each checked bit for bit
against the plain single-GPU search (itself compared with the oracle in test_gpu_parity.py /
test_gpu_golden.py). All calls go through the C ABI (paper_2107_01715_b200.bcts)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2107_01715_b200 as P  # noqa: E402
from synth.inputs import config  # noqa: E402

DEV = torch.device("cuda", 0)
KEYS = ("actions", "root_q", "vanilla_q", "terms", "best_leaf")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).copy()).to(DEV)


def run(h, roots_np, d, cfg, corr=1, roots=None):
    n = roots_np.shape[0]
    out = h.search(dev(roots_np) if roots is None else roots, n, d, cfg.gamma, cfg.beta, corr, extra=True)
    torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in out.items()}


def same(a, b):
    for k in KEYS:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


@pytest.mark.parametrize("cname,n,d", [("C2", 5, 3), ("C5", 1, 3), ("C3", 2, 2)])
def test_nccl_one_rank_communicator_matches_plain_search(cname, n, d):
    """A handle with a one-rank NCCL communicator runs the collective path (shard range = all leaves,
    ncclAllReduce(ncclInt64, ncclMax) of the keys on the handle's stream): identical outputs; and
    the same call repeated (graph replay including the NCCL node) stays identical."""
    cfg = config(cname)
    roots = cfg.roots(n)
    plain = P.Handle.from_config(cfg)
    coll = P.Handle.from_config(cfg, nccl_id=P.nccl_unique_id(), rank=0, world=1)
    ref = run(plain, roots, d, cfg)
    rd = dev(roots)
    for _ in range(4):   # eager, eager + capture, replay, replay
        same(run(coll, roots, d, cfg, roots=rd), ref)
    plain.close()
    coll.close()


def test_caller_owned_workspace():
    """bcts_workspace_size + bcts_set_workspace: the search runs in torch-owned memory with the same
    result; a too-small buffer is rejected with BUDGET before anything is enqueued; NULL returns
    to library-owned memory."""
    cfg = config("C5")
    roots = cfg.roots(1)
    h = P.Handle.from_config(cfg)
    ref = run(h, roots, 3, cfg)
    need = h.workspace_size(1, 3)
    assert need > h.workspace_size(1, 2) > 0
    buf = torch.empty(need, dtype=torch.uint8, device=DEV)
    g = P.Handle.from_config(cfg)
    g.set_workspace(buf)
    same(run(g, roots, 3, cfg), ref)
    with pytest.raises(P.BctsError) as e:   # depth 4 needs more tree workspace than depth 3's buffer
        g.search(dev(roots), 1, 4, cfg.gamma, cfg.beta, 1)
    assert e.value.status == 4
    g.set_workspace(None)
    same(run(g, roots, 3, cfg), ref)
    with pytest.raises(P.BctsError):        # smaller than the net scratch
        g.set_workspace(torch.empty(1 << 20, dtype=torch.uint8, device=DEV))
    h.close()
    g.close()


def test_device_graph_replay_reads_current_inputs():
    """bcts_search_ex replays a CUDA graph once the same arguments repeat: every replay must read
    the roots buffer's CURRENT contents and write the outputs (compared with a graph-free handle)."""
    cfg = config("C5")
    h = P.Handle.from_config(cfg)
    nog = P.Handle.from_config(cfg, flags=P.F_NO_GRAPH)
    rbuf = torch.empty(2, P.RECORD_BYTES[P.ENV_ATARI_HASH], dtype=torch.uint8, device=DEV)
    out = h._outputs(2, True)
    launches = []
    for seed in (31, 32, 33, 34, 35):
        from synth.inputs import atari_roots
        r = atari_roots(2, seed)
        rbuf.copy_(torch.from_numpy(r.view(np.uint8).reshape(2, -1)))
        o = h.search(rbuf, 2, 3, cfg.gamma, cfg.beta, 1, extra=True, out=out)
        torch.cuda.synchronize()
        got = {k: v.cpu().numpy() for k, v in o.items() if k != "stats"}
        same(got, run(nog, r, 3, cfg))
        launches.append(o["stats"]["kernel_launches"])
    assert len(set(launches)) == 1 and launches[0] > 0   # replayed calls report the captured call's stats
    h.close()
    nog.close()


def test_stats_phase_times_when_profiling():
    cfg = config("C5")
    h = P.Handle.from_config(cfg)
    roots = cfg.roots(1)
    st = run(h, roots, 3, cfg)["stats"]
    assert st["ms_total"] == 0.0          # not profiling: the call stays asynchronous
    h.profile(True)
    st = run(h, roots, 3, cfg)["stats"]
    h.profile(False)
    assert st["ms_total"] > 0 and st["ms_leaf"] > 0 and st["ms_expand"] > 0 and st["ms_backup"] > 0
    assert st["ms_leaf"] + st["ms_expand"] + st["ms_backup"] <= st["ms_total"] * 1.05
    assert st["ms_comm"] == 0.0
    h.close()


@pytest.mark.parametrize("cname,n,d", [("C5", 1, 3), ("C4", 4, 3)])
def test_prologue_fold_bit_identical(cname, n, d):
    """The depth-0/1 rows evaluated inside the last leaf batch (PrologueFold) or in their own launches
    (BCTS_F_NO_PROLOGUE_FOLD) give identical outputs (ranks of a multi-GPU run can take
    either path)."""
    cfg = config(cname)
    roots = cfg.roots(n)
    a = P.Handle.from_config(cfg)
    b = P.Handle.from_config(cfg, flags=P.F_NO_PROLOGUE_FOLD | P.F_SEPARATE_BACKUP)
    ra, rb = run(a, roots, d, cfg), run(b, roots, d, cfg)
    same(ra, rb)
    assert ra["stats"]["kernel_launches"] < rb["stats"]["kernel_launches"]
    a.close()
    b.close()


def test_host_composed_sharding_on_handle_stream():
    """parallel.sharded_search on a handle with its own (non-default) stream: one rank covers every
    leaf, and the result equals the library search bit for bit (stream ordering)."""
    from paper_2107_01715_b200.parallel import sharded_search
    cfg = config("C5")
    roots = cfg.roots(1)
    ref = run(P.Handle.from_config(cfg), roots, 3, cfg)
    s = torch.cuda.Stream(DEV)
    h = P.Handle.from_config(cfg, stream=s)
    out = sharded_search(h, dev(roots), 1, 3, cfg.gamma, cfg.beta, 1, extra=True)
    torch.cuda.synchronize()
    same({k: v.cpu().numpy() for k, v in out.items() if k in KEYS}, ref)
    h.close()
