"""World-size-2 gloo test of the multi-GPU host path, on CPU.

Each rank takes its leaf range from bcts_shard_range (the library's host
logic), scores those leaves with the oracle (test infrastructure, standing in
for the GPU shard kernel), folds them into packed int64 keys with the
library's bcts_pack_key, and the ranks combine with
paper_2107_01715_b200.parallel.reduce_partials (all_reduce MAX). The reduced
keys must decode to exactly the single-process oracle's vanilla Q and lowest
best leaf, for root sharding (n % W == 0) and leaf-range sharding (C5-style).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, case, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2107_01715_b200 as P
    from paper_2107_01715_b200.parallel import reduce_partials
    from oracle import Oracle
    from synth.inputs import config
    name, n, d = case
    cfg = config(name)
    o = Oracle.from_config(cfg)
    roots = cfg.roots(n)
    A = cfg.A
    g = float(np.float32(cfg.gamma))
    lpr = A ** d
    b, e = P.shard_range(n, d, A, rank, world)
    keys = torch.full((n * A,), -(2 ** 63), dtype=torch.int64)
    for L in range(b, e):                       # this rank's leaves only
        r, within = divmod(L, lpr)
        tot = o.leaf_total(roots[r], d, within, g, mode=1)
        slot = r * A + within // (lpr // A)     # (root, root action) segment
        keys[slot] = max(int(keys[slot]), P.pack_key(tot, within))
    reduce_partials(keys)
    if rank == 0:
        out_q.put(keys.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", [("C2", 4, 2), ("C2", 3, 3), ("C2", 1, 3)])
def test_gloo_world2_reduction_matches_single_process(case):
    """(C2,4,2): root sharding; (C2,3,3) and (C2,1,3): leaf ranges split inside a root (C5-style)."""
    import paper_2107_01715_b200 as P
    from oracle import Oracle
    from synth.inputs import config
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    keys = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    name, n, d = case
    cfg = config(name)
    ref = Oracle.from_config(cfg).search(cfg.roots(n), d, float(np.float32(cfg.gamma)), 1.0, 0, mode=1)
    vals = np.array([P.key_value(int(k)) for k in keys]).reshape(n, cfg.A)
    leaves = np.array([P.key_leaf(int(k)) for k in keys]).reshape(n, cfg.A)
    np.testing.assert_array_equal(vals, ref["vanilla_q"].astype(np.float32))
    np.testing.assert_array_equal(leaves, ref["best_leaf"])

