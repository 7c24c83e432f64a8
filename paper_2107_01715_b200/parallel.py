"""Multi-GPU partition of the search.

One process per GPU. Every rank holds the full roots and calls with identical
arguments; rank g expands and scores only its contiguous leaf range
(bcts_shard_range: whole roots per rank when n_roots % world == 0, otherwise
balanced leaf ranges -- the single-root C5 case). The only exchange is ONE
max all-reduce of the n_roots*A packed int64 keys (value, lowest leaf index)
-- a few hundred bytes over NVLink -- after which every rank applies the
identical BCTS correction, so all ranks return bit-identical outputs.

The host logic (range plan + reduction + finalize order) is shared with the
world-size-2 gloo tests through ``reduce_partials``.
"""
from __future__ import annotations

from . import bcts as _b


def reduce_partials(keys, group=None):
    """All-reduce MAX over ranks of int64 keys (signed order == (value, lowest index))."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(keys, op=dist.ReduceOp.MAX, group=group)
    return keys


def sharded_search(handle: "_b.Handle", roots, n_roots: int, depth: int, gamma: float, beta: float,
                   correction: int, group=None, extra: bool = False, keys=None):
    """Collective search: every rank passes the same arguments and gets the full outputs."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if depth == 0:
        return handle.finalize(roots, n_roots, 0, gamma, beta, correction, None, extra=extra)
    if keys is None:
        keys = torch.empty(n_roots * handle.A, dtype=torch.int64, device=torch.device("cuda", handle.device))
    b, e = _b.shard_range(n_roots, depth, handle.A, rank, world)
    handle.keys_init(keys)
    st = handle.search_shard(roots, n_roots, depth, gamma, b, e, keys)
    reduce_partials(keys, group)
    out = handle.finalize(roots, n_roots, depth, gamma, beta, correction, keys, extra=extra)
    out["stats"] = {k: out["stats"].get(k, 0) + st.get(k, 0) for k in set(st) | set(out["stats"])}
    out["leaf_range"] = (b, e)
    return out
