"""B200-native Batch-BFS + BCTS (arXiv 2107.01715) hot path.

The compute lives in csrc/ (CUDA for sm_100a) behind the C ABI in
include/bcts.h; bcts.py is the thin ctypes binding. See DESIGN.md.
"""
from .bcts import (Handle, BctsError, Stats, lib, pack_key, key_value, key_leaf, shard_range, nccl_unique_id,  # noqa: F401
                   ENV_TABULAR, ENV_INT_HASH, ENV_ATARI_HASH, ENV_DNN, NET_TABLE, NET_MLP2_F32, NET_NATURE_BF16,
                   NET_RAINBOW_BF16, F_CLAMP_PENALTY, F_SIMT_NET, F_MATERIALIZE_LEAVES, F_SEPARATE_BACKUP, F_NO_PROLOGUE_FOLD,
                   F_NO_GRAPH, F_TF32, RECORD_BYTES,
                   EXPORTS,
                   Prune, PRUNE_NONE, PRUNE_BOUND, PRUNE_BEAM)
