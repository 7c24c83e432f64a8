"""Thin ctypes binding over libbcts.so (include/bcts.h). Argument marshalling only.

Every step of the search runs in the CUDA kernels of csrc/. There is no CPU
fallback: importing this module without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbcts.so")

ENV_TABULAR, ENV_INT_HASH, ENV_ATARI_HASH, ENV_DNN = 1, 2, 3, 4
NET_TABLE, NET_MLP2_F32, NET_NATURE_BF16, NET_RAINBOW_BF16 = 1, 2, 3, 4
F_CLAMP_PENALTY, F_SIMT_NET, F_MATERIALIZE_LEAVES, F_SEPARATE_BACKUP = 0x1, 0x2, 0x4, 0x8
F_NO_PROLOGUE_FOLD, F_NO_GRAPH, F_TF32 = 0x10, 0x20, 0x40
ABI_VERSION = 6
PRUNE_NONE, PRUNE_BOUND, PRUNE_BEAM = 0, 1, 2
STATUS = {0: "BCTS_OK", 1: "BCTS_ERR_INVALID_ARG", 2: "BCTS_ERR_UNSUPPORTED", 3: "BCTS_ERR_OUT_OF_MEMORY",
          4: "BCTS_ERR_BUDGET", 5: "BCTS_ERR_CUDA", 6: "BCTS_ERR_NCCL", 7: "BCTS_ERR_NUMERIC"}
RECORD_BYTES = {ENV_TABULAR: 4, ENV_INT_HASH: 64, ENV_ATARI_HASH: 28240, ENV_DNN: 400}

# every symbol include/bcts.h declares (checked by tests/test_abi.py)
EXPORTS = ["bcts_create", "bcts_destroy", "bcts_abi_version", "bcts_root_record_bytes", "bcts_status_string",
           "bcts_last_error", "bcts_search", "bcts_search_ex", "bcts_search_host", "bcts_keys_init",
           "bcts_search_shard", "bcts_finalize", "bcts_expand", "bcts_q_rows", "bcts_pack_key",
           "bcts_key_value", "bcts_key_leaf", "bcts_shard_range", "bcts_profile_enable", "bcts_profile_read",
           "bcts_pv_targets", "bcts_search_pruned", "bcts_nccl_unique_id", "bcts_workspace_size",
           "bcts_set_workspace"]


class BctsError(RuntimeError):
    def __init__(self, status, detail=""):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {detail}")


class Config(C.Structure):
    _fields_ = [("abi_version", C.c_uint32), ("device", C.c_int32), ("cuda_stream", C.c_void_p),
                ("env", C.c_int32), ("num_actions", C.c_int32), ("num_states", C.c_int32),
                ("tab_next", C.c_void_p), ("tab_reward", C.c_void_p), ("tab_q", C.c_void_p),
                ("net", C.c_int32), ("weights", C.c_void_p), ("weights_count", C.c_int64),
                ("mlp_in", C.c_int32), ("mlp_hidden", C.c_int32), ("atoms", C.c_int32),
                ("v_min", C.c_float), ("v_max", C.c_float), ("workspace_bytes_max", C.c_int64),
                ("flags", C.c_uint32), ("env_weights", C.c_void_p), ("env_weights_count", C.c_int64),
                ("nccl_unique_id", C.c_void_p), ("rank", C.c_int32), ("world", C.c_int32)]


class KernelProfile(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("ms", C.c_double), ("work", C.c_double),
                ("unit", C.c_int32), ("big_launches", C.c_int64), ("big_ms", C.c_double), ("big_work", C.c_double)]


class Prune(C.Structure):
    _fields_ = [("rule", C.c_int32), ("first_level", C.c_int32), ("beam", C.c_int64), ("r_lo", C.c_float),
                ("r_hi", C.c_float), ("q_lo", C.c_float), ("q_hi", C.c_float)]


class Stats(C.Structure):
    _fields_ = [("transitions", C.c_int64), ("leaves", C.c_int64), ("evaluated", C.c_int64),
                ("kernel_launches", C.c_int64), ("chunks", C.c_int64), ("level_launches", C.c_int64),
                ("ms_total", C.c_float), ("ms_expand", C.c_float), ("ms_leaf", C.c_float), ("ms_backup", C.c_float),
                ("ms_comm", C.c_float)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    """Load libbcts.so; raises if it was not built (no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_2107_01715_b200/build.py (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        P, I32, I64, F = C.c_void_p, C.c_int32, C.c_int64, C.c_float
        sig = {
            "bcts_create": ([C.POINTER(Config), C.POINTER(P)], I32),
            "bcts_destroy": ([P], None),
            "bcts_abi_version": ([], I32),
            "bcts_root_record_bytes": ([P], C.c_size_t),
            "bcts_status_string": ([I32], C.c_char_p),
            "bcts_last_error": ([P], C.c_char_p),
            "bcts_search": ([P, P, I64, I32, I32, F, F, I32, P, P], I32),
            "bcts_search_ex": ([P, P, I64, I32, I32, F, F, I32, P, P, P, P, P, C.POINTER(Stats)], I32),
            "bcts_search_host": ([P, P, I64, I32, I32, F, F, I32, P, P], I32),
            "bcts_keys_init": ([P, P, I64], I32),
            "bcts_search_shard": ([P, P, I64, I32, I32, F, I64, I64, P, C.POINTER(Stats)], I32),
            "bcts_finalize": ([P, P, I64, I32, I32, F, F, I32, P, P, P, P, P, P, C.POINTER(Stats)], I32),
            "bcts_expand": ([P, P, I64, I32, I32, F, P, P], I32),
            "bcts_q_rows": ([P, P, I64, P], I32),
            "bcts_pack_key": ([F, I64], I64),
            "bcts_key_value": ([I64], F),
            "bcts_key_leaf": ([I64], I64),
            "bcts_shard_range": ([I64, I32, I32, I32, I32, C.POINTER(I64), C.POINTER(I64)], I32),
            "bcts_profile_enable": ([P, I32], I32),
            "bcts_profile_read": ([P, C.POINTER(KernelProfile), I32], I32),
            "bcts_pv_targets": ([P, I64, I32, P, P, P, P, P], I32),
            "bcts_search_pruned": ([P, P, I64, I32, I32, F, F, I32, C.POINTER(Prune), P, P, P, P, P, P,
                                    C.POINTER(Stats)], I32),
            "bcts_nccl_unique_id": ([P], I32),
            "bcts_workspace_size": ([P, I64, I32, C.POINTER(C.c_size_t)], I32),
            "bcts_set_workspace": ([P, P, C.c_size_t], I32),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        if L.bcts_abi_version() != ABI_VERSION:
            raise ImportError("libbcts ABI version mismatch")
        _lib = L
    return _lib


def _p(t):
    """Device (or host) pointer of a torch tensor / numpy array / None."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data_as(C.c_void_p)
    return C.c_void_p(t.data_ptr())


def pack_key(value: float, leaf: int) -> int:
    return lib().bcts_pack_key(float(value), int(leaf))


def key_value(key: int) -> float:
    return lib().bcts_key_value(int(key))


def key_leaf(key: int) -> int:
    return lib().bcts_key_leaf(int(key))


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (bcts_nccl_unique_id; needs no GPU). Make it on one rank and give the
    same bytes to every rank's Handle(..., nccl_id=..., rank=r, world=W)."""
    buf = C.create_string_buffer(128)
    s = lib().bcts_nccl_unique_id(buf)
    if s:
        raise BctsError(s, "bcts_nccl_unique_id")
    return buf.raw


def shard_range(n_roots: int, depth: int, A: int, rank: int, world: int) -> tuple[int, int]:
    b, e = C.c_int64(), C.c_int64()
    s = lib().bcts_shard_range(n_roots, depth, A, rank, world, C.byref(b), C.byref(e))
    if s:
        raise BctsError(s, "bcts_shard_range")
    return b.value, e.value


class Handle:
    """One bcts handle: env + value net on one device/stream."""

    def __init__(self, env: int, A: int, net: int, *, weights=None, tab=None, device: int = 0, stream=None,
                 mlp_in: int = 64, mlp_hidden: int = 256, atoms: int = 51, v_min: float = -10.0,
                 v_max: float = 10.0, workspace_bytes_max: int = 0, flags: int = 0, env_weights=None,
                 nccl_id: bytes | None = None, rank: int = 0, world: int = 1):
        import torch
        self.env, self.A, self.net, self.device = env, A, net, device
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        cfg = Config()
        cfg.abi_version = ABI_VERSION
        cfg.device = device
        cfg.cuda_stream = stream.cuda_stream
        cfg.env, cfg.num_actions, cfg.net = env, A, net
        keep = []
        if tab is not None:
            nxt = np.ascontiguousarray(tab.next, np.int32)
            rew = np.ascontiguousarray(tab.reward, np.float32)
            q = np.ascontiguousarray(tab.q, np.float32)
            keep += [nxt, rew, q]
            cfg.num_states = tab.nS
            cfg.tab_next, cfg.tab_reward, cfg.tab_q = _p(nxt).value, _p(rew).value, _p(q).value
        if weights is not None:
            w = np.ascontiguousarray(weights, np.float32)
            keep.append(w)
            cfg.weights, cfg.weights_count = _p(w).value, w.size
        if env_weights is not None:
            ew = np.ascontiguousarray(env_weights, np.float32)
            keep.append(ew)
            cfg.env_weights, cfg.env_weights_count = _p(ew).value, ew.size
        cfg.mlp_in, cfg.mlp_hidden, cfg.atoms = mlp_in, mlp_hidden, atoms
        cfg.v_min, cfg.v_max = v_min, v_max
        cfg.workspace_bytes_max = workspace_bytes_max
        cfg.flags = flags
        if nccl_id is not None:   # collective create: every rank passes the same id (bcts_nccl_unique_id)
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
            keep.append(idbuf)
            cfg.nccl_unique_id = C.cast(idbuf, C.c_void_p).value
        cfg.rank, cfg.world = rank, world
        self.rank, self.world = rank, world
        self._ws = None
        h = C.c_void_p()
        s = lib().bcts_create(C.byref(cfg), C.byref(h))
        if s:
            raise BctsError(s, "bcts_create")
        self._h = h
        self.record_bytes = lib().bcts_root_record_bytes(h)

    @classmethod
    def from_config(cls, cfg, tab=None, **kw):
        from synth.inputs import make_env_weights  # input generators only
        nk = cfg.net_kw()
        w = cfg.weights()[0]
        if cfg.env == ENV_DNN:
            kw.setdefault("env_weights", make_env_weights(cfg))
        return cls(cfg.env, cfg.A, cfg.net, weights=w, tab=tab, **{**nk, **kw})

    def close(self):
        if getattr(self, "_h", None):
            lib().bcts_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, s, what):
        if s:
            raise BctsError(s, f"{what}: {lib().bcts_last_error(self._h).decode()}")

    # ---- device-tensor API --------------------------------------------------
    def _outputs(self, n, extra):
        import torch
        dev = torch.device("cuda", self.device)
        out = {"actions": torch.empty(n, dtype=torch.int32, device=dev),
               "root_q": torch.empty(n, self.A, dtype=torch.float32, device=dev)}
        if extra:
            out["vanilla_q"] = torch.empty(n, self.A, dtype=torch.float32, device=dev)
            out["terms"] = torch.empty(n, 4, dtype=torch.float32, device=dev)
            out["best_leaf"] = torch.empty(n, self.A, dtype=torch.int64, device=dev)
        return out

    def search(self, roots, n_roots: int, depth: int, gamma: float, beta: float = 1.0, correction: int = 1,
               extra: bool = False, out=None):
        """roots: device uint8 tensor of n_roots records. Returns dict of device tensors (+ stats)."""
        out = out or self._outputs(n_roots, extra)
        st = Stats()
        s = lib().bcts_search_ex(self._h, _p(roots), n_roots, depth, self.A, gamma, beta, correction,
                                 _p(out["actions"]), _p(out["root_q"]), _p(out.get("vanilla_q")),
                                 _p(out.get("terms")), _p(out.get("best_leaf")), C.byref(st))
        self._check(s, "bcts_search_ex")
        out["stats"] = st.as_dict()
        return out

    def search_pruned(self, roots, n_roots: int, depth: int, gamma: float, rule: int, first_level: int = 1,
                      beam: int = 1, r_lo: float = 0.0, r_hi: float = 0.0, q_lo: float = 0.0, q_hi: float = 0.0,
                      beta: float = 1.0, correction: int = 1):
        """Early-pruned search (NEXT-4, include/bcts.h bcts_search_pruned). Returns device outputs
        (actions, root_q, vanilla_q, terms, best_leaf), 'survivors' (numpy [depth+1]) and 'stats'."""
        out = self._outputs(n_roots, True)
        pr = Prune(rule, first_level, beam, r_lo, r_hi, q_lo, q_hi)
        surv = np.zeros(depth + 1, np.int64)
        st = Stats()
        s = lib().bcts_search_pruned(self._h, _p(roots), n_roots, depth, self.A, gamma, beta, correction,
                                     C.byref(pr), _p(out["actions"]), _p(out["root_q"]), _p(out["vanilla_q"]),
                                     _p(out["terms"]), _p(out["best_leaf"]), _p(surv), C.byref(st))
        self._check(s, "bcts_search_pruned")
        out["survivors"] = surv
        out["stats"] = st.as_dict()
        return out

    def search_plain(self, roots, n_roots, depth, gamma, beta, correction, actions, root_q):
        self._check(lib().bcts_search(self._h, _p(roots), n_roots, depth, self.A, gamma, beta, correction,
                                      _p(actions), _p(root_q)), "bcts_search")

    def search_host(self, roots_host, n_roots, depth, gamma, beta, correction, actions_host, root_q_host):
        """Host buffers in and out (pinned torch tensors or numpy arrays); synchronous."""
        self._check(lib().bcts_search_host(self._h, _p(roots_host), n_roots, depth, self.A, gamma, beta,
                                           correction, _p(actions_host), _p(root_q_host)), "bcts_search_host")

    def keys_init(self, keys):
        self._check(lib().bcts_keys_init(self._h, _p(keys), keys.numel()), "bcts_keys_init")

    def search_shard(self, roots, n_roots, depth, gamma, leaf_begin, leaf_end, keys):
        st = Stats()
        self._check(lib().bcts_search_shard(self._h, _p(roots), n_roots, depth, self.A, gamma, leaf_begin,
                                            leaf_end, _p(keys), C.byref(st)), "bcts_search_shard")
        return st.as_dict()

    def finalize(self, roots, n_roots, depth, gamma, beta, correction, keys, extra=True):
        out = self._outputs(n_roots, extra)
        st = Stats()
        self._check(lib().bcts_finalize(self._h, _p(roots), n_roots, depth, self.A, gamma, beta, correction,
                                        _p(keys), _p(out["actions"]), _p(out["root_q"]),
                                        _p(out.get("vanilla_q")), _p(out.get("terms")),
                                        _p(out.get("best_leaf")), C.byref(st)), "bcts_finalize")
        out["stats"] = st.as_dict()
        return out

    def expand(self, roots, n_roots, level, gamma):
        import torch
        dev = torch.device("cuda", self.device)
        cnt = n_roots * self.A ** level
        states = torch.empty(cnt, self.record_bytes, dtype=torch.uint8, device=dev)
        cum = torch.empty(cnt, dtype=torch.float32, device=dev)
        self._check(lib().bcts_expand(self._h, _p(roots), n_roots, level, self.A, gamma, _p(states), _p(cum)),
                    "bcts_expand")
        return states, cum

    def profile(self, on: bool):
        self._check(lib().bcts_profile_enable(self._h, 1 if on else 0), "bcts_profile_enable")

    def profile_read(self):
        """{class: {launches, ms, work, unit}} accumulated since profile(True)."""
        buf = (KernelProfile * 32)()
        k = lib().bcts_profile_read(self._h, buf, 32)
        return {buf[i].name.decode(): {"launches": buf[i].launches, "ms": buf[i].ms, "work": buf[i].work,
                                       "unit": "flop" if buf[i].unit else "byte",
                                       "big_launches": buf[i].big_launches, "big_ms": buf[i].big_ms,
                                       "big_work": buf[i].big_work} for i in range(k)}

    def pv_targets(self, actions, vanilla_q, best_leaf, n, depth):
        """PV training target (App. B.3) of the executed actions + the best-leaf action path."""
        import torch
        dev = torch.device("cuda", self.device)
        target = torch.empty(n, dtype=torch.float32, device=dev)
        path = torch.empty(n, depth, dtype=torch.int32, device=dev)
        self._check(lib().bcts_pv_targets(self._h, n, depth, _p(actions), _p(vanilla_q), _p(best_leaf), _p(target),
                                          _p(path)), "bcts_pv_targets")
        return target, path

    def workspace_size(self, n_roots: int, depth: int) -> int:
        """Device bytes a search of n_roots roots at `depth` needs (net scratch + tree workspace)."""
        b = C.c_size_t()
        self._check(lib().bcts_workspace_size(self._h, n_roots, depth, C.byref(b)), "bcts_workspace_size")
        return b.value

    def set_workspace(self, buf):
        """Caller-owned device memory (a torch uint8 tensor on this device, or None to return to
        library-owned memory); the handle keeps a reference while it may use it."""
        self._check(lib().bcts_set_workspace(self._h, _p(buf), 0 if buf is None else buf.numel() * buf.element_size()),
                    "bcts_set_workspace")
        self._ws = buf

    def q_rows(self, states, n):
        import torch
        q = torch.empty(n, self.A, dtype=torch.float32, device=torch.device("cuda", self.device))
        self._check(lib().bcts_q_rows(self._h, _p(states), n, _p(q)), "bcts_q_rows")
        return q
