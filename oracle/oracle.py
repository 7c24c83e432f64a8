"""ctypes wrapper over liboracle.so (TEST INFRASTRUCTURE ONLY; see __init__)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "bcts_oracle.c")
LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

ENV_TABULAR, ENV_INT_HASH, ENV_ATARI_HASH, ENV_DNN = 1, 2, 3, 4
NET_TABLE, NET_MLP2_F32, NET_NATURE_BF16, NET_RAINBOW_BF16 = 1, 2, 3, 4


def build(force: bool = False) -> str:
    """Compile liboracle.so: -O2 -ffp-contract=off (no FMA contraction), OpenMP."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", LIB_PATH, SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = C.CDLL(LIB_PATH)
            P, L, I, D = C.c_void_p, C.c_long, C.c_int, C.c_double
            lib.oracle_create.restype = P
            lib.oracle_create.argtypes = [I, I, I, P, P, I, P, P, L, I, I, I, D, D]
            lib.oracle_destroy.argtypes = [P]
            lib.oracle_record_bytes.restype = L
            lib.oracle_record_bytes.argtypes = [P]
            lib.oracle_step.restype = I
            lib.oracle_step.argtypes = [P, P, I, P, C.POINTER(D)]
            lib.oracle_qrow.restype = I
            lib.oracle_qrow.argtypes = [P, P, I, P]
            lib.oracle_search.restype = I
            lib.oracle_search.argtypes = [P, P, L, I, D, D, I, I, I, P, P, P, P, P]
            lib.oracle_search_bruteforce.restype = I
            lib.oracle_search_bruteforce.argtypes = [P, P, L, I, D, D, I, I, P, P, P, P, P]
            lib.oracle_node.restype = I
            lib.oracle_node.argtypes = [P, P, I, C.c_int64, D, I, P, C.POINTER(D)]
            lib.oracle_penalty_eq5.restype = D
            lib.oracle_penalty_eq5.argtypes = [D, D, I, I]
            lib.oracle_bias_gap_eq4.restype = D
            lib.oracle_bias_gap_eq4.argtypes = [D, D, I, I]
            lib.oracle_bf16_round.restype = D
            lib.oracle_bf16_round.argtypes = [D]
            lib.oracle_terms.restype = I
            lib.oracle_terms.argtypes = [P, P, L, I, D, I, P, P]
            lib.oracle_search_subtrees.restype = I
            lib.oracle_search_subtrees.argtypes = [P, P, I, D, I, I, L, L, P]
            lib.oracle_leaf_total.restype = I
            lib.oracle_leaf_total.argtypes = [P, P, I, C.c_int64, D, I, C.POINTER(D)]
            for fn in ("oracle_inv_norm_cdf", "oracle_B_n"):
                getattr(lib, fn).restype = D
                getattr(lib, fn).argtypes = [D]
            lib.oracle_bias_exact.restype = D
            lib.oracle_bias_exact.argtypes = [D, D, I, I]
            lib.oracle_set_env_weights.restype = I
            lib.oracle_set_env_weights.argtypes = [P, P, L]
            lib.oracle_max_threads.restype = I
            lib.oracle_search_pruned.restype = I
            lib.oracle_search_pruned.argtypes = [P, P, L, I, D, D, I, I, I, I, L, D, D, D, D,
                                                 P, P, P, P, P, P]
            _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def bf16_round(x: float) -> float:
    return _load().oracle_bf16_round(float(x))


def penalty_eq5(delta_e: float, delta_o: float, A: int, d: int) -> float:
    return _load().oracle_penalty_eq5(float(delta_e), float(delta_o), int(A), int(d))


def inv_norm_cdf(p: float) -> float:
    return _load().oracle_inv_norm_cdf(float(p))


def B_n(n: float) -> float:
    return _load().oracle_B_n(float(n))


def bias_exact(sigma_o: float, sigma_e: float, A: int, d: int) -> float:
    """Lemma 2 exact gap B_e - B_o."""
    return _load().oracle_bias_exact(float(sigma_o), float(sigma_e), int(A), int(d))


def bias_gap_eq4(sigma_o: float, sigma_e: float, A: int, d: int) -> float:
    return _load().oracle_bias_gap_eq4(float(sigma_o), float(sigma_e), int(A), int(d))


class Oracle:
    """One model (env + value net). Modes: 0 = fp64 reference, 1 = fp32 mirror."""

    def __init__(self, env: int, A: int, net: int, tab=None, weights=None,
                 mlp_in=64, mlp_hidden=256, atoms=51, v_min=-10.0, v_max=10.0, env_weights=None):
        lib = _load()
        self.env, self.A, self.net = env, A, net
        nS = 0
        tn = tr = tq = None
        if tab is not None:
            nS = tab.nS
            tn = np.ascontiguousarray(tab.next, np.int32)
            tr = np.ascontiguousarray(tab.reward, np.float64)
            tq = np.ascontiguousarray(tab.q, np.float64)
        w = None if weights is None else np.ascontiguousarray(weights, np.float32)
        self._keep = (tn, tr, tq, w)
        self._h = lib.oracle_create(env, A, nS, _ptr(tn), _ptr(tr), net, _ptr(tq), _ptr(w),
                                    0 if w is None else w.size, mlp_in, mlp_hidden, atoms,
                                    v_min, v_max)
        if not self._h:
            raise ValueError("oracle_create rejected the model")
        if env_weights is not None:
            ew = np.ascontiguousarray(env_weights, np.float32)
            self._keep = self._keep + (ew,)
            if lib.oracle_set_env_weights(self._h, _ptr(ew), ew.size):
                raise ValueError("oracle_set_env_weights rejected the blob")
        self.record_bytes = lib.oracle_record_bytes(self._h)

    @classmethod
    def from_config(cls, cfg, tab=None):
        from synth.inputs import make_env_weights  # input generators only
        w = cfg.weights()[0]
        ew = make_env_weights(cfg) if cfg.env == ENV_DNN else None
        return cls(cfg.env, cfg.A, cfg.net, tab=tab, weights=w, env_weights=ew, **cfg.net_kw())

    def close(self):
        if getattr(self, "_h", None):
            _load().oracle_destroy(self._h)
            self._h = None

    __del__ = close

    def _records(self, roots) -> np.ndarray:
        a = np.ascontiguousarray(roots)
        return a.view(np.uint8).reshape(-1, self.record_bytes) if a.size else a.reshape(0, self.record_bytes)

    def step(self, rec, a: int):
        rec = self._records(rec)[0]
        out = np.zeros(self.record_bytes, np.uint8)
        r = C.c_double()
        if _load().oracle_step(self._h, _ptr(rec), a, _ptr(out), C.byref(r)):
            raise ValueError("domain error in oracle_step")
        return out, r.value

    def qrow(self, rec, mode: int = 0) -> np.ndarray:
        rec = self._records(rec)[0]
        q = np.zeros(self.A, np.float64)
        if _load().oracle_qrow(self._h, _ptr(rec), mode, _ptr(q)):
            raise ValueError("domain error in oracle_qrow")
        return q

    def node(self, root_rec, level: int, index: int, gamma: float, mode: int = 0):
        rec = self._records(root_rec)[0]
        out = np.zeros(self.record_bytes, np.uint8)
        R = C.c_double()
        if _load().oracle_node(self._h, _ptr(rec), level, int(index), gamma, mode, _ptr(out), C.byref(R)):
            raise ValueError("domain error in oracle_node")
        return out, R.value

    def search(self, roots, depth: int, gamma: float, beta: float = 1.0, correction: int = 1,
               mode: int = 0, threads: int = 1, brute: bool = False) -> dict:
        recs = self._records(roots)
        n = recs.shape[0]
        A = self.A
        act = np.zeros(n, np.int32)
        rq = np.zeros(n * A, np.float64)
        van = np.zeros(n * A, np.float64)
        terms = np.zeros(n * 4, np.float64)
        bl = np.zeros(n * A, np.int64)
        lib = _load()
        if brute:
            rc = lib.oracle_search_bruteforce(self._h, _ptr(recs), n, depth, gamma, beta, correction,
                                              mode, _ptr(act), _ptr(rq), _ptr(van), _ptr(terms), _ptr(bl))
        else:
            rc = lib.oracle_search(self._h, _ptr(recs), n, depth, gamma, beta, correction, mode,
                                   threads, _ptr(act), _ptr(rq), _ptr(van), _ptr(terms), _ptr(bl))
        if rc:
            raise ValueError("oracle search failed (domain error)")
        return {"actions": act, "root_q": rq.reshape(n, A), "vanilla_q": van.reshape(n, A),
                "terms": terms.reshape(n, 4), "best_leaf": bl.reshape(n, A)}

    def search_pruned(self, roots, depth: int, gamma: float, rule: int, first: int = 1, beam: int = 1,
                      r_lo: float = 0.0, r_hi: float = 0.0, q_lo: float = 0.0, q_hi: float = 0.0,
                      beta: float = 1.0, correction: int = 1, mode: int = 0) -> dict:
        """Early-pruned search (rule 0 none, 1 BOUND, 2 BEAM; see bcts_oracle.c)."""
        recs = self._records(roots)
        n = recs.shape[0]
        A = self.A
        act = np.zeros(n, np.int32)
        rq = np.zeros(n * A, np.float64)
        van = np.zeros(n * A, np.float64)
        terms = np.zeros(n * 4, np.float64)
        bl = np.zeros(n * A, np.int64)
        surv = np.zeros(depth + 1, np.int64)
        rc = _load().oracle_search_pruned(self._h, _ptr(recs), n, depth, gamma, beta, correction, mode, rule,
                                          first, beam, r_lo, r_hi, q_lo, q_hi, _ptr(act), _ptr(rq), _ptr(van),
                                          _ptr(terms), _ptr(bl), _ptr(surv))
        if rc:
            raise ValueError("oracle_search_pruned failed")
        return {"actions": act, "root_q": rq.reshape(n, A), "vanilla_q": van.reshape(n, A),
                "terms": terms.reshape(n, 4), "best_leaf": bl.reshape(n, A), "survivors": surv}

    def leaf_total(self, root_rec, depth: int, index: int, gamma: float, mode: int = 0) -> float:
        rec = self._records(root_rec)[0]
        t = C.c_double()
        if _load().oracle_leaf_total(self._h, _ptr(rec), depth, int(index), gamma, mode, C.byref(t)):
            raise ValueError("oracle_leaf_total failed")
        return t.value

    def terms(self, roots, depth: int, gamma: float, mode: int = 0):
        """(pi_o, delta_o, delta_e, B) per root and the root rows Q_hat(s0, .)."""
        recs = self._records(roots)
        n = recs.shape[0]
        t = np.zeros(n * 4, np.float64)
        q0 = np.zeros(n * self.A, np.float64)
        if _load().oracle_terms(self._h, _ptr(recs), n, depth, gamma, mode, _ptr(t), _ptr(q0)):
            raise ValueError("oracle_terms failed")
        return t.reshape(n, 4), q0.reshape(n, self.A)

    def subtrees(self, root, depth: int, gamma: float, t_begin: int, t_end: int, mode: int = 0,
                 threads: int = 1) -> np.ndarray:
        """Max leaf total of each depth-2 subtree t = a0*A + a1 in [t_begin, t_end) (bounded sample)."""
        rec = self._records(root)[0]
        out = np.zeros(max(t_end - t_begin, 1), np.float64)
        if _load().oracle_search_subtrees(self._h, _ptr(rec), depth, gamma, mode, threads, t_begin, t_end,
                                          _ptr(out)):
            raise ValueError("oracle_search_subtrees failed")
        return out[:t_end - t_begin]

    @staticmethod
    def max_threads() -> int:
        return _load().oracle_max_threads()
