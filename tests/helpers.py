"""Shared test helpers: comparison rules of DESIGN.md §2 (R18, R19)."""
import numpy as np


def rel_err(gpu_q, ora_q):
    """|gpu - oracle| / max(max_a |oracle_q[r, a]|, 1e-6), per root (R18)."""
    gpu_q = np.asarray(gpu_q, np.float64)
    ora_q = np.asarray(ora_q, np.float64)
    scale = np.maximum(np.abs(ora_q).max(axis=-1, keepdims=True), 1e-6)
    return np.abs(gpu_q - ora_q) / scale


def action_agreement(gpu_actions, ora_q, rtol):
    """Near-tie rule (R19): the GPU action is accepted if it is the oracle's
    argmax, or if its oracle value is within 2*rtol*scale of the oracle max.
    Returns (fraction accepted, number of exact matches, number of near-ties)."""
    ora_q = np.asarray(ora_q, np.float64)
    gpu_actions = np.asarray(gpu_actions)
    n = ora_q.shape[0]
    scale = np.maximum(np.abs(ora_q).max(axis=1), 1e-6)
    best = ora_q.max(axis=1)
    mine = ora_q[np.arange(n), gpu_actions]
    exact = gpu_actions == ora_q.argmax(axis=1)
    near = (~exact) & (best - mine <= 2 * rtol * scale)
    return float((exact | near).mean()) if n else 1.0, int(exact.sum()), int(near.sum())
