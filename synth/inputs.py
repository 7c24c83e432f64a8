"""Seeded synthetic inputs: root records, weight blobs, tabular fixtures, configs.

Only input generation lives here. The forward model, the value
nets, the search and the BCTS correction are implemented twice and
independently: in ``oracle/`` (plain C, test infrastructure) and in
``paper_2107_01715_b200/csrc`` (CUDA). Neither imports the other; both consume
the arrays this module produces.

Root-record layouts (the C-ABI ``roots`` buffer):
  * TABULAR    : int32 state id                                   (4 B)
  * INT_HASH   : uint32[16] state words                           (64 B)
  * ATARI_HASH : uint64 key, uint64 pad(=0), uint32 w[7056]        (28,240 B)
                 w[p] packs the 4-frame stack of pixel p = y*84+x:
                 byte c of w[p] is frame c (c=0 oldest, c=3 newest).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "MASK64", "mix64", "ENV_TABULAR", "ENV_INT_HASH", "ENV_ATARI_HASH", "ENV_DNN", "DNN_STATE",
    "dnn_roots", "make_env_weights",
    "NET_TABLE", "NET_MLP2_F32", "NET_NATURE_BF16", "NET_RAINBOW_BF16",
    "ATARI_WORDS", "ATARI_RECORD_BYTES", "INT_RECORD_BYTES",
    "atari_roots", "int_roots", "tabular_roots", "weight_specs", "make_weights",
    "Tabular", "chain_c1", "worked_w1", "worked_w2", "Config", "CONFIGS", "config",
]

MASK64 = (1 << 64) - 1
ENV_TABULAR, ENV_INT_HASH, ENV_ATARI_HASH, ENV_DNN = 1, 2, 3, 4
DNN_STATE = 100
NET_TABLE, NET_MLP2_F32, NET_NATURE_BF16, NET_RAINBOW_BF16 = 1, 2, 3, 4

ATARI_H = ATARI_W = 84
ATARI_WORDS = ATARI_H * ATARI_W            # 7056 packed pixel words
ATARI_RECORD_BYTES = 16 + 4 * ATARI_WORDS  # 28,240
INT_RECORD_BYTES = 64


def mix64(z):
    """splitmix64 finalizer on uint64 numpy arrays (seed hashing only)."""
    z = np.asarray(z, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


# ---------------------------------------------------------------- root records
def atari_roots(n: int, seed: int) -> np.ndarray:
    """n ATARI_HASH root records as a uint8 array [n, 28240].

    key_r = mix64(seed ^ mix64(r+1)); byte c of w[p] =
    (mix64(key_r + ((c+1)<<40) + (p>>3)) >> 8*(p&7)) & 0xFF  (uniform bytes).
    """
    out = np.zeros((n, ATARI_RECORD_BYTES), dtype=np.uint8)
    if n == 0:
        return out
    r = np.arange(n, dtype=np.uint64)
    keys = mix64(np.uint64(seed & MASK64) ^ mix64(r + np.uint64(1)))
    out[:, 0:8] = keys.view(np.uint8).reshape(n, 8)
    groups = np.arange(ATARI_WORDS // 8, dtype=np.uint64)
    planes = np.empty((n, 4, ATARI_WORDS), dtype=np.uint8)
    with np.errstate(over="ignore"):
        for c in range(4):
            h = mix64(keys[:, None] + np.uint64((c + 1) << 40) + groups[None, :])
            planes[:, c, :] = h.view(np.uint8).reshape(n, ATARI_WORDS)
    words = np.ascontiguousarray(planes.transpose(0, 2, 1)).reshape(n, 4 * ATARI_WORDS)
    out[:, 16:] = words
    return out


def int_roots(n: int, seed: int) -> np.ndarray:
    """n INT_HASH root records, uint32 [n, 16]: s[w] = low32(mix64(seed ^ mix64((r<<8)|w)))."""
    r = np.arange(n, dtype=np.uint64)[:, None]
    w = np.arange(16, dtype=np.uint64)[None, :]
    h = mix64(np.uint64(seed & MASK64) ^ mix64((r << np.uint64(8)) | w))
    return (h & np.uint64(0xFFFFFFFF)).astype(np.uint32)


def dnn_roots(n: int, seed: int) -> np.ndarray:
    """n DNN-env root states, float32 [n, 100]: uniform in [-1, 1) from mix64(seed ^ mix64((r<<8)|j))."""
    r = np.arange(n, dtype=np.uint64)[:, None]
    j = np.arange(DNN_STATE, dtype=np.uint64)[None, :]
    h = mix64(np.uint64(seed & MASK64) ^ mix64((r << np.uint64(8)) | j))
    u = (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return (2.0 * u - 1.0).astype(np.float32)


def tabular_roots(ids) -> np.ndarray:
    return np.asarray(ids, dtype=np.int32)


# ---------------------------------------------------------------- weights
def weight_specs(net: int, A: int, mlp_in: int = 64, mlp_hidden: int = 256, atoms: int = 51):
    """[(name, shape, fan_in)] in canonical PyTorch order for a net kind."""
    if net == NET_MLP2_F32:
        return [("l1.w", (mlp_hidden, mlp_in), mlp_in), ("l1.b", (mlp_hidden,), mlp_in),
                ("l2.w", (A, mlp_hidden), mlp_hidden), ("l2.b", (A,), mlp_hidden)]
    trunk = [("conv1.w", (32, 4, 8, 8), 256), ("conv1.b", (32,), 256),
             ("conv2.w", (64, 32, 4, 4), 512), ("conv2.b", (64,), 512),
             ("conv3.w", (64, 64, 3, 3), 576), ("conv3.b", (64,), 576)]
    if net == NET_NATURE_BF16:
        return trunk + [("fc1.w", (512, 3136), 3136), ("fc1.b", (512,), 3136),
                        ("fc2.w", (A, 512), 512), ("fc2.b", (A,), 512)]
    if net == NET_RAINBOW_BF16:
        return trunk + [("fc_h_v.w", (512, 3136), 3136), ("fc_h_v.b", (512,), 3136),
                        ("fc_h_a.w", (512, 3136), 3136), ("fc_h_a.b", (512,), 3136),
                        ("fc_z_v.w", (atoms, 512), 512), ("fc_z_v.b", (atoms,), 512),
                        ("fc_z_a.w", (A * atoms, 512), 512), ("fc_z_a.b", (A * atoms,), 512)]
    raise ValueError(f"no weights for net kind {net}")


def env_weight_specs(A: int):
    """Random-DNN forward model: 3 hidden layers of width 100 over [state(100); onehot(a)],
    linear output 101 = (next state, reward) (R27)."""
    S = DNN_STATE
    return [("g1.w", (S, S + A), S + A), ("g1.b", (S,), S + A), ("g2.w", (S, S), S), ("g2.b", (S,), S),
            ("g3.w", (S, S), S), ("g3.b", (S,), S), ("g4.w", (S + 1, S), S), ("g4.b", (S + 1,), S)]


def _blob(specs, wseed, scale_first=None):
    parts = []
    for t, (name, shape, fan_in) in enumerate(specs):
        cnt = int(np.prod(shape))
        e = np.arange(cnt, dtype=np.uint64)
        h = mix64(np.uint64(wseed & MASK64) ^ mix64((np.uint64(t) << np.uint64(40)) | e))
        u = (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        parts.append(((2.0 * u - 1.0) / math.sqrt(fan_in)).astype(np.float32))
    return np.concatenate(parts)


def make_env_weights(cfg) -> np.ndarray:
    """Canonical fp32 blob of the random-DNN forward model (same element recipe as make_weights)."""
    return _blob(env_weight_specs(cfg.A), cfg.extra.get("env_wseed", cfg.wseed + 7))


HEAD_TENSORS = ("fc2.w", "fc_z_v.w", "fc_z_a.w")   # the output layers (Nature fc2; Rainbow z_v, z_a)


def make_weights(net: int, A: int, wseed: int, head_scale: float = 1.0, **kw) -> tuple[np.ndarray, dict]:
    """Canonical fp32 weight blob (concatenation in weight_specs order) + views.

    Element e of tensor t: u = (mix64(wseed ^ mix64((t<<40)|e)) >> 11) * 2^-53,
    value = (2u-1)/sqrt(fan_in)  (PyTorch's default Linear/Conv bound);
    conv1.w is additionally scaled by 1/255 (input /255 folded in, R15).
    head_scale (test-only "spread" weights): the output layers' weights
    (HEAD_TENSORS) are multiplied by it. Random-init Q-hat is nearly flat across leaves
    (max |Q| ~ 0.05, leaf-to-leaf spread ~ 0.004); x64 spreads it (~1.5 / ~0.25) so a
    parity test at the search tolerance can tell a broken trunk from rounding.
    """
    specs = weight_specs(net, A, **kw)
    parts, views = [], {}
    for t, (name, shape, fan_in) in enumerate(specs):
        cnt = int(np.prod(shape))
        e = np.arange(cnt, dtype=np.uint64)
        h = mix64(np.uint64(wseed & MASK64) ^ mix64((np.uint64(t) << np.uint64(40)) | e))
        u = (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        v = (2.0 * u - 1.0) / math.sqrt(fan_in)
        if name == "conv1.w":
            v = v / 255.0
        if head_scale != 1.0 and name in HEAD_TENSORS:
            v = v * head_scale
        parts.append(v.astype(np.float32))
    blob = np.concatenate(parts) if parts else np.zeros(0, np.float32)
    off = 0
    for (name, shape, _), p in zip(specs, parts):
        views[name] = blob[off:off + p.size].reshape(shape)
        off += p.size
    return blob, views


# ---------------------------------------------------------------- tabular fixtures
@dataclass
class Tabular:
    """A literal deterministic MDP + tabular Q-hat (inputs, not results)."""
    A: int
    next: np.ndarray      # int32 [nS*A]
    reward: np.ndarray    # float64 [nS*A]
    q: np.ndarray         # float64 [nS*A]

    @property
    def nS(self) -> int:
        return self.next.size // self.A


def _tab(A, nxt, rew, q):
    return Tabular(A, np.asarray(nxt, np.int32).ravel(), np.asarray(rew, np.float64).ravel(),
                   np.asarray(q, np.float64).ravel())


def chain_c1(exact: bool = False) -> Tabular:
    """SPEC chain-grid L=5, A=2 (0=LEFT, 1=RIGHT), goal 4 absorbing.

    Entering state 4 gives r=1; LEFT at 0 stays at 0. Q-hat = Q* except the two
    over-estimated entries of SURVEY §8c (C1-chain) unless ``exact``.
    """
    nxt = [[0, 1], [0, 2], [1, 3], [2, 4], [4, 4]]
    rew = [[0, 0], [0, 0], [0, 0], [0, 1], [0, 0]]
    q = [[0.6561, 0.729], [0.6561, 0.81], [0.729, 0.9], [0.81, 1.0], [0.0, 0.0]]
    q = np.array(q)
    if not exact:
        q[0, 0] = 0.4561
        q[2, 1] = 1.1
    return _tab(2, nxt, rew, q)


def worked_w1() -> Tabular:
    """A=2, d=1, gamma=0.5. States 0=s0, 1=s1^0, 2=s1^1."""
    nxt = [[1, 2], [1, 1], [2, 2]]
    rew = [[0, 1], [0, 0], [0, 0]]
    q = [[1.0, 0.5], [2.0, 1.0], [0.0, 3.0]]
    return _tab(2, nxt, rew, q)


def worked_w2() -> Tabular:
    """A=2, d=2, gamma=0.5. Leaf i=2*a0+a1 is state 3+i."""
    nxt = [[1, 2], [3, 4], [5, 6], [3, 3], [4, 4], [5, 5], [6, 6]]
    rew = [[0, 1], [2, 0], [0, -1], [0, 0], [0, 0], [0, 0], [0, 0]]
    q = [[1.5, 1.0], [3, 1], [1, 2], [1, 0], [4, 2], [0, 2], [6, 6]]
    return _tab(2, nxt, rew, q)


# ---------------------------------------------------------------- configs
@dataclass
class Config:
    name: str
    env: int
    net: int
    A: int
    depth: int
    n_roots: int
    gamma: float
    beta: float
    seed: int = 0
    wseed: int = 0
    correction: tuple = (0, 1)
    note: str = ""
    extra: dict = field(default_factory=dict)

    def roots(self, n: int | None = None) -> np.ndarray:
        n = self.n_roots if n is None else n
        if self.env == ENV_ATARI_HASH:
            return atari_roots(n, self.seed)
        if self.env == ENV_INT_HASH:
            return int_roots(n, self.seed)
        if self.env == ENV_DNN:
            return dnn_roots(n, self.seed)
        return tabular_roots([0] * n)

    def net_kw(self) -> dict:
        """Net shape arguments beyond the defaults (the DNN env's MLP reads 100 float features)."""
        return {"mlp_in": DNN_STATE} if self.env == ENV_DNN else {}

    def weights(self):
        """The value net's canonical weight blob and views (None for the table net)."""
        if self.net == NET_TABLE:
            return None, {}
        return make_weights(self.net, self.A, self.wseed, head_scale=self.extra.get("head_scale", 1.0),
                            **self.net_kw())


CONFIGS = {
    "C1": Config("C1", ENV_TABULAR, NET_TABLE, 2, 3, 1, 0.9, 1.0,
                 note="SPEC chain-grid L=5, tabular Q-hat, 1 root"),
    "C2": Config("C2", ENV_INT_HASH, NET_MLP2_F32, 4, 4, 256, 0.99, 1.0, seed=2, wseed=102,
                 note="integer hash env, MLP2 64-256-4 fp32"),
    "C3": Config("C3", ENV_ATARI_HASH, NET_NATURE_BF16, 18, 3, 64, 0.99, 1.0, seed=3, wseed=103,
                 note="Atari-shaped 4x84x84 uint8, Nature-DQN A=18 bf16"),
    "C4": Config("C4", ENV_ATARI_HASH, NET_RAINBOW_BF16, 6, 5, 1024, 0.99, 1.0, seed=4, wseed=104,
                 correction=(1,), note="Rainbow A=6 bf16, d=5, 1024 roots"),
    "C5": Config("C5", ENV_ATARI_HASH, NET_RAINBOW_BF16, 18, 4, 1, 0.99, 1.0, seed=5, wseed=105,
                 correction=(1,), note="Rainbow A=18 bf16, d=4, 1 root (headline)"),
    # NEXT-1: the paper's second runtime workload, a random DNN as learned forward model,
    # Fig. 4 right: A in {2, 10}; leaf value = MLP2 100-256-A fp32
    "D2": Config("D2", ENV_DNN, NET_MLP2_F32, 2, 8, 64, 0.99, 1.0, seed=21, wseed=121,
                 note="random-DNN forward model, A=2"),
    "D10": Config("D10", ENV_DNN, NET_MLP2_F32, 10, 4, 64, 0.99, 1.0, seed=22, wseed=122,
                  note="random-DNN forward model, A=10"),
}


# test-only "spread" variants (head_scale, see make_weights): same envs / roots, output layers x64
for _n in ("C3", "C4", "C5"):
    _c = CONFIGS[_n]
    CONFIGS[_n + "S"] = Config(_n + "S", _c.env, _c.net, _c.A, _c.depth, _c.n_roots, _c.gamma, _c.beta, _c.seed,
                               _c.wseed, _c.correction, _c.note + "; output layers x64 (spread Q-hat, tests only)",
                               {"head_scale": 64.0})


def config(name: str) -> Config:
    return CONFIGS[name]
