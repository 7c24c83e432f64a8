"""CPU-side checks of the C-ABI library: it builds, loads, exports every symbol
include/bcts.h declares, and its host-only logic (packed keys, shard plan,
argument validation that precedes any CUDA call) behaves. No GPU compute."""
import os
import re
import struct

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2107_01715_b200 import build
    build.build()
    import paper_2107_01715_b200 as P
    return P


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "bcts.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(bcts_[a-z_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(L):
    import subprocess
    syms = header_symbols()
    assert len(syms) >= 18
    nm = subprocess.run(["nm", "-D", "--defined-only", L.bcts.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (bcts_\w+)", nm))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert sorted(L.EXPORTS) == syms
    lib = L.lib()
    for s in syms:
        assert hasattr(lib, s)
    assert lib.bcts_abi_version() == 1


def test_status_strings(L):
    lib = L.lib()
    assert lib.bcts_status_string(0) == b"BCTS_OK"
    assert lib.bcts_status_string(4) == b"BCTS_ERR_BUDGET"


def test_config_struct_layout(L):
    """ctypes mirror of bcts_config has the C layout (natural alignment, 8-byte pointers)."""
    C = L.bcts.Config
    offs = {n: getattr(C, n).offset for n, _ in C._fields_}
    assert offs["cuda_stream"] == 8 and offs["env"] == 16 and offs["tab_next"] == 32
    assert offs["net"] == 56 and offs["weights"] == 64 and offs["weights_count"] == 72
    assert offs["workspace_bytes_max"] == 104 and offs["flags"] == 112
    import ctypes
    assert ctypes.sizeof(C) == 120


def f32(x):
    return struct.unpack("f", struct.pack("f", x))[0]


def test_packed_key_order(L):
    """Key order == (value, then LOWEST leaf index) under signed int64 max (R4, §6)."""
    rng = np.random.default_rng(0)
    vals = [f32(v) for v in np.concatenate([rng.normal(size=200) * 10, [0.0, -0.0, 1e-30, -1e-30, 3e38, -3e38]])]
    items = [(v, int(i)) for v in vals for i in rng.integers(0, 2 ** 32 - 1, size=3)]
    keys = [L.pack_key(v, i) for v, i in items]
    for (v, i), k in zip(items, keys):
        assert L.key_value(k) == (0.0 if v == 0.0 else v) and L.key_leaf(k) == i
    order = sorted(range(len(items)), key=lambda j: keys[j])
    expect = sorted(range(len(items)), key=lambda j: (items[j][0], -items[j][1]))
    assert [items[j] for j in order] == [items[j] for j in expect]
    assert L.pack_key(-0.0, 5) == L.pack_key(0.0, 5)
    assert L.pack_key(-3e38, 2 ** 32 - 1) > -(2 ** 63)   # the empty key (INT64_MIN) is below every real key


@pytest.mark.parametrize("n,d,A", [(1, 4, 18), (1024, 5, 6), (64, 3, 18), (7, 2, 4), (3, 1, 2)])
def test_shard_range_plan(L, n, d, A):
    total = n * A ** d
    for W in (1, 2, 3, 4, 8):
        rs = [L.shard_range(n, d, A, r, W) for r in range(W)]
        assert rs[0][0] == 0 and rs[-1][1] == total
        assert all(rs[i][1] == rs[i + 1][0] for i in range(W - 1))
        sizes = [e - b for b, e in rs]
        if n % W == 0:
            assert all(b % A ** d == 0 for b, _ in rs)        # whole roots per rank (C4)
            assert len(set(sizes)) == 1
        else:
            assert max(sizes) - min(sizes) <= 1               # balanced leaf ranges (C5)


def test_create_rejects_bad_config_without_gpu(L):
    import ctypes
    lib = L.lib()
    cfg = L.bcts.Config()
    h = ctypes.c_void_p()
    cfg.abi_version = 99
    assert lib.bcts_create(ctypes.byref(cfg), ctypes.byref(h)) == 1
    cfg.abi_version = 1
    cfg.num_actions = 1                                        # A >= 2
    assert lib.bcts_create(ctypes.byref(cfg), ctypes.byref(h)) == 1
    cfg.num_actions, cfg.env, cfg.net = 4, 2, 1                # INT_HASH + TABLE: unsupported pair
    assert lib.bcts_create(ctypes.byref(cfg), ctypes.byref(h)) == 2
    assert not h.value
    assert lib.bcts_search(None, None, 0, 1, 2, 0.9, 1.0, 1, None, None) == 1


def test_no_cpu_fallback_in_product_path():
    """The product package never imports, links or loads the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2107_01715_b200")
    pat = re.compile(r"(import\s+oracle|from\s+oracle|liboracle|oracle_search|oracle_qrow)")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                assert not pat.search(open(os.path.join(dirpath, f)).read()), f
