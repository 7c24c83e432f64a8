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
    ver = int(re.search(r"#define BCTS_ABI_VERSION (\d+)", open(os.path.join(ROOT, "include", "bcts.h")).read())[1])
    assert lib.bcts_abi_version() == ver == L.bcts.ABI_VERSION


@pytest.mark.parametrize("struct", ["Config", "Stats", "KernelProfile", "Prune"])
def test_ctypes_structs_match_c_layout(L, struct, tmp_path):
    """The binding's ctypes mirrors of bcts_config / bcts_stats / bcts_kernel_profile have the C
    compiler's size and field offsets (gcc on include/bcts.h)."""
    import ctypes
    import subprocess
    cname = {"Config": "bcts_config", "Stats": "bcts_stats", "KernelProfile": "bcts_kernel_profile",
             "Prune": "bcts_prune"}[struct]
    py = getattr(L.bcts, struct)
    lines = [f'printf("size %zu\\n", sizeof({cname}));']
    lines += [f'printf("{f} %zu\\n", offsetof({cname}, {f}));' for f, _ in py._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "bcts.h"\nint main(void) {\n'
                   + "\n".join(lines) + "\nreturn 0; }\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n") if l)
    assert int(got["size"]) == ctypes.sizeof(py)
    for f, _ in py._fields_:
        assert int(got[f]) == getattr(py, f).offset, f


def test_status_strings(L):
    lib = L.lib()
    assert lib.bcts_status_string(0) == b"BCTS_OK"
    assert lib.bcts_status_string(4) == b"BCTS_ERR_BUDGET"


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
    cfg.abi_version = L.bcts.ABI_VERSION
    cfg.num_actions = 1                                        # A >= 2
    assert lib.bcts_create(ctypes.byref(cfg), ctypes.byref(h)) == 1
    cfg.num_actions, cfg.env, cfg.net = 4, 2, 1                # INT_HASH + TABLE: unsupported pair
    assert lib.bcts_create(ctypes.byref(cfg), ctypes.byref(h)) == 2
    cfg.env, cfg.net, cfg.mlp_in, cfg.mlp_hidden = 4, 2, 100, 256   # DNN without env weights
    assert lib.bcts_create(ctypes.byref(cfg), ctypes.byref(h)) == 1
    ew = np.zeros(40501 + 100 * 4 - 1, np.float32)                # one float short
    cfg.env_weights, cfg.env_weights_count = ew.ctypes.data, ew.size
    assert lib.bcts_create(ctypes.byref(cfg), ctypes.byref(h)) == 1
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


def test_nccl_unique_id_without_gpu(L):
    """bcts_nccl_unique_id needs no GPU (NCCL resolved at run time): 128 bytes, fresh per call."""
    a, b = L.nccl_unique_id(), L.nccl_unique_id()
    assert len(a) == len(b) == 128 and a != b
    assert L.lib().bcts_nccl_unique_id(None) == 1


def test_world_and_workspace_argument_checks_without_gpu(L):
    """Argument checks that precede any CUDA call: rank/world of a multi-GPU config, NULL handles
    of the workspace entry points."""
    import ctypes
    lib = L.lib()
    cfg = L.bcts.Config()
    cfg.abi_version = L.bcts.ABI_VERSION
    cfg.env, cfg.net, cfg.num_actions, cfg.mlp_in, cfg.mlp_hidden = 2, 2, 4, 64, 256
    h = ctypes.c_void_p()
    cfg.world, cfg.rank = 2, 0                     # world > 1 needs the unique id
    assert lib.bcts_create(ctypes.byref(cfg), ctypes.byref(h)) == 1
    idbuf = ctypes.create_string_buffer(L.nccl_unique_id(), 128)
    cfg.nccl_unique_id = ctypes.cast(idbuf, ctypes.c_void_p).value
    cfg.rank = 2                                   # rank outside [0, world)
    assert lib.bcts_create(ctypes.byref(cfg), ctypes.byref(h)) == 1
    cfg.rank = -1
    assert lib.bcts_create(ctypes.byref(cfg), ctypes.byref(h)) == 1
    assert not h.value
    size = ctypes.c_size_t()
    assert lib.bcts_workspace_size(None, 1, 4, ctypes.byref(size)) == 1
    assert lib.bcts_set_workspace(None, None, 0) == 1
    assert lib.bcts_status_string(6) == b"BCTS_ERR_NCCL"


def test_bench_self_launches_world2_reference_on_cpu():
    """`bench.py --gpus 2 --impl reference` outside torchrun re-runs itself as 2 ranks (gloo on CPU for
    the reference arm): rank 0 prints one JSON line with n_gpus 2, the other rank exits 0."""
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--config", "C2", "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                       timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


def test_python_flags_match_header():
    """The binding's BCTS_F_* constants are the header's (argument marshalling only)."""
    import paper_2107_01715_b200 as P
    hdr = open(os.path.join(ROOT, "include", "bcts.h")).read()
    for name in ("CLAMP_PENALTY", "SIMT_NET", "MATERIALIZE_LEAVES", "SEPARATE_BACKUP", "NO_PROLOGUE_FOLD", "NO_GRAPH",
                 "TF32"):
        v = int(re.search(r"#define BCTS_F_%s (0x[0-9a-fA-F]+)u" % name, hdr)[1], 16)
        assert getattr(P, "F_" + name) == v, name
