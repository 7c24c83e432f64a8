"""The C ABI from plain C99 (`examples/bcts_example.c`): it compiles warning-free against include/bcts.h
(CPU), and on a GPU the linked program's search equals the oracle's on the inputs it wrote (Alg. 1
return rule; fp32 INT_HASH + MLP2 path: actions and corrected Q vs the oracle, R18)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "examples", "bcts_example.c")
LIBDIR = os.path.join(ROOT, "paper_2107_01715_b200")
A, IN, HID, N_ROOTS, DEPTH = 4, 64, 256, 8, 3


def test_example_compiles_as_c99(tmp_path):
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"), "-c", SRC,
                    "-o", str(tmp_path / "ex.o")], check=True)


@pytest.mark.gpu
def test_example_search_matches_oracle(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2107_01715_b200 as P
    from oracle import Oracle
    from synth.inputs import ENV_INT_HASH, NET_MLP2_F32
    P.lib()   # built
    exe = tmp_path / "bcts_example"
    subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), SRC, "-L", LIBDIR, "-lbcts",
                    "-Wl,-rpath," + LIBDIR, "-lm", "-o", str(exe)], check=True)
    inputs = tmp_path / "inputs.bin"
    r = subprocess.run([str(exe), str(inputs)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rows = [l.split() for l in r.stdout.splitlines() if l.strip()]
    assert len(rows) == N_ROOTS
    actions = np.array([int(x[0]) for x in rows])
    root_q = np.array([[float(v) for v in x[1:]] for x in rows])
    raw = inputs.read_bytes()
    nw = HID * IN + HID + A * HID + A
    w = np.frombuffer(raw[:4 * nw], dtype=np.float32)
    roots = np.frombuffer(raw[4 * nw:], dtype=np.uint32).reshape(N_ROOTS, 16)
    o = Oracle(ENV_INT_HASH, A, NET_MLP2_F32, weights=w, mlp_in=IN, mlp_hidden=HID)
    g = float(np.float32(0.99))
    m = o.search(roots, DEPTH, g, 1.0, 1, mode=1, threads=os.cpu_count() or 1)
    ref = o.search(roots, DEPTH, g, 1.0, 1, mode=0, threads=os.cpu_count() or 1)
    np.testing.assert_array_equal(actions, m["actions"])
    scale = np.maximum(np.abs(ref["root_q"]).max(axis=1, keepdims=True), 1e-6)
    assert (np.abs(root_q - ref["root_q"]) / scale).max() <= 1e-5
