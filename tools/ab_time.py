"""Same-box A/B timing of a package copy: python tools/ab_time.py PKG_ROOT [CONFIG] [STEPS] [ROUNDS] [tf32]

PKG_ROOT holds a paper_2107_01715_b200/ (e.g. gpurun_exp/base built from HEAD, or . for the working tree).
Prints the device-timed step (L2 flushed before each step, CUDA events) and the per-class kernel times
of a profiled repeat, like bench.py, for ROUNDS alternating rounds when several roots are given
separated by commas (A,B,A,B...)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(pkg_root, cname, steps, tf32=False):
    sys.path.insert(0, os.path.abspath(pkg_root))
    sys.path.insert(1, ROOT)
    import numpy as np
    import torch
    import paper_2107_01715_b200 as P
    assert P.__file__.startswith(os.path.abspath(pkg_root)), P.__file__
    from synth.inputs import config
    cfg = config(cname)
    h = P.Handle.from_config(cfg, flags=P.F_TF32 if tf32 else 0)
    roots = torch.from_numpy(cfg.roots().view(np.uint8).copy()).cuda()
    n = roots.shape[0]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        h.search(roots, n, cfg.depth, cfg.gamma, cfg.beta, 1)
    torch.cuda.synchronize()
    ts = []
    for i in range(steps):
        flush.fill_(i & 0xFF)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        h.search(roots, n, cfg.depth, cfg.gamma, cfg.beta, 1)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    h.profile(True)
    for i in range(steps):
        flush.fill_(i & 0xFF)
        h.search(roots, n, cfg.depth, cfg.gamma, cfg.beta, 1)
    torch.cuda.synchronize()
    prof = h.profile_read()
    h.profile(False)
    cls = " ".join(f"{k} {v['ms'] / steps:.4f}" for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]))
    print(f"{pkg_root}: {cname}{' tf32' if tf32 else ''} step mean {np.mean(ts):.4f} ms median {np.median(ts):.4f} | {cls}", flush=True)


if __name__ == "__main__":
    import subprocess
    roots = sys.argv[1].split(",")
    cname = sys.argv[2] if len(sys.argv) > 2 else "C5"
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    tf32 = len(sys.argv) > 5 and sys.argv[5] == "tf32"
    if len(roots) == 1 and rounds == 1:
        run(roots[0], cname, steps, tf32)
    else:   # one fresh process per measurement (each imports its own package copy)
        for _ in range(rounds):
            for r in roots:
                subprocess.run([sys.executable, os.path.abspath(__file__), r, cname, str(steps), "1"] + (["tf32"] if tf32 else []),
                               check=True)
