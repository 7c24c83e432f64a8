"""Bit-exactness of two package copies on one search: python tools/ab_bitexact.py PKG_A PKG_B [CONFIG] [N_ROOTS] [DEPTH]
(each copy runs in its own process; the outputs are compared byte for byte)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(pkg, cname, n, d, out):
    sys.path.insert(0, os.path.abspath(pkg))
    sys.path.insert(1, ROOT)
    import numpy as np
    import torch
    import paper_2107_01715_b200 as P
    from synth.inputs import config
    cfg = config(cname)
    h = P.Handle.from_config(cfg)
    roots = torch.from_numpy(cfg.roots(n).view(np.uint8).copy()).cuda()
    r = h.search(roots, n, d, cfg.gamma, cfg.beta, 1, extra=True)
    torch.cuda.synchronize()
    np.savez(out, **{k: v.cpu().numpy() for k, v in r.items() if hasattr(v, "cpu")})


if __name__ == "__main__":
    if sys.argv[1] == "--one":
        one(sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5]), sys.argv[6])
        sys.exit(0)
    import numpy as np
    a, b = sys.argv[1], sys.argv[2]
    cname = sys.argv[3] if len(sys.argv) > 3 else "C5"
    n = sys.argv[4] if len(sys.argv) > 4 else "1"
    d = sys.argv[5] if len(sys.argv) > 5 else "4"
    outs = []
    for i, pkg in enumerate((a, b)):
        f = f"/tmp/ab_bitexact_{i}.npz"
        subprocess.run([sys.executable, __file__, "--one", pkg, cname, n, d, f], check=True)
        outs.append(np.load(f))
    same = all(np.array_equal(outs[0][k], outs[1][k]) for k in outs[0].files)
    print(f"{cname} n={n} d={d}: {'BIT-IDENTICAL' if same else 'DIFFERENT'} ({', '.join(outs[0].files)})")
    for k in outs[0].files:
        if not np.array_equal(outs[0][k], outs[1][k]):
            print("  differs:", k, np.abs(outs[0][k].astype(np.float64) - outs[1][k].astype(np.float64)).max())
