"""Debug: GPU act3 (dense [49][64] bf16 per image, after conv1 -> conv2+conv3) vs torch float64 convs with
bf16 rounding of weights and activations (the R17 reading) on a few Atari-shaped states."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2107_01715_b200 as P  # noqa: E402
from synth.inputs import atari_roots, config  # noqa: E402

F = torch.nn.functional
cfg = config(sys.argv[1] if len(sys.argv) > 1 else "C5")
h = P.Handle.from_config(cfg)
_, w = cfg.weights()
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
recs = atari_roots(n, 99)
dev = torch.device("cuda", 0)
q = h.q_rows(torch.from_numpy(recs.view(np.uint8).copy()).to(dev), n)
torch.cuda.synchronize()
buf = torch.empty(n * 3136 * 2, dtype=torch.uint8, device=dev)
got = P.lib().bcts_debug_net_buffer(h._h, 2, ctypes.c_void_p(buf.data_ptr()), n * 3136 * 2)
torch.cuda.synchronize()
a3 = buf.cpu().view(torch.bfloat16).to(torch.float64).reshape(n, 7, 7, 64).permute(0, 3, 1, 2)


def bf(t):
    return t.to(torch.float32).to(torch.bfloat16).to(torch.float64)


def W(k):
    return torch.from_numpy(w[k].astype(np.float64))


for i in sorted(set([0, 1, n // 2, n - 1, 148, 149, 300, n - 149, n - 148, n - 2, 148 * 40 + 7, 148 * 41 + 7])):
    if i >= n: continue
    words = recs[i, 16:].view(np.uint32).reshape(84, 84)
    x = torch.from_numpy(np.stack([(words >> (8 * c)) & 0xFF for c in range(4)]).astype(np.float64)[None])
    h1 = bf(F.relu(F.conv2d(x, bf(W("conv1.w")), W("conv1.b"), stride=4)))
    h2 = bf(F.relu(F.conv2d(h1, bf(W("conv2.w")), W("conv2.b"), stride=2)))
    h3 = bf(F.relu(F.conv2d(h2, bf(W("conv3.w")), W("conv3.b"), stride=1)))[0]
    d = (a3[i] - h3).abs()
    print(f"img {i}: max|act3 - ref| {d.max():.4g} (ref max {h3.abs().max():.4g}); "
          f"frac > 2^-7 rel: {(d > h3.abs() * 2 ** -7 + 1e-3).double().mean():.4f}")
    if i == 0:
        bad = (d > h3.abs() * 2 ** -7 + 1e-3).nonzero()[:10].tolist()
        print("first bad (c, y, x):", bad)
        per_c = (d > h3.abs() * 2 ** -7 + 1e-3).double().mean(dim=(1, 2))
        print("bad fraction per channel:", np.round(per_c.numpy(), 2).tolist())
        per_p = (d > h3.abs() * 2 ** -7 + 1e-3).double().mean(dim=0)
        print("bad fraction per pixel:\n", np.round(per_p.numpy(), 2))
