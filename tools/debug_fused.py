"""Debug: act3 of the fused leaf path (k_conv1_sib -> k_conv23) vs torch float64 convs (R17 rounding)
on the leaves of a small search (corr = 0, so the last net batch is the leaf level)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2107_01715_b200 as P  # noqa: E402
from synth.inputs import config  # noqa: E402

F = torch.nn.functional
cfg = config(sys.argv[1] if len(sys.argv) > 1 else "C3")
d = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n = 1
h = P.Handle.from_config(cfg)
_, w = cfg.weights()
dev = torch.device("cuda", 0)
roots = cfg.roots(n)
rd = torch.from_numpy(roots.view(np.uint8).copy()).to(dev)
h.search(rd, n, d, cfg.gamma, 1.0, 0, extra=True)
torch.cuda.synchronize()
nl = n * cfg.A ** d
buf = torch.empty(nl * 3136 * 2, dtype=torch.uint8, device=dev)
P.lib().bcts_debug_net_buffer(h._h, 2, ctypes.c_void_p(buf.data_ptr()), nl * 3136 * 2)
torch.cuda.synchronize()
a3 = buf.cpu().view(torch.bfloat16).to(torch.float64).reshape(nl, 7, 7, 64).permute(0, 3, 1, 2)
st, cum = h.expand(rd, n, d, np.float32(cfg.gamma))
st = st.cpu().numpy()


def bf(t):
    return t.to(torch.float32).to(torch.bfloat16).to(torch.float64)


def W(k):
    return torch.from_numpy(w[k].astype(np.float64))


words = torch.from_numpy(st[:, 16:].copy().view(np.uint32).reshape(nl, 84, 84).astype(np.int64))
x = torch.stack([(words >> (8 * c)) & 0xFF for c in range(4)], dim=1).double()
h1 = bf(F.relu(F.conv2d(x, bf(W("conv1.w")), W("conv1.b"), stride=4)))
h2 = bf(F.relu(F.conv2d(h1, bf(W("conv2.w")), W("conv2.b"), stride=2)))
ref = bf(F.relu(F.conv2d(h2, bf(W("conv3.w")), W("conv3.b"), stride=1)))
for rep in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
    h.search(rd, n, d, cfg.gamma, 1.0, 0, extra=True)
    torch.cuda.synchronize()
    P.lib().bcts_debug_net_buffer(h._h, 2, ctypes.c_void_p(buf.data_ptr()), nl * 3136 * 2)
    torch.cuda.synchronize()
    a3 = buf.cpu().view(torch.bfloat16).to(torch.float64).reshape(nl, 7, 7, 64).permute(0, 3, 1, 2)
    dd = (a3 - ref).abs()
    bad = dd > ref.abs() * 2 ** -6 + 2e-3
    badimg = bad.flatten(1).any(1)
    print(f"rep {rep}: {int(badimg.sum())} of {nl} leaves outside bf16 rounding; max diff {dd.max():.4g}")
    if badimg.any():
        i = int(badimg.nonzero()[0])
        print(f" first bad leaf {i} (CTA {i % 148}, li {i // 148}); per pixel:\n", bad[i].double().mean(dim=0).numpy().round(2))
        print(" per channel:", bad[i].double().mean(dim=(1, 2)).numpy().round(2).tolist())
        print(" bad leaves:", badimg.nonzero().flatten()[:20].tolist())
