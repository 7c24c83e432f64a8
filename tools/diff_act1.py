"""act1 of the last trunk batch: fused conv1 (k_conv1_sib) vs materialised leaves + conv_sw<G1>."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2107_01715_b200 as P
from synth.inputs import config
lib = P.lib()
lib.bcts_debug_net_buffer.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64]
lib.bcts_debug_net_buffer.restype = ctypes.c_int64
cfg = config("C5")
n, d = 1, 2                                   # 324 leaves: one trunk batch
IMG = 36864
roots = torch.from_numpy(cfg.roots(n).view(np.uint8).reshape(n, -1).copy()).cuda()
out = {}
for tag, flags in (("fused", 0), ("mat", P.F_MATERIALIZE_LEAVES)):
    h = P.Handle.from_config(cfg, flags=flags)
    h.search(roots, n, d, cfg.gamma, 1.0, 0)
    torch.cuda.synchronize()
    buf = torch.zeros(324 * IMG, dtype=torch.uint8, device="cuda")
    assert lib.bcts_debug_net_buffer(h._h, 0, buf.data_ptr(), buf.numel()) > 0
    cum = torch.zeros(324, dtype=torch.float32, device="cuda")
    lib.bcts_debug_net_buffer(h._h, 3, cum.data_ptr(), 324 * 4)
    out[tag] = (buf.cpu().numpy().reshape(324, IMG), cum.cpu().numpy())
    h.close()
a, b = out["fused"][0], out["mat"][0]
print("leaf R_d equal:", np.array_equal(out["fused"][1], out["mat"][1]))
# valid region: 2 blocks x 100 rows x 128 B at block stride 18432
def valid(x):
    return np.concatenate([x[:, q * 18432: q * 18432 + 12800] for q in range(2)], axis=1)
va, vb = valid(a).view(np.uint16), valid(b).view(np.uint16)
fa = (va.astype(np.uint32) << 16).view(np.float32); fb = (vb.astype(np.uint32) << 16).view(np.float32)
diff = fa != fb
print("images with any diff:", diff.any(1).sum(), "/ 324; elements differing:", diff.sum(), "of", diff.size)
if diff.any():
    i = int(np.argmax(diff.any(1)))
    idx = np.nonzero(diff[i])[0][:12]
    print("first image", i, "element idx", idx, "fused", fa[i, idx], "mat", fb[i, idx])
    # per (block,row,chunk) pattern of diffs, image i
    e = np.nonzero(diff[i])[0]
    blk, rem = e // 6400, e % 6400
    row, col = rem // 64, rem % 64
    print("rows with diffs:", sorted(set(row.tolist()))[:40])
    print("16B chunks (phys) with diffs:", sorted(set((col // 8).tolist())))
    print("rel err max:", np.max(np.abs(fa - fb)[diff] / np.maximum(np.abs(fb[diff]), 1e-6)))
