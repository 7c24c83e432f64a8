"""Which computation does the fused conv1 (k_conv1_sib) output match? act1 vs torch conv1 variants."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2107_01715_b200 as P
from synth.inputs import config
lib = P.lib()
lib.bcts_debug_net_buffer.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64]
cfg = config("C5")
n, d = 1, 2
IMG = 36864
roots = torch.from_numpy(cfg.roots(n).view(np.uint8).reshape(n, -1).copy()).cuda()
h = P.Handle.from_config(cfg)
h.search(roots, n, d, cfg.gamma, 1.0, 0)
torch.cuda.synchronize()
buf = torch.zeros(324 * IMG, dtype=torch.uint8, device="cuda")
lib.bcts_debug_net_buffer(h._h, 0, buf.data_ptr(), buf.numel())
act = buf.cpu().numpy().reshape(324, IMG)
# decode act1 (s2d(2) SW128, 2 blocks x 100 rows x 8 chunks) -> [324][20][20][32]
def decode(a):
    out = np.zeros((a.shape[0], 20, 20, 32), np.float32)
    for oy in range(20):
        for ox in range(20):
            row = (oy >> 1) * 10 + (ox >> 1); sub = ((oy & 1) << 1) | (ox & 1)
            for cq in range(4):
                chunk = sub * 4 + cq
                off = (chunk >> 3) * 18432 + row * 128 + (((chunk & 7) ^ (row & 7)) << 4)
                v = a[:, off:off + 16].copy().view(np.uint16).astype(np.uint32) << 16
                out[:, oy, ox, cq * 8:cq * 8 + 8] = v.view(np.float32)
    return out
f = decode(act)
# leaf frames via expand (level 2 records: key, pad, w[7056] packed 4 frames)
st, cum = h.expand(roots, n, 2, np.float32(cfg.gamma))
rec = st.cpu().numpy().reshape(324, -1)
w = rec[:, 16:].copy().view(np.uint32).reshape(324, 84, 84)
frames = np.stack([(w >> (8 * c)) & 0xFF for c in range(4)], 1).astype(np.float32)   # [324][4][84][84]
from synth.inputs import make_weights
_, views = make_weights(cfg.net, cfg.A, cfg.wseed)
W1 = torch.from_numpy(views["conv1.w"].astype(np.float32)).cuda()
W1 = W1.to(torch.bfloat16).to(torch.float32)
b1 = torch.from_numpy(views["conv1.b"].astype(np.float32)).cuda()
def conv(fr):
    x = torch.from_numpy(fr).cuda()
    y = torch.nn.functional.conv2d(x, W1, b1, stride=4)
    return torch.relu(y).to(torch.bfloat16).to(torch.float32).permute(0, 2, 3, 1).cpu().numpy()
hyps = {"correct [f0 f1 f2 f3]": frames,
        "no-noise new frame": None}
ref = conv(frames)
print("fused vs correct: mean|diff|", np.abs(f - ref).mean(), "max", np.abs(f - ref).max(), "mean|ref|", np.abs(ref).mean())
# parent frames (level 1) to test the shared part hypothesis
st1, _ = h.expand(roots, n, 1, np.float32(cfg.gamma))
r1 = st1.cpu().numpy().reshape(18, -1)
w1 = r1[:, 16:].copy().view(np.uint32).reshape(18, 84, 84)
pf = np.stack([(w1 >> (8 * c)) & 0xFF for c in range(4)], 1).astype(np.float32)
par = np.repeat(pf, 18, axis=0)
for name, fr in [("shared=parent f0..2", np.concatenate([par[:, 0:3], frames[:, 3:4]], 1)),
                 ("shared=parent f1..3 (correct)", np.concatenate([par[:, 1:4], frames[:, 3:4]], 1)),
                 ("new = parent newest (no xor)", np.concatenate([frames[:, 0:3], par[:, 3:4]], 1)),
                 ("new frame zero", np.concatenate([frames[:, 0:3], 0 * frames[:, 3:4]], 1)),
                 ("shared zero", np.concatenate([0 * frames[:, 0:3], frames[:, 3:4]], 1))]:
    r = conv(fr)
    print(f"{name:32s} mean|fused - hyp| = {np.abs(f - r).mean():.5f}")
# channel / position structure of the error
e = np.abs(f - ref).mean(axis=(0, 1, 2))
print("per-channel mean err:", np.round(e, 4))
e2 = np.abs(f - ref).mean(axis=(0, 3))
print("per-row mean err:", np.round(e2.mean(1), 4))
print("per-col mean err:", np.round(e2.mean(0), 4))
