"""Phase timeline of the shifted-window conv kernel (CTA 0), one layer launch."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2107_01715_b200 as P
from synth.inputs import atari_roots, config
h = P.Handle.from_config(config("C5"))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
recs = torch.from_numpy(atari_roots(n, 1).copy()).cuda()
h.q_rows(recs, n); torch.cuda.synchronize()
buf = torch.zeros(64 * 4, dtype=torch.int64, device="cuda")
layer = int(sys.argv[2]) if len(sys.argv) > 2 else 0
lib = P.lib(); lib.bcts_debug_conv_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
lib.bcts_debug_conv_trace(buf.data_ptr(), layer)
if layer in (9, 10):   # fused conv1: run a real search (d=2 -> 324 leaves per root)
    roots = torch.from_numpy(config("C5").roots(1).copy()).cuda()
    h.search(roots, 1, 4, 0.99, 1.0, 1); torch.cuda.synchronize()
else:
    h.q_rows(recs, n); torch.cuda.synchronize()
lib.bcts_debug_conv_trace(None, -1)
t = buf.cpu().numpy().reshape(64, 4).astype(np.float64)
t0 = t[0, 0]
if layer == 10:
    print("k_conv1_sib trace in SM cycles: child start (converter), conversion start, conversion end, MMAs issued")
    for i in range(64):
        if t[i, 0] == 0: break
        prev = t[i - 1, 0] if i else t0
        print(f"{i:3d} period {t[i,0]-prev:7.0f}  k2+noise+bars {t[i,1]-t[i,0]:6.0f}  convert {t[i,2]-t[i,1]:6.0f}  "
              f"->mma {t[i,3]-t[i,2]:7.0f}")
    sys.exit(0)
print("img  t0 t1 t2 t3 [copy_issued/conv_start, input_ready/conv_done, mma_issued, epi_done]   (us from first copy; layer out_mode %d, last sub-batch)" % layer + "")
for i in range(64):
    if t[i, 0] == 0: break
    print(f"{i:3d} " + " ".join(f"{(x - t0) / 1e3:11.2f}" for x in t[i]))
