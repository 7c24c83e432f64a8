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
layer = int(sys.argv[2]) if len(sys.argv) > 2 else 0   # 10 + 100*dbg: k_conv1_sib with debug switches
dbg, layer_arg, layer = layer // 100, layer, layer % 100
buf = torch.zeros(64 * (10 if layer == 10 else 4), dtype=torch.int64, device="cuda")
lib = P.lib(); lib.bcts_debug_conv_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
lib.bcts_debug_conv_trace(buf.data_ptr(), layer_arg)
if layer in (9, 10):   # fused conv1: run a real search (d=2 -> 324 leaves per root)
    roots = torch.from_numpy(config("C5").roots(1).copy()).cuda()
    h.search(roots, 1, 4, 0.99, 1.0, 1); torch.cuda.synchronize()
else:
    h.q_rows(recs, n); torch.cuda.synchronize()
lib.bcts_debug_conv_trace(None, -1)
if dbg:
    lib.bcts_debug_conv_trace(None, 100 * 0 - 1)
t = buf.cpu().numpy().reshape(64, -1).astype(np.float64)
t0 = t[0, 0]
if layer == 10:
    print("k_conv1_sib trace, SM cycles relative to child 0's start: conv start, conv begin (n_empty ok), conv end, "
          "mma: loop top, new ready, C free, issued; epi: C ready, C released, stored")
    for i in range(64):
        if t[i, 0] == 0: break
        print(f"{i:3d} " + " ".join(f"{x - t0:8.0f}" for x in t[i, :10]))
    n = int((t[:, 0] != 0).sum())
    d7 = np.diff(t[2:n, 7])
    md = lambda a, b: np.median(t[2:n, b] - t[2:n, a])
    print(f"dbg={dbg}: median C-ready spacing {np.median(d7):.0f} cycles, mean {d7.mean():.0f}; medians: "
          f"issue->C ready {md(6, 7):.0f}, loop top->new ready {md(3, 4):.0f}, new ready->C free {md(4, 5):.0f}, "
          f"C free->issued {md(5, 6):.0f}, issued->next loop top {np.median(t[3:n, 3] - t[2:n - 1, 6]):.0f}, "
          f"conv begin->end {md(1, 2):.0f}, conv end->MMA new ready {md(2, 4):.0f}")
    sys.exit(0)
print("img  t0 t1 t2 t3 [copy_issued/conv_start, input_ready/conv_done, mma_issued, epi_done]   (us from first copy; layer out_mode %d, last sub-batch)" % layer + "")
for i in range(64):
    if t[i, 0] == 0: break
    print(f"{i:3d} " + " ".join(f"{(x - t0) / 1e3:11.2f}" for x in t[i]))
