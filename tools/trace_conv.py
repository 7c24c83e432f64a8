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
if layer == 11:
    buf = torch.zeros(64 * 8, dtype=torch.int64, device="cuda")
    lib.bcts_debug_conv_trace(buf.data_ptr(), layer_arg)
if layer in (9, 10, 11):   # fused conv1 / conv2+conv3: run a real search
    roots = torch.from_numpy(config("C5").roots(1).copy()).cuda()
    h.search(roots, 1, 4, 0.99, 1.0, 1); torch.cuda.synchronize()
else:
    h.q_rows(recs, n); torch.cuda.synchronize()
lib.bcts_debug_conv_trace(None, -1)
if dbg:
    lib.bcts_debug_conv_trace(None, 100 * 0 - 1)
t = buf.cpu().numpy().reshape(64, -1).astype(np.float64)
t0 = t[0, 0]
if layer == 11:
    print("k_conv23 trace (cycles rel. to image 0): conv2 wait begin, act1 landed, T2 free, conv2 issued, "
          "conv3 wait begin, act2 ready, conv3 issued, conv2 done (epi)")
    for i in range(64):
        if t[i, 0] == 0: break
        print(f"{i:3d} " + " ".join(f"{x - t0:8.0f}" for x in t[i]))
    n = int((t[:, 0] != 0).sum())
    md = lambda a, b, lo=2: np.median(t[lo:n, b] - t[lo:n, a])
    print(f"median period (conv2 issued) {np.median(np.diff(t[2:n, 3])):.0f}; conv2 wait->act1 {md(0, 1):.0f}, "
          f"act1->T2 free {md(1, 2):.0f}, T2 free->conv2 issued {md(2, 3):.0f}, conv3 wait->act2 ready {md(4, 5):.0f}, "
          f"act2->conv3 issued {md(5, 6):.0f}")
    sys.exit(0)
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
