"""Per-image timeline of k_conv23 (clock64 stamps per role) in a patched COPY of the package.

  python tools/c23_trace.py build      # here: copy the package to gpurun_exp/trace/, patch, build
  python tools/c23_trace.py run        # on the GPU box: one C5 search, print per-role waits

The product source is untouched: the stamps exist only in the copy (gpurun_exp/ is git-ignored but
travels with gpurun). Stamps (CTA 0..7, images 0..kMax-1), all in SM cycles of the CTA's SM:
  0 producer in_empty wait start   1 producer load issued
  2 conv2 issuer in_full wait start 3 in_full passed        4 t2empty passed (issue start)
  5 epi2 t2full passed             6 epi2 T2 loaded (t2empty arrive) 7 epi2 a2empty passed 8 epi2 a2full arrive
  9 conv3 issuer a2full passed     10 t3empty passed (issue start)
  11 epi3 t3full passed            12 epi3 staging free (after wait_group.read)  13 epi3 bulk store issued
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DST = os.path.join(ROOT, "gpurun_exp", "trace")
NS = 14
KMAX = 160
NCTA = 8


def patch(src: str) -> str:
    head = (f"\n#define C23T_NS {NS}\n#define C23T_KMAX {KMAX}\n#define C23T_NCTA {NCTA}\n"
            "__device__ unsigned long long g_c23t[C23T_NCTA * C23T_KMAX * C23T_NS];\n"
            "#define C23T(li, k) do { if (blockIdx.x < C23T_NCTA && (li) < C23T_KMAX) "
            "g_c23t[(blockIdx.x * C23T_KMAX + (li)) * C23T_NS + (k)] = clock64(); } while (0)\n"
            "__device__ unsigned long long g_c23g[1024 * 4];\n"
            "__device__ __forceinline__ unsigned long long c23_gt() { unsigned long long t; "
            "asm volatile(\"mov.u64 %0, %globaltimer;\" : \"=l\"(t)); return t; }\n")
    anchor = "constexpr int kC3tOutBytes"
    assert anchor in src
    src = src.replace(anchor, head + anchor, 1)
    reps = [
        ("        mbar_wait_spin(&in_empty[b], ph ^ 1u);\n        mbar_expect_tx(&in_full[b], 2u * 12800u);",
         "        C23T(li, 0);\n        mbar_wait_spin(&in_empty[b], ph ^ 1u);\n        mbar_expect_tx(&in_full[b], 2u * 12800u);"),
        ("                   12800u, &in_full[b]);\n      }",
         "                   12800u, &in_full[b]);\n        C23T(li, 1);\n      }"),
        ("    mbar_wait_spin(&w2ready, 0);   // W2 in TMEM (tcgen05.st by the conv2-epilogue warps)",
         "    mbar_wait_spin(&w2ready, 0);\n    if (elected) { g_c23g[blockIdx.x * 4] = c23_gt(); g_c23g[blockIdx.x * 4 + 1] = clock64(); }"),
        ("      commit_pred(&t2full, elected);\n      __syncwarp();\n    }",
         "      commit_pred(&t2full, elected);\n      __syncwarp();\n    }\n"
         "    if (elected) { g_c23g[blockIdx.x * 4 + 2] = c23_gt(); g_c23g[blockIdx.x * 4 + 3] = clock64(); }"),
        ("      mbar_wait_spin(&in_full[bi], phi);\n      mbar_wait_spin(&t2empty, (li & 1u) ^ 1u);",
         "      if (elected) C23T(li, 2);\n      mbar_wait_spin(&in_full[bi], phi);\n      if (elected) C23T(li, 3);\n"
         "      mbar_wait_spin(&t2empty, (li & 1u) ^ 1u);\n      if (elected) C23T(li, 4);"),
        ("      mbar_wait_spin(&t2full, li & 1u);\n      tc_fence_after();\n      uint32_t v[48];",
         "      mbar_wait_spin(&t2full, li & 1u);\n      if (threadIdx.x == 64) C23T(li, 5);\n      tc_fence_after();\n      uint32_t v[48];"),
        ("      tc_fence_before();\n      mbar_arrive(&t2empty);",
         "      tc_fence_before();\n      mbar_arrive(&t2empty);\n      if (threadIdx.x == 64) C23T(li, 6);"),
        ("      mbar_wait_spin(&a2empty[b], ph ^ 1u);              // conv3 of image li-2 is done with sA2[b]",
         "      mbar_wait_spin(&a2empty[b], ph ^ 1u);\n      if (threadIdx.x == 64) C23T(li, 7);"),
        ("      asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n      mbar_arrive(&a2full[b]);",
         "      asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n      mbar_arrive(&a2full[b]);\n"
         "      if (threadIdx.x == 64) C23T(li, 8);"),
        ("      mbar_wait_spin(&a2full[b], ph);\n      mbar_wait_spin(&t3empty, (jj & 1u) ^ 1u);",
         "      mbar_wait_spin(&a2full[b], ph);\n      if (elected) C23T(jj, 9);\n      mbar_wait_spin(&t3empty, (jj & 1u) ^ 1u);\n"
         "      if (elected) C23T(jj, 10);"),
        ("      mbar_wait_spin(&t3full, li & 1u);\n      tc_fence_after();\n      uint32_t v[64];",
         "      mbar_wait_spin(&t3full, li & 1u);\n      if (lead) C23T(li, 11);\n      tc_fence_after();\n      uint32_t v[64];"),
        ("      if (lead) asm volatile(\"cp.async.bulk.wait_group.read 1;\" ::: \"memory\");",
         "      if (lead) asm volatile(\"cp.async.bulk.wait_group.read 1;\" ::: \"memory\");\n      if (lead) C23T(li, 12);"),
        ("        asm volatile(\"cp.async.bulk.commit_group;\" ::: \"memory\");\n      }\n    }\n    if (lead) asm volatile(\"cp.async.bulk.wait_group 0;\"",
         "        asm volatile(\"cp.async.bulk.commit_group;\" ::: \"memory\");\n        C23T(li, 13);\n      }\n    }\n"
         "    if (lead) asm volatile(\"cp.async.bulk.wait_group 0;\""),
    ]
    for a, b in reps:
        assert src.count(a) == 1, a[:80]
        src = src.replace(a, b)
    src += ("\nextern \"C\" int c23_trace_read(void *host, size_t bytes) {\n"
            "  return (int)cudaMemcpyFromSymbol(host, bcts::g_c23t, bytes);\n}\n"
            "extern \"C\" int c23_g_read(void *host) {\n"
            "  return (int)cudaMemcpyFromSymbol(host, bcts::g_c23g, sizeof(bcts::g_c23g));\n}\n"
            "extern \"C\" int c23_trace_clear() {\n"
            "  static unsigned long long z[C23T_NCTA * C23T_KMAX * C23T_NS];\n"
            "  return (int)cudaMemcpyToSymbol(bcts::g_c23t, z, sizeof(z));\n}\n")
    return src


def build():
    pkg = os.path.join(DST, "paper_2107_01715_b200")
    if os.path.exists(DST):
        shutil.rmtree(DST)
    shutil.copytree(os.path.join(ROOT, "paper_2107_01715_b200"), pkg,
                    ignore=shutil.ignore_patterns("build", "*.so", "__pycache__"))
    f = os.path.join(pkg, "csrc", "qnet_conv.cu")
    txt = patch(open(f).read())
    open(f, "w").write(txt)
    # the copy's build.py resolves include/ relative to its parent: give it the header
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(DST, "include"))
    subprocess.run([sys.executable, "-c", "import sys; sys.path.insert(0, %r); "
                    "from paper_2107_01715_b200 import build; build.build(force=True)" % DST], check=True)
    print("built", os.path.join(pkg, "libbcts.so"))


def run():
    sys.path.insert(0, DST)
    sys.path.insert(1, ROOT)
    import ctypes
    import numpy as np
    import torch
    import paper_2107_01715_b200 as P
    assert P.__file__.startswith(DST), P.__file__
    from synth.inputs import config
    cfg = config("C5")
    h = P.Handle.from_config(cfg)
    roots = torch.from_numpy(cfg.roots(1).view(np.uint8).copy()).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    L = P.lib()
    buf = np.zeros(NCTA * KMAX * NS, np.uint64)
    for _ in range(4):
        h.search(roots, 1, 4, cfg.gamma, cfg.beta, 1)
    torch.cuda.synchronize()
    res = []
    for rep in range(3):
        flush.fill_(rep)
        torch.cuda.synchronize()
        assert L.c23_trace_clear() == 0
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        h.search(roots, 1, 4, cfg.gamma, cfg.beta, 1)
        e.record()
        torch.cuda.synchronize()
        assert L.c23_trace_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
        res.append(buf.copy().reshape(NCTA, KMAX, NS).astype(np.int64))
        print(f"rep {rep}: search {s.elapsed_time(e):.3f} ms")
    t = res[-1]
    names = ["prod wait start", "prod issued", "c2 wait in_full", "c2 in_full ok", "c2 issue", "e2 t2full",
             "e2 T2 loaded", "e2 a2empty ok", "e2 a2full", "c3 a2full ok", "c3 issue", "e3 t3full", "e3 stage free",
             "e3 stored"]
    lo, hi = 20, KMAX - 1
    for cta in range(NCTA):
        x = t[cta]
        per = np.diff(x[lo:hi, 4]).mean()
        d = lambda a, b, off=0: (x[lo:hi, b] - x[lo - off:hi - off, a]).astype(float)
        print(f"CTA {cta}: cycles/image (conv2 issue to issue) {per:.0f}")
        print("   producer in_empty wait   %6.0f" % d(0, 1).mean())
        print("   load issue -> c2 in_full ok (latency upper bound) %6.0f" % d(1, 3).mean())
        print("   c2 waits in_full          %6.0f  (frac waiting %.2f)" % (d(2, 3).mean(), (d(2, 3) > 50).mean()))
        print("   c2 waits t2empty          %6.0f" % d(3, 4).mean())
        print("   c2 issue -> e2 t2full     %6.0f" % d(4, 5).mean())
        print("   e2 t2full -> T2 loaded    %6.0f" % d(5, 6).mean())
        print("   e2 T2 loaded -> a2empty ok %6.0f" % d(6, 7).mean())
        print("   e2 a2empty -> a2full      %6.0f" % d(7, 8).mean())
        print("   e2 a2full -> c3 a2full ok %6.0f" % d(8, 9).mean())
        print("   c3 waits t3empty          %6.0f" % d(9, 10).mean())
        print("   c3 issue -> e3 t3full     %6.0f" % d(10, 11).mean())
        print("   e3 t3full -> stage free   %6.0f" % d(11, 12).mean())
        print("   e3 stage free -> stored   %6.0f" % d(12, 13).mean())
        print("   c2 issue(i) -> c3 issue(i) %6.0f" % d(4, 10).mean())
        print("   c3 issue(i) -> c2 issue(i+1) %6.0f" % (x[lo + 1:hi + 1, 4] - x[lo:hi, 10]).mean())
    np.save(os.path.join(ROOT, "gpurun_out", "c23_trace.npy"), np.stack(res))
    g = np.zeros(1024 * 4, np.uint64)
    assert L.c23_g_read(g.ctypes.data_as(ctypes.c_void_p)) == 0
    g = g.reshape(1024, 4).astype(np.int64)[:148]
    ns = g[:, 2] - g[:, 0]
    cyc = g[:, 3] - g[:, 1]
    print(f"per CTA conv2-issuer span: {ns.min() / 1e3:.1f}..{ns.max() / 1e3:.1f} us; SM clock over it "
          f"{(cyc / ns).min():.3f}..{(cyc / ns).max():.3f} GHz (median {np.median(cyc / ns):.3f}); "
          f"start spread {(g[:, 0].max() - g[:, 0].min()) / 1e3:.1f} us, end spread {(g[:, 2].max() - g[:, 2].min()) / 1e3:.1f} us")
    np.save(os.path.join(ROOT, "gpurun_out", "c23_g.npy"), g)


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
