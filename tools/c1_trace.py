"""Per-child timeline of k_conv1_sib (clock64 stamps per role) in a patched COPY of the package.

  python tools/c1_trace.py build      # here: copy the package to gpurun_exp/trace1/, patch, build
  python tools/c1_trace.py run        # on the GPU box: one C5 search, print per-role waits

Same scheme as tools/c23_trace.py (product source untouched). Stamps for CTA 0..7, children j < KMAX
(events 0-10) or parents q < KMAX (events 11-13), in SM cycles:
  MMA issuer:  0 before n_full wait   1 n_full passed   2 c_empty passed (issue)   3 commits done
  converter 0: 4 before n_empty wait  5 n_empty passed  6 new image written (n_full arrive)
  epilogue 0:  7 c_full passed        8 staging free    9 C loaded (c_empty arrive) 10 bulk store issued
  parent q:    11 load_parent begin   12 load_parent end (shared image + next parent issued)
               13 issue_shared(q) by the MMA issuer
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DST = os.path.join(ROOT, "gpurun_exp", "trace1")
NS = 14
KMAX = 160
NCTA = 8


def patch(src: str) -> str:
    head = (f"\n#define C1T_NS {NS}\n#define C1T_KMAX {KMAX}\n#define C1T_NCTA {NCTA}\n"
            "__device__ unsigned long long g_c1t[C1T_NCTA * C1T_KMAX * C1T_NS];\n"
            "__device__ unsigned long long g_c1g[1024 * 4];\n"
            "__device__ __forceinline__ unsigned long long c1_gt() { unsigned long long t; "
            "asm volatile(\"mov.u64 %0, %globaltimer;\" : \"=l\"(t)); return t; }\n"
            "#define C1T(li, k) do { if (blockIdx.x < C1T_NCTA && (int64_t)(li) < C1T_KMAX) "
            "g_c1t[(blockIdx.x * C1T_KMAX + (li)) * C1T_NS + (k)] = clock64(); } while (0)\n")
    anchor = "constexpr float kSibScale"
    assert src.count(anchor) == 1
    src = src.replace(anchor, head + anchor, 1)
    reps = [
        ("        mbar_wait_spin(&n_full[nb], nph);\n        mbar_wait_spin(&c_empty[cb], cph ^ 1u);\n        tc_fence_after();",
         "        if (elected) C1T(j, 0);\n        mbar_wait_spin(&n_full[nb], nph);\n        if (elected) C1T(j, 1);\n"
         "        mbar_wait_spin(&c_empty[cb], cph ^ 1u);\n        if (elected) C1T(j, 2);\n        tc_fence_after();"),
        ("        commit_pred(&n_empty[nb], elected);\n        commit_pred(&c_full[cb], elected);",
         "        commit_pred(&n_empty[nb], elected);\n        commit_pred(&c_full[cb], elected);\n        if (elected) C1T(j, 3);"),
        ("        mbar_wait(&n_empty[nb], nph ^ 1u);\n        uint8_t *nw = sNw + nb * kNewBytes;",
         "        if (t == 0) C1T(img - i0, 4);\n        mbar_wait(&n_empty[nb], nph ^ 1u);\n        if (t == 0) C1T(img - i0, 5);\n"
         "        uint8_t *nw = sNw + nb * kNewBytes;"),
        ("        asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n        mbar_arrive(&n_full[nb]);",
         "        asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n        mbar_arrive(&n_full[nb]);\n"
         "        if (t == 0) C1T(img - i0, 6);"),
        ("      mbar_wait(&c_full[cb], cph);\n      tc_fence_after();\n      uint8_t *oimg",
         "      mbar_wait(&c_full[cb], cph);\n      if (threadIdx.x == 32) C1T(j, 7);\n      tc_fence_after();\n      uint8_t *oimg"),
        ("      if (threadIdx.x == 32) asm volatile(\"cp.async.bulk.wait_group.read 1;\" ::: \"memory\");\n      epi_bar();",
         "      if (threadIdx.x == 32) asm volatile(\"cp.async.bulk.wait_group.read 1;\" ::: \"memory\");\n      epi_bar();\n"
         "      if (threadIdx.x == 32) C1T(j, 8);"),
        ("        if (hf == 1) {\n          tc_fence_before();\n          mbar_arrive(&c_empty[cb]);\n        }",
         "        if (hf == 1) {\n          tc_fence_before();\n          mbar_arrive(&c_empty[cb]);\n"
         "          if (threadIdx.x == 32) C1T(j, 9);\n        }"),
        ("        asm volatile(\"cp.async.bulk.commit_group;\" ::: \"memory\");\n      }\n      }   // children",
         "        asm volatile(\"cp.async.bulk.commit_group;\" ::: \"memory\");\n        C1T(j, 10);\n      }\n      }   // children"),
        ("    auto load_parent = [&](int64_t q) {\n      const uint32_t sb",
         "    auto load_parent = [&](int64_t q) {\n      if (t == 0) C1T(q, 11);\n      const uint32_t sb"),
        ("      if (t == 0 && q + 1 < npar) {",
         "      if (t == 0) C1T(q, 12);\n      if (t == 0 && q + 1 < npar) {"),
        ("    auto issue_shared = [&](int q) {\n      const uint32_t sb = (uint32_t)q & 1u;",
         "    auto issue_shared = [&](int q) {\n      if (elected) C1T(q, 13);\n      const uint32_t sb = (uint32_t)q & 1u;"),
        ("    mbar_wait(&wbar, 0);\n    const uint64_t wsh",
         "    mbar_wait(&wbar, 0);\n    if (elected) { g_c1g[blockIdx.x * 4] = c1_gt(); g_c1g[blockIdx.x * 4 + 1] = clock64(); }\n"
         "    const uint64_t wsh"),
        ("      a0 = 0;\n    }\n  } else if (warp < 9) {",
         "      a0 = 0;\n    }\n    if (elected) { g_c1g[blockIdx.x * 4 + 2] = c1_gt(); g_c1g[blockIdx.x * 4 + 3] = clock64(); }\n"
         "  } else if (warp < 9) {"),
    ]
    for a, b in reps:
        assert src.count(a) == 1, a[:80]
        src = src.replace(a, b)
    src += ("\nextern \"C\" int c1_trace_read(void *host, size_t bytes) {\n"
            "  return (int)cudaMemcpyFromSymbol(host, bcts::g_c1t, bytes);\n}\n"
            "extern \"C\" int c1_g_read(void *host) {\n"
            "  return (int)cudaMemcpyFromSymbol(host, bcts::g_c1g, sizeof(bcts::g_c1g));\n}\n"
            "extern \"C\" int c1_trace_clear() {\n"
            "  static unsigned long long z[C1T_NCTA * C1T_KMAX * C1T_NS];\n"
            "  return (int)cudaMemcpyToSymbol(bcts::g_c1t, z, sizeof(z));\n}\n")
    return src


def build():
    pkg = os.path.join(DST, "paper_2107_01715_b200")
    if os.path.exists(DST):
        shutil.rmtree(DST)
    shutil.copytree(os.path.join(ROOT, "paper_2107_01715_b200"), pkg,
                    ignore=shutil.ignore_patterns("build", "*.so", "__pycache__"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(DST, "include"))
    f = os.path.join(pkg, "csrc", "qnet_conv.cu")
    txt = patch(open(f).read())
    open(f, "w").write(txt)
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
    for rep in range(3):
        flush.fill_(rep)
        torch.cuda.synchronize()
        assert L.c1_trace_clear() == 0
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        h.search(roots, 1, 4, cfg.gamma, cfg.beta, 1)
        e.record()
        torch.cuda.synchronize()
        print(f"rep {rep}: search {s.elapsed_time(e):.3f} ms")
    assert L.c1_trace_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
    t = buf.reshape(NCTA, KMAX, NS).astype(np.int64)
    g = np.zeros(1024 * 4, np.uint64)
    assert L.c1_g_read(g.ctypes.data_as(ctypes.c_void_p)) == 0
    g = g.reshape(1024, 4).astype(np.int64)[:148]
    ns, cyc = g[:, 2] - g[:, 0], g[:, 3] - g[:, 1]
    print(f"per CTA MMA-issuer span {ns.min() / 1e3:.1f}..{ns.max() / 1e3:.1f} us; SM clock "
          f"{(cyc / ns).min():.3f}..{(cyc / ns).max():.3f} GHz (median {np.median(cyc / ns):.3f})")
    lo, hi = 20, KMAX - 1
    for cta in range(4):
        x = t[cta]
        d = lambda a, b: (x[lo:hi, b] - x[lo:hi, a]).astype(float)
        print(f"CTA {cta}: cycles/child (issue to issue) {np.diff(x[lo:hi, 2]).mean():.0f}")
        print("   MMA waits n_full   %6.0f   waits c_empty %6.0f   issue->commit %6.0f" % (d(0, 1).mean(), d(1, 2).mean(), d(2, 3).mean()))
        print("   conv waits n_empty %6.0f   writes new image %6.0f" % (d(4, 5).mean(), d(5, 6).mean()))
        print("   conv n_full(j) -> MMA issue(j) %6.0f" % d(6, 2).mean())
        print("   MMA issue(j) -> epi c_full(j) %6.0f" % d(2, 7).mean())
        print("   epi c_full -> stage free %6.0f   -> C loaded %6.0f   -> store issued %6.0f" % (d(7, 8).mean(), d(8, 9).mean(), d(9, 10).mean()))
        print("   epi store(j) -> c_full(j+1) wait start..end: %6.0f" % (x[lo + 1:hi + 1, 7] - x[lo:hi, 10]).mean())
        print("   conv loop: n_full arrive(j) -> n_empty wait start(j+1) %6.0f" % (x[lo + 1:hi + 1, 4] - x[lo:hi, 6]).mean())
        pq = x[:, 11:14]
        ok = (pq[:, 0] > 0) & (pq[:, 1] > 0)
        print("   load_parent duration (per parent) %6.0f (n=%d)" % ((pq[ok, 1] - pq[ok, 0]).mean() if ok.any() else -1, ok.sum()))
    np.save(os.path.join(ROOT, "gpurun_out", "c1_trace.npy"), t)


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
