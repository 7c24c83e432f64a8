"""Per-job timeline of k_zhead (clock64 stamps) in a patched COPY of the package (product source untouched).

  python tools/head_trace.py build      # here: copy to gpurun_exp/traceh/, patch, build
  python tools/head_trace.py run        # on the GPU box: one C5 search, print where each tile's time goes

Stamps for CTA 0..7, tiles tl < 12, jobs j < 8 (0 = v, 1 = mean, 2.. = z_a chunks), in SM cycles:
  0 MMA issuer before tempty wait   1 after tempty wait   2 after a_full wait (j = 1)   3 job issued (commit)
  4 sum over the job's k-blocks of the ring (full) waits
  5 epilogue (thread 64) after tfull wait   6 epilogue job done (tempty arrive)
Per tile: 7 producer before a_empty wait (slot j = 0), 8 after it (h_a load issued) (slot j = 1)
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DST = os.path.join(ROOT, "gpurun_exp", "traceh")
NT, NJ, NS, NCTA = 12, 8, 10, 8


def patch(src):
    head = (f"\n#define HT_NT {NT}\n#define HT_NJ {NJ}\n#define HT_NS {NS}\n#define HT_NCTA {NCTA}\n"
            "__device__ long long g_ht[HT_NCTA * HT_NT * HT_NJ * HT_NS];\n"
            "__device__ unsigned long long g_hg[1024 * 4];\n"
            "__device__ __forceinline__ unsigned long long ht_gt() { unsigned long long t; "
            "asm volatile(\"mov.u64 %0, %globaltimer;\" : \"=l\"(t)); return t; }\n"
            "#define HT(tl, j, k) do { if (blockIdx.x < HT_NCTA && (tl) < HT_NT && (j) < HT_NJ) "
            "g_ht[((blockIdx.x * HT_NT + (tl)) * HT_NJ + (j)) * HT_NS + (k)] = clock64(); } while (0)\n"
            "#define HTADD(tl, j, k, v) do { if (blockIdx.x < HT_NCTA && (tl) < HT_NT && (j) < HT_NJ) "
            "g_ht[((blockIdx.x * HT_NT + (tl)) * HT_NJ + (j)) * HT_NS + (k)] += (v); } while (0)\n")
    anchor = "constexpr int kHeadStages = 3"
    assert src.count(anchor) == 1
    src = src.replace(anchor, head + anchor, 1)
    reps = [
        ("        mbar_wait_spin(&a_empty, (tl & 1u) ^ 1u);      // previous tile's MMAs are done with sA",
         "        HT(tl, 0, 7);\n        mbar_wait_spin(&a_empty, (tl & 1u) ^ 1u);\n        HT(tl, 1, 8);"),
        ("        mbar_wait_spin(&tempty[b], ((job >> 1) & 1u) ^ 1u);\n        tc_fence_after();\n        if (j == 1) {\n"
         "          mbar_wait_spin(&a_full, tl & 1u);\n          tc_fence_after();\n        }",
         "        if (elected) HT(tl, j, 0);\n        mbar_wait_spin(&tempty[b], ((job >> 1) & 1u) ^ 1u);\n"
         "        if (elected) HT(tl, j, 1);\n        tc_fence_after();\n        if (j == 1) {\n"
         "          mbar_wait_spin(&a_full, tl & 1u);\n          if (elected) HT(tl, j, 2);\n          tc_fence_after();\n        }"),
        ("          mbar_wait_spin(&full[st], (it / nst) & 1u);\n          tc_fence_after();\n          const uint32_t slot = saddr(sRing + st * kHeadSlot);\n          const uint64_t ad",
         "          const long long fw0 = clock64();\n          mbar_wait_spin(&full[st], (it / nst) & 1u);\n"
         "          if (elected) HTADD(tl, j, 4, clock64() - fw0);\n          tc_fence_after();\n"
         "          const uint32_t slot = saddr(sRing + st * kHeadSlot);\n          const uint64_t ad"),
        ("        commit_pred(&tfull[b], elected);\n        __syncwarp();\n      }\n      commit_pred(&a_empty, elected);",
         "        commit_pred(&tfull[b], elected);\n        if (elected) HT(tl, j, 3);\n        __syncwarp();\n      }\n"
         "      commit_pred(&a_empty, elected);"),
    ]
    for a, b in reps:
        assert src.count(a) == 1, a[:70]
        src = src.replace(a, b)
    # epilogue: job v, mean, chunks (thread 64 = warp 2 lane 0, group 0)
    ev = [("        mbar_wait_spin(&tfull[b], (job >> 1) & 1u);\n        tc_fence_after();\n        tmem_ld64(tmem + b * 256 + lanes, x);\n"
           "        tc_fence_before();\n        mbar_arrive(&tempty[b]);\n        ++job;\n#pragma unroll\n        for (int t = 0; t < ATOMS; ++t) v[t] = __uint_as_float(x[t]) + hb.v[t];",
           "        mbar_wait_spin(&tfull[b], (job >> 1) & 1u);\n        if (threadIdx.x == 64) HT(tl, 0, 5);\n        tc_fence_after();\n"
           "        tmem_ld64(tmem + b * 256 + lanes, x);\n        tc_fence_before();\n        mbar_arrive(&tempty[b]);\n"
           "        if (threadIdx.x == 64) HT(tl, 0, 6);\n        ++job;\n#pragma unroll\n        for (int t = 0; t < ATOMS; ++t) v[t] = __uint_as_float(x[t]) + hb.v[t];"),
          ("        mbar_wait_spin(&tfull[b], (job >> 1) & 1u);\n        tc_fence_after();\n        tmem_ld64(tmem + b * 256 + lanes, x);\n"
           "        tc_fence_before();\n        mbar_arrive(&tempty[b]);\n        ++job;\n#pragma unroll\n        for (int t = 0; t < ATOMS; ++t) v[t] = v[t] -",
           "        mbar_wait_spin(&tfull[b], (job >> 1) & 1u);\n        if (threadIdx.x == 64) HT(tl, 1, 5);\n        tc_fence_after();\n"
           "        tmem_ld64(tmem + b * 256 + lanes, x);\n        tc_fence_before();\n        mbar_arrive(&tempty[b]);\n"
           "        if (threadIdx.x == 64) HT(tl, 1, 6);\n        ++job;\n#pragma unroll\n        for (int t = 0; t < ATOMS; ++t) v[t] = v[t] -"),
          ("        mbar_wait_spin(&tfull[b], (job >> 1) & 1u);\n        tc_fence_after();\n        const int na = min(4, A - 4 * c);",
           "        mbar_wait_spin(&tfull[b], (job >> 1) & 1u);\n        if (threadIdx.x == 64) HT(tl, 2 + c - c_lo, 5);\n        tc_fence_after();\n"
           "        const int na = min(4, A - 4 * c);"),
          ("        tc_fence_before();\n        mbar_arrive(&tempty[b]);\n      }\n      if (mode != MODE_ROWS) {",
           "        tc_fence_before();\n        mbar_arrive(&tempty[b]);\n        if (threadIdx.x == 64) HT(tl, 2 + c - c_lo, 6);\n      }\n      if (mode != MODE_ROWS) {")]
    for a, b in ev:
        assert src.count(a) == 1, a[:70]
        src = src.replace(a, b)
    # kernel span (MMA issuer) for the SM clock
    a = "    const uint32_t elected = elect_one();\n    uint32_t it = 0, job = 0, tl = 0;"
    assert src.count(a) == 1
    src = src.replace(a, a + "\n    if (elected) { g_hg[blockIdx.x * 4] = ht_gt(); g_hg[blockIdx.x * 4 + 1] = clock64(); }")
    a = "      commit_pred(&a_empty, elected);   // sA free once this tile's MMAs have completed\n      __syncwarp();\n    }"
    assert src.count(a) == 1
    src = src.replace(a, a + "\n    if (elected) { g_hg[blockIdx.x * 4 + 2] = ht_gt(); g_hg[blockIdx.x * 4 + 3] = clock64(); }")
    src += ("\nextern \"C\" int ht_read(void *host, size_t bytes) { return (int)cudaMemcpyFromSymbol(host, bcts::g_ht, bytes); }\n"
            "extern \"C\" int hg_read(void *host) { return (int)cudaMemcpyFromSymbol(host, bcts::g_hg, sizeof(bcts::g_hg)); }\n"
            "extern \"C\" int ht_clear() { static long long z[HT_NCTA * HT_NT * HT_NJ * HT_NS]; "
            "return (int)cudaMemcpyToSymbol(bcts::g_ht, z, sizeof(z)); }\n")
    return src


def build():
    pkg = os.path.join(DST, "paper_2107_01715_b200")
    if os.path.exists(DST):
        shutil.rmtree(DST)
    shutil.copytree(os.path.join(ROOT, "paper_2107_01715_b200"), pkg,
                    ignore=shutil.ignore_patterns("build", "*.so", "__pycache__"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(DST, "include"))
    f = os.path.join(pkg, "csrc", "qnet_tma.cu")
    txt = patch(open(f).read())
    open(f, "w").write(txt)
    subprocess.run([sys.executable, "-c", "import sys; sys.path.insert(0, %r); "
                    "from paper_2107_01715_b200 import build; build.build(force=True)" % DST], check=True)
    print("built")


def run():
    sys.path.insert(0, DST)
    sys.path.insert(1, ROOT)
    import ctypes
    import numpy as np
    import torch
    import paper_2107_01715_b200 as P
    assert P.__file__.startswith(DST)
    from synth.inputs import config
    cfg = config("C5")
    h = P.Handle.from_config(cfg)
    roots = torch.from_numpy(cfg.roots(1).view(np.uint8).copy()).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    L = P.lib()
    for _ in range(4):
        h.search(roots, 1, 4, cfg.gamma, cfg.beta, 1)
    torch.cuda.synchronize()
    flush.fill_(1)
    torch.cuda.synchronize()
    assert L.ht_clear() == 0
    h.search(roots, 1, 4, cfg.gamma, cfg.beta, 1)
    torch.cuda.synchronize()
    buf = np.zeros(NCTA * NT * NJ * NS, np.int64)
    assert L.ht_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
    t = buf.reshape(NCTA, NT, NJ, NS)
    g = np.zeros(1024 * 4, np.uint64)
    assert L.hg_read(g.ctypes.data_as(ctypes.c_void_p)) == 0
    g = g.reshape(1024, 4).astype(np.int64)[:148]
    ok = g[:, 2] > 0
    ns, cyc = g[ok, 2] - g[ok, 0], g[ok, 3] - g[ok, 1]
    print(f"MMA-issuer span {ns.min() / 1e3:.1f}..{ns.max() / 1e3:.1f} us, SM clock median {np.median(cyc / ns):.3f} GHz")
    names = ["v", "mean", "c0", "c1", "c2", "c3", "c4", "-"]
    for cta in range(2):
        print(f"CTA {cta}")
        for tl in range(1, 5):
            x = t[cta, tl]
            if x[0, 0] == 0:
                continue
            t0 = x[0, 0]
            print(f"  tile {tl}: producer a_empty wait {x[1, 8] - x[0, 7]:6d} (at +{x[0, 7] - t0}); "
                  f"tile span {t[cta, tl + 1, 0, 0] - t0 if t[cta, tl + 1, 0, 0] else -1}")
            for j in range(7):
                if x[j, 0] == 0:
                    continue
                print(f"    {names[j]:4s} issuer: tempty wait {x[j, 1] - x[j, 0]:6d} a_full wait "
                      f"{(x[j, 2] - x[j, 1]) if j == 1 else 0:6d} ring waits {x[j, 4]:6d} issue->commit "
                      f"{x[j, 3] - (x[j, 2] if j == 1 else x[j, 1]):6d} | epi tfull at +{x[j, 5] - t0:6d} done +{x[j, 6] - t0:6d}")


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
