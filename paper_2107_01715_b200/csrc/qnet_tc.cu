// qnet_tc.cu -- K2 on the 5th-gen tensor cores: one implicit-GEMM layer
//   out[m][n] = act( sum_k X[m][k] * W[n][k] + b[n] )
// for every conv / fc layer of the leaf Q-net (Alg. 1 leaf line).
//
// Per CTA: a 128-row M tile x BN columns. Warp roles:
//   warps 0-3 (128 threads): producers -- thread t gathers row t of the
//       im2col'd A tile (128 contiguous bytes per k-block: NHWC makes 64
//       consecutive k = (ky, kx, c) contiguous in memory; conv1 converts two
//       32-byte uint8 pixel rows to bf16 on the fly) and its share of the
//       weight rows, and stores both into shared memory in the canonical
//       K-major SWIZZLE_128B layout; then the same warps run the epilogue
//       (tcgen05.ld TMEM -> registers -> bias, ReLU, bf16 RNE -> global).
//   warp 4: allocates the TMEM accumulator; one elected thread issues the
//       tcgen05.mma.cta_group::1.kind::f16 (M=128, N=BN, K=16) and signals
//       smem-slot release / accumulator completion with tcgen05.commit.
// A kStages-deep mbarrier ring (full: 128 producer arrivals; empty: one
// tcgen05.commit) overlaps the gather of k-block i+1.. with the MMAs of i.
#include <algorithm>

#include "engine.h"

namespace bcts {
namespace {

constexpr int kStages = 4;
constexpr int kBM = 128;        // UMMA M
constexpr int kBK = 64;         // bf16 per k-block = one 128-byte swizzle-atom row
constexpr int kThreads = 160;

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(saddr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor (tcgen05): start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version 1 [46,48), base offset [49,52), layout [61,64).
// K-major SWIZZLE_128B: 8-row x 128-byte atoms, atoms 1024 B apart (SBO); LBO unused.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;                 // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO
  d |= (uint64_t)1 << 46;                 // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}
// Instruction descriptor, kind::f16: D=F32 [4,6), A=BF16 [7,10), B=BF16 [10,13),
// K-major A and B, N>>3 [17,23), M>>4 [24,29).
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// uint8 word (4 pixels' bytes) -> two packed bf16x2 words (exact: v < 256).
__device__ __forceinline__ uint32_t u8pair_bf16(uint32_t w, int sh) {
  const uint32_t lo = __float_as_uint((float)((w >> sh) & 0xFFu)) >> 16;
  const uint32_t hi = __float_as_uint((float)((w >> (sh + 8)) & 0xFFu)) >> 16;
  return lo | (hi << 16);
}
__device__ __forceinline__ uint4 u8x8_to_bf16(uint32_t w0, uint32_t w1) {
  return make_uint4(u8pair_bf16(w0, 0), u8pair_bf16(w0, 16), u8pair_bf16(w1, 0), u8pair_bf16(w1, 16));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async16_cg(uint32_t dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Persistent, warp-specialized layer kernel.
//   warps 0-3 : producers (A gather + streamed B)   -> smem ring (kStages)
//   warp  4   : TMEM allocator + single-thread MMA issuer
//   warps 5-8 : epilogue (TMEM -> regs -> global), double-buffered accumulator
// BRES: the whole weight matrix ([Npad][K], <= 72 KB) is loaded once per CTA
// and stays resident in shared memory; otherwise B streams with A per k-block.
constexpr int kThreads2 = 288;
constexpr int kLag = 2;   // cp.async groups kept in flight per producer thread

template <int BN, bool U8, bool BRES>
struct Cfg {
  static constexpr int A_BYTES = kBM * 128;
  static constexpr int B_STAGE = BRES ? 0 : BN * 128;
  static constexpr int STAGE = A_BYTES + B_STAGE;
  static constexpr int STAGES = BRES ? 6 : 4;
  static constexpr uint32_t TCOLS = 2 * BN < 32 ? 32 : 2 * BN;
  static int smem_bytes(int bres_bytes) { return STAGES * STAGE + (BRES ? bres_bytes : 0) + 1024; }
};

template <int BN, bool U8, bool BRES>
__global__ void __launch_bounds__(kThreads2, 1) k_layer_tc(Layer L, const void *__restrict__ in, int64_t M,
                                                           void *__restrict__ out, int n_m, int n_n) {
  using C = Cfg<BN, U8, BRES>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base, derived from smem_raw by an OFFSET so the compiler keeps the
  // shared address space (a uintptr_t round trip turns every access into a generic LD/ST)
  uint8_t *smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  uint8_t *sB_res = smem + C::STAGES * C::STAGE;   // resident weights (BRES)
  __shared__ __align__(8) uint64_t full[C::STAGES], empty[C::STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nk = L.K / kBK;
  const int n_tiles = n_m * n_n;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 128);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_slot)),
                 "r"(C::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (BRES) {
    // all threads: weights -> smem, one [Npad x 128 B] swizzled block per k-block
    const int chunks = L.Npad * nk * 8;
    for (int e = threadIdx.x; e < chunks; e += kThreads2) {
      const int j = e & 7, kb = (e >> 3) % nk, n = (e >> 3) / nk;
      const uint4 w = __ldg((const uint4 *)(L.Wt + (int64_t)n * L.K + (int64_t)kb * kBK) + j);
      uint8_t *row = sB_res + (size_t)kb * L.Npad * 128 + (uint32_t)(n >> 3) * 1024u + (uint32_t)(n & 7) * 128u;
      *(uint4 *)(row + (uint32_t)((j ^ (n & 7)) << 4)) = w;
    }
    fence_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp < 4) {
    // ------------------------------------------------------------ producers
    const int t = threadIdx.x;
    const int sw = t & 7;
    const uint32_t a_row_off = (uint32_t)(t >> 3) * 1024u + (uint32_t)sw * 128u;
    const int64_t rows = (int64_t)L.OH * L.OW;
    const int kwc = L.KW * L.C;
    uint32_t it = 0;
    // U8 (conv1) software pipeline: raw[] holds this tile's 4 k-blocks of raw
    // bytes, nxt[] the next tile's, whose loads are in flight meanwhile.
    uint4 raw[16], nxt[16];
    auto load_u8_tile = [&](int tile_idx, uint4 (&dst)[16]) {
      const int64_t mm = (int64_t)(tile_idx / n_n) * kBM + t;
      if (tile_idx < n_tiles && mm < M) {
        const int64_t im = mm / rows;
        const int ps = (int)(mm - im * rows);
        const int yy = ps / L.OW, xx = ps - yy * L.OW;
        const uint8_t *base = (const uint8_t *)in + im * L.in_img_stride + ((int64_t)(yy * L.S) * L.W + xx * L.S) * 4;
#pragma unroll
        for (int ky = 0; ky < 8; ++ky) {
          const uint4 *p = (const uint4 *)(base + (int64_t)ky * L.W * 4);
          dst[2 * ky] = __ldg(p);
          dst[2 * ky + 1] = __ldg(p + 1);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) dst[j] = make_uint4(0, 0, 0, 0);
      }
    };
    if (U8) load_u8_tile(blockIdx.x, raw);
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const int mt = tile / n_n, ntile = tile - mt * n_n;
      const int64_t m = (int64_t)mt * kBM + t;
      const bool valid = m < M;
      if (U8) load_u8_tile(tile + gridDim.x, nxt);
      const int n0 = ntile * BN;
      const int nt = min(BN, L.Npad - n0);
      int64_t img = 0;
      int oy = 0, ox = 0;
      if (valid) {
        img = m / rows;
        const int pos = (int)(m - img * rows);
        oy = pos / L.OW;
        ox = pos - oy * L.OW;
      }
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = it % C::STAGES;
        const uint32_t ph = (it / C::STAGES) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        uint8_t *sa = smem + s * C::STAGE;
        const uint32_t sa_u = saddr(sa);
        if (U8) {
          // conv1: two 32-byte uint8 pixel rows per k-block -> 64 bf16 (exact).
          // The whole tile's raw bytes (nk <= 4 k-blocks, 16 x 16 B) were loaded
          // into registers one tile ahead (software pipeline, see below).
          uint4 v[8];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 x;
            switch (kb) {   // constant-indexed register selection (no local memory)
              case 0: x = raw[j]; break;
              case 1: x = raw[4 + j]; break;
              case 2: x = raw[8 + j]; break;
              default: x = raw[12 + j]; break;
            }
            v[2 * j] = u8x8_to_bf16(x.x, x.y);
            v[2 * j + 1] = u8x8_to_bf16(x.z, x.w);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) *(uint4 *)(sa + a_row_off + (uint32_t)((j ^ sw) << 4)) = v[j];
          fence_async_smem();
          mbar_arrive(&full[s]);
          if (kb == nk - 1) {
#pragma unroll
            for (int j = 0; j < 16; ++j) raw[j] = nxt[j];
          }
        } else {
          // bf16: 128 contiguous bytes per row per k-block -> cp.async (L1-cached: im2col reuse)
          const void *src = in;
          if (valid) {
            const int k0 = kb * kBK;
            const int ky = k0 / kwc, r = k0 - ky * kwc;
            const int kx = r / L.C, c = r - kx * L.C;
            src = (const __nv_bfloat16 *)in + img * L.in_img_stride + L.in_col_off +
                  ((int64_t)(oy * L.S + ky) * L.W + (ox * L.S + kx)) * L.C + c;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            cp_async16(sa_u + a_row_off + (uint32_t)((j ^ sw) << 4), (const uint4 *)src + (valid ? j : 0),
                       valid ? 16u : 0u);
          if (!BRES) {
            const uint32_t sb_u = sa_u + C::A_BYTES;
            for (int n = t; n < nt; n += 128) {
              const uint4 *p = (const uint4 *)(L.Wt + (int64_t)(n0 + n) * L.K + (int64_t)kb * kBK);
              const uint32_t rowp = sb_u + (uint32_t)(n >> 3) * 1024u + (uint32_t)(n & 7) * 128u;
#pragma unroll
              for (int j = 0; j < 8; ++j) cp_async16_cg(rowp + (uint32_t)((j ^ (n & 7)) << 4), p + j);
            }
          }
          cp_async_commit();
          if (it >= (uint32_t)kLag) {
            cp_async_wait<kLag>();
            fence_async_smem();
            mbar_arrive(&full[(it - kLag) % C::STAGES]);
          }
        }
      }
    }
    if (!U8) {
      cp_async_wait<0>();
      fence_async_smem();
      for (uint32_t j = (it >= (uint32_t)kLag ? it - kLag : 0); j < it; ++j) mbar_arrive(&full[j % C::STAGES]);
    }
  } else if (warp == 4) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      uint32_t it = 0, acc_it = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++acc_it) {
        const int ntile = tile % n_n;
        const int n0 = ntile * BN;
        const int nt = min(BN, L.Npad - n0);
        const uint32_t idesc = idesc_bf16(kBM, nt);
        const uint32_t a = acc_it & 1u, aph = (acc_it >> 1) & 1u;
        mbar_wait(&tempty[a], aph ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + a * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % C::STAGES;
          const uint32_t ph = (it / C::STAGES) & 1u;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a0 = saddr(smem + s * C::STAGE);
          const uint32_t b0 = BRES ? saddr(sB_res + (size_t)kb * L.Npad * 128 + (size_t)n0 * 128)
                                   : a0 + C::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk)
            mma_bf16(d, sw128_desc(a0 + kk * 32), sw128_desc(b0 + kk * 32), idesc, (kb | kk) != 0);
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[a]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;               // TMEM lane quarter this warp may access
    const int r = q * 32 + lane;          // tile row
    uint32_t acc_it = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++acc_it) {
      const int mt = tile / n_n, ntile = tile - mt * n_n;
      const int64_t m = (int64_t)mt * kBM + r;
      const int n0 = ntile * BN;
      const int nt = min(BN, L.Npad - n0);
      const uint32_t a = acc_it & 1u, aph = (acc_it >> 1) & 1u;
      mbar_wait(&tfull[a], aph);
      tc_fence_after();
      const uint32_t trow = tmem + a * BN + ((uint32_t)(q * 32) << 16);
      for (int c = 0; c < nt; c += 16) {
        uint32_t v[16];
        tmem_ld16(trow + (uint32_t)c, v);
        if (m >= M) continue;
        const float *bias = L.bias + n0 + c;
        if (L.relu_bf16) {
          uint32_t pk[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float x = __uint_as_float(v[2 * i]) + __ldg(bias + 2 * i);
            float y = __uint_as_float(v[2 * i + 1]) + __ldg(bias + 2 * i + 1);
            __nv_bfloat162 h = __floats2bfloat162_rn(x > 0.0f ? x : 0.0f, y > 0.0f ? y : 0.0f);
            pk[i] = *(uint32_t *)&h;
          }
          uint4 *dst = (uint4 *)((__nv_bfloat16 *)out + m * L.out_ld + n0 + c);
          dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        } else {
          float4 *dst = (float4 *)((float *)out + m * L.out_ld + n0 + c);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_float4(__uint_as_float(v[4 * i]) + __ldg(bias + 4 * i),
                                 __uint_as_float(v[4 * i + 1]) + __ldg(bias + 4 * i + 1),
                                 __uint_as_float(v[4 * i + 2]) + __ldg(bias + 4 * i + 2),
                                 __uint_as_float(v[4 * i + 3]) + __ldg(bias + 4 * i + 3));
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[a]);
    }
  }
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TCOLS));
  }
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, bool U8, bool BRES>
void launch(const Layer &L, const void *in, int64_t M, void *out, cudaStream_t st) {
  using C = Cfg<BN, U8, BRES>;
  const int bres = BRES ? L.Npad * L.K * 2 : 0;
  const int smem = C::smem_bytes(bres);
  static int attr_for = -1;
  if (attr_for < smem) {
    cudaFuncSetAttribute(k_layer_tc<BN, U8, BRES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_for = smem;
  }
  const int n_m = (int)((M + kBM - 1) / kBM), n_n = (L.Npad + BN - 1) / BN;
  const int per_sm = smem <= 110 * 1024 ? 2 : 1;
  const int grid = std::min<int64_t>((int64_t)n_m * n_n, (int64_t)num_sms() * per_sm);
  k_layer_tc<BN, U8, BRES><<<grid, kThreads2, smem, st>>>(L, in, M, out, n_m, n_n);
}

}  // namespace

bool tc_supported(const Layer &L) {
  if (L.K % kBK != 0 || L.Npad % 16 != 0 || L.Npad < 16) return false;
  if (L.in_u8) return L.C == 4 && L.KW == 8 && L.KH % 2 == 0 && L.Npad <= 32 && L.in_img_stride % 16 == 0;
  return (L.KW * L.C) % kBK == 0 && L.C % 8 == 0 && L.in_col_off % 8 == 0 && L.in_img_stride % 8 == 0;
}

void launch_layer_tc(const Layer &L, const void *in, int64_t n_img, void *out, cudaStream_t st) {
  const int64_t M = n_img * L.rows_per_img();
  if (M <= 0) return;
  const bool res = (int64_t)L.Npad * L.K * 2 <= 80 * 1024;   // weights fit: keep them resident
  if (L.in_u8) {
    launch<32, true, true>(L, in, M, out, st);
  } else if (L.Npad <= 32) {
    if (res) launch<32, false, true>(L, in, M, out, st);
    else launch<32, false, false>(L, in, M, out, st);
  } else if (L.Npad <= 64) {
    if (res) launch<64, false, true>(L, in, M, out, st);
    else launch<64, false, false>(L, in, M, out, st);
  } else {
    launch<256, false, false>(L, in, M, out, st);
  }
}

}  // namespace bcts
