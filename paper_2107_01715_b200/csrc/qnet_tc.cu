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

template <int BN, bool U8>
__global__ void __launch_bounds__(kThreads, 1) k_layer_tc(Layer L, const void *__restrict__ in, int64_t M,
                                                          void *__restrict__ out) {
  constexpr int A_BYTES = kBM * 128;
  constexpr int B_BYTES = BN * 128;
  constexpr int STAGE = A_BYTES + B_BYTES;
  constexpr uint32_t TCOLS = BN < 32 ? 32 : BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], done;
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t m0 = (int64_t)blockIdx.x * kBM;
  const int n0 = blockIdx.y * BN;
  const int nt = min(BN, L.Npad - n0);
  const int nk = L.K / kBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 128);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_slot)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp < 4) {
    // ------------------------------------------------------------ producer
    const int t = threadIdx.x;
    const int64_t m = m0 + t;
    const bool valid = m < M;
    const int64_t rows = (int64_t)L.OH * L.OW;
    int64_t img = 0;
    int oy = 0, ox = 0;
    if (valid) {
      img = m / rows;
      const int pos = (int)(m - img * rows);
      oy = pos / L.OW;
      ox = pos - oy * L.OW;
    }
    const int sw = t & 7;
    const uint32_t a_row_off = (uint32_t)(t >> 3) * 1024u + (uint32_t)sw * 128u;
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kStages;
      const uint32_t ph = (uint32_t)(kb / kStages) & 1u;
      mbar_wait(&empty[s], ph ^ 1u);
      uint8_t *sa = smem + s * STAGE;
      uint8_t *sb = sa + A_BYTES;
      uint4 v[8];
      if (valid) {
        if (U8) {
          // conv1: k = (ky, kx, c) with C = 4, KW = 8: a k-block = two ky rows of 32 bytes
          const uint8_t *base = (const uint8_t *)in + img * L.in_img_stride +
                                ((int64_t)(oy * L.S) * L.W + ox * L.S) * 4;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint4 *p = (const uint4 *)(base + (int64_t)(2 * kb + h) * L.W * 4);
            const uint4 x0 = __ldg(p), x1 = __ldg(p + 1);
            v[4 * h + 0] = u8x8_to_bf16(x0.x, x0.y);
            v[4 * h + 1] = u8x8_to_bf16(x0.z, x0.w);
            v[4 * h + 2] = u8x8_to_bf16(x1.x, x1.y);
            v[4 * h + 3] = u8x8_to_bf16(x1.z, x1.w);
          }
        } else {
          const int k0 = kb * kBK;
          const int kwc = L.KW * L.C;
          const int ky = k0 / kwc, r = k0 - ky * kwc;
          const int kx = r / L.C, c = r - kx * L.C;
          const uint4 *p = (const uint4 *)((const __nv_bfloat16 *)in + img * L.in_img_stride + L.in_col_off +
                                           ((int64_t)(oy * L.S + ky) * L.W + (ox * L.S + kx)) * L.C + c);
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = __ldg(p + j);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) *(uint4 *)(sa + a_row_off + (uint32_t)((j ^ sw) << 4)) = v[j];
      // weight rows n = t, t + 128 (K-major [Npad][K] bf16)
      for (int n = t; n < nt; n += 128) {
        const uint4 *p = (const uint4 *)(L.Wt + (int64_t)(n0 + n) * L.K + (int64_t)kb * kBK);
        uint8_t *rowp = sb + (uint32_t)(n >> 3) * 1024u + (uint32_t)(n & 7) * 128u;
        uint4 w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = __ldg(p + j);
#pragma unroll
        for (int j = 0; j < 8; ++j) *(uint4 *)(rowp + (uint32_t)((j ^ (n & 7)) << 4)) = w[j];
      }
      fence_async_smem();   // make the generic-proxy stores visible to the tensor core (async proxy)
      mbar_arrive(&full[s]);
    }
    // ------------------------------------------------------------ epilogue
    mbar_wait(&done, 0);
    tc_fence_after();
    const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < nt; c += 16) {
      uint32_t r[16];
      tmem_ld16(trow + (uint32_t)c, r);
      if (!valid) continue;
      const float *bias = L.bias + n0 + c;
      if (L.relu_bf16) {
        uint32_t pk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float a = __uint_as_float(r[2 * i]) + bias[2 * i];
          float b = __uint_as_float(r[2 * i + 1]) + bias[2 * i + 1];
          a = a > 0.0f ? a : 0.0f;
          b = b > 0.0f ? b : 0.0f;
          __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
          pk[i] = *(uint32_t *)&h;
        }
        uint4 *dst = (uint4 *)((__nv_bfloat16 *)out + m * L.out_ld + n0 + c);
        dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      } else {
        float f[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(r[i]) + bias[i];
        float4 *dst = (float4 *)((float *)out + m * L.out_ld + n0 + c);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
      }
    }
    tc_fence_before();
  } else {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(kBM, nt);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kStages;
        const uint32_t ph = (uint32_t)(kb / kStages) & 1u;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a0 = saddr(smem + s * STAGE), b0 = a0 + A_BYTES;
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)   // K = 16 per MMA: +32 bytes inside the swizzle atom
          mma_bf16(tmem, sw128_desc(a0 + kk * 32), sw128_desc(b0 + kk * 32), idesc, (kb | kk) != 0);
        mma_commit(&empty[s]);                   // frees the smem slot once these MMAs retire
      }
      mma_commit(&done);                         // accumulator complete
    }
    __syncwarp();
  }
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
  }
}

template <int BN, bool U8>
void launch(const Layer &L, const void *in, int64_t M, void *out, cudaStream_t st) {
  constexpr int smem = kStages * (kBM * 128 + BN * 128) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_layer_tc<BN, U8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid((unsigned)((M + kBM - 1) / kBM), (unsigned)((L.Npad + BN - 1) / BN));
  k_layer_tc<BN, U8><<<grid, kThreads, smem, st>>>(L, in, M, out);
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
  if (L.in_u8) {
    launch<32, true>(L, in, M, out, st);
  } else if (L.Npad <= 32) {
    launch<32, false>(L, in, M, out, st);
  } else if (L.Npad <= 64) {
    launch<64, false>(L, in, M, out, st);
  } else {
    launch<256, false>(L, in, M, out, st);
  }
}

}  // namespace bcts
