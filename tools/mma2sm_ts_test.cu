// tools/mma2sm_ts_test.cu -- semantics of tcgen05.mma.cta_group::2 with the A operand in TMEM
// (kind::f16 bf16, M = 128 = 64 rows per CTA, N = 128 with B split along N: 64 rows per CTA, K = 16):
// which TMEM lanes of each CTA hold its A rows, and which lanes / columns of each CTA's TMEM
// receive D. A is written with tcgen05.st under two lane hypotheses (hyp 1: local row m at lane
// (m / 16) * 32 + m % 16, the cta_group::1 M = 64 layout; hyp 2: lane m). Each CTA dumps all 128
// lanes x 128 columns of D; the host matches every dumped lane against the reference rows.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma2sm_ts_test tools/mma2sm_ts_test.cu
#include <cuda_bf16.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_planar(uint32_t addr, uint32_t lbo) {
  uint64_t d = (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)(lbo >> 4) << 16;
  d |= (uint64_t)(128 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
constexpr int MH = 64, NH = 64, K = 16;   // per-CTA halves
__host__ __device__ float aval(int g, int k) { return (float)(((g * 31 + k * 17 + g * k) % 61) - 30) * 0.125f; }   // A row g
__host__ __device__ float bval(int n, int k) { return (float)(((n * 23 + k * 29 + n * k * 3) % 59) - 29) * 0.125f; }  // B row n
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(lo)) |
         ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(hi)) << 16);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void __cluster_dims__(2, 1, 1) k(float *D, int hyp) {
  __shared__ __align__(1024) uint8_t sB[NH * K * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int e = threadIdx.x; e < NH * K; e += blockDim.x) {   // this CTA's B half: global rows 64r + n
    const int n = e / K, kk = e % K;
    *(__nv_bfloat16 *)(sB + (kk / 8) * (NH * 16) + n * 16 + (kk % 8) * 2) = __float2bfloat16_rn(bval(64 * rank + n, kk));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  {   // A (this CTA's 64 rows, global rows 64r + m) into TMEM columns [0, 8)
    const int l = warp * 32 + lane;
    int m = -1;
    if (hyp == 1) m = (l % 32 < 16) ? (l / 32) * 16 + l % 32 : -1;
    else m = l < 64 ? l : -1;
    uint32_t r[8];
    for (int j = 0; j < 8; ++j) r[j] = m >= 0 ? pack2(aval(64 * rank + m, 2 * j), aval(64 * rank + m, 2 * j + 1)) : 0u;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                     tmem + ((uint32_t)(warp * 32) << 16)),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (rank == 0 && threadIdx.x == 0) {
    const uint64_t bd = desc_planar(saddr(sB), NH * 16);
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + 64),
        "r"(tmem), "l"(bd), "r"(idesc_bf16(128, 128)));
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            saddr(&bar)),
        "h"((uint16_t)3)
        : "memory");
  }
  asm volatile(
      "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(saddr(&bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c = 0; c < 128; c += 8) {   // D: all 128 lanes x 128 columns of this CTA's TMEM, from column 64
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + 64 + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) D[((size_t)rank * 128 + warp * 32 + lane) * 128 + c + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

static float bf(float x) {   // host bf16 RNE of the small exact test values (they are exact already)
  return x;
}

int main() {
  float *dD;
  cudaMalloc(&dD, 2 * 128 * 128 * 4);
  std::vector<float> D(2 * 128 * 128), ref(128 * 128);
  for (int g = 0; g < 128; ++g)
    for (int n = 0; n < 128; ++n) {
      double s = 0;
      for (int kk = 0; kk < K; ++kk) s += (double)bf(aval(g, kk)) * bf(bval(n, kk));
      ref[g * 128 + n] = (float)s;
    }
  for (int hyp = 1; hyp <= 2; ++hyp) {
    cudaMemset(dD, 0, 2 * 128 * 128 * 4);
    k<<<2, 128>>>(dD, hyp);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("hyp %d: %s\n", hyp, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    printf("hyp %d (A row m at lane %s):\n", hyp, hyp == 1 ? "(m/16)*32 + m%16" : "m");
    for (int r = 0; r < 2; ++r) {
      int matched = 0, first = -1, last = -1;
      printf("  CTA %d lane->A row (global), '.' = zero lane, '?' = no match:\n   ", r);
      for (int l = 0; l < 128; ++l) {
        const float *row = &D[((size_t)r * 128 + l) * 128];
        bool zero = true;
        for (int n = 0; n < 128; ++n) zero &= row[n] == 0.0f;
        int hit = -1;
        for (int g = 0; g < 128 && hit < 0 && !zero; ++g) {
          bool ok = true;
          for (int n = 0; n < 128 && ok; ++n) ok = fabsf(row[n] - ref[g * 128 + n]) <= 1e-3f;
          if (ok) hit = g;
        }
        if (zero) printf(" .");
        else if (hit < 0) printf(" ?");
        else {
          printf(" %d", hit);
          ++matched;
          if (first < 0) first = l;
          last = l;
        }
        if (l % 32 == 31) printf("\n   ");
      }
      printf("matched %d lanes (first %d, last %d)\n", matched, first, last);
      // 64-column halves: which global A row g and B offset (0 or 64) reproduce D[l][c .. c+63]?
      for (int l = 0; l < 128; l += 1) {
        const float *row = &D[((size_t)r * 128 + l) * 128];
        for (int half = 0; half < 2; ++half) {
          bool zero = true;
          for (int c = 0; c < 64; ++c) zero &= row[half * 64 + c] == 0.0f;
          if (zero) continue;
          int hit = -1, off = -1;
          for (int g = 0; g < 128 && hit < 0; ++g)
            for (int o = 0; o < 128 && hit < 0; o += 64) {
              bool ok = true;
              for (int c = 0; c < 64 && ok; ++c) ok = fabsf(row[half * 64 + c] - ref[g * 128 + o + c]) <= 1e-3f;
              if (ok) hit = g, off = o;
            }
          if (l < 4 || (l % 16) == 0) printf("   CTA %d lane %3d cols %3d..%3d: A row %d x B rows %d..%d\n", r, l, half * 64,
                                             half * 64 + 63, hit, off, off + 63);
        }
      }
    }
  }
  return 0;
}
