// tools/mma2sm_test.cu -- semantics check of the 2-SM MMA (tcgen05.mma.cta_group::2) on a CTA pair:
// D[256 x 256] = A[256 x K] . B[256 x K]^T, K = 64, bf16, SWIZZLE_NONE K-major operands written by
// threads into each CTA's SMEM. Hypothesis: CTA r holds A rows 128r..128r+127 and B rows (N)
// 128r..128r+127 (N split), the leader (rank 0) issues, each CTA's TMEM receives its own 128 rows x
// all 256 columns. Prints max |D - ref| per CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma2sm_test tools/mma2sm_test.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <cmath>

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_planar(uint32_t addr, uint32_t lbo) {
  uint64_t d = (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)(lbo >> 4) << 16;
  d |= (uint64_t)(128 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
constexpr int MH = 128, NH = 128, N = 256, K = 64;   // per-CTA A rows, per-CTA B rows, total N, K
__device__ float aval(int m, int k) { return (float)(((m * 3 + k * 7) % 11) - 5) * 0.5f; }
__device__ float bval(int n, int k) { return (float)(((n * 5 + k * 3) % 13) - 6) * 0.25f; }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(float *D, int variant) {
  __shared__ __align__(1024) uint8_t sA[MH * K * 2];
  __shared__ __align__(1024) uint8_t sB[NH * K * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  // operand halves of this CTA (K-major, no swizzle: chunk j = k/8 at j * rows * 16)
  for (int e = threadIdx.x; e < MH * K; e += blockDim.x) {
    const int m = e / K, kk = e % K;
    *(__nv_bfloat16 *)(sA + (kk / 8) * (MH * 16) + m * 16 + (kk % 8) * 2) = __float2bfloat16_rn(aval(MH * rank + m, kk));
  }
  for (int e = threadIdx.x; e < NH * K; e += blockDim.x) {
    const int n = e / K, kk = e % K;
    const int ng = variant == 0 ? NH * (int)rank + n : n;   // variant 0: N split; variant 1: full B rows 0..127 in both
    *(__nv_bfloat16 *)(sB + (kk / 8) * (NH * 16) + n * 16 + (kk % 8) * 2) = __float2bfloat16_rn(bval(ng, kk));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(saddr(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  if (rank == 0 && threadIdx.x == 0) {
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint64_t ad = desc_planar(saddr(sA) + ks * 2 * (MH * 16), MH * 16);
      const uint64_t bd = desc_planar(saddr(sB) + ks * 2 * (NH * 16), NH * 16);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(ks));
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     saddr(&bar)),
                 "h"((uint16_t)3)
                 : "memory");
  }
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(
                   saddr(&bar))
               : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t ta = tmem + ((uint32_t)((threadIdx.x / 32) * 32) << 16);
  for (int c = 0; c < N; c += 32) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(ta + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int m = MH * rank + threadIdx.x;
    for (int i = 0; i < 32; ++i) D[m * N + c + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  float *d, *h = new float[256 * N];
  cudaMalloc(&d, 256 * N * 4);
  for (int variant = 0; variant < 2; ++variant) {
    cudaMemset(d, 0, 256 * N * 4);
    k<<<2, 128>>>(d, variant);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 256 * N * 4, cudaMemcpyDeviceToHost);
    double err[2] = {0, 0};
    for (int m = 0; m < 256; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int kk = 0; kk < K; ++kk) {
          const double a = (double)(((m * 3 + kk * 7) % 11) - 5) * 0.5;
          const int ng = variant == 0 ? n : n % 128;
          const double b = (double)(((ng * 5 + kk * 3) % 13) - 6) * 0.25;
          ref += a * b;
        }
        const double e2 = fabs(h[m * N + n] - ref);
        if (e2 > err[m / 128]) err[m / 128] = e2;
      }
    printf("variant %d (%s): %s; max|D-ref| CTA0 rows %g, CTA1 rows %g; D[0][0..3] = %g %g %g %g\n", variant,
           variant == 0 ? "B split along N" : "B rows 0..127 in both CTAs", cudaGetErrorString(e), err[0], err[1], h[0],
           h[1], h[2], h[3]);
  }
  return 0;
}
