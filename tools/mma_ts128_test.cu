// tools/mma_ts128_test.cu -- (copy of mma_ts_test.cu at M = 128) semantics + speed of tcgen05.mma with A in TMEM (M = 128,
// N = 64, K = 16, kind::f16 bf16) for conv3's weights. A is written with tcgen05.st
// (32x32b.x8: 8 columns = 16 bf16 per lane) under two lane-layout hypotheses:
//   H1: row m at lane (m / 16) * 32 + m % 16  (the measured M = 64 accumulator layout)
//   H2: row m at lane m                         (rows 0..63 in lanes 0..63)
// B: SWIZZLE_NONE K-major in SMEM. D read back with the M = 64 accumulator layout (H1).
// Then times 4096 ts-MMAs vs ss-MMAs (A in SMEM) at M = 64, N = 64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_ts_test tools/mma_ts_test.cu
#include <cuda_bf16.h>
#include <cmath>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_planar(uint32_t addr, uint32_t lbo) {
  uint64_t d = (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)(lbo >> 4) << 16;
  d |= (uint64_t)(128 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
constexpr int M = 128, N = 64, K = 16;
__device__ float aval(int m, int k) { return (float)(((m * 3 + k * 7) % 11) - 5) * 0.5f; }
__device__ float bval(int n, int k) { return (float)(((n * 5 + k * 3) % 13) - 6) * 0.25f; }
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(lo)) | ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(hi)) << 16);
}

__global__ void k(float *D, int hyp, int timing, long long *cyc) {
  __shared__ __align__(1024) uint8_t sB[N * K * 2];
  __shared__ __align__(1024) uint8_t sA[128 * K * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    const int n = e / K, kk = e % K;
    *(__nv_bfloat16 *)(sB + (kk / 8) * (N * 16) + n * 16 + (kk % 8) * 2) = __float2bfloat16_rn(bval(n, kk));
  }
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) {   // SMEM copy of A for the ss timing
    const int m = e / K, kk = e % K;
    *(__nv_bfloat16 *)(sA + (kk / 8) * (M * 16) + m * 16 + (kk % 8) * 2) = __float2bfloat16_rn(aval(m, kk));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  // A into TMEM columns [0, 8): each warp writes its lane quarter
  {
    const int l = warp * 32 + lane;   // TMEM lane
    int m = -1;
    if (hyp == 1) m = (l % 32) * 4 + l / 32;
    else m = l;
    uint32_t r[8];
    for (int j = 0; j < 8; ++j) r[j] = m >= 0 ? pack2(aval(m, 2 * j), aval(m, 2 * j + 1)) : 0u;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                     tmem + ((uint32_t)(warp * 32) << 16)),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  const uint64_t bd = desc_planar(saddr(sB), N * 16), ad = desc_planar(saddr(sA), M * 16);
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    const int iters = timing ? 4096 : 1;
    for (int i = 0; i < iters; ++i) {
      if (timing == 2)   // ss reference: A from SMEM
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                         tmem + 256),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(i));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
                         tmem + 256),
                     "r"(tmem), "l"(bd), "r"(idesc), "r"(i));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar)) : "memory");
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(saddr(&bar))
                 : "memory");
    *cyc = (clock64() - t0) / iters;
  }
  __syncthreads();
  asm volatile("{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W2;\n}\n" ::"r"(saddr(&bar))
               : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  // D (M = 64 layout): row m at lane (m / 16) * 32 + m % 16, columns 256 + n
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16) + 256 + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    {
      const int m = warp * 32 + lane;
      for (int i = 0; i < 16; ++i) D[m * N + c + i] = __uint_as_float(r[i]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  float *d, h[M * N];
  long long *c, hc;
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&c, 8);
  for (int hyp = 1; hyp <= 2; ++hyp) {
    cudaMemset(d, 0, sizeof(h));
    k<<<1, 128>>>(d, hyp, 0, c);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double err = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int kk = 0; kk < K; ++kk)
          ref += ((double)(((m * 3 + kk * 7) % 11) - 5) * 0.5) * ((double)(((n * 5 + kk * 3) % 13) - 6) * 0.25);
        err = fmax(err, fabs(h[m * N + n] - ref));
      }
    printf("H%d (%s): %s, max|D-ref| = %g\n", hyp, hyp == 1 ? "row m at lane (m%4)*32+m/4" : "row m at lane m",
           cudaGetErrorString(e), err);
  }
  for (int t = 1; t <= 2; ++t) {
    k<<<1, 128>>>(d, 2, t, c);
    cudaDeviceSynchronize();
    cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("%s M=128 N=64 K=16: %lld cycles/MMA (issue-loop, 4096 dependent MMAs)\n", t == 1 ? "ts (A in TMEM)" : "ss (A in SMEM)", hc);
  }
  return 0;
}
