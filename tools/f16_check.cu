// tools/f16_check.cu -- correctness microtest: tcgen05.mma kind::f16 with fp16 vs bf16
// operands (SWIZZLE_NONE K-major), and the PRMT+HADD2 byte -> fp16 conversion.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f16_check tools/f16_check.cu && ./f16_check
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

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
__device__ __forceinline__ uint32_t h2_minus1024(uint32_t u) {
  uint32_t r;
  asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(u), "r"(0xE400E400u));
  return r;
}

constexpr int M = 128, N = 32, K = 16;

// A[m][k], B[n][k] as 16-bit patterns (fp16 or bf16), planar K-major: chunk j = k/8 at j*LBO
template <bool F16>
__global__ void kmma(const uint16_t *A, const uint16_t *B, float *D, int fmt_override) {
  __shared__ __align__(1024) uint8_t sA[M * K * 2];
  __shared__ __align__(1024) uint8_t sB[N * K * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
    const int m = e / K, k = e % K;
    *(uint16_t *)(sA + (k / 8) * (M * 16) + m * 16 + (k % 8) * 2) = A[e];
  }
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    const int n = e / K, k = e % K;
    *(uint16_t *)(sB + (k / 8) * (N * 16) + n * 16 + (k % 8) * 2) = B[e];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(saddr(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t fmt = fmt_override >= 0 ? (uint32_t)fmt_override : (F16 ? 0u : 1u);
  const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (threadIdx.x == 0) {
    const uint64_t ad = desc_planar(saddr(sA), M * 16), bd = desc_planar(saddr(sB), N * 16);
    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar))
                 : "memory");
  }
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(
                   saddr(&bar))
               : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[32];
  const uint32_t taddr = tmem + ((uint32_t)((threadIdx.x / 32) * 32) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int n = 0; n < N; ++n) D[threadIdx.x * N + n] = __uint_as_float(r[n]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

__global__ void kconv(float *out) {   // all 256 bytes through PRMT(0x64) + HADD2(-1024)
  const uint32_t w = threadIdx.x * 0x01010101u;
  const uint32_t h = h2_minus1024(__byte_perm(w, 0x64646464u, 0x4140u));
  out[threadIdx.x] = __half2float(__ushort_as_half((unsigned short)(h & 0xFFFF)));
}

int main() {
  uint16_t hA16[M * K], hB16[N * K], hA[M * K], hB[N * K];
  double ref[M * N];
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < K; ++k) {
      const float v = (float)((m * 7 + k * 13) % 256);
      __half hh = __float2half_rn(v);
      __nv_bfloat16 bb = __float2bfloat16_rn(v);
      hA16[m * K + k] = *(uint16_t *)&hh;
      hA[m * K + k] = *(uint16_t *)&bb;
    }
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) {
      const float v = (float)((n * 5 + k * 3) % 9 - 4) * 0.25f;
      __half hh = __float2half_rn(v);
      __nv_bfloat16 bb = __float2bfloat16_rn(v);
      hB16[n * K + k] = *(uint16_t *)&hh;
      hB[n * K + k] = *(uint16_t *)&bb;
    }
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)((m * 7 + k * 13) % 256) * ((double)((n * 5 + k * 3) % 9 - 4) * 0.25);
      ref[m * N + n] = s;
    }
  uint16_t *dA, *dB;
  float *dD, *dC;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dD, M * N * 4);
  cudaMalloc(&dC, 256 * 4);
  float hD[M * N];
  for (int variant = 0; variant < 3; ++variant) {
    const bool f16 = variant != 1;
    cudaMemcpy(dA, f16 ? hA16 : hA, sizeof(hA), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, f16 ? hB16 : hB, sizeof(hB), cudaMemcpyHostToDevice);
    if (variant == 0) kmma<true><<<1, 128>>>(dA, dB, dD, -1);
    else if (variant == 1) kmma<false><<<1, 128>>>(dA, dB, dD, -1);
    else kmma<true><<<1, 128>>>(dA, dB, dD, 1);   // fp16 data read as bf16 (should be wrong)
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
    double maxerr = 0;
    int bad = 0;
    for (int i = 0; i < M * N; ++i) {
      const double err = fabs(hD[i] - ref[i]);
      if (err > maxerr) maxerr = err;
      if (err > 1e-3) ++bad;
    }
    printf("%s: err=%s max|D-ref| = %g, bad %d / %d; D[0..3] = %g %g %g %g ref %g %g %g %g\n",
           variant == 0 ? "fp16 data, fp16 idesc" : variant == 1 ? "bf16 data, bf16 idesc" : "fp16 data, bf16 idesc",
           cudaGetErrorString(e), maxerr, bad, M * N, hD[0], hD[1], hD[2], hD[3], ref[0], ref[1], ref[2], ref[3]);
  }
  kconv<<<1, 256>>>(dC);
  float hc[256];
  cudaMemcpy(hc, dC, sizeof(hc), cudaMemcpyDeviceToHost);
  int cbad = 0;
  for (int i = 0; i < 256; ++i) cbad += hc[i] != (float)i;
  printf("byte->fp16 conversion: %d / 256 wrong (e.g. 200 -> %g)\n", cbad, hc[200]);
  return 0;
}
