// tools/m64_layout.cu -- where does tcgen05.mma (cta_group::1, kind::f16) put an M=64 accumulator
// in TMEM? A[m][k] = (k == 0 ? m : 0), B[n][k] = (k == 0 ? n + 1 : 0) -> D[m][n] = m * (n + 1).
// Reads 128 lanes x 32 columns and prints which (m, n) each (lane, column) holds.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_planar(uint32_t addr, uint32_t lbo) {
  uint64_t d = (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)(lbo >> 4) << 16;
  d |= (uint64_t)(128 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
constexpr int M = 64, N = 64, K = 16;
__global__ void k(float *D) {
  __shared__ __align__(1024) uint8_t sA[M * K * 2];
  __shared__ __align__(1024) uint8_t sB[N * K * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
    const int m = e / K, kk = e % K;
    __nv_bfloat16 v = __float2bfloat16_rn(kk == 0 ? (float)m : 0.0f);
    *(__nv_bfloat16 *)(sA + (kk / 8) * (M * 16) + m * 16 + (kk % 8) * 2) = v;
  }
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    const int n = e / K, kk = e % K;
    __nv_bfloat16 v = __float2bfloat16_rn(kk == 0 ? (float)(n + 1) : 0.0f);
    *(__nv_bfloat16 *)(sB + (kk / 8) * (N * 16) + n * 16 + (kk % 8) * 2) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(saddr(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  // zero the accumulator region first (so untouched lanes read 0)
  {
    uint32_t z[32] = {0};
    const uint32_t ta = tmem + ((uint32_t)((threadIdx.x / 32) * 32) << 16);
    for (int c = 0; c < 128; c += 32)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta + c),
          "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]), "r"(z[7]), "r"(z[8]),
          "r"(z[9]), "r"(z[10]), "r"(z[11]), "r"(z[12]), "r"(z[13]), "r"(z[14]), "r"(z[15]), "r"(z[16]),
          "r"(z[17]), "r"(z[18]), "r"(z[19]), "r"(z[20]), "r"(z[21]), "r"(z[22]), "r"(z[23]), "r"(z[24]),
          "r"(z[25]), "r"(z[26]), "r"(z[27]), "r"(z[28]), "r"(z[29]), "r"(z[30]), "r"(z[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
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
  const uint32_t ta = tmem + ((uint32_t)((threadIdx.x / 32) * 32) << 16);
  for (int c = 0; c < 128; c += 32) {
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
    for (int i = 0; i < 32; ++i) D[threadIdx.x * 128 + c + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}
int main() {
  float *d, h[128 * 128];
  cudaMalloc(&d, sizeof(h));
  k<<<1, 128>>>(d);
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  // decode: value v = m * (n + 1): report (m, n) for lanes 0..127, first few columns
  for (int lane = 0; lane < 128; lane += 1) {
    int nz = 0;
    for (int c = 0; c < 128; ++c) nz += h[lane * 128 + c] != 0.0f;
    if (lane % 8 == 0 || nz)
      printf("lane %3d: nonzero cols %3d; col0..3 = %g %g %g %g; col 64..65 = %g %g\n", lane, nz, h[lane * 128],
             h[lane * 128 + 1], h[lane * 128 + 2], h[lane * 128 + 3], h[lane * 128 + 64], h[lane * 128 + 65]);
  }
  return 0;
}
