// tools/mma_shift_bench.cu -- cycles per tcgen05.mma (M=128, N=32, K=16, kind::f16, SS) for the
// shifted-window A operands of k_conv1_sib: SWIZZLE_NONE K-major "chunk-planar" A (8 fp16 per
// 16-byte row, plane stride LBO) whose start row is offset by r rows (16*r bytes) from a
// 128-byte boundary, versus SW128 A. Tells whether misaligned window starts slow the MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_shift_bench tools/mma_shift_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_none(uint32_t addr, uint32_t lbo) {
  uint64_t d = (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)(lbo >> 4) << 16;
  d |= (uint64_t)(128 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  uint64_t d = (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int N>
__global__ void kb(int iters, int mode, int shift, uint32_t lbo, int bf16, int samea, long long *out) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t *sm = sm_raw + ((1024u - (saddr(sm_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) ((uint32_t *)sm)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int wid = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0);
  if (wid == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(saddr(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t idesc = (1u << 4) | (bf16 ? (1u << 7) | (1u << 10) : 0u) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t A = saddr(sm), B = saddr(sm + 140 * 1024);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    uint64_t ad[4], bd[4];
#pragma unroll
    for (int tap = 0; tap < 4; ++tap) {   // descriptors hoisted: the loop only issues MMAs
      const int tp = samea ? 0 : tap;
      const int row = (mode == 0) ? ((tp >> 1) * 21 + (tp & 1) + shift) : (mode == 1 ? 8 * tp : 0);
      ad[tap] = mode == 2 ? desc_sw128(A + (uint32_t)tp * 16384u) : desc_none(A + (uint32_t)row * 16u, lbo);
      bd[tap] = desc_sw128(B + (uint32_t)(tp & 1) * 32u);
    }
    t0 = clock64();
    for (int i = 0; i < iters; i += 4) {
#pragma unroll
      for (int tap = 0; tap < 4; ++tap)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                         tmem + (uint32_t)(tap * N)),
                     "l"(ad[tap]), "l"(bd[tap]), "r"(idesc), "r"(i > 0 ? 1 : 0));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar)) : "memory");
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(saddr(&bar))
                 : "memory");
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (wid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

int main() {
  long long *d, h[148];
  cudaMalloc(&d, 148 * 8);
  const int iters = 8192, smem = 170 * 1024;
  cudaFuncSetAttribute(kb<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct Case { int mode, shift; uint32_t lbo; const char *what; int bf16 = 0, samea = 0; };
  const Case cases[] = {
      {2, 0, 0, "SW128 A, bf16 idesc", 1},
      {2, 0, 0, "SW128 A, bf16 idesc, same A/B every MMA", 1, 1},
      {2, 0, 0, "SW128 A, f16, same A/B every MMA", 0, 1},
      {2, 0, 0, "SW128 A (reference)"},
      {1, 0, 8576, "NOSWZ A, rows 8*tap (128B-aligned), LBO 8576"},
      {0, 0, 8576, "NOSWZ A, conv1 taps {0,1,21,22}, LBO 8576 (k_conv1_sib)"},
      {0, 0, 8192, "NOSWZ A, conv1 taps, LBO 8192"},
      {0, 0, 9216, "NOSWZ A, conv1 taps, LBO 9216"},
      {0, 0, 4096 + 128, "NOSWZ A, conv1 taps, LBO 4224"},
  };
  for (const Case &c : cases) {
    for (int grid : {1}) {
      kb<32><<<grid, 128, smem>>>(iters, c.mode, c.shift, c.lbo, c.bf16, c.samea, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
      printf("%-60s grid %3d: %6.1f cyc/MMA (%s)\n", c.what, grid, (double)h[0] / iters, cudaGetErrorString(e));
    }
  }
  return 0;
}
