// tools/mma_bench.cu -- microbenchmark of tcgen05.mma issue/throughput on B200.
// Measures cycles per MMA (M=128, K=16, bf16, SS) for N in {32,64,128,256},
// for 1..8 independent TMEM accumulators (round-robin), SW128 vs SWIZZLE_NONE
// A operand, and warp-uniform vs lane-0 issue.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench tools/mma_bench.cu && ./mma_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, int sw) {
  uint64_t d = (uint64_t)((addr & 0x3FFFFu) >> 4);
  if (sw) {
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)2 << 61;
  } else {
    d |= (uint64_t)(4096 >> 4) << 16;  // LBO: K chunk stride
    d |= (uint64_t)(128 >> 4) << 32;   // SBO
  }
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t *b, uint32_t par) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(saddr(b)), "r"(par) : "memory");
}

template <int N>
__global__ void kbench(int iters, int nacc, int sw, int uniform, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t *A = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint8_t *B = A + 32768;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t *)A)[i] = 0x3f803f80u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x < 32) {
    const uint32_t a0 = saddr(A), b0 = saddr(B);
    if (uniform) {
      t0 = clock64();
      for (int i = 0; i < iters; ++i) {
        const uint32_t d = tmem + (uint32_t)((i % nacc) * N);
        const uint64_t ad = desc(a0 + (uint32_t)((i & 3) * 32), sw), bd = desc(b0 + (uint32_t)((i & 3) * 32), 1);
        uint32_t pred;
        asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(pred));
        if (pred) mma(d, ad, bd, idesc, i >= nacc);
        __syncwarp();
      }
      if (threadIdx.x == 0) commit(&bar);
      __syncwarp();
      wait(&bar, 0);
      t1 = clock64();
    } else if (threadIdx.x == 0) {
      t0 = clock64();
      for (int i = 0; i < iters; ++i) {
        const uint32_t d = tmem + (uint32_t)((i % nacc) * N);
        mma(d, desc(a0 + (uint32_t)((i & 3) * 32), sw), desc(b0 + (uint32_t)((i & 3) * 32), 1), idesc, i >= nacc);
      }
      commit(&bar);
      wait(&bar, 0);
      t1 = clock64();
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

__device__ __forceinline__ void mma_pred(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc,
                                         uint32_t issue) {
  asm volatile("{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nsetp.ne.b32 q, %5, 0;\n"
               "@q tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(issue));
}

// V: 0 = lane-0 unrolled-by-4 with constant descriptor increments;
//    1 = warp-uniform loop (warp id via shfl), elected lane computed once,
//        predicated tcgen05.mma (no branch), uniform descriptor arithmetic.
template <int N, int NACC, int V>
__global__ void kbench2(int iters, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t *A = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint8_t *B = A + 32768;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t *)A)[i] = 0x3f803f80u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int wid = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0);
  if (wid == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = 0, t1 = 0;
  const uint64_t ad0 = desc(saddr(A), 1), bd0 = desc(saddr(B), 1);
  if (wid == 0) {
    uint32_t elected = 0;
    asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(elected));
    if (V == 0) {
      if (threadIdx.x == 0) {
        t0 = clock64();
        for (int i = 0; i < iters; i += 4 * NACC) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int a = 0; a < NACC; ++a) mma(tmem + a * N, ad0 + 2 * j, bd0 + 2 * j, idesc, i > 0 || j > 0);
        }
        commit(&bar);
        wait(&bar, 0);
        t1 = clock64();
      }
    } else {
      t0 = clock64();
      for (int i = 0; i < iters; i += 4 * NACC) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int a = 0; a < NACC; ++a) mma_pred(tmem + a * N, ad0 + 2 * j, bd0 + 2 * j, idesc, i > 0 || j > 0, elected);
      }
      if (elected) commit(&bar);
      __syncwarp();
      wait(&bar, 0);
      t1 = clock64();
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  __syncthreads();
  if (wid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int N, int NACC, int V>
void run2(long long *d, int grid) {
  const int iters = 4096;
  cudaFuncSetAttribute(kbench2<N, NACC, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  kbench2<N, NACC, V><<<grid, 128, 70000>>>(iters, d);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double cyc = (double)c / iters;
  const double tf = 2.0 * 128 * N * 16 / cyc * 1.965e9 * 148 / 1e12;
  printf("V%d N=%3d nacc=%d grid=%3d : %7.1f cyc/MMA (~%6.0f TFLOP/s chip @1.965GHz)\n", V, N, NACC, grid, cyc, tf);
}

template <int N>
void run(long long *d, int grid) {
  const int iters = 4096;
  cudaFuncSetAttribute(kbench<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int uni = 0; uni < 2; ++uni)
    for (int sw = 1; sw >= 0; --sw)
      for (int nacc : {1, 2, 4, 8}) {
        if (nacc * N > 512) continue;
        kbench<N><<<grid, 128, 70000>>>(iters, nacc, sw, uni, d);
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        const double cyc = (double)c / iters;
        const double tf = 2.0 * 128 * N * 16 / cyc * 1.965e9 * 148 / 1e12;
        printf("N=%3d grid=%3d %s %-8s nacc=%d : %7.1f cyc/MMA  (~%6.0f TFLOP/s chip @1.965GHz)\n", N, grid,
               uni ? "warp-uniform" : "lane0-only  ", sw ? "SW128" : "NOSWZ", nacc, cyc, tf);
      }
}

int main() {
  long long *d;
  cudaMalloc(&d, 8);
  for (int grid : {1, 148}) {
    run2<32, 1, 0>(d, grid); run2<32, 4, 0>(d, grid); run2<32, 1, 1>(d, grid); run2<32, 4, 1>(d, grid);
    run2<64, 1, 0>(d, grid); run2<64, 4, 0>(d, grid); run2<64, 1, 1>(d, grid); run2<64, 4, 1>(d, grid);
    run2<128, 1, 0>(d, grid); run2<128, 2, 1>(d, grid);
    run2<256, 1, 0>(d, grid); run2<256, 1, 1>(d, grid);
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
