// tools/expand_bench.cu -- store-pattern study for the ATARI_HASH level expansion (k_expand_atari):
// the same child frames (frames 1..3 shifted down, newest = old newest ^ noise) written with
//   v0: each thread owns one 8-pixel group = two 16-B stores 16 B apart (lane stride 32 B)
//   v1: each thread owns one 16-B chunk (a warp stores 512 contiguous bytes per instruction);
//       the group hash is recomputed by both threads of a group
//   v2: v1's arithmetic into an SMEM staging buffer, written by one bulk (TMA) store per child,
//       double buffered
// at the C5 level-3 shape (324 parents x 18) and the C3 level-2 shape (1152 x 18), for several
// children-per-CTA splits. Prints GB/s of algorithmic bytes (children written + parents read).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/expand_bench tools/expand_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kPix = 7056, kFrame = 4 * kPix, kGroups = kPix / 8, kChunks = kFrame / 16;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra WAIT_%=;\n}\n" ::"r"(
          saddr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint4 step4(uint4 v, uint32_t nz) {
  v.x = (v.x >> 8) | ((v.x ^ (nz << 24)) & 0xFF000000u);
  v.y = (v.y >> 8) | ((v.y ^ ((nz >> 8) << 24)) & 0xFF000000u);
  v.z = (v.z >> 8) | ((v.z ^ ((nz >> 16) << 24)) & 0xFF000000u);
  v.w = (v.w >> 8) | ((v.w ^ (nz & 0xFF000000u)) & 0xFF000000u);
  return v;
}

template <int V, int T>
__global__ void __launch_bounds__(T) kexp(const uint8_t *par, const uint64_t *pkey, int A, int split, uint8_t *out,
                                          uint64_t *okey) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint4 *sframe = (uint4 *)sm;
  __shared__ __align__(8) uint64_t bar;
  const int p = blockIdx.x / split;
  const int per = (A + split - 1) / split, a_lo = (blockIdx.x % split) * per;
  const int a_hi = min(A, a_lo + per);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&bar)), "r"(kFrame) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     saddr(sframe)),
                 "l"(par + (size_t)p * kFrame), "r"(kFrame), "r"(saddr(&bar))
                 : "memory");
  }
  const uint64_t key = pkey[p];
  __syncthreads();
  mbar_wait(&bar, 0);
  for (int a = a_lo; a < a_hi; ++a) {
    const uint64_t k2 = mix64(key ^ (0x9E3779B97F4A7C15ull * (uint64_t)(a + 1)));
    const size_t ci = (size_t)p * A + a;
    uint4 *dst = (uint4 *)(out + ci * kFrame);
    if (V == 0) {
      for (int g = threadIdx.x; g < kGroups; g += T) {
        const uint64_t h = mix64(k2 + (uint64_t)g);
        dst[2 * g] = step4(sframe[2 * g], (uint32_t)h);
        dst[2 * g + 1] = step4(sframe[2 * g + 1], (uint32_t)(h >> 32));
      }
    } else if (V == 1) {
#pragma unroll 4
      for (int j = threadIdx.x; j < kChunks; j += T) {
        const uint64_t h = mix64(k2 + (uint64_t)(j >> 1));
        dst[j] = step4(sframe[j], (uint32_t)(h >> (32 * (j & 1))));
      }
    } else {
      uint4 *stg = sframe + kChunks + ((a - a_lo) & 1) * kChunks;
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncthreads();
#pragma unroll 4
      for (int j = threadIdx.x; j < kChunks; j += T) {
        const uint64_t h = mix64(k2 + (uint64_t)(j >> 1));
        stg[j] = step4(sframe[j], (uint32_t)(h >> (32 * (j & 1))));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(saddr(stg)),
                     "r"(kFrame)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (threadIdx.x == 0) okey[ci] = k2;
  }
  if (V == 2 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int V, int T>
float run(const uint8_t *par, const uint64_t *pk, int np, int A, int split, uint8_t *out, uint64_t *ok, uint8_t *flush,
          size_t flush_bytes) {
  const int smem = kFrame * (V == 2 ? 3 : 1);
  cudaFuncSetAttribute(kexp<V, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f, tot = 0;
  const int reps = 10;
  for (int r = 0; r < reps + 2; ++r) {
    cudaMemsetAsync(flush, r, flush_bytes);
    cudaEventRecord(e0);
    kexp<V, T><<<np * split, T, smem>>>(par, pk, A, split, out, ok);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 2) {
      tot += ms;
      best = ms < best ? ms : best;
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return tot / reps;
}

int main() {
  const int A = 18;
  const int shapes[2] = {324, 1152};
  uint8_t *par, *out, *flush;
  uint64_t *pk, *ok;
  const size_t flush_bytes = 256u << 20;
  cudaMalloc(&par, (size_t)1152 * kFrame);
  cudaMalloc(&pk, 1152 * 8);
  cudaMalloc(&out, (size_t)1152 * A * kFrame);
  cudaMalloc(&ok, (size_t)1152 * A * 8);
  cudaMalloc(&flush, flush_bytes);
  cudaMemset(par, 0x5a, (size_t)1152 * kFrame);
  cudaMemset(pk, 0x33, 1152 * 8);
  // reference output of v0 for the equality check
  uint8_t *ref;
  cudaMalloc(&ref, (size_t)1152 * A * kFrame);
  for (int s = 0; s < 2; ++s) {
    const int np = shapes[s];
    const double bytes = (double)np * (A + 1) * (kFrame + 12);
    printf("shape: %d parents x %d children (%.1f MB algorithmic)\n", np, A, bytes / 1e6);
    run<0, 256>(par, pk, np, A, 2, ref, ok, flush, flush_bytes);
    for (int split : {1, 2, 3, 6, 9, 18}) {
      float t[5];
      t[0] = run<0, 256>(par, pk, np, A, split, out, ok, flush, flush_bytes);
      t[1] = run<1, 256>(par, pk, np, A, split, out, ok, flush, flush_bytes);
      t[2] = run<1, 512>(par, pk, np, A, split, out, ok, flush, flush_bytes);
      t[3] = run<2, 256>(par, pk, np, A, split, out, ok, flush, flush_bytes);
      t[4] = run<2, 512>(par, pk, np, A, split, out, ok, flush, flush_bytes);
      // equality of the last variant's output with v0's
      cudaDeviceSynchronize();
      static uint8_t h0[64], h1[64];
      size_t off = (size_t)(np * A - 1) * kFrame + 1000;
      cudaMemcpy(h0, ref + off, 64, cudaMemcpyDeviceToHost);
      cudaMemcpy(h1, out + off, 64, cudaMemcpyDeviceToHost);
      int same = 1;
      for (int i = 0; i < 64; ++i) same &= h0[i] == h1[i];
      printf("  split %2d (%5d CTAs): v0/256 %7.1f  v1/256 %7.1f  v1/512 %7.1f  v2/256 %7.1f  v2/512 %7.1f GB/s  %s\n",
             split, np * split, bytes / t[0] / 1e6, bytes / t[1] / 1e6, bytes / t[2] / 1e6, bytes / t[3] / 1e6,
             bytes / t[4] / 1e6, same ? "" : "MISMATCH");
    }
  }
  return 0;
}
