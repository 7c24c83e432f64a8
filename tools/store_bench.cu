// tools/store_bench.cu -- cost of the conv1 epilogue's output paths on B200: 8 warps per CTA, one
// CTA per SM, each warp storing 4 KB per "image" as 16-byte lanes in several address patterns,
// vs staging through SMEM + bulk store. Prints cycles per image per CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_bench tools/store_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// mode 0: lane stride 128 B (32 lines / instruction)   mode 1: lane stride 32 B (8 lines)
// mode 2: contiguous 512 B per instruction (4 lines)    mode 3: STS to staging + bulk store
__global__ void __launch_bounds__(256, 1) kst(uint8_t *out, int n_img, int mode, int l2only, long long *cyc) {
  extern __shared__ __align__(128) uint8_t stage[];
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  long long t0 = clock64();
  for (int img = 0; img < n_img; ++img) {
    uint8_t *o = out + ((size_t)blockIdx.x * (l2only ? 1 : n_img) + (l2only ? 0 : img)) * 32768;
    const uint4 v = make_uint4(img, l, w, 7);
    if (mode == 3) {
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {   // 8 x 16 B per lane = 4 KB per warp, 32 KB per CTA
      uint32_t off;
      if (mode == 0) off = (uint32_t)(w * 4096 + ((i * 32 + l) % 32) * 128 + (i * 16) % 128);
      else if (mode == 1) off = (uint32_t)(w * 4096 + (i >> 2) * 1024 + l * 32 + (i & 1) * 16 + ((i >> 1) & 1) * 2048 * 0);
      else off = (uint32_t)(w * 4096 + i * 512 + l * 16);
      if (mode == 1) off = (uint32_t)(w * 4096 + (i >> 1) * 1024 + l * 32 + (i & 1) * 16);
      if (mode == 3) *(uint4 *)(stage + off % 32768) = v;
      else *(uint4 *)(o + off) = v;
    }
    if (mode == 3) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(o), "r"(saddr(stage)), "r"(32768)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  const int n_img = 256, grid = 148;
  uint8_t *out;
  long long *cyc, h[148];
  cudaMalloc(&out, (size_t)grid * n_img * 32768);
  cudaMalloc(&cyc, grid * 8);
  cudaFuncSetAttribute(kst, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  const char *names[] = {"lane stride 128 B (32 lines/instr)", "lane stride 32 B (8 lines/instr)",
                         "contiguous 512 B/instr (4 lines)", "STS staging + bulk store"};
  for (int l2 = 0; l2 < 2; ++l2)
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 4; ++mode) {
      kst<<<grid, 256, 32768>>>(out, n_img, mode, l2, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
      double m = 0;
      for (int i = 0; i < grid; ++i) m += h[i];
      m /= grid;
      if (rep) printf("%s %-40s: %7.0f cycles per 32 KB image per CTA (%.1f B/clk/SM) %s\n", l2 ? "L2-resident" : "HBM stream ", names[mode], m / n_img,
                      32768.0 * n_img / m, cudaGetErrorString(e));
    }
  return 0;
}
