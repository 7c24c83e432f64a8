// ffma_bench.cu -- fp32 FFMA issue rate on this GPU (the "alu" roofline of the
// fixed-order fmaf kernels). Variants: 3-register FFMA (both
// multiplicands in registers, like k_expand_dnn's inner loop) and immediate-form.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma_bench ffma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int REG>
__global__ void k_ffma(const float *in, float *out, int iters) {
  float a[8], b[8], c[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    a[j] = in[(threadIdx.x + j) & 63];
    b[j] = in[(threadIdx.x + j + 17) & 63];
    c[j] = in[(threadIdx.x + j + 33) & 63];
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (REG) c[j] = fmaf(a[j], b[(j + u) & 7], c[j]);
        else c[j] = fmaf(c[j], 1.0001f, 0.5f);
      }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j];
  if (s == 1234.5f) out[0] = s;
}

int main() {
  float *in, *out;
  cudaMalloc(&in, 256);
  cudaMalloc(&out, 4);
  cudaMemset(in, 0, 256);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int reg = 1; reg >= 0; --reg) {
    for (int tpb : {256, 512, 1024}) {
      const int blocks = sms * (2048 / tpb);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (reg) k_ffma<1><<<blocks, tpb>>>(in, out, iters);
        else k_ffma<0><<<blocks, tpb>>>(in, out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flop = 2.0 * 16 * 8 * (double)iters * blocks * tpb;
        if (rep) printf("%s tpb=%d blocks=%d: %.3f ms, %.1f TFLOP/s (%.1f FFMA/clk/SM at 1965 MHz)\n",
                        reg ? "3-reg FFMA" : "imm FFMA  ", tpb, blocks, ms, flop / ms / 1e9,
                        flop / 2 / (ms * 1e-3) / sms / 1.965e9);
      }
    }
  }
  return 0;
}
