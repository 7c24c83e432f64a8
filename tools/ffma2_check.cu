// tools/ffma2_check.cu -- fma.rn.f32x2 (FFMA2) vs two fmaf: bit-identical? (random operands)
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(*(const uint64_t *)&a), "l"(*(const uint64_t *)&b), "l"(*(const uint64_t *)&c));
  return *(const float2 *)&r;
}
__global__ void k(const float *x, int n, int *bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i * 6 + 5 >= n) return;
  const float *p = x + i * 6;
  float2 r = ffma2(make_float2(p[0], p[1]), make_float2(p[2], p[3]), make_float2(p[4], p[5]));
  float u = fmaf(p[0], p[2], p[4]), v = fmaf(p[1], p[3], p[5]);
  if (__float_as_uint(r.x) != __float_as_uint(u) || __float_as_uint(r.y) != __float_as_uint(v)) atomicAdd(bad, 1);
}
int main() {
  const int n = 6 << 20;
  float *h = new float[n];
  uint32_t s = 12345;
  for (int i = 0; i < n; ++i) { s = s * 1664525u + 1013904223u; h[i] = (float)((int)(s >> 8) - (1 << 23)) * 1e-5f; }
  float *d; int *b; cudaMalloc(&d, n * 4); cudaMalloc(&b, 4); cudaMemset(b, 0, 4);
  cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
  k<<<(n / 6 + 255) / 256, 256>>>(d, n, b);
  int hb = -1; cudaMemcpy(&hb, b, 4, cudaMemcpyDeviceToHost);
  printf("ffma2 vs fmaf mismatches: %d of %d pairs (%s)\n", hb, n / 6, cudaGetErrorString(cudaGetLastError()));
}
