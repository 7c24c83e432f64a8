#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t h2_minus1024(uint32_t u) {
  uint32_t r;
  asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(u), "r"(0xE400E400u));
  return r;
}
__global__ void k(float *o) {
  const uint32_t w = 0x44332211u, u = 0xDDCCBBAAu;
  uint32_t r[5];
  r[0] = h2_minus1024(__byte_perm(w, 0x64646464u, 0x4140u));
  r[1] = h2_minus1024(__byte_perm(w, 0x64646464u, 0x4342u));
  for (int b = 1; b <= 3; ++b) {
    const uint32_t s2 = (uint32_t)b | ((uint32_t)(b + 4) << 8);
    r[1 + b] = h2_minus1024(__byte_perm(__byte_perm(u, w, s2), 0x6464u, 0x5140u));
  }
  for (int i = 0; i < 5; ++i) {
    o[2 * i] = __half2float(__ushort_as_half((unsigned short)(r[i] & 0xFFFF)));
    o[2 * i + 1] = __half2float(__ushort_as_half((unsigned short)(r[i] >> 16)));
  }
}
int main() {
  float *d, h[10];
  cudaMalloc(&d, 40);
  k<<<1, 1>>>(d);
  cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
  printf("0x4140 on 0x44332211: %g %g (want 17 34)\n", h[0], h[1]);
  printf("0x4342 on 0x44332211: %g %g (want 51 68)\n", h[2], h[3]);
  printf("hp b=1: %g %g (want 187 34)\nhp b=2: %g %g (want 204 51)\nhp b=3: %g %g (want 221 68)\n", h[4], h[5], h[6], h[7],
         h[8], h[9]);
}
