// common.cuh -- shared device/host helpers of the CUDA path (NOT shared with oracle/).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <utility>

#include <string>

#include "bcts.h"

namespace bcts {

// ------------------------------------------------ programmatic dependent launch
// Trunk kernels are launched with programmatic stream serialization: a kernel may be
// scheduled while its stream predecessor drains, runs its prologue (barriers, TMEM,
// weight bulk copies -- nothing the predecessor writes), then pdl_wait()s for the
// predecessor's completion before touching its outputs. pdl_trigger() lets the next
// kernel be scheduled as this one's CTAs retire.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
inline bool pdl_enabled() { return true; }

// Per-device launch configuration (defined in bcts.cu): the SM count of the current device, and
// the dynamic-SMEM opt-in of a kernel on the current device (cudaFuncSetAttribute is per device:
// every device a handle runs on gets it; thread-safe, once per (kernel, device, size)).
int sm_count_current();
cudaError_t smem_optin(const void *kernel, int bytes);
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

constexpr int kImg = 84;
constexpr int kPix = kImg * kImg;             // 7056 packed pixel words per frame stack
constexpr int kFrameBytes = 4 * kPix;         // 28,224
constexpr int kAtariRecord = 16 + kFrameBytes;  // 28,240
constexpr int kMaxA = 64;
constexpr int kMaxDepth = 12;

// ------------------------------------------------------------------ hashing
// ENV_SPEC: splitmix64 finalizer and murmur3 fmix32.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
__host__ __device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}
// Synthetic reward from the top 3 bits of a child key: +1 if 7, -1 if 0, else 0.
__host__ __device__ __forceinline__ float atari_reward(uint64_t child_key) {
  uint32_t t = (uint32_t)(child_key >> 61);
  return t == 7u ? 1.0f : (t == 0u ? -1.0f : 0.0f);
}
__host__ __device__ __forceinline__ uint64_t atari_child_key(uint64_t key, int a) {
  return mix64(key ^ (0x9E3779B97F4A7C15ull * (uint64_t)(a + 1)));
}

// ------------------------------------------------------------ packed keys
// (value, lowest leaf index) -> int64 that orders correctly under SIGNED max.
// -0.0 is canonicalised to +0.0 first (R4).
__host__ __device__ __forceinline__ uint32_t float_orderable(float v) {
  uint32_t u;
#ifdef __CUDA_ARCH__
  u = __float_as_uint(v == 0.0f ? 0.0f : v);
#else
  float w = (v == 0.0f) ? 0.0f : v;
  memcpy(&u, &w, 4);
#endif
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ __forceinline__ float orderable_float(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  memcpy(&f, &u, 4);
  return f;
#endif
}
__host__ __device__ __forceinline__ int64_t pack_key(float v, int64_t leaf) {
  uint64_t hi = (uint64_t)(float_orderable(v) ^ 0x80000000u);
  uint64_t lo = 0xFFFFFFFFull - (uint64_t)(uint32_t)leaf;
  return (int64_t)((hi << 32) | lo);
}
__host__ __device__ __forceinline__ float key_value(int64_t k) {
  return orderable_float((uint32_t)((uint64_t)k >> 32) ^ 0x80000000u);
}
__host__ __device__ __forceinline__ int64_t key_leaf(int64_t k) {
  return (int64_t)(0xFFFFFFFFull - ((uint64_t)k & 0xFFFFFFFFull));
}
constexpr int64_t kKeyEmpty = INT64_MIN;

// --------------------------------------------------------------- node views
// A level of the tree as device arrays. For level 0 the view points into the
// caller's root records (strided); deeper levels are contiguous SoA.
struct NodeView {
  const uint8_t *state = nullptr;  // ids (int32) / words (u32[16]) / frames (u32[7056])
  int64_t state_stride = 0;        // bytes between consecutive nodes' states
  const uint64_t *key = nullptr;   // ATARI only
  int64_t key_stride = 0;          // bytes
  const float *cum = nullptr;      // nullable: cumulative reward 0
};

struct NodeOut {
  uint8_t *state = nullptr;
  int64_t state_stride = 0;
  uint64_t *key = nullptr;
  float *cum = nullptr;
};

}  // namespace bcts
