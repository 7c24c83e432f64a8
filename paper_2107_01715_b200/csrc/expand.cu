// expand.cu -- K1: fused level expansion (replicate x A + env step + reward
// accumulation), Alg. 1 loop body:
//   S <- S x A, R <- R x A;  r, S' = G([S, A]);  R <- R + gamma^k r.
// Tree indices stay implicit, base A: child c of level k+1 has parent c / A
// and action c % A (R1). No pointers are stored.
#include <algorithm>

#include "engine.h"
#include "ptx.cuh"

namespace bcts {

// ------------------------------------------------------------ PTX helpers (the rest: ptx.cuh)
__device__ __forceinline__ void st_v4(uint4 *p, const uint4 &v) {
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// ---------------------------------------------------------------- TABULAR
__global__ void k_expand_tabular(NodeView par, int64_t p_first, int64_t c_begin, int64_t n_child, int A, float gk,
                                 const int32_t *__restrict__ tnext, const float *__restrict__ trew, NodeOut out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_child) return;
  int64_t c = c_begin + i, p = c / A;
  int a = (int)(c - p * A);
  int64_t pl = p - p_first;
  int32_t s = *(const int32_t *)(par.state + pl * par.state_stride);
  float R = par.cum ? par.cum[pl] : 0.0f;
  ((int32_t *)out.state)[i] = tnext[(int64_t)s * A + a];
  out.cum[i] = fmaf(gk, trew[(int64_t)s * A + a], R);
}

// --------------------------------------------------------------- INT_HASH
// s'[w] = fmix32(s[w] ^ rotl32(s[(w+1)&15], 13) ^ 0x9E3779B9*(a+1) ^ 0x85EBCA6B*w);
// r from the top two bits of s'[0]: +1 if 3, -1 if 0, else 0.
__global__ void k_expand_int(NodeView par, int64_t p_first, int64_t c_begin, int64_t n_child, int A, float gk,
                             NodeOut out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_child) return;
  int64_t c = c_begin + i, p = c / A;
  int a = (int)(c - p * A);
  int64_t pl = p - p_first;
  const uint4 *src = (const uint4 *)(par.state + pl * par.state_stride);
  uint32_t s[16], o[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 v = __ldg(src + q);
    s[4 * q] = v.x; s[4 * q + 1] = v.y; s[4 * q + 2] = v.z; s[4 * q + 3] = v.w;
  }
  const uint32_t ka = 0x9E3779B9u * (uint32_t)(a + 1);
#pragma unroll
  for (int w = 0; w < 16; ++w) o[w] = fmix32(s[w] ^ __funnelshift_l(s[(w + 1) & 15], s[(w + 1) & 15], 13) ^ ka ^
                                             (0x85EBCA6Bu * (uint32_t)w));
  uint4 *dst = (uint4 *)(out.state + i * out.state_stride);
#pragma unroll
  for (int q = 0; q < 4; ++q) dst[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
  uint32_t t = o[0] >> 30;
  float r = t == 3u ? 1.0f : (t == 0u ? -1.0f : 0.0f);
  float R = par.cum ? par.cum[pl] : 0.0f;
  out.cum[i] = fmaf(gk, r, R);
}

// ------------------------------------------------------------- ATARI_HASH
// One CTA per parent: the parent's 28,224-byte frame stack is staged in shared
// memory by one bulk copy (TMA engine), then the CTA writes its A children with
// coalesced 128-bit stores. Per child: k' = mix64(key ^ C*(a+1)); for the 8
// pixels of group g, h = mix64(k' + g) supplies one noise byte each;
// w' = (w >> 8) | ((w ^ (byte << 24)) & 0xFF000000)  (frames 1..3 shift down,
// the new newest frame is the old newest XOR noise; frame stack P:355).
constexpr int kExpandThreads = 256;
constexpr int kGroups = kPix / 8;  // 882 groups of 8 pixel words (32 B)

// split: CTAs per parent (each takes a contiguous slice of the parent's A children), so a
// small level still spreads over every SM and no SM drains a long tail of whole parents.
__global__ void __launch_bounds__(kExpandThreads) k_expand_atari(NodeView par, int64_t p_first, int64_t c_begin,
                                                                   int64_t c_end, int A, float gk, NodeOut out,
                                                                   int split) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint4 *sframe = (uint4 *)smem_raw;  // 1764 x 16 B
  __shared__ __align__(8) uint64_t bar;
  const unsigned us = (unsigned)split;
  const int64_t p = c_begin / A + (int64_t)(blockIdx.x / us);
  const int per = (A + split - 1) / split, s0 = (int)(blockIdx.x % us) * per;
  const int64_t cfirst = p * (int64_t)A;                               // child index of action 0
  const int64_t lo64 = c_begin > cfirst ? c_begin - cfirst : 0;        // this level call's children
  const int64_t hi64 = c_end < cfirst + A ? c_end - cfirst : (int64_t)A;
  const int a_lo = (int)(lo64 > (int64_t)s0 ? lo64 : (int64_t)s0);
  const int a_hi = (int)(hi64 < (int64_t)(s0 + per) ? hi64 : (int64_t)(s0 + per));
  if (a_lo >= a_hi) return;
  const int64_t pl = p - p_first;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&bar, kFrameBytes);
    bulk_g2s(saddr(sframe), par.state + pl * par.state_stride, kFrameBytes, &bar);   // one UBLKCP
  }
  const uint64_t key = *(const uint64_t *)((const uint8_t *)par.key + pl * par.key_stride);
  const float R = par.cum ? par.cum[pl] : 0.0f;
  __syncthreads();          // mbarrier init visible before anyone waits on it
  mbar_wait_spin(&bar, 0);
  for (int a = a_lo; a < a_hi; ++a) {
    const uint64_t k2 = atari_child_key(key, a);
    const int64_t ci = p * A + a - c_begin;
    uint4 *dst = (uint4 *)(out.state + ci * out.state_stride);
    // one 16-byte chunk (4 pixel words) per thread: a warp stores 512 contiguous bytes per
    // instruction (tools/expand_bench.cu: 1.7x the bandwidth of two stores 16 B apart); both
    // threads of an 8-pixel group hash it and each keeps its half of the 8 noise bytes
#pragma unroll 4
    for (int j = threadIdx.x; j < 2 * kGroups; j += kExpandThreads) {
      const uint32_t nz = (uint32_t)(mix64(k2 + (uint64_t)(j >> 1)) >> (32 * (j & 1)));
      uint4 v = sframe[j];
      v.x = (v.x >> 8) | ((v.x ^ (nz << 24)) & 0xFF000000u);
      v.y = (v.y >> 8) | ((v.y ^ ((nz >> 8) << 24)) & 0xFF000000u);
      v.z = (v.z >> 8) | ((v.z ^ ((nz >> 16) << 24)) & 0xFF000000u);
      v.w = (v.w >> 8) | ((v.w ^ (nz & 0xFF000000u)) & 0xFF000000u);
      st_v4(dst + j, v);
    }
    if (threadIdx.x == 0) {
      out.key[ci] = k2;
      out.cum[ci] = fmaf(gk, atari_reward(k2), R);
    }
  }
}

void launch_expand(int env, const NodeView &par, int64_t p_first, int64_t c_begin, int64_t c_end, int A, float gk,
                   const EnvModel &em, const NodeOut &out, cudaStream_t st, Profiler *prof) {
  const int64_t n = c_end - c_begin;
  if (n <= 0) return;
  const int64_t nparents = (c_end - 1) / A - c_begin / A + 1;
  if (env == BCTS_ENV_DNN) {
    if (em.dnn_tc) launch_expand_dnn_tc(par, p_first, c_begin, c_end, A, gk, em.dnn_tc, em.dnn_tc_bias, out, st, prof);
    else launch_expand_dnn(par, p_first, c_begin, c_end, A, gk, em.dnn, out, st, prof);
    return;
  }
  // algorithmic bytes: every child node written once + every parent node read once
  const double nb = env == BCTS_ENV_TABULAR ? 8.0 : env == BCTS_ENV_INT_HASH ? 68.0 : (double)kFrameBytes + 12.0;
  if (prof) prof->begin(env == BCTS_ENV_TABULAR ? KC_EXPAND_TAB : env == BCTS_ENV_INT_HASH ? KC_EXPAND_INT
                                                                                             : KC_EXPAND_ATARI,
                        nb * (double)(n + nparents), st);
  if (env == BCTS_ENV_TABULAR) {
    k_expand_tabular<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(par, p_first, c_begin, n, A, gk, em.tab_next,
                                                                   em.tab_rew, out);
  } else if (env == BCTS_ENV_INT_HASH) {
    k_expand_int<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(par, p_first, c_begin, n, A, gk, out);
  } else {
    smem_optin((const void *)k_expand_atari, kFrameBytes);
    // about 6 CTAs per SM (8 fit by SMEM) and at most ~6 children per CTA (measured best at the
    // C5 level-3 and C3 level-2 shapes, tools/expand_bench.cu)
    const int64_t want = std::max<int64_t>((6 * 148 + nparents - 1) / nparents, (A + 5) / 6);
    int split = (int)std::max<int64_t>(1, std::min<int64_t>(A, want));
    k_expand_atari<<<(unsigned)(nparents * split), kExpandThreads, kFrameBytes, st>>>(par, p_first, c_begin, c_end, A, gk,
                                                                             out, split);
  }
  if (prof) prof->end(st);
}

}  // namespace bcts

// ================================================================ s2d frames
// Space-to-depth(4) bf16 layout of a frame stack for the conv1 tensor-core
// layer: S[Y][X][c'] with Y, X in [0, 21) and c' = (dy*4 + dx)*4 + c holds
// frame byte c of pixel (4Y+dy, 4X+dx). conv1 (8x8, stride 4, 4 channels)
// becomes a 2x2 stride-1 conv over 64 channels whose im2col the TMA engine
// gathers (qnet_tma.cu). The 16 bytes of one (Y, X, dy) row segment are
// contiguous in the NHWC frame, so each segment converts with one 16-byte
// load. u8 -> bf16 is exact: f = as_float(0x4B0000bb) - 2^23 (PRMT + FADD).
namespace bcts {

constexpr int kS2dPix = 21 * 21;              // 441 s2d pixels
constexpr int kS2dElems = kS2dPix * 64;       // 28,224 bf16 per image

__device__ __forceinline__ uint32_t u8pair_to_bf16x2(uint32_t w, uint32_t i) {
  const float f0 = __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7540u + i)) - 8388608.0f;
  const float f1 = __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7540u + i + 1)) - 8388608.0f;
  return __byte_perm(__float_as_uint(f0), __float_as_uint(f1), 0x7632u);
}
__device__ __forceinline__ void u8x16_to_bf16(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint4 &lo,
                                              uint4 &hi) {
  lo = make_uint4(u8pair_to_bf16x2(w0, 0), u8pair_to_bf16x2(w0, 2), u8pair_to_bf16x2(w1, 0), u8pair_to_bf16x2(w1, 2));
  hi = make_uint4(u8pair_to_bf16x2(w2, 0), u8pair_to_bf16x2(w2, 2), u8pair_to_bf16x2(w3, 0), u8pair_to_bf16x2(w3, 2));
}

// images [first, first + n) of view v -> s2d (one task per (image, s2d pixel, dy))
__device__ __forceinline__ void s2d_store(void *out, uint32_t planar, int layout, int64_t img, int pix, int dy,
                                          const uint4 &lo, const uint4 &hi) {
  if (planar) {   // trunk layout: channels dy*16 .. dy*16+15 = chunks 2dy, 2dy+1 of row pix
    uint8_t *base = (uint8_t *)out + img * (int64_t)(8 * planar);
    *(uint4 *)(base + act_off(layout, planar, pix, 2 * dy)) = lo;
    *(uint4 *)(base + act_off(layout, planar, pix, 2 * dy + 1)) = hi;
  } else {
    uint4 *dst = (uint4 *)((__nv_bfloat16 *)out + img * kS2dElems + pix * 64 + dy * 16);
    dst[0] = lo;
    dst[1] = hi;
  }
}

__global__ void k_s2d_convert(NodeView v, int64_t first, int64_t n, void *__restrict__ out, uint32_t planar,
                              int layout) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * kS2dPix * 4) return;
  const int64_t img = t / (kS2dPix * 4);
  const int rem = (int)(t - img * (kS2dPix * 4));
  const int pix = rem >> 2, dy = rem & 3;
  const int Y = pix / 21, X = pix - Y * 21;
  const uint4 w = __ldg((const uint4 *)(v.state + (first + img) * v.state_stride) + ((4 * Y + dy) * 84 + 4 * X) / 4);
  uint4 lo, hi;
  u8x16_to_bf16(w.x, w.y, w.z, w.w, lo, hi);
  s2d_store(out, planar, layout, img, pix, dy, lo, hi);
}

void launch_s2d_convert(const NodeView &v, int64_t first, int64_t n, void *out, uint32_t planar, cudaStream_t st,
                        int layout) {
  const int64_t tasks = n * kS2dPix * 4;
  if (tasks > 0) k_s2d_convert<<<(unsigned)((tasks + 255) / 256), 256, 0, st>>>(v, first, n, out, planar, layout);
}

// Fused last-level expansion (Alg. 1 loop body at i_d = d-1) that
// writes each child's frame stack directly as the conv1 input (s2d bf16) plus
// its R_d: the leaf level is never materialised as uint8 frames in HBM. One
// task per (child, s2d pixel, dy): the 16 parent bytes come straight from L2
// (siblings share the parent, which stays cached), one mix64 supplies the 4
// noise bytes, and the child's 16 bytes convert to 16 bf16.
__global__ void k_expand_s2d(NodeView par, int64_t p_first, int64_t c_begin, int64_t n, int A, float gk,
                             void *__restrict__ out, uint32_t planar, float *__restrict__ cum_out, int layout) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * kS2dPix * 4) return;
  const int64_t ci = t / (kS2dPix * 4);
  const int rem = (int)(t - ci * (kS2dPix * 4));
  const int pix = rem >> 2, dy = rem & 3;
  const int64_t c = c_begin + ci, p = c / A;
  const int a = (int)(c - p * A);
  const int64_t pl = p - p_first;
  const uint64_t k2 = atari_child_key(*(const uint64_t *)((const uint8_t *)par.key + pl * par.key_stride), a);
  const int Y = pix / 21, X = pix - Y * 21;
  const int p0 = (4 * Y + dy) * 84 + 4 * X;                // first of 4 pixels, p0 % 4 == 0
  const uint4 x = __ldg((const uint4 *)(par.state + pl * par.state_stride) + (p0 >> 2));
  const uint32_t nz = (uint32_t)(mix64(k2 + (uint64_t)(p0 >> 3)) >> (8 * (p0 & 7)));
  const uint32_t w0 = (x.x >> 8) | ((x.x ^ (nz << 24)) & 0xFF000000u);
  const uint32_t w1 = (x.y >> 8) | ((x.y ^ ((nz >> 8) << 24)) & 0xFF000000u);
  const uint32_t w2 = (x.z >> 8) | ((x.z ^ ((nz >> 16) << 24)) & 0xFF000000u);
  const uint32_t w3 = (x.w >> 8) | ((x.w ^ (nz & 0xFF000000u)) & 0xFF000000u);
  uint4 lo, hi;
  u8x16_to_bf16(w0, w1, w2, w3, lo, hi);
  s2d_store(out, planar, layout, ci, pix, dy, lo, hi);
  if (rem == 0) cum_out[ci] = fmaf(gk, atari_reward(k2), par.cum ? par.cum[pl] : 0.0f);
}

void launch_expand_s2d(const NodeView &par, int64_t p_first, int64_t c_begin, int64_t c_end, int A, float gk,
                       void *out, uint32_t planar, float *cum_out, cudaStream_t st, Profiler *prof, int layout) {
  const int64_t n = c_end - c_begin;
  if (n <= 0) return;
  const int64_t nparents = (c_end - 1) / A - c_begin / A + 1;
  // algorithmic bytes: parent frames read once + children written (s2d bf16 + R)
  if (prof) prof->begin(KC_EXPAND_ATARI, (double)nparents * (kFrameBytes + 12) + (double)n * (2.0 * kS2dElems + 4), st);
  const int64_t tasks = n * kS2dPix * 4;
  k_expand_s2d<<<(unsigned)((tasks + 255) / 256), 256, 0, st>>>(par, p_first, c_begin, n, A, gk, out, planar, cum_out,
                                                                 layout);
  if (prof) prof->end(st);
}

}  // namespace bcts
