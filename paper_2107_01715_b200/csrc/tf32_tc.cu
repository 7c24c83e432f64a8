// tf32_tc.cu -- NEXT-1 on the tensor cores (opt-in, BCTS_F_TF32): the random-DNN forward model
// (level expansion, Alg. 1 P:318-321 with the learned model of P:340-341, R27) and the
// MLP2 leaf net as tcgen05 kind::tf32 GEMMs with TMEM-resident activations.
//
// The default fp32 kernels (ffma_tiles.cu) reproduce the oracle's fmaf chains bit for bit; this
// path trades that for the tensor pipe: operands are rounded to tf32 (10-bit mantissa, round to
// nearest, ties away) and accumulated in fp32 in the MMA's own order, so results are compared with
// the fp64 oracle within the tolerance derived in DESIGN.md R34.
//
// Both kernels keep a 128-node tile's activations in TMEM as the A operand of the next layer:
//   D (fp32, lanes = nodes, columns = units) --tcgen05.ld--> bias / ReLU / tf32 rounding in
//   registers --tcgen05.st--> A columns (lanes = nodes, columns = inputs)
// so no activation touches shared or global memory between layers. The weights of every layer
// are resident in SMEM (one bulk copy per CTA) as K-major SWIZZLE_NONE tf32 images:
//   byte(n, k) = (k / 4) * (Npad * 16) + n * 16 + (k % 4) * 4
// (8-row x 16-byte core matrices; LBO = one 4-wide K chunk = Npad * 16 B, SBO = 128 B); an MMA
// (K = 8) reads two chunks.
#include <algorithm>
#include <type_traits>
#include <vector>

#include <cooperative_groups.h>

#include "engine.h"
#include "ptx.cuh"

namespace cg = cooperative_groups;

namespace bcts {
namespace {

constexpr int kTcThreadsDnn = 640;   // warp 0 MMA issuer; warps 4-11 / 12-19: epilogue of tile slot 0 / 1
constexpr int kTcThreadsMlp = 384;   // warp 0 MMA issuer; warps 4-11: epilogue (lane quarter x column half)
constexpr int kTcK = 104;            // DNN state width 100 padded to a multiple of 8 (tf32 MMA K)
constexpr int kTcN = 112;            // DNN layer outputs (100, or 101 for the last) padded to 16
constexpr uint32_t kTcPlane = kTcN * 16;                       // one 4-wide K chunk of a DNN layer
constexpr uint32_t kTcLayerBytes = (kTcK / 4) * kTcPlane;      // 46,592 B per DNN layer image
constexpr int kTcDnnFloats = (int)(4 * kTcLayerBytes / 4) + 4 * kTcN;   // 4 layers + biases [4][112]
static_assert(kDnnTcBiasOffset == 4 * kTcLayerBytes / 4 && kTcN == 112, "engine.h's bias offset");

// K-major SWIZZLE_NONE descriptor: LBO = K-chunk stride, SBO = 8-row-group stride (128 B).
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t addr, uint32_t plane_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((plane_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)(128 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// kind::tf32: c_format F32, a_format = b_format = TF32 (2), K-major A and B
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// D[tmem] (+)= A[tmem] x B[smem]^T, kind::tf32, issued by the elected lane of a converged warp
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc,
                                            uint32_t issue) {
  asm volatile(
      "{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nsetp.ne.b32 q, %5, 0;\n"
      "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc), "r"(issue));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
// fp32 -> tf32 (round to nearest, ties away from zero; low 13 bits cleared): the integer form of
// cvt.rna.tf32.f32 for finite inputs (the PTX instruction is emulated with an extra Inf/NaN test)
__device__ __forceinline__ uint32_t tf32_bits(float x) { return (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u; }
// one bulk copy per 32 KB piece (the whole image completes `bar`)
__device__ __forceinline__ void load_weights(uint8_t *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  mbar_expect_tx(bar, bytes);
  for (uint32_t o = 0; o < bytes; o += 32768u)
    bulk_g2s(saddr(dst + o), (const uint8_t *)src + o, min(32768u, bytes - o), bar);
}

// ------------------------------------------------------------------ DNN forward model, one level
// Tile = 128 children (child c: parent c / A, action c % A, R1). Per tile and slot s (two tiles
// in flight, one per epilogue warpgroup): A0 = the parent's state (100 -> 104 columns, tf32) ->
// L1 = relu(W1s.s + W1[:, 100 + a] + b1) -> L2, L3 = relu(W.h + b) -> L4 = W4.h + b4: units
// 0..99 = s', unit 100 = r; R' = fmaf(gk, r, R). The action part of layer 1 is the one-hot column
// W1[:, 100 + a], added in fp32 in the epilogue (exact: the one-hot product is the weight itself).
// TMEM per slot s: A at columns 256 s .. +104, D at 256 s + 128 .. +112.
struct DnnTcBias {   // the four layers' biases as a kernel parameter: constant-bank operands of the FADDs
  float b[4][kTcN];
};
// One launch may expand several consecutive levels (DnnTcLevels.n > 1, cooperative launch): every CTA
// keeps the weights and TMEM across the levels and a grid-wide barrier separates them (level k+1's
// parents are level k's children, written by other CTAs). Parent states are read through L2 (ld.cg),
// never the non-coherent path, since they may have been written earlier in the same launch.
__global__ void __launch_bounds__(kTcThreadsDnn, 1)
    k_dnn_tc(const __grid_constant__ DnnTcLevels levels, int A, const float *__restrict__ img,
             const __grid_constant__ DnnTcBias bias) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((128u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 127u)) & 127u);
  const float *sB = (const float *)(smem + 4 * kTcLayerBytes);   // biases [4][112]
  const float *sW1A = sB + 4 * kTcN;                               // one-hot columns [A][100]
  __shared__ __align__(8) uint64_t wbar, a_ready[2], d_full[2];
  __shared__ uint32_t tmem_slot;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&wbar, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&a_ready[s], 256);
      mbar_init(&d_full[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    load_weights(smem, img, (uint32_t)(kTcDnnFloats + A * kDnnS) * 4u, &wbar);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();      // parent states: the previous kernel's output (the weight copy above overlaps its tail)
  pdl_trigger();
  for (int lv = 0; lv < levels.n; ++lv) {
  const DnnTcLevel &LV = levels.lv[lv];
  const NodeView &par = LV.par;
  const NodeOut &out = LV.out;
  const int64_t p_first = LV.p_first, c_begin = LV.c_begin, c_end = LV.c_end;
  const float gk = LV.gk;
  const int64_t n = c_end - c_begin, ntiles = (n + 127) / 128;

  if (warp == 0) {   // ---------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = idesc_tf32(128, kTcN);
    const uint32_t elected = elect_one();
    mbar_wait_spin(&wbar, 0);
    const uint32_t wbase = saddr(smem);
    // tiles in pairs (slot 0: t, slot 1: t + grid), layers interleaved across the pair so one
    // slot's MMAs run while the other slot's epilogue works. Each slot's barriers complete four
    // times per tile, so the parity of layer L's wait is L & 1.
    for (int64_t t0 = blockIdx.x; t0 < ntiles; t0 += 2 * (int64_t)gridDim.x) {
      const int nslot = t0 + gridDim.x < ntiles ? 2 : 1;
      for (int L = 0; L < 4; ++L)
        for (int s = 0; s < nslot; ++s) {
          mbar_wait_spin(&a_ready[s], (uint32_t)L & 1u);
          tc_fence_after();
          const uint32_t tA = tmem + 256u * s, tD = tA + 128u;
#pragma unroll
          for (int kk = 0; kk < kTcK / 8; ++kk)
            mma_tf32_ts(tD, tA + 8u * kk,
                        desc_kmajor(wbase + (uint32_t)L * kTcLayerBytes + (uint32_t)(2 * kk) * kTcPlane, kTcPlane),
                        idesc, kk != 0, elected);
          commit_pred(&d_full[s], elected);
          __syncwarp();
        }
    }
  } else if (warp >= 4) {   // ------------------------------------------ epilogue, slot s
    // 8 warps per slot: lane quarter q (= warp % 4, the TMEM lanes a warp may access) x column half h
    // (h = 0: units / inputs 0..63, h = 1: 64..111), so each thread handles half of one node's row;
    // the half is a compile-time constant of each instantiation (warp-uniform dispatch below)
    const int s = (warp - 4) >> 3, q = warp & 3, m = q * 32 + lane;
    const uint32_t tA = tmem + ((uint32_t)(q * 32) << 16) + 256u * s, tD = tA + 128u;
    auto epilogue = [&](auto half) {
      constexpr int h = decltype(half)::value;
      constexpr int j_lo = h ? 64 : 0, j_hi = h ? kTcN : 64, a_hi = h ? kTcK : 64;
      constexpr int nf4 = ((h ? kDnnS : 64) - j_lo) / 4;   // float4 of the parent state this half loads
      for (int64_t t = blockIdx.x + (int64_t)s * gridDim.x; t < ntiles; t += 2 * (int64_t)gridDim.x) {
        const int64_t c = c_begin + t * 128 + m;
        const bool valid = c < c_end;
        const int64_t p = valid ? c / A : c_begin / A;
        const int a = valid ? (int)(c - p * A) : 0;
        {   // A0: the parent's state (this half's columns) rounded to tf32; columns 100..103, invalid rows: 0
          const float4 *ps = (const float4 *)(par.state + (p - p_first) * par.state_stride) + j_lo / 4;
          float4 x4[nf4];   // the half row's loads in flight at once (one L2 round trip)
#pragma unroll
          for (int e = 0; e < nf4; ++e) x4[e] = valid ? __ldcg(ps + e) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int j = j_lo; j < a_hi; j += 8) {
            const int e = (j - j_lo) / 4;
            const float4 v0 = e < nf4 ? x4[e] : make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 v1 = e + 1 < nf4 ? x4[e + 1] : make_float4(0.f, 0.f, 0.f, 0.f);
            const uint32_t r8[8] = {tf32_bits(v0.x), tf32_bits(v0.y), tf32_bits(v0.z), tf32_bits(v0.w),
                                    tf32_bits(v1.x), tf32_bits(v1.y), tf32_bits(v1.z), tf32_bits(v1.w)};
            tmem_st8(tA + (uint32_t)j, r8);
          }
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&a_ready[s]);
        }
        const float rpar = valid && par.cum ? __ldcg(par.cum + (p - p_first)) : 0.0f;
        float *srow = (float *)(out.state + (valid ? c - c_begin : 0) * out.state_stride);
#pragma unroll
        for (int L = 0; L < 4; ++L) {
          mbar_wait_spin(&d_full[s], (uint32_t)L & 1u);
          tc_fence_after();
          const float *b = bias.b[L];
#pragma unroll
          for (int j2 = j_lo; j2 < j_hi; j2 += 32) {   // two 16-column loads per wait (register budget)
            uint32_t v[2][16];
#pragma unroll
            for (int u = 0; u < 2; ++u)
              if (j2 + 16 * u < j_hi) tmem_ld16_nw(tD + (uint32_t)(j2 + 16 * u), v[u]);
#pragma unroll
            for (int u = 0; u < 2; ++u)
              if (j2 + 16 * u < j_hi) tmem_wait16(v[u]);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int j0 = j2 + 16 * u;
              if (j0 >= j_hi) continue;
              if (L < 3) {   // hidden layer: relu(D + b (+ W1[:, 100 + a])) -> tf32 -> A columns j0..
                uint32_t r[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                  const int uu = j0 + e;
                  float x = 0.0f;
                  if (uu < kDnnS) {
                    x = __uint_as_float(v[u][e]) + b[uu];
                    if (L == 0) x += sW1A[a * kDnnS + uu];
                    x = fmaxf(x, 0.0f);
                  }
                  r[e] = tf32_bits(x);
                }
                if (j0 + 16 <= kTcK) {
                  tmem_st8(tA + (uint32_t)j0, *(const uint32_t(*)[8])r);
                  tmem_st8(tA + (uint32_t)j0 + 8u, *(const uint32_t(*)[8])(r + 8));
                } else if (j0 < kTcK) {
                  tmem_st8(tA + (uint32_t)j0, *(const uint32_t(*)[8])r);
                }
              } else if (valid) {   // output layer: s' (units 0..99) and r (unit 100)
#pragma unroll
                for (int e = 0; e < 16; e += 4) {
                  const int uu = j0 + e;
                  if (uu < kDnnS)
                    *(float4 *)(srow + uu) =
                        make_float4(__uint_as_float(v[u][e]) + b[uu], __uint_as_float(v[u][e + 1]) + b[uu + 1],
                                    __uint_as_float(v[u][e + 2]) + b[uu + 2], __uint_as_float(v[u][e + 3]) + b[uu + 3]);
                }
                if (j0 <= kDnnS && kDnnS < j0 + 16)
                  out.cum[c - c_begin] = fmaf(gk, __uint_as_float(v[u][kDnnS - j0]) + b[kDnnS], rpar);
              }
            }
          }
          if (L < 3) {
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&a_ready[s]);
          }
        }
      }
    };
    if (((warp - 4) >> 2) & 1) epilogue(std::integral_constant<int, 1>{});
    else epilogue(std::integral_constant<int, 0>{});
  }
  if (lv + 1 < levels.n) {   // the whole level written before any CTA reads it as parents
    __threadfence();
    cg::this_grid().sync();
  }
  }   // levels
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ------------------------------------------------------------------ MLP2 leaf / row net
// Q(x, .) = W2 relu(W1 x + b1) + b2 over 128-node tiles; x = 100 fp32 state values (DNN env) or
// 64 state bytes / 256 (INT_HASH, exact in tf32). TMEM: A0 at column 0 (IK = I padded to 8),
// D1 = A1 at column 128 (H units), D2 at column 384 (NA = A padded to 16). One tile at a time.
struct MlpTcShape {
  int I, IK, H, A, NA;
  uint32_t w1_bytes, b1_off, w2_off, w2_bytes, b2_off, total;   // image layout (bytes)
};
__host__ __device__ inline MlpTcShape mlp_tc_shape(int I, int H, int A) {
  MlpTcShape s;
  s.I = I;
  s.IK = (I + 7) / 8 * 8;
  s.H = H;
  s.A = A;
  s.NA = (A + 15) / 16 * 16;
  s.w1_bytes = (uint32_t)(s.IK / 4) * (uint32_t)H * 16u;
  s.b1_off = s.w1_bytes;
  s.w2_off = s.b1_off + (uint32_t)H * 4u;
  s.w2_bytes = (uint32_t)(H / 4) * (uint32_t)s.NA * 16u;
  s.b2_off = s.w2_off + s.w2_bytes;
  s.total = s.b2_off + (uint32_t)s.NA * 4u;
  return s;
}

// A0 of node `node` (features -> tf32; columns I..IK-1 and rows past n zero) into TMEM columns 0..,
// in two steps: mlp_fetch_a0 issues the row's loads into registers (a tile ahead of their use),
// mlp_store_a0 rounds and stores them. Half H of the epilogue handles columns 64 H .. 64 H + 63:
// fp32 features (DNN env) 0..63 / 64..99 (+ zero padding to IK); the 64 state bytes (INT_HASH,
// exact in tf32 after / 256) all belong to half 0 and travel in the first four float4 as raw bits.
template <int H>
struct MlpA0 {
  float4 x[H ? (kDnnS - 64) / 4 : 16];
};
template <int H>
__device__ __forceinline__ void mlp_fetch_a0(const uint8_t *__restrict__ states, int64_t stride, int64_t node,
                                             int64_t n, int feat_f32, MlpA0<H> &r) {
  constexpr int nf4 = H ? (kDnnS - 64) / 4 : 16;
  const bool valid = node < n;
  const uint8_t *srow = states + (valid ? node : 0) * stride;
  if (feat_f32) {   // fp32 state values 64 H .. (DNN env)
#pragma unroll
    for (int e = 0; e < nf4; ++e)
      r.x[e] = valid ? __ldg((const float4 *)srow + 16 * H + e) : make_float4(0.f, 0.f, 0.f, 0.f);
  } else if (H == 0) {   // 64 state bytes (INT_HASH)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint4 w = valid ? __ldg((const uint4 *)srow + e) : make_uint4(0u, 0u, 0u, 0u);
      r.x[e] = make_float4(__uint_as_float(w.x), __uint_as_float(w.y), __uint_as_float(w.z), __uint_as_float(w.w));
    }
  }
}
template <int H>
__device__ __forceinline__ void mlp_store_a0(const MlpA0<H> &r, int feat_f32, uint32_t tl) {
  constexpr int nf4 = H ? (kDnnS - 64) / 4 : 16;
  if (feat_f32) {
#pragma unroll
    for (int j = 64 * H; j < (H ? kTcK : 64); j += 8) {
      const int e = (j - 64 * H) / 4;
      const float4 v0 = e < nf4 ? r.x[e] : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 v1 = e + 1 < nf4 ? r.x[e + 1] : make_float4(0.f, 0.f, 0.f, 0.f);
      const uint32_t q[8] = {tf32_bits(v0.x), tf32_bits(v0.y), tf32_bits(v0.z), tf32_bits(v0.w),
                             tf32_bits(v1.x), tf32_bits(v1.y), tf32_bits(v1.z), tf32_bits(v1.w)};
      tmem_st8(tl + (uint32_t)j, q);
    }
  } else if (H == 0) {   // bytes / 256: exact in tf32
#pragma unroll
    for (int j0 = 0; j0 < 64; j0 += 8) {
      const float4 w = r.x[j0 / 16];
      const uint32_t lo = __float_as_uint((j0 & 8) ? w.z : w.x), hi = __float_as_uint((j0 & 8) ? w.w : w.y);
      uint32_t q[8];
#pragma unroll
      for (int e = 0; e < 8; ++e)
        q[e] = __float_as_uint((float)((((e < 4 ? lo : hi) >> (8 * (e & 3))) & 0xFFu)) * (1.0f / 256.0f));
      tmem_st8(tl + (uint32_t)j0, q);
    }
  }
}

// The next tile's A0 is loaded while the current tile's layer-2 MMAs run (A0's columns are free
// once layer 1 is done); each barrier completes once per tile, so tile i waits parity i & 1.
__global__ void __launch_bounds__(kTcThreadsMlp, 1)
    k_mlp_tc(const uint8_t *__restrict__ states, int64_t stride, const uint8_t *__restrict__ img, MlpTcShape sh,
             int64_t n, int mode, float gd, const float *__restrict__ cum, float *__restrict__ out, int feat_f32) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((128u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 127u)) & 127u);
  const float *sb1 = (const float *)(smem + sh.b1_off), *sb2 = (const float *)(smem + sh.b2_off);
  __shared__ __align__(8) uint64_t wbar, a0_ready, a1_ready, d1_full, d2_full;
  __shared__ uint32_t tmem_slot;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&wbar, 1);
    mbar_init(&a0_ready, 256);
    mbar_init(&a1_ready, 256);
    mbar_init(&d1_full, 1);
    mbar_init(&d2_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    load_weights(smem, img, sh.total, &wbar);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();      // node states: the previous kernel's output (the weight copy above overlaps its tail)
  pdl_trigger();
  const int64_t ntiles = (n + 127) / 128;

  if (warp == 0) {   // ---------------------------------------------------------- MMA issuer
    const uint32_t elected = elect_one();
    const uint32_t id1 = idesc_tf32(128, sh.H), id2 = idesc_tf32(128, sh.NA);
    const uint32_t w1 = saddr(smem), w2 = saddr(smem + sh.w2_off);
    const uint32_t p1 = (uint32_t)sh.H * 16u, p2 = (uint32_t)sh.NA * 16u;
    mbar_wait_spin(&wbar, 0);
    uint32_t i = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      mbar_wait_spin(&a0_ready, i & 1u);
      if (i) mbar_wait_spin(&d2_full, (i - 1) & 1u);   // the previous tile's layer 2 has read A1 (= D1's columns)
      tc_fence_after();
      for (int kk = 0; kk < sh.IK / 8; ++kk)
        mma_tf32_ts(tmem + 128u, tmem + 8u * kk, desc_kmajor(w1 + (uint32_t)(2 * kk) * p1, p1), id1, kk != 0, elected);
      commit_pred(&d1_full, elected);
      __syncwarp();
      mbar_wait_spin(&a1_ready, i & 1u);
      tc_fence_after();
      for (int kk = 0; kk < sh.H / 8; ++kk)
        mma_tf32_ts(tmem + 384u, tmem + 128u + 8u * kk, desc_kmajor(w2 + (uint32_t)(2 * kk) * p2, p2), id2, kk != 0,
                    elected);
      commit_pred(&d2_full, elected);
      __syncwarp();
    }
  } else if (warp >= 4) {   // ------------------------------------------------- epilogue
    // 8 warps: lane quarter q (= warp % 4) x column half (features 0..63 / 64.., hidden units
    // [0, hs) / [hs, H)); layer 2 (NA <= 64 columns) is read by half 0 alone
    const int q = warp & 3, m = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    const int hs = (sh.H / 2 + 15) / 16 * 16;
    auto epilogue = [&](auto half) {
      constexpr int h = decltype(half)::value;
      const int u_lo = h ? hs : 0, u_hi = h ? sh.H : hs;
      MlpA0<h> a0;
      if (blockIdx.x < ntiles) {
        mlp_fetch_a0<h>(states, stride, (int64_t)blockIdx.x * 128 + m, n, feat_f32, a0);
        mlp_store_a0<h>(a0, feat_f32, tl);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&a0_ready);
      }
      uint32_t i = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int64_t node = t * 128 + m;
        // the next tile's row: loads in flight during this tile's layer 1, stored after it
        const bool has_next = t + gridDim.x < ntiles;
        if (has_next) mlp_fetch_a0<h>(states, stride, (t + gridDim.x) * 128 + m, n, feat_f32, a0);
        // layer 1: relu(D1 + b1) -> tf32 -> A1 (the same columns), four 16-column loads per wait
        mbar_wait_spin(&d1_full, i & 1u);
        tc_fence_after();
        for (int j0 = u_lo; j0 < u_hi; j0 += 64) {
          uint32_t v[4][16];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (j0 + 16 * u < u_hi) tmem_ld16_nw(tl + 128u + (uint32_t)(j0 + 16 * u), v[u]);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (j0 + 16 * u < u_hi) tmem_wait16(v[u]);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (j0 + 16 * u >= u_hi) break;
            uint32_t lo[8], hi[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              lo[e] = tf32_bits(fmaxf(__uint_as_float(v[u][e]) + sb1[j0 + 16 * u + e], 0.0f));
              hi[e] = tf32_bits(fmaxf(__uint_as_float(v[u][e + 8]) + sb1[j0 + 16 * u + e + 8], 0.0f));
            }
            tmem_st8(tl + 128u + (uint32_t)(j0 + 16 * u), lo);
            tmem_st8(tl + 128u + (uint32_t)(j0 + 16 * u) + 8u, hi);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&a1_ready);
        // the next tile's features while layer 2 runs
        if (has_next) {
          mlp_store_a0<h>(a0, feat_f32, tl);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&a0_ready);
        }
        if (h == 0) {   // layer 2: Q = D2 + b2 -> rows / max / total
          mbar_wait_spin(&d2_full, i & 1u);
          tc_fence_after();
          float best = -INFINITY;
          const bool valid = node < n;
          for (int j0 = 0; j0 < sh.NA; j0 += 16) {
            uint32_t v[16];
            tmem_ld16_nw(tl + 384u + (uint32_t)j0, v);
            tmem_wait16(v);
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int a = j0 + e;
              if (a < sh.A) {
                const float qv = __uint_as_float(v[e]) + sb2[a];
                best = fmaxf(best, qv);
                if (valid && mode == MODE_ROWS) out[node * sh.A + a] = qv;
              }
            }
          }
          if (valid && mode != MODE_ROWS) out[node] = mode == MODE_ROWMAX ? best : fmaf(gd, best, cum ? cum[node] : 0.0f);
          tc_fence_before();
        }
      }
    };
    if (((warp - 4) >> 2) & 1) epilogue(std::integral_constant<int, 1>{});
    else epilogue(std::integral_constant<int, 0>{});
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// host: fp32 -> tf32, round to nearest with ties away from zero (= cvt.rna.tf32.f32)
float tf32_round_host(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) != 0x7F800000u) u = (u + 0x1000u) & 0xFFFFE000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}
// element (n, k) of a K-major SWIZZLE_NONE image with Npad rows
inline size_t kmajor_index(int n, int k, int npad) { return (size_t)(k / 4) * npad * 4 + (size_t)n * 4 + (k % 4); }

}  // namespace

// canonical DNN blob (include/bcts.h: g1.w [100][100+A], g1.b, g2.w, g2.b, g3.w, g3.b, g4.w [101][100],
// g4.b [101]) -> the k_dnn_tc image: 4 layer images (tf32-rounded), biases [4][112], W1A [A][100]
size_t dnn_tc_image_floats(int A) { return (size_t)kTcDnnFloats + (size_t)kDnnS * A; }
void dnn_tc_repack(const float *blob, int A, float *out) {
  const int S = kDnnS, I1 = S + A;
  memset(out, 0, dnn_tc_image_floats(A) * 4);
  const float *g1w = blob, *g1b = g1w + (size_t)S * I1, *g2w = g1b + S, *g2b = g2w + S * S, *g3w = g2b + S,
              *g3b = g3w + S * S, *g4w = g3b + S, *g4b = g4w + (S + 1) * S;
  const float *W[4] = {g1w, g2w, g3w, g4w}, *B[4] = {g1b, g2b, g3b, g4b};
  const int ld[4] = {I1, S, S, S}, nout[4] = {S, S, S, S + 1};
  for (int L = 0; L < 4; ++L) {
    float *img = out + (size_t)L * (kTcLayerBytes / 4);
    for (int u = 0; u < nout[L]; ++u)
      for (int i = 0; i < S; ++i) img[kmajor_index(u, i, kTcN)] = tf32_round_host(W[L][(size_t)u * ld[L] + i]);
    for (int u = 0; u < nout[L]; ++u) out[4 * (kTcLayerBytes / 4) + L * kTcN + u] = B[L][u];
  }
  float *w1a = out + kTcDnnFloats;
  for (int a = 0; a < A; ++a)
    for (int u = 0; u < S; ++u) w1a[a * S + u] = g1w[(size_t)u * I1 + S + a];
}

static size_t dnn_tc_smem(int A) { return dnn_tc_image_floats(A) * 4 + 128; }

void launch_expand_dnn_tc(const NodeView &par, int64_t p_first, int64_t c_begin, int64_t c_end, int A, float gk,
                          const float *img, const float *bias_host, const NodeOut &out, cudaStream_t st,
                          Profiler *prof) {
  DnnTcLevel lv;
  lv.par = par;
  lv.p_first = p_first;
  lv.c_begin = c_begin;
  lv.c_end = c_end;
  lv.gk = gk;
  lv.out = out;
  launch_expand_dnn_tc_levels(&lv, 1, A, img, bias_host, st, prof);
}

int launch_expand_dnn_tc_levels(const DnnTcLevel *lvs, int nlev, int A, const float *img, const float *bias_host,
                                cudaStream_t st, Profiler *prof) {
  DnnTcLevels L;
  L.n = 0;
  double flops = 0.0;
  int64_t max_tiles = 0;
  for (int k = 0; k < nlev; ++k) {
    const int64_t n = lvs[k].c_end - lvs[k].c_begin;
    if (n <= 0) continue;
    const int64_t nparents = (lvs[k].c_end - 1) / A - lvs[k].c_begin / A + 1;
    // the same algorithmic FLOPs as the fp32 path (launch_expand_dnn)
    flops += 2.0 * (30100.0 * (double)n + 10000.0 * (double)nparents);
    max_tiles = std::max<int64_t>(max_tiles, (n + 127) / 128);
    L.lv[L.n++] = lvs[k];
  }
  if (!L.n) return 0;
  if (prof) prof->begin(KC_EXPAND_DNN, flops, st);
  const size_t smem = dnn_tc_smem(A);
  smem_optin((const void *)k_dnn_tc, (int)smem);
  const unsigned grid = (unsigned)std::min<int64_t>((max_tiles + 1) / 2, sm_count_current());
  DnnTcBias bias;
  memcpy(bias.b, bias_host, sizeof(bias.b));
  cudaError_t e;
  if (L.n == 1) {
    e = launch_pdl(k_dnn_tc, dim3(grid), dim3(kTcThreadsDnn), smem, st, L, A, img, bias);
  } else {   // grid-wide barriers between the levels: every CTA must be resident (one per SM)
    void *args[] = {(void *)&L, (void *)&A, (void *)&img, (void *)&bias};
    e = cudaLaunchCooperativeKernel((const void *)k_dnn_tc, dim3(grid), dim3(kTcThreadsDnn), args, smem, st);
  }
  if (prof) prof->end(st);
  return e == cudaSuccess ? 0 : -1;
}

bool dnn_tc_ok(int A) { return dnn_tc_smem(A) <= 227 * 1024 - 1024; }

// MLP2 weights (w1 [H][I], b1 [H], w2 [A][H], b2 [A]) -> the k_mlp_tc image
size_t mlp_tc_image_bytes(int I, int H, int A) { return mlp_tc_shape(I, H, A).total; }
bool mlp_tc_ok(int I, int H, int A) {
  const MlpTcShape s = mlp_tc_shape(I, H, A);
  return s.IK <= 128 && H % 16 == 0 && H <= 256 && s.NA <= 64 && s.total + 128 <= 227 * 1024 - 1024;
}
void mlp_tc_repack(const float *w1, const float *b1, const float *w2, const float *b2, int I, int H, int A,
                   uint8_t *out) {
  const MlpTcShape s = mlp_tc_shape(I, H, A);
  memset(out, 0, s.total);
  float *W1 = (float *)out, *B1 = (float *)(out + s.b1_off), *W2 = (float *)(out + s.w2_off),
        *B2 = (float *)(out + s.b2_off);
  for (int u = 0; u < H; ++u)
    for (int i = 0; i < I; ++i) W1[kmajor_index(u, i, H)] = tf32_round_host(w1[(size_t)u * I + i]);
  for (int u = 0; u < H; ++u) B1[u] = b1[u];
  for (int a = 0; a < A; ++a)
    for (int u = 0; u < H; ++u) W2[kmajor_index(a, u, s.NA)] = tf32_round_host(w2[(size_t)a * H + u]);
  for (int a = 0; a < A; ++a) B2[a] = b2[a];
}

void launch_mlp_tc(const NodeView &v, int64_t n, const uint8_t *img, int I, int H, int A, int mode, float gd,
                   float *out, int feat_f32, cudaStream_t st) {
  if (n <= 0) return;
  const MlpTcShape sh = mlp_tc_shape(I, H, A);
  const size_t smem = sh.total + 128;
  smem_optin((const void *)k_mlp_tc, (int)smem);
  const unsigned grid = (unsigned)std::min<int64_t>((n + 127) / 128, sm_count_current());
  launch_pdl(k_mlp_tc, dim3(grid), dim3(kTcThreadsMlp), smem, st, v.state, v.state_stride, img, sh, n, mode, gd, v.cum,
             out, feat_f32);
}

}  // namespace bcts
