// prune.cu -- NEXT-4 early pruning ("Efficient pruning can be done by maintaining an
// index array of unpruned states which are updated with each pruning step. These indices are
// then used for tracing the optimal action at the root."; R30-R33).
//
// A pruned level is a compacted array of survivors. Each node carries f, its index in the
// UNPRUNED tree (global over the roots of the call): the index array. Its group (root, root
// action) is f / A^(k-1) and a leaf's key slot is f / A^(d-1), exactly as in the implicit
// layout, so best_leaf keeps its meaning and the backup stays a max over packed keys.
//
//   k_child_index  f(child c) = f(parent c / A) * A + c % A          (Alg. 1 replicate, R1)
//   k_bound_*      BOUND rule (R31): per-group max of the lower bounds, then keep iff the node's
//                  upper bound reaches it. Bound arithmetic in IEEE double with explicit _rn
//                  intrinsics (no FMA contraction), the oracle's operation order.
//   k_beam_keep    BEAM rule (R32): rank of fmaf(g_k, max_a Q, R) inside the group.
//   compaction     cub::DeviceSelect::Flagged over the node indices, then one gather of the
//                  survivors' states / keys / cum / f (memory-bound copies, 16-byte vectors).
//   k_segmax_f     backup of leaf totals whose f is explicit.
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "engine.h"

namespace bcts {

__global__ void k_iota64(int64_t *__restrict__ f, int64_t first, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = first + i;
}

__global__ void k_child_index(const int64_t *__restrict__ pf, int64_t n_child, int A, int64_t *__restrict__ cf) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n_child) {
    const int64_t p = c / A;
    cf[c] = pf[p] * A + (c - p * A);
  }
}

void launch_prune_iota(int64_t *f, int64_t first, int64_t n, cudaStream_t st) {
  if (n > 0) k_iota64<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(f, first, n);
}

void launch_child_index(const int64_t *pf, int64_t n_child, int A, int64_t *cf, cudaStream_t st) {
  if (n_child > 0) k_child_index<<<(unsigned)((n_child + 255) / 256), 256, 0, st>>>(pf, n_child, A, cf);
}

// ------------------------------------------------------------------ BOUND (R31)
// Monotone map double -> uint64 (total order of the non-NaN doubles; 0 is below -inf's image).
__device__ __forceinline__ unsigned long long ord_f64(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double unord_f64(unsigned long long o) {
  const unsigned long long u = (o >> 63) ? (o & 0x7FFFFFFFFFFFFFFFull) : ~o;
  return __longlong_as_double((long long)u);
}
// s = 2^-16 (|R| + S): exact power-of-two scaling, as ldexp in the oracle
__device__ __forceinline__ double bound_margin(double R, double S) { return __dmul_rn(__dadd_rn(fabs(R), S), 0x1p-16); }

__global__ void k_bound_max(const float *__restrict__ cum, const int64_t *__restrict__ f, int64_t n, BoundRule b,
                            unsigned long long *__restrict__ gmax) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double R = (double)cum[i];
  const double lb = __dsub_rn(__dadd_rn(R, b.L), bound_margin(R, b.S));
  atomicMax(&gmax[f[i] / b.gsz - b.g0], ord_f64(lb));
}

__global__ void k_bound_keep(const float *__restrict__ cum, const int64_t *__restrict__ f, int64_t n, BoundRule b,
                             const unsigned long long *__restrict__ gmax, uint8_t *__restrict__ keep) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double R = (double)cum[i];
  const double ub = __dadd_rn(__dadd_rn(R, b.U), bound_margin(R, b.S));
  keep[i] = !(ub < unord_f64(gmax[f[i] / b.gsz - b.g0]));
}

void launch_bound_keep(const float *cum, const int64_t *f, int64_t n, const BoundRule &b, unsigned long long *gmax,
                       uint8_t *keep, cudaStream_t st, Profiler *prof) {
  if (n <= 0) return;
  if (prof) prof->begin(KC_PRUNE, 2.0 * 12.0 * (double)n + (double)n, st);   // cum + f read twice, flag written
  cudaMemsetAsync(gmax, 0, (size_t)b.groups * 8, st);
  const unsigned g = (unsigned)((n + 255) / 256);
  k_bound_max<<<g, 256, 0, st>>>(cum, f, n, b, gmax);
  k_bound_keep<<<g, 256, 0, st>>>(cum, f, n, b, gmax, keep);
  if (prof) prof->end(st);
}

// ------------------------------------------------------------------- BEAM (R32)
// Groups are contiguous runs of G nodes (every group of a level has the same size: the rule keeps
// min(beam, G) per group). rank(i) = #{j in group : v_j > v_i or (v_j == v_i and j < i)}, j in f
// order (compaction preserves it); keep iff rank < beam.
__global__ void k_beam_keep(const float *__restrict__ m, const float *__restrict__ cum, float gk, int64_t n, int64_t G,
                            int64_t beam, uint8_t *__restrict__ keep) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t g0 = (i / G) * G;
  const float vi = fmaf(gk, m[i], cum[i]);
  int64_t rank = 0;
  for (int64_t j = g0; j < g0 + G && rank < beam; ++j) {
    const float vj = fmaf(gk, m[j], cum[j]);
    rank += (vj > vi) || (vj == vi && j < i);
  }
  keep[i] = rank < beam;
}

void launch_beam_keep(const float *m, const float *cum, float gk, int64_t n, int64_t G, int64_t beam, uint8_t *keep,
                      cudaStream_t st, Profiler *prof) {
  if (n <= 0) return;
  if (prof) prof->begin(KC_PRUNE, 9.0 * (double)n, st);
  k_beam_keep<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(m, cum, gk, n, G, beam, keep);
  if (prof) prof->end(st);
}

// ------------------------------------------------------------------ compaction
size_t compact_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::CountingInputIterator<int64_t> it(0);
  cub::DeviceSelect::Flagged(nullptr, bytes, it, (const uint8_t *)nullptr, (int64_t *)nullptr, (int64_t *)nullptr,
                             n, (cudaStream_t)0);
  return bytes;
}

void launch_compact(const uint8_t *keep, int64_t n, int64_t *sel, int64_t *d_count, void *temp, size_t temp_bytes,
                    cudaStream_t st) {
  cub::CountingInputIterator<int64_t> it(0);
  cub::DeviceSelect::Flagged(temp, temp_bytes, it, keep, sel, d_count, n, st);
}

template <typename V>
__global__ void k_gather_states(const uint8_t *__restrict__ src, int64_t src_stride, const int64_t *__restrict__ sel,
                                int64_t n_out, int per, uint8_t *__restrict__ dst, int64_t dst_stride) {
  const int64_t total = n_out * per;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / per;
    const int w = (int)(e - j * per);
    const V *s = (const V *)(src + sel[j] * src_stride);
    ((V *)(dst + j * dst_stride))[w] = s[w];
  }
}

__global__ void k_gather_meta(const uint64_t *__restrict__ key, const float *__restrict__ cum,
                              const int64_t *__restrict__ f, const int64_t *__restrict__ sel, int64_t n,
                              uint64_t *__restrict__ okey, float *__restrict__ ocum, int64_t *__restrict__ of) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t i = sel[j];
  if (key) okey[j] = key[i];
  ocum[j] = cum[i];
  of[j] = f[i];
}

void launch_gather_level(int64_t state_bytes, const NodeView &src, const int64_t *f, const int64_t *sel, int64_t n_out,
                         const NodeOut &dst, int64_t *f_out, cudaStream_t st, Profiler *prof) {
  if (n_out <= 0) return;
  const double node = (double)state_bytes + (src.key ? 8.0 : 0.0) + 4.0 + 8.0;
  if (prof) prof->begin(KC_PRUNE, 2.0 * node * (double)n_out + 8.0 * (double)n_out, st);
  const bool v16 = state_bytes % 16 == 0 && src.state_stride % 16 == 0 && dst.state_stride % 16 == 0 &&
                   ((uintptr_t)src.state % 16) == 0 && ((uintptr_t)dst.state % 16) == 0;
  const int per = (int)(v16 ? state_bytes / 16 : state_bytes / 4);
  const int64_t total = n_out * per;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (v16)
    k_gather_states<uint4><<<grid, 256, 0, st>>>(src.state, src.state_stride, sel, n_out, per, dst.state,
                                                 dst.state_stride);
  else
    k_gather_states<uint32_t><<<grid, 256, 0, st>>>(src.state, src.state_stride, sel, n_out, per, dst.state,
                                                    dst.state_stride);
  k_gather_meta<<<(unsigned)((n_out + 255) / 256), 256, 0, st>>>(src.key, src.cum, f, sel, n_out, dst.key, dst.cum,
                                                                 f_out);
  if (prof) prof->end(st);
}

// ---------------------------------------------------------------------- backup
// Leaf c has unpruned index f[c] (global over the call's roots): slot = f / A^(d-1) = root*A + a0,
// key = (total, index within the root) -- the same keys as k_segmax over the implicit layout.
__global__ void k_segmax_f(const float *__restrict__ totals, const int64_t *__restrict__ f, int64_t n, int64_t lpr,
                           int64_t seg, int64_t *__restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x % 32;
  int64_t key = kKeyEmpty, slot = -1;
  if (i < n) {
    const int64_t L = f[i];
    slot = L / seg;
    key = pack_key(totals[i], L - (L / lpr) * lpr);
  }
  const int64_t s0 = __shfl_sync(0xffffffffu, slot, 0);
  const bool uniform = __all_sync(0xffffffffu, slot == s0 || slot < 0);
  if (uniform) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int64_t other = __shfl_xor_sync(0xffffffffu, key, o);
      key = other > key ? other : key;
    }
    if (lane == 0 && s0 >= 0) atomicMax((long long *)&keys[s0], (long long)key);
  } else if (slot >= 0) {
    atomicMax((long long *)&keys[slot], (long long)key);
  }
}

void launch_segmax_f(const float *totals, const int64_t *f, int64_t n, int64_t lpr, int64_t seg, int64_t *keys,
                     cudaStream_t st, Profiler *prof) {
  if (n <= 0) return;
  if (prof) prof->begin(KC_SEGMAX, 12.0 * (double)n, st);   // one fp32 total + one int64 index per leaf
  k_segmax_f<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(totals, f, n, lpr, seg, keys);
  if (prof) prof->end(st);
}

}  // namespace bcts
