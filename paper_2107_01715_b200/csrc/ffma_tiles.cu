// ffma_tiles.cu -- the fixed-order fp32 FMA kernels: the random-DNN forward
// model (level expansion, Alg. 1 P:318-321 with the learned model of
// P:340-341) and the MLP2 leaf net (Q_theta on the hash / DNN envs).
//
// Both are fp32 contractions whose every output is ONE fmaf chain from the
// bias over the inputs in index order, so they match the oracle's fp32 mirror
// bit for bit (R27, R16). That fixes the summation order per output,
// which rules out split-K and tensor cores (their accumulation order is not
// this chain); what is left is a register-tiled SIMT kernel whose ceiling is
// the FFMA issue rate ("alu" roofline).
//
// Shape shared by both kernels: persistent CTAs (one per SM), the transposed
// weight image put in shared memory ONCE per CTA by a single bulk copy (TMA
// engine, cp.async.bulk), then a loop over tiles of T nodes. Activations live
// in shared memory as [input][T] (node index contiguous). A thread owns a
// 4-output x 8-node register tile: per input i it reads one float4 of weights
// (WT[i][4u..4u+3]) and two float4 of activations (X[i][8c..8c+7]) for 32 FFMA.
#include <algorithm>

#include "engine.h"

namespace bcts {
namespace {

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// One bulk copy of `bytes` (multiple of 16) global -> shared, then every thread waits for it.
__device__ __forceinline__ void load_image(float *dst, const float *src, uint32_t bytes, uint64_t *bar) {
  if (threadIdx.x == 0) {
    bar_init(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(bar))
        : "memory");
  }
  __syncthreads();
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(su32(bar))
      : "memory");
}

// Column layout of an activation row X[i][0..T) (node index within the tile):
// CPT = 8 tiles use a PERMUTED layout -- logical node 8cg + 4j + k sits at
// column j*(T/2) + 4cg + k -- so that the 8 node groups a warp reads with one
// LDS.128 are 8 consecutive float4 (one conflict-free wavefront) instead of 8
// float4 32 bytes apart (2-way bank conflicts). Other CPT: plain, CPT*cg + c.
template <int T, int CPT>
__device__ __forceinline__ int xcol(int c) {
  if constexpr (CPT == 8) return ((c >> 2) & 1) * (T / 2) + (c >> 3) * 4 + (c & 3);
  else return c;
}

// acc[c][j] = fmaf chain over i = 0..nin-1 of WT[i][4ug + j] * X[i][node CPT*cg + c], from b[4ug + j].
// The operands of step i+1 are loaded before the 4*CPT FFMAs of step i (register double buffer).
template <int T, int CPT>
__device__ __forceinline__ void ffma_tile(const float *__restrict__ WT, int ldw, const float *__restrict__ b,
                                          const float *__restrict__ X, int nin, int ug, int cg,
                                          float (&acc)[CPT][4]) {
  static_assert(CPT == 8 || CPT == 2, "tile shapes: 4x8 (permuted columns) or 4x2 (plain)");
  const float4 bb = *(const float4 *)(b + 4 * ug);
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    acc[c][0] = bb.x; acc[c][1] = bb.y; acc[c][2] = bb.z; acc[c][3] = bb.w;
  }
  const float *w = WT + 4 * ug;
  const float *x = X + (CPT == 8 ? 4 * cg : CPT * cg);
  float4 wv = *(const float4 *)w;
  float xv[CPT];
  auto ldx = [&](const float *p, float (&v)[CPT]) {
    if constexpr (CPT == 8) {
      const float4 a = *(const float4 *)p, b2 = *(const float4 *)(p + T / 2);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b2.x; v[5] = b2.y; v[6] = b2.z; v[7] = b2.w;
    } else {
      const float2 a = *(const float2 *)p;
      v[0] = a.x; v[1] = a.y;
    }
  };
  ldx(x, xv);
#pragma unroll 2
  for (int i = 0; i < nin; ++i) {
    const int nx = i + 1 < nin ? i + 1 : i;
    const float4 wn = *(const float4 *)(w + nx * ldw);
    float xn[CPT];
    ldx(x + nx * T, xn);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      acc[c][0] = fmaf(wv.x, xv[c], acc[c][0]);
      acc[c][1] = fmaf(wv.y, xv[c], acc[c][1]);
      acc[c][2] = fmaf(wv.z, xv[c], acc[c][2]);
      acc[c][3] = fmaf(wv.w, xv[c], acc[c][3]);
    }
    wv = wn;
#pragma unroll
    for (int c = 0; c < CPT; ++c) xv[c] = xn[c];
  }
}

// Y[4ug + j][node CPT*cg + c] = (relu) acc[c][j], in the xcol layout
template <int T, int CPT>
__device__ __forceinline__ void store_tile(float *Y, int ug, int cg, const float (&acc)[CPT][4], bool relu) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float v[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) v[c] = relu ? fmaxf(acc[c][j], 0.0f) : acc[c][j];
    float *y = Y + (4 * ug + j) * T;
    if constexpr (CPT == 8) {
      *(float4 *)(y + 4 * cg) = make_float4(v[0], v[1], v[2], v[3]);
      *(float4 *)(y + T / 2 + 4 * cg) = make_float4(v[4], v[5], v[6], v[7]);
    } else {
      *(float2 *)(y + 2 * cg) = make_float2(v[0], v[1]);
    }
  }
}

}  // namespace

// =================================================================== DNN env
// Random-DNN learned forward model of the runtime study (R27):
// x = [s(100); onehot(a)] -> 3 x (Linear 100 + ReLU) -> Linear 101 = (s', r).
// Sibling sharing: the state part of layer 1, pre[u] = chain over s only, is
// computed once per parent; child a finishes the chain with the one-hot tail,
// where fmaf(w, 0, acc) = acc and fmaf(w, 1, acc) = acc + w (only a signed
// zero can differ, and ReLU maps both zeros to +0).
// Device image (floats): W1T[100][100] | W2T | W3T | W4T[100][104] |
// b1[100] b2[100] b3[100] b4[104]  (kDnnImg, one bulk copy), then W1A[A][100]
// (the one-hot columns, read through L1).
// Tiles: 10 groups of CPT children x 25 groups of 4 units = 250 tasks on
// warps 0-7 (warp 8 computes the reward unit); T = 10*CPT children per tile. CPT = 8 (T = 80, the largest tile
// whose two [100][T] activation buffers fit beside the 163 KB image) for big
// levels; CPT = 2 (T = 20, 4x shorter per-tile latency, 4x more CTAs) for
// levels too small to fill the GPU with 80-child tiles.
constexpr int kDnnThreads = 288, kDnnCg = 10;   // warps 0-7: 250 tile tasks; warp 8: reward unit
constexpr int kDnnPf = 4;                         // parent float4 prefetched per thread (<= 42 parents)
constexpr int kDnnOff2 = 10000, kDnnOff3 = 20000, kDnnOff4 = 30000, kDnnOffB = 40400;
template <int CPT>
constexpr size_t dnn_smem() { return (size_t)kDnnImg * 4 + 2 * (size_t)kDnnS * (kDnnCg * CPT) * 4; }

int64_t dnn_env_weights_count(int A) { return 40501 + 100LL * A; }

void dnn_repack(const float *blob, int A, float *out) {
  const int S = kDnnS, I1 = S + A;
  const float *g1w = blob, *g1b = g1w + S * I1, *g2w = g1b + S, *g2b = g2w + S * S, *g3w = g2b + S,
              *g3b = g3w + S * S, *g4w = g3b + S, *g4b = g4w + (S + 1) * S;
  memset(out, 0, ((size_t)kDnnImg + (size_t)S * A) * 4);
  for (int u = 0; u < S; ++u)
    for (int i = 0; i < S; ++i) {
      out[i * S + u] = g1w[u * I1 + i];
      out[kDnnOff2 + i * S + u] = g2w[u * S + i];
      out[kDnnOff3 + i * S + u] = g3w[u * S + i];
    }
  for (int u = 0; u <= S; ++u)
    for (int i = 0; i < S; ++i) out[kDnnOff4 + i * 104 + u] = g4w[u * S + i];
  for (int u = 0; u < S; ++u) {
    out[kDnnOffB + u] = g1b[u];
    out[kDnnOffB + 100 + u] = g2b[u];
    out[kDnnOffB + 200 + u] = g3b[u];
  }
  for (int u = 0; u <= S; ++u) out[kDnnOffB + 300 + u] = g4b[u];
  for (int a = 0; a < A; ++a)
    for (int u = 0; u < S; ++u) out[kDnnImg + a * S + u] = g1w[u * I1 + S + a];
}

namespace {
// Task -> (unit group ug < 25, node group cg < 10). CPT = 8: tasks 0..199 are
// warps of 8 node groups x 4 unit groups (cg 0..7; 3 wavefronts per step),
// tasks 200..249 cover cg 8, 9 as 2 x 16 blocks. CPT = 2: cg = task % 10.
template <int CPT>
__device__ __forceinline__ void dnn_task(int task, int &ug, int &cg) {
  if constexpr (CPT == 8) {
    if (task < 200) { cg = task & 7; ug = task >> 3; }
    else { cg = 8 + ((task - 200) & 1); ug = (task - 200) >> 1; }
  } else {
    cg = task % kDnnCg; ug = task / kDnnCg;
  }
}

// hidden layer: Y[u][c] = relu(chain) for u < 100, all T columns
template <int T, int CPT>
__device__ __forceinline__ void dnn_hidden(const float *WT, const float *b, const float *X, float *Y) {
  const int task = threadIdx.x;
  if (task < 25 * kDnnCg) {
    int ug, cg;
    dnn_task<CPT>(task, ug, cg);
    float acc[CPT][4];
    ffma_tile<T, CPT>(WT, kDnnS, b, X, kDnnS, ug, cg, acc);
    store_tile<T, CPT>(Y, ug, cg, acc, true);
  }
}

template <int CPT>
__global__ void __launch_bounds__(kDnnThreads, 1)
    k_expand_dnn(NodeView par, int64_t p_first, int64_t c_begin, int64_t c_end, int A, float gk,
                 const float *__restrict__ img, NodeOut out) {
  constexpr int T = kDnnCg * CPT;
  extern __shared__ __align__(128) float dsm[];
  float *W = dsm, *Bs = dsm + kDnnOffB;
  float *bufA = dsm + kDnnImg, *bufB = bufA + kDnnS * T;
  __shared__ __align__(8) uint64_t bar;
  const float *W1A = img + kDnnImg;
  load_image(dsm, img, kDnnImg * 4, &bar);
  const int64_t n = c_end - c_begin, ntiles = (n + T - 1) / T;
  // parent states of a tile, 25 float4 each, fetched into registers one tile ahead
  float4 pf[kDnnPf];
  auto fetch = [&](int64_t tt) {
    if (tt >= ntiles) return;
    const int64_t cb = c_begin + tt * T, pb = cb / A;
    const int npp = (int)((cb + min((int64_t)T, c_end - cb) - 1) / A - pb + 1);
#pragma unroll
    for (int k = 0; k < kDnnPf; ++k) {
      const int e = threadIdx.x + k * kDnnThreads;
      if (e < npp * 25) {
        const int p = e / 25, q = e - p * 25;
        pf[k] = __ldg((const float4 *)(par.state + (pb + p - p_first) * par.state_stride) + q);
      }
    }
  };
  fetch(blockIdx.x);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t c0 = c_begin + t * T;
    const int nc = (int)min((int64_t)T, c_end - c0);
    const int64_t p0 = c0 / A;
    const int np = (int)((c0 + nc - 1) / A - p0 + 1);   // <= T/A + 2 <= 42 (A >= 2)
    // 0: parent states (prefetched) -> bufA[i][p] (columns past np are never read back)
#pragma unroll
    for (int k = 0; k < kDnnPf; ++k) {
      const int e = threadIdx.x + k * kDnnThreads;
      if (e < np * 25) {
        const int p = e / 25, q = e - p * 25;
        bufA[(4 * q + 0) * T + p] = pf[k].x;
        bufA[(4 * q + 1) * T + p] = pf[k].y;
        bufA[(4 * q + 2) * T + p] = pf[k].z;
        bufA[(4 * q + 3) * T + p] = pf[k].w;
      }
    }
    __syncthreads();
    fetch(t + gridDim.x);
    // 1: pre[u][p] = b1[u] + chain over the 100 state inputs, once per parent -> bufB (4x2 tiles)
    {
      const int n_pg = (np + 1) / 2;
      for (int task = threadIdx.x; task < 25 * n_pg; task += kDnnThreads) {
        const int pg = task % n_pg, ug = task / n_pg;
        float acc[2][4];
        ffma_tile<T, 2>(W, kDnnS, Bs, bufA, kDnnS, ug, pg, acc);
        store_tile<T, 2>(bufB, ug, pg, acc, false);
      }
    }
    __syncthreads();
    // 2: h1[u][c] = relu(pre[u][parent(c)] + W1[u][100 + a(c)]) -> bufA (children past nc: zeros)
#pragma unroll 4
    for (int e = threadIdx.x; e < kDnnS * T; e += kDnnThreads) {
      const int u = e / T, c = e % T;
      float h = 0.0f;
      if (c < nc) {
        const int64_t cc = c0 + c, p = cc / A;
        const int a = (int)(cc - p * A);
        h = fmaxf(__fadd_rn(bufB[u * T + (int)(p - p0)], __ldg(W1A + a * kDnnS + u)), 0.0f);
      }
      bufA[u * T + xcol<T, CPT>(c)] = h;
    }
    __syncthreads();
    dnn_hidden<T, CPT>(W + kDnnOff2, Bs + 100, bufA, bufB);   // 3: layer 2
    __syncthreads();
    dnn_hidden<T, CPT>(W + kDnnOff3, Bs + 200, bufB, bufA);   // 4: layer 3
    __syncthreads();
    // 5: layer 4 (no ReLU): units 0..99 = s' -> out.state (250 tile tasks); unit 100 = r -> out.cum,
    //    one child chain per lane of warp 8
    const int task = threadIdx.x;
    if (task < 25 * kDnnCg) {
      int ug, cg;
      dnn_task<CPT>(task, ug, cg);
      float acc[CPT][4];
      ffma_tile<T, CPT>(W + kDnnOff4, 104, Bs + 300, bufA, kDnnS, ug, cg, acc);
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const int cl = CPT * cg + c;
        if (cl < nc)
          *(float4 *)((float *)(out.state + (c0 + cl - c_begin) * out.state_stride) + 4 * ug) =
              make_float4(acc[c][0], acc[c][1], acc[c][2], acc[c][3]);
      }
    } else if (task >= 256) {
      for (int cl = task - 256; cl < nc; cl += 32) {
        const float *x = bufA + xcol<T, CPT>(cl);
        float r = Bs[400];
        for (int i = 0; i < kDnnS; ++i) r = fmaf(W[kDnnOff4 + i * 104 + 100], x[i * T], r);
        const int64_t p = (c0 + cl) / A;
        out.cum[c0 + cl - c_begin] = fmaf(gk, r, par.cum ? par.cum[p - p_first] : 0.0f);
      }
    }
    __syncthreads();   // bufA/bufB reuse by the next tile
  }
}

int sm_count() { return sm_count_current(); }
}  // namespace

void launch_expand_dnn(const NodeView &par, int64_t p_first, int64_t c_begin, int64_t c_end, int A, float gk,
                       const float *img, const NodeOut &out, cudaStream_t st, Profiler *prof) {
  const int64_t n = c_end - c_begin;
  if (n <= 0) return;
  const int64_t nparents = (c_end - 1) / A - c_begin / A + 1;
  // algorithmic FLOPs: per child 2*(100*100 + 100*100 + 101*100) (layers 2-4; the layer-1 tail is
  // one add), per parent 2*100*100 (the shared state part of layer 1)
  if (prof) prof->begin(KC_EXPAND_DNN, 2.0 * (30100.0 * (double)n + 10000.0 * (double)nparents), st);
  smem_optin((const void *)k_expand_dnn<8>, (int)dnn_smem<8>());
  smem_optin((const void *)k_expand_dnn<2>, (int)dnn_smem<2>());
  const int sms = sm_count();
  const int64_t tiles80 = (n + 79) / 80;
  if (tiles80 >= 2 * sms) {
    const unsigned grid = (unsigned)std::min<int64_t>(tiles80, sms);
    k_expand_dnn<8><<<grid, kDnnThreads, dnn_smem<8>(), st>>>(par, p_first, c_begin, c_end, A, gk, img, out);
  } else {
    const unsigned grid = (unsigned)std::min<int64_t>((n + 19) / 20, sms);
    k_expand_dnn<2><<<grid, kDnnThreads, dnn_smem<2>(), st>>>(par, p_first, c_begin, c_end, A, gk, img, out);
  }
  if (prof) prof->end(st);
}

// ============================================================== MLP2, tiled
// Q(s, .) = W2 relu(W1 x + b1) + b2 over T nodes per tile; x_j = byte j / 256
// (INT_HASH) or the j-th fp32 state value (DNN env). Device image (floats):
// W1T[I][H] | b1[H] | W2T[H][A4] | b2[A4] (A4 = A rounded up to 4, zero pad).
// Layer 1 uses the 4x8 register tile; layer 2 (A outputs) gives each thread
// one node x 4 actions, a 256-long chain per output.
int mlp_image_floats(int I, int H, int A) {
  const int A4 = (A + 3) / 4 * 4;
  return I * H + H + H * A4 + A4;
}

void mlp_repack(const float *w1, const float *b1, const float *w2, const float *b2, int I, int H, int A,
                float *out) {
  const int A4 = (A + 3) / 4 * 4;
  memset(out, 0, (size_t)mlp_image_floats(I, H, A) * 4);
  for (int u = 0; u < H; ++u)
    for (int i = 0; i < I; ++i) out[i * H + u] = w1[u * I + i];
  for (int u = 0; u < H; ++u) out[I * H + u] = b1[u];
  float *w2t = out + I * H + H;
  for (int a = 0; a < A; ++a)
    for (int u = 0; u < H; ++u) w2t[u * A4 + a] = w2[a * H + u];
  for (int a = 0; a < A; ++a) w2t[H * A4 + a] = b2[a];
}

namespace {
constexpr int kMlpThreads = 256;
constexpr size_t kMlpSmemMax = 227 * 1024 - 1024;   // dynamic budget left beside the static barrier

template <int T>
size_t mlp_smem(int I, int H, int A) {
  const int A4 = (A + 3) / 4 * 4;
  return (size_t)mlp_image_floats(I, H, A) * 4 + ((size_t)I * T + (size_t)H * T + (size_t)T * A4) * 4;
}

template <int T>
__global__ void __launch_bounds__(kMlpThreads, 1)
    k_mlp_tiled(const uint8_t *__restrict__ states, int64_t stride, const float *__restrict__ img, int I, int H,
                int A, int64_t n, int mode, float gd, const float *__restrict__ cum, float *__restrict__ out,
                int feat_f32) {
  extern __shared__ __align__(128) float msm[];
  __shared__ __align__(8) uint64_t bar;
  const int A4 = (A + 3) / 4 * 4, nimg = I * H + H + H * A4 + A4;
  const float *W1T = msm, *b1 = msm + I * H, *W2T = b1 + H, *b2 = W2T + H * A4;
  float *X = msm + nimg, *Hs = X + I * T, *Q = Hs + H * T;
  load_image(msm, img, (uint32_t)nimg * 4, &bar);
  const int64_t ntiles = (n + T - 1) / T;
  const int n_ug = H / 4, n_ag = A4 / 4;
  // features of a tile in 16-byte chunks (4 fp32 or 16 u8 features), fetched into
  // registers one tile ahead so the HBM latency hides under the previous tile's math
  constexpr int KF = (T * 32 + kMlpThreads - 1) / kMlpThreads;   // chunks per thread (I <= 128)
  const int nq = feat_f32 ? I / 4 : I / 16;
  uint4 pf[KF];
  auto fetch = [&](int64_t tt) {
    if (tt >= ntiles) return;
    const int ntt = (int)min((int64_t)T, n - tt * T);
#pragma unroll
    for (int k = 0; k < KF; ++k) {
      const int e = threadIdx.x + k * kMlpThreads;
      if (e < ntt * nq) {
        const int c = e / nq, q = e - c * nq;
        pf[k] = __ldg((const uint4 *)(states + (tt * T + c) * stride) + q);
      }
    }
  };
  fetch(blockIdx.x);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t first = t * T;
    const int nt = (int)min((int64_t)T, n - first);
    // features (prefetched) -> X[i][xcol(c)]
#pragma unroll
    for (int k = 0; k < KF; ++k) {
      const int e = threadIdx.x + k * kMlpThreads;
      if (e < nt * nq) {
        const int c = e / nq, q = e - c * nq, col = xcol<T, 8>(c);
        const uint32_t w[4] = {pf[k].x, pf[k].y, pf[k].z, pf[k].w};
        if (feat_f32) {
#pragma unroll
          for (int j = 0; j < 4; ++j) X[(4 * q + j) * T + col] = __uint_as_float(w[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) X[(16 * q + j) * T + col] = (float)((w[j / 4] >> (8 * (j % 4))) & 0xFFu) / 256.0f;
        }
      }
    }
    __syncthreads();
    fetch(t + gridDim.x);
    // layer 1: Hs[u][c] = relu(b1[u] + chain_i W1[u][i] x_i)
    for (int task = threadIdx.x; task < n_ug * (T / 8); task += kMlpThreads) {
      const int cg = task % (T / 8), ug = task / (T / 8);
      float acc[8][4];
      ffma_tile<T, 8>(W1T, H, b1, X, I, ug, cg, acc);
      store_tile<T, 8>(Hs, ug, cg, acc, true);
    }
    __syncthreads();
    // layer 2: Q[c][a] = b2[a] + chain_u W2[a][u] h_u
    for (int task = threadIdx.x; task < n_ag * T; task += kMlpThreads) {
      const int c = task % T, ag = task / T;
      if (c >= nt) continue;
      const float4 bb = *(const float4 *)(b2 + 4 * ag);
      float q0 = bb.x, q1 = bb.y, q2 = bb.z, q3 = bb.w;
      const float *w = W2T + 4 * ag;
      const float *hc = Hs + xcol<T, 8>(c);
#pragma unroll 8
      for (int u = 0; u < H; ++u) {
        const float h = hc[u * T];
        const float4 wv = *(const float4 *)(w + u * A4);
        q0 = fmaf(wv.x, h, q0);
        q1 = fmaf(wv.y, h, q1);
        q2 = fmaf(wv.z, h, q2);
        q3 = fmaf(wv.w, h, q3);
      }
      *(float4 *)(Q + c * A4 + 4 * ag) = make_float4(q0, q1, q2, q3);
    }
    __syncthreads();
    if (mode == MODE_ROWS) {
      for (int e = threadIdx.x; e < nt * A; e += kMlpThreads) {
        const int c = e / A, a = e - c * A;
        out[(first + c) * A + a] = Q[c * A4 + a];
      }
    } else {
      for (int c = threadIdx.x; c < nt; c += kMlpThreads) {
        float m = Q[c * A4];
        for (int a = 1; a < A; ++a) m = fmaxf(m, Q[c * A4 + a]);
        out[first + c] = mode == MODE_ROWMAX ? m : fmaf(gd, m, cum ? cum[first + c] : 0.0f);
      }
    }
    __syncthreads();   // X / Hs / Q reuse by the next tile
  }
}
}  // namespace

bool mlp_tiled_ok(int I, int H, int A) {
  // I is 64 (INT_HASH bytes, 4 x 16-byte chunks) or 100 (DNN floats, 25 chunks): net_build checks it
  return H % 4 == 0 && I % 4 == 0 && I <= 128 && mlp_smem<32>(I, H, A) <= kMlpSmemMax;
}

void launch_mlp_tiled(const NodeView &v, int64_t n, const float *img, int I, int H, int A, int mode, float gd,
                      float *out, int feat_f32, cudaStream_t st) {
  if (n <= 0) return;
  // the attribute is raised to what this launch needs (static smem counts against the same 227 KB)
  if (mlp_smem<64>(I, H, A) <= kMlpSmemMax) {
    const size_t sm = mlp_smem<64>(I, H, A);
    smem_optin((const void *)k_mlp_tiled<64>, (int)sm);
    const unsigned grid = (unsigned)std::min<int64_t>((n + 63) / 64, sm_count());
    k_mlp_tiled<64><<<grid, kMlpThreads, sm, st>>>(v.state, v.state_stride, img, I, H, A, n, mode, gd, v.cum, out,
                                                   feat_f32);
  } else {
    const size_t sm = mlp_smem<32>(I, H, A);
    smem_optin((const void *)k_mlp_tiled<32>, (int)sm);
    const unsigned grid = (unsigned)std::min<int64_t>((n + 31) / 32, sm_count());
    k_mlp_tiled<32><<<grid, kMlpThreads, sm, st>>>(v.state, v.state_stride, img, I, H, A, n, mode, gd, v.cum, out,
                                                   feat_f32);
  }
}

}  // namespace bcts
