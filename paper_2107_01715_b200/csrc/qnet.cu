// qnet.cu -- K2: the leaf value network Q_theta (Alg. 1 leaf line, P:323:
// R <- R + gamma^d max_a Q_theta(S, a)), its weight repack (E2) and the
// non-tensor-core pieces: TABLE gather, fp32 MLP (fixed-order fmaf chains,
// DESIGN.md R3), the SIMT reference implicit-GEMM layer, and the heads
// (Nature fc2 / Rainbow dueling C51 expectation) with fused max_a and
// fmaf(g_d, max_a Q, R) epilogue. The tcgen05 layer lives in qnet_tc.cu.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include <cuda_fp16.h>

#include "engine.h"

namespace bcts {

// ------------------------------------------------------------------ TABLE
__global__ void k_table(const int32_t *__restrict__ ids, int64_t stride_bytes, const float *__restrict__ tq, int A,
                        int64_t n, int mode, float gd, const float *__restrict__ cum, float *__restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t s = *(const int32_t *)((const uint8_t *)ids + i * stride_bytes);
  const float *q = tq + (int64_t)s * A;
  float m = q[0];
  for (int a = 0; a < A; ++a) {
    if (mode == MODE_ROWS) out[i * A + a] = q[a];
    m = q[a] > m ? q[a] : m;
  }
  if (mode == MODE_ROWMAX) out[i] = m;
  if (mode == MODE_TOTAL) out[i] = fmaf(gd, m, cum ? cum[i] : 0.0f);
}

// ------------------------------------------------------------------ MLP2
// One warp per state. x_j = byte j of the state / 256 (exact; INT_HASH) or the
// j-th fp32 state component (DNN env, feat_f32); hidden unit u:
// acc = b1[u]; acc = fmaf(W1[u][i], x_i, acc) for i = 0..in-1; h = acc > 0 ? acc : 0.
// Output a: acc = b2[a]; acc = fmaf(W2[a][u], h_u, acc) for u = 0..hid-1.
constexpr int kMlpWarps = 4;
__global__ void __launch_bounds__(32 * kMlpWarps)
    k_mlp(const uint8_t *__restrict__ states, int64_t stride_bytes, const float *__restrict__ w1,
          const float *__restrict__ b1, const float *__restrict__ w2, const float *__restrict__ b2, int IN, int H,
          int A, int64_t n, int mode, float gd, const float *__restrict__ cum, float *__restrict__ out,
          int feat_f32) {
  __shared__ float xs[kMlpWarps][128];
  __shared__ float hs[kMlpWarps][1024];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t i = (int64_t)blockIdx.x * kMlpWarps + warp;
  if (i >= n) return;
  const uint8_t *s = states + i * stride_bytes;
  if (feat_f32)
    for (int j = lane; j < IN; j += 32) xs[warp][j] = ((const float *)s)[j];
  else
    for (int j = lane; j < IN; j += 32) xs[warp][j] = (float)s[j] / 256.0f;
  __syncwarp();
  for (int u = lane; u < H; u += 32) {
    float acc = b1[u];
    const float *w = w1 + (int64_t)u * IN;
    for (int k = 0; k < IN; ++k) acc = fmaf(w[k], xs[warp][k], acc);
    hs[warp][u] = acc > 0.0f ? acc : 0.0f;
  }
  __syncwarp();
  float m = -INFINITY;
  for (int a0 = 0; a0 < A; a0 += 32) {
    const int a = a0 + lane;
    float q = -INFINITY;
    if (a < A) {
      float acc = b2[a];
      const float *w = w2 + (int64_t)a * H;
      for (int u = 0; u < H; ++u) acc = fmaf(w[u], hs[warp][u], acc);
      q = acc;
      if (mode == MODE_ROWS) out[i * A + a] = q;
    }
    m = fmaxf(m, q);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) {
    if (mode == MODE_ROWMAX) out[i] = m;
    if (mode == MODE_TOTAL) out[i] = fmaf(gd, m, cum ? cum[i] : 0.0f);
  }
}

// ------------------------------------------------------- SIMT implicit GEMM
// Reference layer (BCTS_F_SIMT_NET, and the parity baseline for tcgen05):
// 64x64 output tile per CTA, K step 32, fp32 FMA accumulation of bf16 operands.
__device__ __forceinline__ float gather_x(const Layer &L, const void *in, int64_t m, int k) {
  const int64_t rows = (int64_t)L.OH * L.OW;
  const int64_t img = m / rows;
  const int pos = (int)(m - img * rows);
  const int oy = pos / L.OW, ox = pos - oy * L.OW;
  const int kwc = L.KW * L.C;
  const int ky = k / kwc, r = k - ky * kwc;
  const int kx = r / L.C, c = r - kx * L.C;
  const int64_t idx =
      img * L.in_img_stride + L.in_col_off + ((int64_t)(oy * L.S + ky) * L.W + (ox * L.S + kx)) * L.C + c;
  if (L.in_u8) return (float)((const uint8_t *)in)[idx];
  return __bfloat162float(((const __nv_bfloat16 *)in)[idx]);
}

constexpr int kSimtBM = 64, kSimtBN = 64, kSimtBK = 32;
__global__ void __launch_bounds__(256) k_layer_simt(Layer L, const void *__restrict__ in, int64_t M,
                                                    void *__restrict__ out) {
  __shared__ float As[kSimtBK][kSimtBM + 4];
  __shared__ float Bs[kSimtBK][kSimtBN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = (int64_t)blockIdx.x * kSimtBM;
  const int n0 = blockIdx.y * kSimtBN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < L.K; k0 += kSimtBK) {
    for (int e = threadIdx.x; e < kSimtBM * kSimtBK; e += 256) {
      const int mm = e / kSimtBK, kk = e % kSimtBK;
      const int64_t m = m0 + mm;
      const int k = k0 + kk;
      As[kk][mm] = (m < M && k < L.K) ? gather_x(L, in, m, k) : 0.0f;
      const int n = n0 + mm;
      Bs[kk][mm] = (n < L.Npad && k < L.K) ? __bfloat162float(L.Wt[(int64_t)n * L.K + k]) : 0.0f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < kSimtBK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= L.Npad) continue;
      const float v = acc[i][j] + L.bias[n];
      if (L.relu_bf16)
        ((__nv_bfloat16 *)out)[m * L.out_ld + n] = __float2bfloat16_rn(v > 0.0f ? v : 0.0f);
      else
        ((float *)out)[m * L.out_ld + n] = v;
    }
  }
}

void launch_layer_simt(const Layer &L, const void *in, int64_t n_img, void *out, cudaStream_t st) {
  const int64_t M = n_img * L.rows_per_img();
  dim3 grid((unsigned)((M + kSimtBM - 1) / kSimtBM), (unsigned)((L.Npad + kSimtBN - 1) / kSimtBN));
  k_layer_simt<<<grid, 256, 0, st>>>(L, in, M, out);
}

// ------------------------------------------------------------------ heads
// One warp per image. Nature: q_a = z[a]. Rainbow (dueling C51, R15):
// logits[a][i] = v_i + adv[a][i] - mean_a adv[a][i]; p = softmax_i; q_a = sum_i z_i p.
template <bool RAINBOW>
__global__ void __launch_bounds__(128) k_head(const float *__restrict__ zv, int64_t ldv, const float *__restrict__ za,
                                              int64_t lda, int A, int atoms, float vmin, float dz, int64_t n, int mode,
                                              float gd, const float *__restrict__ cum, float *__restrict__ out) {
  const int lane = threadIdx.x % 32;
  const int64_t i = (int64_t)blockIdx.x * 4 + threadIdx.x / 32;
  if (i >= n) return;
  float best = -INFINITY;
  if (!RAINBOW) {
    for (int a0 = 0; a0 < A; a0 += 32) {
      const int a = a0 + lane;
      float q = -INFINITY;
      if (a < A) {
        q = za[i * lda + a];
        if (mode == MODE_ROWS) out[i * A + a] = q;
      }
      best = fmaxf(best, q);
    }
    for (int o = 16; o > 0; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
  } else {
    const float *v = zv + i * ldv;
    const float *adv = za + i * lda;
    float vi[2], mean[2], zi[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int at = lane + 32 * t;
      vi[t] = 0.f; mean[t] = 0.f; zi[t] = 0.f;
      if (at < atoms) {
        vi[t] = v[at];
        float s = 0.f;
        for (int a = 0; a < A; ++a) s += adv[a * atoms + at];
        mean[t] = s / (float)A;
        zi[t] = vmin + (float)at * dz;
      }
    }
    for (int a = 0; a < A; ++a) {
      float lg[2], mx = -INFINITY;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int at = lane + 32 * t;
        lg[t] = at < atoms ? vi[t] + adv[a * atoms + at] - mean[t] : -INFINITY;
        mx = fmaxf(mx, lg[t]);
      }
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      float den = 0.f, num = 0.f;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int at = lane + 32 * t;
        if (at < atoms) {
          const float e = expf(lg[t] - mx);
          den += e;
          num += zi[t] * e;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        den += __shfl_xor_sync(0xffffffffu, den, o);
        num += __shfl_xor_sync(0xffffffffu, num, o);
      }
      const float q = num / den;
      if (mode == MODE_ROWS && lane == 0) out[i * A + a] = q;
      best = fmaxf(best, q);
    }
  }
  if (lane == 0) {
    if (mode == MODE_ROWMAX) out[i] = best;
    if (mode == MODE_TOTAL) out[i] = fmaf(gd, best, cum ? cum[i] : 0.0f);
  }
}

// Rainbow head, block-staged: 8 leaves per CTA. Their z rows are loaded into
// shared memory with coalesced float4 loads, then one thread per (leaf, action)
// computes the softmax expectation over the atoms (mean_a adv[a][i] shared per
// leaf); fused max_a and fmaf(g_d, max, R_d).
constexpr int kHeadLeaves = 8;
template <int ATOMS>
__global__ void __launch_bounds__(256) k_head_rainbow(const float *__restrict__ zv, int64_t ldv,
                                                      const float *__restrict__ za, int64_t lda, int A, float vmin,
                                                      float dz, int64_t n, int mode, float gd,
                                                      const float *__restrict__ cum, float *__restrict__ out) {
  extern __shared__ float hsm[];
  const int AN = (A * ATOMS + 3) & ~3;              // smem row stride (float4 staging; lda >= AN)
  float *sa = hsm;                                  // [kHeadLeaves][AN]
  float *svm = sa + kHeadLeaves * AN;               // [kHeadLeaves][ATOMS]: v_i - mean_a adv[a][i]
  float *sq = svm + kHeadLeaves * ATOMS;            // [kHeadLeaves][A]
  const int64_t l0 = (int64_t)blockIdx.x * kHeadLeaves;
  const int nl = n - l0 < kHeadLeaves ? (int)(n - l0) : kHeadLeaves;
  // coalesced staging (lda and AN are multiples of 4 floats)
  for (int l = 0; l < nl; ++l) {
    const float4 *src = (const float4 *)(za + (l0 + l) * lda);
    float4 *dst = (float4 *)(sa + l * AN);
    for (int e = threadIdx.x; e < AN / 4; e += blockDim.x) dst[e] = src[e];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nl * ATOMS; e += blockDim.x) {
    const int l = e / ATOMS, t = e - l * ATOMS;
    float s = 0.0f;
    for (int a = 0; a < A; ++a) s += sa[l * AN + a * ATOMS + t];
    svm[e] = zv[(l0 + l) * ldv + t] - s / (float)A;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nl * A; e += blockDim.x) {
    const int l = e / A, a = e - l * A;
    const float *ad = sa + l * AN + a * ATOMS;
    const float *vm = svm + l * ATOMS;
    float mx = -INFINITY;
#pragma unroll 17
    for (int t = 0; t < ATOMS; ++t) mx = fmaxf(mx, vm[t] + ad[t]);
    float den = 0.0f, num = 0.0f;
#pragma unroll 17
    for (int t = 0; t < ATOMS; ++t) {
      const float ex = expf(vm[t] + ad[t] - mx);
      den += ex;
      num += (vmin + (float)t * dz) * ex;
    }
    const float q = num / den;
    sq[e] = q;
    if (mode == MODE_ROWS) out[(l0 + l) * A + a] = q;
  }
  __syncthreads();
  if (mode != MODE_ROWS && threadIdx.x < nl) {
    const int l = threadIdx.x;
    float best = -INFINITY;
    for (int a = 0; a < A; ++a) best = fmaxf(best, sq[l * A + a]);
    if (mode == MODE_ROWMAX) out[l0 + l] = best;
    else out[l0 + l] = fmaf(gd, best, cum ? cum[l0 + l] : 0.0f);
  }
}

// ------------------------------------------------------------ build / eval
static int round_up(int x, int m) { return (x + m - 1) / m * m; }

static cudaError_t upload(Net &net, const void *h, size_t bytes, void **d) {
  cudaError_t e = cudaMalloc(d, bytes ? bytes : 16);
  if (e != cudaSuccess) return e;
  net.allocs.push_back(*d);
  return cudaMemcpy(*d, h, bytes, cudaMemcpyHostToDevice);
}

// Repack an OIHW conv weight (or [N][K] linear) into [Npad][K] bf16 with
// k = (ky, kx, c); rows >= O are zero. src_index(o, ky, kx, c) -> canonical index.
template <class F>
static std::vector<__nv_bfloat16> repack(int O, int Npad, int KH, int KW, int C, F src_index, const float *w) {
  const int K = KH * KW * C;
  std::vector<__nv_bfloat16> out((size_t)Npad * K, __float2bfloat16_rn(0.0f));
  for (int o = 0; o < O; ++o)
    for (int ky = 0; ky < KH; ++ky)
      for (int kx = 0; kx < KW; ++kx)
        for (int c = 0; c < C; ++c)
          out[(size_t)o * K + (ky * KW + kx) * C + c] = __float2bfloat16_rn(w[(int64_t)src_index(o, ky, kx, c)]);
  return out;
}

static int make_layer(Net &net, Layer &L, std::vector<__nv_bfloat16> &&wt, const float *bias, int N, int Npad,
                      std::string &err) {
  std::vector<float> b((size_t)Npad, 0.0f);
  for (int i = 0; i < N; ++i) b[i] = bias[i];
  void *dw = nullptr, *db = nullptr;
  if (upload(net, wt.data(), wt.size() * sizeof(__nv_bfloat16), &dw) != cudaSuccess ||
      upload(net, b.data(), b.size() * sizeof(float), &db) != cudaSuccess) {
    err = "cudaMalloc/cudaMemcpy of weights failed";
    return -1;
  }
  L.Wt = (const __nv_bfloat16 *)dw;
  L.bias = (const float *)db;
  L.N = N;
  L.Npad = Npad;
  return 0;
}

int net_build(Net &net, const bcts_config &cfg, std::string &err) {
  net.kind = cfg.net;
  net.A = cfg.num_actions;
  const int A = net.A;
  if (cfg.net == BCTS_NET_TABLE) {
    if (!cfg.tab_q || cfg.num_states <= 0) { err = "TABLE net needs tab_q and num_states"; return -1; }
    void *d = nullptr;
    if (upload(net, cfg.tab_q, sizeof(float) * (size_t)cfg.num_states * A, &d) != cudaSuccess) {
      err = "upload tab_q failed";
      return -1;
    }
    net.tq = (const float *)d;
    net.nS = cfg.num_states;
    return 0;
  }
  if (!cfg.weights) { err = "weights required"; return -1; }
  const float *w = cfg.weights;
  if (cfg.net == BCTS_NET_MLP2_F32) {
    const int I = cfg.mlp_in, H = cfg.mlp_hidden;
    const int want_in = cfg.env == BCTS_ENV_DNN ? kDnnS : 64;
    if (I != want_in || H < 1 || H > 1024) {
      err = "MLP2 needs mlp_in == 64 (INT_HASH) / 100 (DNN) and 1 <= mlp_hidden <= 1024";
      return -1;
    }
    net.feat_f32 = cfg.env == BCTS_ENV_DNN;
    const int64_t need = (int64_t)H * I + H + (int64_t)A * H + A;
    if (cfg.weights_count != need) { err = "weights_count mismatch for MLP2"; return -1; }
    void *p[4];
    const size_t sz[4] = {(size_t)H * I, (size_t)H, (size_t)A * H, (size_t)A};
    for (int t = 0; t < 4; ++t) {
      if (upload(net, w, sz[t] * sizeof(float), &p[t]) != cudaSuccess) { err = "upload MLP failed"; return -1; }
      w += sz[t];
    }
    net.l1w = (const float *)p[0]; net.l1b = (const float *)p[1];
    net.l2w = (const float *)p[2]; net.l2b = (const float *)p[3];
    net.in = I; net.hid = H;
    if (mlp_tiled_ok(I, H, A)) {
      std::vector<float> img((size_t)mlp_image_floats(I, H, A));
      const float *c = cfg.weights;
      mlp_repack(c, c + (size_t)H * I, c + (size_t)H * I + H, c + (size_t)H * I + H + (size_t)A * H, I, H, A,
                 img.data());
      void *d;
      if (upload(net, img.data(), img.size() * sizeof(float), &d) != cudaSuccess) { err = "upload MLP image"; return -1; }
      net.mlp_img = (const float *)d;
    }
    if (cfg.flags & BCTS_F_TF32) {
      if (!mlp_tc_ok(I, H, A)) { err = "BCTS_F_TF32: MLP2 needs mlp_hidden % 16 == 0, <= 256 and A <= 64"; return -1; }
      std::vector<uint8_t> img(mlp_tc_image_bytes(I, H, A));
      const float *c = cfg.weights;
      mlp_tc_repack(c, c + (size_t)H * I, c + (size_t)H * I + H, c + (size_t)H * I + H + (size_t)A * H, I, H, A,
                    img.data());
      void *d;
      if (upload(net, img.data(), img.size(), &d) != cudaSuccess) { err = "upload tf32 MLP image"; return -1; }
      net.mlp_tc_img = (const uint8_t *)d;
    }
    return 0;
  }
  const bool rainbow = cfg.net == BCTS_NET_RAINBOW_BF16;
  if (!rainbow && cfg.net != BCTS_NET_NATURE_BF16) { err = "unknown net kind"; return -1; }
  const int atoms = rainbow ? cfg.atoms : 0;
  if (rainbow && (atoms < 2 || atoms > 64)) { err = "atoms must be in [2, 64]"; return -1; }
  int64_t need = 32 * 256 + 32 + 64 * 512 + 64 + 64 * 576 + 64;
  need += rainbow ? 2 * (512LL * 3136 + 512) + (int64_t)atoms * 512 + atoms + (int64_t)A * atoms * 512 + A * atoms
                  : 512LL * 3136 + 512 + (int64_t)A * 512 + A;
  if (cfg.weights_count != need) { err = "weights_count mismatch for conv net"; return -1; }
  net.atoms = atoms;
  net.vmin = cfg.v_min;
  net.vmax = cfg.v_max;
  // conv1: OIHW [32][4][8][8] over uint8 NHWC frames, computed as a 2x2
  // stride-1 conv over the space-to-depth(4) bf16 frame S[21][21][64] with
  // c' = (dy*4 + dx)*4 + c:  W'[o][(ty*2 + tx)*64 + c'] = W[o][c][4ty+dy][4tx+dx].
  {
    Layer &L = net.c1;
    L.H = L.W = 21; L.C = 64; L.KH = L.KW = 2; L.S = 1; L.OH = L.OW = 20; L.K = 256;
    L.relu_bf16 = 1; L.out_ld = 32; L.in_img_stride = 21 * 21 * 64;
    auto src = [](int o, int ty, int tx, int cp) {
      const int c = cp & 3, dx = (cp >> 2) & 3, dy = cp >> 4;
      return ((o * 4 + c) * 8 + (4 * ty + dy)) * 8 + (4 * tx + dx);
    };
    if (make_layer(net, L, repack(32, 32, 2, 2, 64, src, w), w + 32 * 256, 32, 32, err)) return -1;
    // sibling-factorised conv1: child frames 0..2 (= parent frames 1..3) and frame 3,
    // channel order (c, dy, dx) inside an s2d pixel:
    //   W_shared[o][tap*48 + c*16 + dy*4 + dx] = W[o][c][4ty+dy][4tx+dx]   (c = 0..2)
    //   W_new[o][tap*16 + dy*4 + dx]           = W[o][3][4ty+dy][4tx+dx]
    // This path runs its MMAs in fp16 (kind::f16, f16 operands): frame bytes are
    // exact in fp16 and convert with one PRMT + one HADD2 per pair. The weights are
    // the bf16 weights of R15 scaled by 2^14: fp16(bf16(w) * 2^14) is EXACT (8
    // significant bits, scaled into fp16's normal range), every product and fp32
    // partial sum is then exactly 2^14 x the bf16 one, and the epilogue's 2^-14
    // undoes it -- the same accumulator as a bf16 MMA, with cheaper conversions.
    {
      auto sw_image = [](const std::vector<__half> &wl, int Nr, int K) {
        std::vector<__half> img((size_t)Nr * K);
        uint8_t *dst = (uint8_t *)img.data();
        for (int n = 0; n < Nr; ++n)
          for (int kb = 0; kb < K / 64; ++kb)
            for (int j = 0; j < 8; ++j)
              memcpy(dst + (size_t)kb * Nr * 128 + (n / 8) * 1024 + (n % 8) * 128 + ((j ^ (n % 8)) * 16),
                     (const uint8_t *)(wl.data() + (size_t)n * K + kb * 64) + j * 16, 16);
        return img;
      };
#ifndef SIB_F16
#define SIB_F16 1
#endif
#if SIB_F16
      auto f16s = [](float x) { return __float2half_rn(__bfloat162float(__float2bfloat16_rn(x)) * 16384.0f); };
#else
      auto f16s = [](float x) { __nv_bfloat16 b = __float2bfloat16_rn(x); return *(__half *)&b; };   // bf16 bits
#endif
      std::vector<__half> wsh((size_t)32 * 192), wnw((size_t)32 * 64);
      for (int o = 0; o < 32; ++o)
        for (int tap = 0; tap < 4; ++tap) {
          const int ty = tap >> 1, tx = tap & 1;
          for (int dy = 0; dy < 4; ++dy)
            for (int dx = 0; dx < 4; ++dx) {
              for (int c = 0; c < 3; ++c)
                wsh[(size_t)o * 192 + tap * 48 + c * 16 + dy * 4 + dx] =
                    f16s(w[((o * 4 + c) * 8 + 4 * ty + dy) * 8 + 4 * tx + dx]);
              wnw[(size_t)o * 64 + tap * 16 + dy * 4 + dx] = f16s(w[((o * 4 + 3) * 8 + 4 * ty + dy) * 8 + 4 * tx + dx]);
            }
        }
      std::vector<__half> a = sw_image(wsh, 32, 192), b = sw_image(wnw, 32, 64);
      void *da = nullptr, *db = nullptr;
      if (upload(net, a.data(), a.size() * 2, &da) != cudaSuccess || upload(net, b.data(), b.size() * 2, &db) != cudaSuccess) {
        err = "upload factorised conv1 weights";
        return -1;
      }
      net.w1_shared = (const uint8_t *)da;
      net.w1_new = (const uint8_t *)db;
    }
    w += 32 * 256 + 32;
  }
  {
    Layer &L = net.c2;
    L.H = L.W = 20; L.C = 32; L.KH = L.KW = 4; L.S = 2; L.OH = L.OW = 9; L.K = 512; L.relu_bf16 = 1; L.out_ld = 64;
    L.in_img_stride = 20 * 20 * 32;
    if (make_layer(net, L, repack(64, 64, 4, 4, 32, [](int o, int ky, int kx, int c) { return ((o * 32 + c) * 4 + ky) * 4 + kx; }, w),
                   w + 64 * 512, 64, 64, err)) return -1;
    // the same conv as a 2x2 stride-1 conv over space-to-depth(2) of act1
    // (c2 = (dy*2 + dx)*32 + c): W'[o][(ty*2 + tx)*128 + c2] = W[o][c][2ty+dy][2tx+dx]
    Layer &S = net.c2s;
    S = L;
    S.H = S.W = 10; S.C = 128; S.KH = S.KW = 2; S.S = 1;
    auto src2 = [](int o, int ty, int tx, int c2) {
      const int c = c2 & 31, dx = (c2 >> 5) & 1, dy = c2 >> 6;
      return ((o * 32 + c) * 4 + (2 * ty + dy)) * 4 + (2 * tx + dx);
    };
    if (make_layer(net, S, repack(64, 64, 2, 2, 128, src2, w), w + 64 * 512, 64, 64, err)) return -1;
    w += 64 * 512 + 64;
  }
  {
    Layer &L = net.c3;
    L.H = L.W = 9; L.C = 64; L.KH = L.KW = 3; L.S = 1; L.OH = L.OW = 7; L.K = 576; L.relu_bf16 = 1; L.out_ld = 64;
    L.in_img_stride = 9 * 9 * 64;
    if (make_layer(net, L, repack(64, 64, 3, 3, 64, [](int o, int ky, int kx, int c) { return ((o * 64 + c) * 3 + ky) * 3 + kx; }, w),
                   w + 64 * 576, 64, 64, err)) return -1;
    w += 64 * 576 + 64;
  }
  // fc over the 7x7x64 conv3 output: PyTorch flattens NCHW (c*49 + y*7 + x) (R25);
  // our activations are NHWC, so k = (y, x, c) <- canonical c*49 + y*7 + x.
  auto fc_src = [](int o, int y, int x, int c) { return (int64_t)o * 3136 + c * 49 + y * 7 + x; };
  const int hidN = rainbow ? 1024 : 512;
  {
    Layer &L = net.fc_h;
    L.H = L.W = 7; L.C = 64; L.KH = L.KW = 7; L.S = 1; L.OH = L.OW = 1; L.K = 3136; L.relu_bf16 = 1; L.out_ld = hidN;
    L.in_img_stride = 3136;
    std::vector<__nv_bfloat16> wt;
    std::vector<float> b(hidN);
    if (!rainbow) {
      wt = repack(512, 512, 7, 7, 64, [&](int o, int y, int x, int c) { return fc_src(o, y, x, c); }, w);
      for (int i = 0; i < 512; ++i) b[i] = w[512 * 3136 + i];
      w += 512 * 3136 + 512;
    } else {
      // rows 0..511 = fc_h_v, 512..1023 = fc_h_a (one GEMM, concatenated)
      const float *wv = w, *bv = w + 512 * 3136, *wa = bv + 512, *ba = wa + 512 * 3136;
      wt = repack(512, 512, 7, 7, 64, fc_src, wv);
      std::vector<__nv_bfloat16> wta = repack(512, 512, 7, 7, 64, fc_src, wa);
      wt.insert(wt.end(), wta.begin(), wta.end());
      for (int i = 0; i < 512; ++i) { b[i] = bv[i]; b[512 + i] = ba[i]; }
      w = ba + 512;
    }
    if (make_layer(net, L, std::move(wt), b.data(), hidN, hidN, err)) return -1;
  }
  if (!rainbow) {
    Layer &L = net.fc2;
    const int Np = round_up(A, 16);
    L.H = L.W = 1; L.C = 512; L.K = 512; L.relu_bf16 = 0; L.out_ld = Np; L.in_img_stride = 512;
    if (make_layer(net, L, repack(A, Np, 1, 1, 512, [](int o, int, int, int c) { return o * 512 + c; }, w),
                   w + A * 512, A, Np, err)) return -1;
    w += A * 512 + A;
    net.ld_za = Np;
  } else {
    Layer &V = net.z_v;
    const int Nv = round_up(atoms, 16);
    V.H = V.W = 1; V.C = 512; V.K = 512; V.relu_bf16 = 0; V.out_ld = Nv; V.in_img_stride = 1024; V.in_col_off = 0;
    if (make_layer(net, V, repack(atoms, Nv, 1, 1, 512, [](int o, int, int, int c) { return o * 512 + c; }, w),
                   w + atoms * 512, atoms, Nv, err)) return -1;
    if (atoms <= 64) {
      for (int t = 0; t < atoms; ++t) net.head.bias.v[t] = w[atoms * 512 + t];
      for (int t = 0; t < 64; ++t)   // the kernel's former in-loop support value, fmaf(t, dz, v_min)
        net.head.bias.z[t] = std::fmaf((float)t, (net.vmax - net.vmin) / (float)(atoms - 1), net.vmin);
    }
    w += atoms * 512 + atoms;
    Layer &Z = net.z_a;
    const int Na = round_up(A * atoms, 16);
    Z.H = Z.W = 1; Z.C = 512; Z.K = 512; Z.relu_bf16 = 0; Z.out_ld = Na; Z.in_img_stride = 1024; Z.in_col_off = 512;
    if (make_layer(net, Z, repack(A * atoms, Na, 1, 1, 512, [](int o, int, int, int c) { return o * 512 + c; }, w),
                   w + A * atoms * 512, A * atoms, Na, err)) return -1;
    if (atoms <= 64) {   // fused-head copy of z_a: action a owns rows a*64 .. a*64+atoms-1 (zero pad)
      std::vector<__nv_bfloat16> wa64((size_t)A * 64 * 512, __float2bfloat16_rn(0.0f));
      std::vector<float> ba64((size_t)A * 64, 0.0f);
      for (int a = 0; a < A; ++a)
        for (int t = 0; t < atoms; ++t) {
          for (int c = 0; c < 512; ++c)
            wa64[((size_t)a * 64 + t) * 512 + c] = __float2bfloat16_rn(w[((size_t)a * atoms + t) * 512 + c]);
          ba64[(size_t)a * 64 + t] = w[(size_t)A * atoms * 512 + a * atoms + t];
        }
      // sum over actions of the bf16 z_a weights (exact in double) as a bf16 hi + lo pair,
      // and of the fp32 biases (double, rounded once)
      std::vector<__nv_bfloat16> ws((size_t)128 * 512, __float2bfloat16_rn(0.0f));
      std::vector<float> bs(64, 0.0f);
      for (int t = 0; t < atoms; ++t) {
        for (int c = 0; c < 512; ++c) {
          double acc = 0.0;
          for (int a = 0; a < A; ++a) acc += (double)__bfloat162float(wa64[((size_t)a * 64 + t) * 512 + c]);
          const __nv_bfloat16 hi = __float2bfloat16_rn((float)acc);
          ws[(size_t)t * 512 + c] = hi;
          ws[(size_t)(64 + t) * 512 + c] = __float2bfloat16_rn((float)(acc - (double)__bfloat162float(hi)));
        }
        double bacc = 0.0;
        for (int a = 0; a < A; ++a) bacc += (double)ba64[(size_t)a * 64 + t];
        bs[t] = (float)bacc;
      }
      // the fused head streams z_a in chunks of 4 actions packed at 51 rows each (chunk c: rows
      // kHeadChunkRows c + 51 s + t for action 4 c + s; rows 204..207 of a chunk zero), so a
      // chunk's MMA is N = 208 instead of 4 x 64 padded rows
      const int nch = (A + 3) / 4;
      std::vector<__nv_bfloat16> wpk((size_t)nch * kHeadChunkRows * 512, __float2bfloat16_rn(0.0f));
      for (int a = 0; a < A; ++a)
        for (int t = 0; t < atoms; ++t)
          for (int c = 0; c < 512; ++c)
            wpk[((size_t)(a / 4) * kHeadChunkRows + (size_t)(a % 4) * atoms + t) * 512 + c] =
                wa64[((size_t)a * 64 + t) * 512 + c];
      void *dw = nullptr, *db = nullptr, *dws = nullptr, *dbs = nullptr;
      if (upload(net, wpk.data(), wpk.size() * 2, &dw) != cudaSuccess ||
          upload(net, ba64.data(), ba64.size() * 4, &db) != cudaSuccess ||
          upload(net, ws.data(), ws.size() * 2, &dws) != cudaSuccess ||
          upload(net, bs.data(), bs.size() * 4, &dbs) != cudaSuccess) {
        err = "upload fused-head weights";
        return -1;
      }
      net.wa64 = (const __nv_bfloat16 *)dw;
      net.ba64 = (const float *)db;
      net.wsum = (const __nv_bfloat16 *)dws;
      net.bsum = (const float *)dbs;
      if (A <= 64) {
        for (int t = 0; t < 64; ++t) net.head.bias.sum[t] = bs[t];
        for (size_t e = 0; e < ba64.size(); ++e) net.head.bias.a64[e] = ba64[e];
      }
    }
    w += (int64_t)A * atoms * 512 + A * atoms;
    net.ld_zv = Nv;
    net.ld_za = Na;
  }
  // Batch capacity = six waves of 128-row M tiles (6 x 148 x 128 = 113,664 images): eval_conv
  // splits a call into equal batches of at most this size (rounded to 128 rows), so no batch is a
  // thin tail. Several tiles per SM let the fc / head kernels overlap one tile's loads with
  // another's math, and fewer batches mean fewer kernel tails (measured on C5: 1 wave 2.41 ms/step,
  // 2 waves 2.33, 3 waves 2.31, 6 waves -- the whole 104,976-leaf level in one batch -- 2.28). The
  // materialised-state path (s2d input, act2) keeps one wave of sub-batch: it only scores small
  // sets. Scratch at 6 waves: ~4.2 GB of act1 + ~1 GB of act3 / hidden / head buffers.
  const int64_t waves = 6;
  net.batch = 148 * 128 * waves;
  net.fc_batch = 148 * 128 * waves;
  net.mat_batch = 148 * 128;
  const int64_t B = net.batch, FB = net.fc_batch, MB = net.mat_batch;
  const bool simt = (cfg.flags & BCTS_F_SIMT_NET) != 0;   // dense NHWC trunk buffers only for the SIMT path
  net.simt = simt;
  // scratch (device memory bound later by net_bind_scratch: library-owned or caller-provided)
  const size_t bytes[kNetScratch] = {simt ? (size_t)MB * 400 * 32 * 2 : 0, simt ? (size_t)MB * 81 * 64 * 2 : 0,
                                     (size_t)FB * 49 * 64 * 2, (size_t)FB * hidN * 2,
                                     (size_t)FB * (rainbow ? net.ld_zv : 16) * 4, (size_t)FB * net.ld_za * 4,
                                     simt ? (size_t)MB * 21 * 21 * 64 * 2 : 0, (size_t)FB * 4, (size_t)MB * kIn1Bytes,
                                     (size_t)B * kIn2Bytes, (size_t)MB * kIn3Bytes};
  for (int t = 0; t < kNetScratch; ++t) net.scratch_sz[t] = bytes[t];
  // shifted-window trunk geometry (qnet_conv.cu)
  {
    ConvSW &a = net.sw1;
    a.N = 32; a.K = 256; a.Cin = 64; a.KH = a.KW = 2; a.W_in = 21; a.OH = a.OW = 20; a.n_mt = (20 * 21 + 127) / 128;
    a.plane = kPlane1; a.in_img_bytes = kIn1Bytes; a.in_rows = 21 * 21;
    a.out_mode = 0; a.out_plane = kPlane2; a.out_w = 10; a.out_img_bytes = kIn2Bytes;
    ConvSW &b = net.sw2;
    b.N = 64; b.K = 512; b.Cin = 128; b.KH = b.KW = 2; b.W_in = 10; b.OH = b.OW = 9; b.n_mt = (9 * 10 + 127) / 128;
    b.plane = kPlane2; b.in_img_bytes = kIn2Bytes; b.in_rows = 10 * 10;
    b.out_mode = 1; b.out_plane = kPlane3; b.out_w = 9; b.out_img_bytes = kIn3Bytes;
    ConvSW &c = net.sw3;
    c.N = 64; c.K = 576; c.Cin = 64; c.KH = c.KW = 3; c.W_in = 9; c.OH = c.OW = 7; c.n_mt = (7 * 9 + 127) / 128;
    c.plane = kPlane3; c.in_img_bytes = kIn3Bytes; c.in_rows = 9 * 9;
    c.out_mode = 2; c.out_plane = 0; c.out_w = 7; c.out_img_bytes = 3136 * 2;
    const int layout = 2;   // SW128 row blocks, address-based swizzle (the compiled MMA loop assumes it)
    a.layout = b.layout = c.layout = layout;
    // weights of each shifted-window layer as the exact SW128 shared-memory
    // image the kernel wants (K/64 blocks of [N rows x 128 B], 16-byte chunk
    // j of row n at (n/8)*1024 + (n%8)*128 + ((j ^ n%8) * 16)): one bulk copy
    ConvSW *cs[3] = {&a, &b, &c};
    const Layer *ls[3] = {&net.c1, &net.c2s, &net.c3};
    for (int t = 0; t < 3; ++t) {
      const int N = cs[t]->N, K = cs[t]->K, nkb = K / 64;
      std::vector<__nv_bfloat16> hw((size_t)N * K), img((size_t)N * K);
      cudaMemcpy(hw.data(), ls[t]->Wt, hw.size() * 2, cudaMemcpyDeviceToHost);
      uint8_t *dst = (uint8_t *)img.data();
      for (int n = 0; n < N; ++n)
        for (int kb = 0; kb < nkb; ++kb)
          for (int j = 0; j < 8; ++j)
            memcpy(dst + (size_t)kb * N * 128 + (n / 8) * 1024 + (n % 8) * 128 + ((j ^ (n % 8)) * 16),
                   (const uint8_t *)(hw.data() + (size_t)n * K + kb * 64) + j * 16, 16);
      void *d = nullptr;
      if (upload(net, img.data(), img.size() * 2, &d) != cudaSuccess) { err = "upload swizzled weights"; return -1; }
      cs[t]->wsw = (const uint8_t *)d;
      if (t == 1) {   // conv2 tap pairs for k_conv23: k-block (pr, kb) = [128 rows x 128 B], row n < 64 =
                      // tap (pr, 0) channel n, row n >= 64 = tap (pr, 1) channel n - 64; K = s2d channels
                      // kb*64 .. kb*64+63 of that tap (k = tap*128 + c2 in hw)
        std::vector<__nv_bfloat16> pimg((size_t)4 * 128 * 64);
        uint8_t *pd = (uint8_t *)pimg.data();
        for (int pr = 0; pr < 2; ++pr)
          for (int kb = 0; kb < 2; ++kb)
            for (int n = 0; n < 128; ++n) {
              const int tap = pr * 2 + (n >> 6), o = n & 63;
              for (int j = 0; j < 8; ++j)
                memcpy(pd + (size_t)(pr * 2 + kb) * 128 * 128 + (n / 8) * 1024 + (n % 8) * 128 + ((j ^ (n % 8)) * 16),
                       (const uint8_t *)(hw.data() + (size_t)o * K + tap * 128 + kb * 64) + j * 16, 16);
            }
        void *dp = nullptr;
        if (upload(net, pimg.data(), pimg.size() * 2, &dp) != cudaSuccess) { err = "upload paired conv2 weights"; return -1; }
        cs[t]->wpair = (const uint8_t *)dp;
      }
    }
  }
  cudaGetLastError();
  return 0;
}

size_t net_scratch_bytes(const Net &net) {
  size_t t = 0;
  for (int i = 0; i < kNetScratch; ++i) t += (net.scratch_sz[i] + 255) / 256 * 256;
  return t;
}

int net_bind_scratch(Net &net, uint8_t *base, std::string &err) {
  void *p[kNetScratch];
  size_t off = 0;
  for (int t = 0; t < kNetScratch; ++t) {
    p[t] = net.scratch_sz[t] && base ? base + off : nullptr;
    off += (net.scratch_sz[t] + 255) / 256 * 256;
  }
  net.act1 = (__nv_bfloat16 *)p[0]; net.act2 = (__nv_bfloat16 *)p[1]; net.act3 = (__nv_bfloat16 *)p[2];
  net.hid_act = (__nv_bfloat16 *)p[3]; net.zv = (float *)p[4]; net.za = (float *)p[5];
  net.s2d = (__nv_bfloat16 *)p[6]; net.leaf_cum = (float *)p[7];
  net.in1p = (uint8_t *)p[8]; net.act1p = (uint8_t *)p[9]; net.act2p = (uint8_t *)p[10];
  net.scratch = base;
  if (!base || (net.kind != BCTS_NET_NATURE_BF16 && net.kind != BCTS_NET_RAINBOW_BF16)) return 0;
  // TMA plans: tensor maps over the scratch buffers (re-encoded whenever the scratch moves)
  const int64_t FB = net.fc_batch, MB = net.mat_batch;
  bool ok = true;
  if (net.simt) {   // dense trunk (SIMT reference path)
    ok &= tma_plan(net.p_c1, net.c1, net.s2d, MB);
    ok &= tma_plan(net.p_c2, net.c2, net.act1, MB);
    ok &= tma_plan(net.p_c3, net.c3, net.act2, MB);
  }
  ok &= tma_plan(net.p_fc_h, net.fc_h, net.act3, FB);
  if (net.kind == BCTS_NET_RAINBOW_BF16) {
    ok &= tma_plan(net.p_z_v, net.z_v, net.hid_act, FB);
    ok &= tma_plan(net.p_z_a, net.z_a, net.hid_act, FB);
    if (net.wa64 && net.atoms == 51 && net.A <= 64) ok &= head_plan(net.head, net.hid_act, FB, net.z_v.Wt, net.wa64, net.wsum, net.A);
  } else {
    ok &= tma_plan(net.p_fc2, net.fc2, net.hid_act, FB);
  }
  if (!ok) {
    err = "TMA tensor-map encoding failed (driver entry point cuTensorMapEncodeTiled)";
    return -1;
  }
  return 0;
}

void net_free(Net &net) {
  for (void *p : net.allocs) cudaFree(p);
  net.allocs.clear();
}

static void run_layer(const Net &net, int cls, const Layer &L, const void *in, int64_t n_img, void *out,
                      cudaStream_t st, const TmaPlan *plan = nullptr) {
  // algorithmic FLOPs: 2 * M * N * K with the true (unpadded) N
  if (net.prof) net.prof->begin(cls, 2.0 * (double)(n_img * L.rows_per_img()) * L.N * L.K, st);
  if (net.tc && plan && plan->ok) launch_layer_tma(*plan, L, n_img, out, st);
  else launch_layer_simt(L, in, n_img, out, st);   // BCTS_F_SIMT_NET (tensor-map plans are checked at bind)
  if (net.prof) net.prof->end(st);
}

// Conv-net evaluation over n images that come either from a view of frame
// stacks (`img`, images [0, n)) or are the children [c_begin, c_begin + n) of
// the parents in `par` (fused last-level expansion). Trunk in L2-sized
// sub-batches: frames -> s2d bf16 -> conv1 -> conv2 -> conv3 (act3 of the fc
// batch); then fc_hidden, the output layer(s) and the head.
static int eval_conv(Net &net, const NodeView *par, const NodeView *img, int64_t p_first, int64_t c_begin, float gk,
                     int64_t n, int mode, float gd, float *out, cudaStream_t st, const KeyFold *kf = nullptr,
                     PrologueFold *pf = nullptr) {
  const int A = net.A;
  const bool rainbow = net.kind == BCTS_NET_RAINBOW_BF16;
  int launches = 0;
  // balanced batches: ceil(n / capacity) of them, equal sizes rounded up to 128 rows
  const int64_t nbat = (n + net.fc_batch - 1) / net.fc_batch;
  const int64_t step = std::min<int64_t>(net.fc_batch, ((n + nbat - 1) / nbat + 127) / 128 * 128);
  for (int64_t f0 = 0; f0 < n; f0 += step) {
    const int64_t nf = n - f0 < step ? n - f0 : step;
    const bool fused_leaf = par && net.tc && net.sw;
    const int64_t tb = fused_leaf ? (net.batch) : net.mat_batch;
    // the prologue's states ride along in this (last) batch when it has room (PrologueFold)
    const int64_t ne = (pf && !pf->done && f0 + nf >= n && fused_leaf && mode == MODE_TOTAL &&
                        net.kind == BCTS_NET_RAINBOW_BF16 && net.head.ok && nf <= tb && nf + pf->ne <= net.batch &&
                        nf + pf->ne <= net.fc_batch && pf->ne <= net.mat_batch)
                           ? pf->ne
                           : 0;
    for (int64_t b0 = 0; b0 < nf; b0 += tb) {
      const int64_t nb = nf - b0 < tb ? nf - b0 : tb;
      const bool sw = net.tc && net.sw;
      void *in1 = sw ? (void *)net.in1p : (void *)net.s2d;
      const uint32_t planar = sw ? kPlane1 : 0;
      const int lay = net.sw1.layout;
      if (par && sw) {   // leaf level generated inside conv1 (never leaves the SM)
        const double fl = 2.0 * (double)nb;
        if (net.prof) net.prof->begin(KC_CONV1, fl * 400 * 32 * 256, st);
        launch_conv1_sib(net.sw1, net.c1, net.w1_shared, net.w1_new, *par, p_first, c_begin + f0 + b0, nb, A, gk,
                         net.act1p, net.leaf_cum + b0, st);
        if (net.prof) net.prof->end(st);
        if (ne) {   // conv1 of the prologue's explicit states, appended after the batch's act1 images
          if (net.prof) net.prof->begin(KC_OTHER, (double)ne * (kFrameBytes + 2.0 * 28224), st);
          launch_s2d_convert(pf->view, 0, ne, net.in1p, kPlane1, st, net.sw1.layout);
          if (net.prof) net.prof->end(st);
          if (net.prof) net.prof->begin(KC_CONV1, 2.0 * (double)ne * 400 * 32 * 256, st);
          launch_conv_sw(net.sw1, net.c1, net.in1p, ne, (uint8_t *)net.act1p + nb * (int64_t)kIn2Bytes, st);
          if (net.prof) net.prof->end(st);
          launches += 2;
        }
        {   // conv2 + conv3 fused: act2 never leaves the SM
          const double fl2 = 2.0 * (double)(nb + ne);
          if (net.prof) net.prof->begin(KC_CONV23, fl2 * (81 * 64 * 512 + 49 * 64 * 576), st);
          launch_conv23(net.sw2, net.c2s, net.sw3, net.c3, net.act1p, nb + ne, net.act3 + b0 * 3136, st);
          if (net.prof) net.prof->end(st);
          launches += 2;
        }
        continue;
      }
      if (par) {
        launch_expand_s2d(*par, p_first, c_begin + f0 + b0, c_begin + f0 + b0 + nb, A, gk, in1, planar,
                          net.leaf_cum + b0, st, net.prof, lay);
      } else {
        if (net.prof) net.prof->begin(KC_OTHER, (double)nb * (kFrameBytes + 2.0 * 28224), st);
        launch_s2d_convert(*img, f0 + b0, nb, in1, planar, st, lay);
        if (net.prof) net.prof->end(st);
      }
      if (sw) {
        const double fl = 2.0 * (double)nb;
        if (net.prof) net.prof->begin(KC_CONV1, fl * 400 * 32 * 256, st);
        launch_conv_sw(net.sw1, net.c1, net.in1p, nb, net.act1p, st);
        if (net.prof) net.prof->end(st);
        if (net.prof) net.prof->begin(KC_CONV23, fl * (81 * 64 * 512 + 49 * 64 * 576), st);
        launch_conv23(net.sw2, net.c2s, net.sw3, net.c3, net.act1p, nb, net.act3 + b0 * 3136, st);
        if (net.prof) net.prof->end(st);
        launches -= 1;
      } else {
        run_layer(net, KC_CONV1, net.c1, net.s2d, nb, net.act1, st, &net.p_c1);
        run_layer(net, KC_CONV2, net.c2, net.act1, nb, net.act2, st, &net.p_c2);
        run_layer(net, KC_CONV3, net.c3, net.act2, nb, net.act3 + b0 * 3136, st, &net.p_c3);
      }
      launches += 4;
    }
    run_layer(net, KC_FC_H, net.fc_h, net.act3, nf + ne, net.hid_act, st, &net.p_fc_h);
    launches += 1;
    float *o = out + (mode == MODE_ROWS ? f0 * A : f0);
    const float *cum = par ? net.leaf_cum : (img->cum ? img->cum + f0 : nullptr);
    if (!rainbow) {
      run_layer(net, KC_FC_OUT, net.fc2, net.hid_act, nf, net.za, st, &net.p_fc2);
      if (net.prof) net.prof->begin(KC_HEAD, (double)nf * 4.0 * (net.ld_za + 1), st);
      k_head<false><<<(unsigned)((nf + 3) / 4), 128, 0, st>>>(nullptr, 0, net.za, net.ld_za, A, 0, 0.f, 0.f, nf, mode,
                                                               gd, cum, o);
      if (net.prof) net.prof->end(st);
      launches += 2;
    } else if (net.tc && net.head.ok) {   // z_v + z_a + dueling C51 head + max_a fused (k_zhead)
      const float dz = (net.vmax - net.vmin) / (float)(net.atoms - 1);
      if (net.prof) net.prof->begin(KC_FC_OUT, 2.0 * (double)(nf + ne) * 512.0 * (double)(net.atoms + A * net.atoms), st);
      KeyFold kb;
      if (kf) {
        kb = *kf;
        kb.leaf0 += f0;
      }
      launch_zhead(net.head, A, net.atoms, nf + ne, net.vmin, dz, mode, gd, cum, o, st, kb, nf,
                   ne ? pf->rows_out : nullptr);
      if (ne) pf->done = true;
      if (net.prof) net.prof->end(st);
      launches += 1;
    } else {
      run_layer(net, KC_FC_OUT, net.z_v, net.hid_act, nf, net.zv, st, &net.p_z_v);
      run_layer(net, KC_FC_OUT, net.z_a, net.hid_act, nf, net.za, st, &net.p_z_a);
      const float dz = (net.vmax - net.vmin) / (float)(net.atoms - 1);
      if (net.prof) net.prof->begin(KC_HEAD, (double)nf * 4.0 * (net.ld_za + net.ld_zv + 1), st);
      if (net.atoms == 51)
        k_head_rainbow<51><<<(unsigned)((nf + kHeadLeaves - 1) / kHeadLeaves), 256,
                             (size_t)kHeadLeaves * (((A * 51 + 3) & ~3) + 51 + A) * 4, st>>>(net.zv, net.ld_zv, net.za, net.ld_za,
                                                                               A, net.vmin, dz, nf, mode, gd, cum, o);
      else
        k_head<true><<<(unsigned)((nf + 3) / 4), 128, 0, st>>>(net.zv, net.ld_zv, net.za, net.ld_za, A, net.atoms,
                                                                net.vmin, dz, nf, mode, gd, cum, o);
      if (net.prof) net.prof->end(st);
      launches += 3;
    }
  }
  return launches;
}

bool net_fuses_leaves(const Net &net) {
  return net.kind == BCTS_NET_NATURE_BF16 || net.kind == BCTS_NET_RAINBOW_BF16;
}

int net_eval_children(Net &net, const NodeView &par, int64_t p_first, int64_t c_begin, int64_t c_end, int A,
                      float gk, int mode, float gd, float *out, cudaStream_t st, const KeyFold *kf, bool *folded,
                      PrologueFold *pf) {
  (void)A;
  const bool fold = kf && kf->keys && mode == MODE_TOTAL && net.kind == BCTS_NET_RAINBOW_BF16 && net.tc &&
                    net.head.ok;
  if (folded) *folded = fold;
  return eval_conv(net, &par, nullptr, p_first, c_begin, gk, c_end - c_begin, mode, gd, out, st, fold ? kf : nullptr,
                   pf);
}

int net_eval(Net &net, const NodeView &v, int64_t n, int mode, float gd, float *out, cudaStream_t st) {
  if (n <= 0) return 0;
  const int A = net.A;
  if (net.kind == BCTS_NET_TABLE) {
    if (net.prof) net.prof->begin(KC_TABLE, (double)n * (8.0 + 4.0 * A), st);
    k_table<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((const int32_t *)v.state, v.state_stride, net.tq, A, n, mode,
                                                          gd, v.cum, out);
    if (net.prof) net.prof->end(st);
    return 1;
  }
  if (net.kind == BCTS_NET_MLP2_F32) {
    if (net.prof) net.prof->begin(KC_MLP, 2.0 * (double)n * ((double)net.in * net.hid + (double)net.hid * A), st);
    if (net.mlp_tc_img) {
      launch_mlp_tc(v, n, net.mlp_tc_img, net.in, net.hid, A, mode, gd, out, net.feat_f32, st);
      if (net.prof) net.prof->end(st);
      return 1;
    }
    if (net.mlp_img) {
      launch_mlp_tiled(v, n, net.mlp_img, net.in, net.hid, A, mode, gd, out, net.feat_f32, st);
      if (net.prof) net.prof->end(st);
      return 1;
    }
    k_mlp<<<(unsigned)((n + kMlpWarps - 1) / kMlpWarps), 32 * kMlpWarps, 0, st>>>(
        v.state, v.state_stride, net.l1w, net.l1b, net.l2w, net.l2b, net.in, net.hid, A, n, mode, gd, v.cum, out,
        net.feat_f32);
    if (net.prof) net.prof->end(st);
    return 1;
  }
  return eval_conv(net, nullptr, &v, 0, 0, 0.0f, n, mode, gd, out, st);
}

}  // namespace bcts
