// engine.h -- internal interfaces between the C-ABI/engine and the kernels.
#pragma once
#include <string>
#include <vector>

#include "common.cuh"

namespace bcts {

// ---------------------------------------------------------------- profiler
// Per-kernel-class CUDA-event timing, enabled with bcts_profile_enable. Each
// record carries the ALGORITHMIC work of its launch (bytes or FLOPs,
// DESIGN.md §5) so bench.py can report achieved = work / duration.
enum KernelClass {
  KC_EXPAND_ATARI = 0, KC_EXPAND_INT, KC_EXPAND_TAB, KC_CONV1, KC_CONV2, KC_CONV3, KC_FC_H, KC_FC_OUT, KC_HEAD,
  KC_MLP, KC_TABLE, KC_SEGMAX, KC_FINALIZE, KC_OTHER, KC_EXPAND_DNN, KC_CONV23, KC_PRUNE, KC_COMM, KC_COUNT
};
struct Profiler {
  bool on = false;
  struct Rec {
    int cls;
    cudaEvent_t a, b;
    double work;
  };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  double ms[KC_COUNT] = {}, work[KC_COUNT] = {};
  int64_t launches[KC_COUNT] = {};
  double big_work[KC_COUNT] = {}, big_ms[KC_COUNT] = {};   // the class's largest launches
  int64_t big_n[KC_COUNT] = {};
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  void begin(int cls, double w, cudaStream_t st) {
    if (!on) return;
    Rec r{cls, get(), get(), w};
    cudaEventRecord(r.a, st);
    pending.push_back(r);
  }
  void end(cudaStream_t st) {
    if (!on || pending.empty()) return;
    cudaEventRecord(pending.back().b, st);
  }
  // Fold completed records into the totals (caller synchronizes first).
  void collect() {
    for (auto &r : pending) {
      float t = 0.f;
      cudaEventElapsedTime(&t, r.a, r.b);
      ms[r.cls] += t;
      work[r.cls] += r.work;
      launches[r.cls] += 1;
      if (r.work > big_work[r.cls]) big_work[r.cls] = r.work, big_ms[r.cls] = 0.0, big_n[r.cls] = 0;
      if (r.work == big_work[r.cls]) big_ms[r.cls] += t, big_n[r.cls] += 1;
      pool.push_back(r.a);
      pool.push_back(r.b);
    }
    pending.clear();
  }
  void reset() {
    collect();
    for (int i = 0; i < KC_COUNT; ++i) ms[i] = work[i] = big_work[i] = big_ms[i] = 0, launches[i] = big_n[i] = 0;
  }
  ~Profiler() {
    for (auto &r : pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

// ---------------------------------------------------------------- K1 expand
// Expand parents (global level-k indices starting at p_first, view `par`) into
// the children with global level-(k+1) indices [c_begin, c_end):
// child c has parent c / A and action c % A (R1); R' = fmaf(gk, r, R).
// Device-resident forward-model parameters (set at bcts_create).
struct EnvModel {
  const int32_t *tab_next = nullptr;  // TABULAR [nS*A]
  const float *tab_rew = nullptr;     // TABULAR [nS*A]
  const float *dnn = nullptr;         // DNN: smem image (kDnnImg floats) followed by W1A [A][100]
  const float *dnn_tc = nullptr;      // DNN, BCTS_F_TF32: the k_dnn_tc image (tf32_tc.cu)
  const float *dnn_tc_bias = nullptr; // DNN, BCTS_F_TF32: HOST copy of the image's biases [4][112] (kernel parameter)
};
constexpr int kDnnS = 100;                         // DNN state width
constexpr int kDnnImg = 3 * 10000 + 10400 + 404;   // W1T|W2T|W3T|W4T[100][104]|b1|b2|b3|b4[104] floats
int64_t dnn_env_weights_count(int A);              // canonical blob size: 40,501 + 100*A
// canonical blob (include/bcts.h) -> device image (host side; out has kDnnImg + 100*A floats)
void dnn_repack(const float *blob, int A, float *out);

void launch_expand(int env, const NodeView &par, int64_t p_first, int64_t c_begin, int64_t c_end, int A,
                   float gk, const EnvModel &em, const NodeOut &out, cudaStream_t st, Profiler *prof = nullptr);
// ffma_tiles.cu: fixed-order fp32 FMA kernels (DNN forward model, tiled MLP2)
void launch_expand_dnn(const NodeView &par, int64_t p_first, int64_t c_begin, int64_t c_end, int A, float gk,
                       const float *img, const NodeOut &out, cudaStream_t st, Profiler *prof);
// tf32_tc.cu: the same two nets on the tensor cores (kind::tf32, opt-in BCTS_F_TF32)
size_t dnn_tc_image_floats(int A);
void dnn_tc_repack(const float *blob, int A, float *out);
bool dnn_tc_ok(int A);
void launch_expand_dnn_tc(const NodeView &par, int64_t p_first, int64_t c_begin, int64_t c_end, int A, float gk,
                          const float *img, const float *bias_host, const NodeOut &out, cudaStream_t st,
                          Profiler *prof);
// several consecutive levels (level k+1's parents = level k's output) in ONE cooperative launch: the
// weights and TMEM stay put and a grid barrier separates the levels; nonzero if the launch failed
struct DnnTcLevel {
  NodeView par;
  int64_t p_first = 0, c_begin = 0, c_end = 0;
  float gk = 0.f;
  NodeOut out;
};
struct DnnTcLevels {
  int n = 0;
  DnnTcLevel lv[kMaxDepth];
};
int launch_expand_dnn_tc_levels(const DnnTcLevel *lvs, int nlev, int A, const float *img, const float *bias_host,
                                cudaStream_t st, Profiler *prof);
constexpr size_t kDnnTcBiasOffset = 4 * 26 * 112 * 4;   // floats of the image before the biases (4 layer images)
size_t mlp_tc_image_bytes(int I, int H, int A);
bool mlp_tc_ok(int I, int H, int A);
void mlp_tc_repack(const float *w1, const float *b1, const float *w2, const float *b2, int I, int H, int A,
                   uint8_t *out);
void launch_mlp_tc(const NodeView &v, int64_t n, const uint8_t *img, int I, int H, int A, int mode, float gd,
                   float *out, int feat_f32, cudaStream_t st);
int mlp_image_floats(int I, int H, int A);
void mlp_repack(const float *w1, const float *b1, const float *w2, const float *b2, int I, int H, int A, float *out);
bool mlp_tiled_ok(int I, int H, int A);

// s2d bf16 frames for the conv1 tensor-core layer (expand.cu)
// planar != 0: write the chunk-planar layout (plane = bytes per 8-channel plane,
// image stride 8*plane); 0: dense [21][21][64] bf16.
void launch_s2d_convert(const NodeView &v, int64_t first, int64_t n, void *out, uint32_t planar, cudaStream_t st,
                        int layout = 0);
void launch_expand_s2d(const NodeView &par, int64_t p_first, int64_t c_begin, int64_t c_end, int A, float gk,
                       void *out, uint32_t planar, float *cum_out, cudaStream_t st, Profiler *prof, int layout = 0);

// -------------------------------------------------------- implicit-GEMM layer
// out[m][n] = act( sum_k X[m][k] * W[n][k] + b[n] ), X gathered im2col-style
// from an NHWC input (k = (ky, kx, c)); used for every conv and fc layer.
struct Layer {
  int in_u8 = 0;            // 1: uint8 input (frames, C=4 packed per pixel word); 0: bf16
  int64_t in_img_stride = 0;  // elements between images (bytes for u8)
  int in_col_off = 0;       // element offset inside an image (fc on a column slice)
  int H = 1, W = 1, C = 0;  // input geometry
  int KH = 1, KW = 1, S = 1, OH = 1, OW = 1;
  int K = 0;                // KH*KW*C
  int N = 0, Npad = 0;      // true / padded output width (rows >= N of W are zero)
  const __nv_bfloat16 *Wt = nullptr;  // [Npad][K], k = (ky, kx, c)
  const float *bias = nullptr;        // [Npad]
  int relu_bf16 = 1;        // 1: ReLU then bf16 RNE store; 0: fp32 store
  int64_t out_ld = 0;       // elements per output row
  int64_t rows_per_img() const { return (int64_t)OH * OW; }
};

// TMA-fed layer (qnet_tma.cu): tensor maps for A (2-D tile or 4-D im2col) and B.
struct TmaPlan {
  bool ok = false;
  int im2col = 0, kb = 64, bn = 64;
  alignas(64) uint8_t mapA[128];
  alignas(64) uint8_t mapB[128];
  bool ok2sm = false;               // mapB2: B with 128-row boxes (2-SM MMA, half an N tile per CTA)
  alignas(64) uint8_t mapB2[128];
  bool ok_small = false;            // mapAs / mapBs: 32-row boxes for fc batches of <= kSmallM rows
  alignas(64) uint8_t mapAs[128];
  alignas(64) uint8_t mapBs[128];
};
constexpr int kSmallM = 32;
bool tma_plan(TmaPlan &P, const Layer &L, const void *in, int64_t cap_img);
// Fused Rainbow head (qnet_tma.cu, k_zhead): z_v + z_a + dueling C51 + max_a in one kernel.
// The head biases travel as a __grid_constant__ kernel parameter: every lane of a warp reads
// the same (action, atom) bias, so they are broadcast constant-bank loads (no L1 latency).
constexpr int kHeadChunkRows = 208;   // fused head: rows per z_a chunk (4 actions x 51 atoms, padded to 16)
struct HeadBias {
  float v[64];         // z_v bias (atoms)
  float sum[64];       // sum over actions of the z_a bias
  float a64[64 * 64];  // z_a bias, 64 slots per action
  float z[64];         // C51 support z_t = v_min + t dz (fp32, as fmaf(t, dz, v_min))
};
struct HeadPlan {
  bool ok = false;
  alignas(64) uint8_t mapAv[128];
  alignas(64) uint8_t mapAa[128];
  alignas(64) uint8_t mapBv[128];
  alignas(64) uint8_t mapBa[128];
  alignas(64) uint8_t mapBs[128];   // sum_a W_a as bf16 hi (rows 0..63) + lo (rows 64..127)
  HeadBias bias;
};
bool head_plan(HeadPlan &H, const __nv_bfloat16 *hid, int64_t cap, const __nv_bfloat16 *wv64, const __nv_bfloat16 *wa64,
               const __nv_bfloat16 *wsum, int A);
// Backup fused into a MODE_TOTAL head epilogue (K3a): leaf row m of the batch is
// global leaf leaf0 + m of root (leaf / lpr), root action (leaf % lpr) / seg; its packed key
// (total, leaf % lpr) is max-folded into keys[root * A + action] (warp max, one atomicMax per
// warp-uniform segment). keys == nullptr: totals only.
struct KeyFold {
  int64_t *keys = nullptr;
  int64_t leaf0 = 0, lpr = 1, seg = 1;
  int A = 0;
};
// rows_out != NULL: rows [mrow0, M) are full-row rows (Q_hat(s, .) -> rows_out[(m - mrow0) * A + a]);
// only rows below mrow0 produce totals / keys.
void launch_zhead(const HeadPlan &H, int A, int atoms, int64_t M, float vmin, float dz, int mode, float gd,
                  const float *cum, float *out, cudaStream_t st, KeyFold kf = KeyFold(), int64_t mrow0 = 0,
                  float *rows_out = nullptr);
void launch_layer_tma(const TmaPlan &P, const Layer &L, int64_t n_img, void *out, cudaStream_t st);

// Shifted-window conv layer (qnet_conv.cu): stride-1 conv over a per-image
// chunk-planar K-major activation (byte(row r, chunk j) = j*plane + r*16).
struct ConvSW {
  int N = 0, K = 0, Cin = 0, KH = 0, KW = 0, W_in = 0, OH = 0, OW = 0, n_mt = 0;
  uint32_t plane = 0, in_img_bytes = 0;        // input: planar, Cin/8 planes
  uint32_t out_img_bytes = 0, out_plane = 0;   // output layout of the next layer
  int out_w = 0, out_mode = 0;                 // 0: s2d(2) planar, 1: planar, 2: dense [row][N]
  const uint8_t *wsw = nullptr;                // weights pre-swizzled as their SW128 smem image
  const uint8_t *wpair = nullptr;              // conv2 only: tap-pair image for k_conv23 (qnet.cu)
  int layout = 0;                              // activation layout (see act_off)
  uint32_t copy_chunks = 1;                    // (unused) bulk copies per input image
  int in_rows = 0;                             // valid input rows per 64-channel block
};
void launch_conv_sw(const ConvSW &P, const Layer &L, const void *in, int64_t n_img, void *out, cudaStream_t st);
// conv2 + conv3 in one kernel (act2 stays in SMEM): act1 planar in, dense act3 out
void launch_conv23(const ConvSW &P2, const Layer &L2, const ConvSW &P3, const Layer &L3, const void *in, int64_t n_img,
                   void *out, cudaStream_t st);
// conv1, sibling-factorised (shared frames once per parent + new frame per child)
void launch_conv1_sib(const ConvSW &P, const Layer &L, const uint8_t *wsh, const uint8_t *wnw, const NodeView &par,
                      int64_t p_first, int64_t c_begin, int64_t n_img, int A, float gk, void *out, float *cum_out,
                      cudaStream_t st);
// Trunk activation layout (runtime, BCTS_CONV_LAYOUT): 0 = chunk-planar
// SWIZZLE_NONE; 1 = SW128 row blocks, descriptor base_offset = row phase;
// 2 = SW128 row blocks, base_offset 0. In the SW128 layouts
//   byte(r, c) = (c/64)*BPLANE + r*128 + ((((c%64)/8) ^ (r%8)) * 16) + (c%8)*2,
// BPLANE = Rpad*128 (same total bytes as the planar layout).
__host__ __device__ __forceinline__ uint32_t act_off(int layout, uint32_t plane16, int r, int chunk) {
  // plane16 = planar plane bytes (Rpad*16); chunk = 8-channel chunk index
  if (layout == 0) return (uint32_t)chunk * plane16 + (uint32_t)r * 16u;
  return (uint32_t)(chunk >> 3) * (plane16 * 8u) + (uint32_t)r * 128u + (uint32_t)(((chunk & 7) ^ (r & 7)) << 4);
}
// planar geometry of the three trunk inputs
constexpr uint32_t kPlane1 = 536 * 16, kIn1Bytes = 8 * kPlane1;      // s2d(4) frame: 21x21 rows, 64 ch
constexpr uint32_t kPlane2 = 144 * 16, kIn2Bytes = 16 * kPlane2;     // s2d(2) act1: 10x10 rows, 128 ch
constexpr uint32_t kPlane3 = 152 * 16, kIn3Bytes = 8 * kPlane3;      // act2: 9x9 rows, 64 ch

// Net output modes.
enum { MODE_ROWS = 0, MODE_ROWMAX = 1, MODE_TOTAL = 2 };

void launch_mlp_tiled(const NodeView &v, int64_t n, const float *img, int I, int H, int A, int mode, float gd,
                      float *out, int feat_f32, cudaStream_t st);

constexpr int kNetScratch = 11;
struct Net {
  int kind = 0, A = 0;
  // TABLE
  const float *tq = nullptr;
  int nS = 0;
  // MLP2
  const float *l1w = nullptr, *l1b = nullptr, *l2w = nullptr, *l2b = nullptr;
  int in = 0, hid = 0;
  int feat_f32 = 0;               // DNN env: features are the fp32 state itself
  const float *mlp_img = nullptr; // tiled-MLP smem image (mlp_repack), null = warp-per-state kernel
  const uint8_t *mlp_tc_img = nullptr;  // BCTS_F_TF32: the k_mlp_tc image (tf32_tc.cu)
  // conv nets
  Layer c1, c2, c3, fc_h, z_v, z_a, fc2;
  int atoms = 51;
  float vmin = -10.f, vmax = 10.f;
  const __nv_bfloat16 *wa64 = nullptr;   // fused head: z_a weights, chunks of 4 actions x 51 rows (kHeadChunkRows)
  const float *ba64 = nullptr;
  const __nv_bfloat16 *wsum = nullptr;   // fused head: sum_a W_a (bf16 hi | lo), [128][512]
  const float *bsum = nullptr;           // fused head: sum_a b_a [64]
  HeadPlan head;
  // scratch: trunk sub-batches of `batch` images (conv activations stay
  // L2-resident), fc layers over `fc_batch` images at a time
  int64_t batch = 0, fc_batch = 0;
  int64_t mat_batch = 0;          // trunk sub-batch of the materialised-state path (s2d input buffer)
  TmaPlan p_c1, p_c2, p_c3, p_fc_h, p_z_v, p_z_a, p_fc2;
  // scratch buffers (net_bind_scratch): sizes fixed at build, memory bound later (library-owned
  // or caller-provided via bcts_set_workspace)
  size_t scratch_sz[kNetScratch] = {};
  uint8_t *scratch = nullptr;
  bool simt = false;
  __nv_bfloat16 *s2d = nullptr;   // [batch][21][21][64] conv1 input (dense; SIMT / TMA paths)
  uint8_t *in1p = nullptr, *act1p = nullptr, *act2p = nullptr;  // planar trunk buffers [batch]
  Layer c2s;                      // conv2 as 2x2 stride-1 over s2d(2) of act1 (shifted windows)
  ConvSW sw1, sw2, sw3;
  const uint8_t *w1_shared = nullptr, *w1_new = nullptr;   // sibling-factorised conv1 weights (SW128 images)
  bool sw = false;                // shifted-window trunk enabled
  float *leaf_cum = nullptr;      // [fc_batch] R_d of fused-expanded leaves
  __nv_bfloat16 *act1 = nullptr, *act2 = nullptr, *act3 = nullptr, *hid_act = nullptr;
  float *zv = nullptr, *za = nullptr;
  int64_t ld_za = 0, ld_zv = 0;
  bool tc = false;          // tensor-core (tcgen05) layers available + enabled
  Profiler *prof = nullptr;
  std::vector<void *> allocs;
};

// Evaluate Q_hat on n nodes of view v. MODE_ROWS: out[n*A]; MODE_ROWMAX:
// out[n] = max_a Q; MODE_TOTAL: out[n] = fmaf(gd, max_a Q, cum[i]).
// Returns the number of kernels launched, or -1 on a CUDA error.
int net_eval(Net &net, const NodeView &v, int64_t n, int mode, float gd, float *out, cudaStream_t st);
// Scratch the conv nets need (0 for the table / MLP nets), and binding it: carve the buffers out
// of `base` (256-byte aligned pieces) and re-encode the TMA tensor maps over them.
size_t net_scratch_bytes(const Net &net);
// NCCL (comm.cu): the multi-GPU handle's communicator; errors as text in err
constexpr int kNcclIdBytes = 128;
bool comm_unique_id(void *out128, std::string &err);
bool comm_init(void **comm, const void *id128, int rank, int world, std::string &err);
bool comm_allreduce_max_i64(void *comm, int64_t *buf, int64_t count, cudaStream_t st, std::string &err);
void comm_destroy(void *comm);
int net_bind_scratch(Net &net, uint8_t *base, std::string &err);
// Conv nets only: evaluate the children [c_begin, c_end) of the parents in view
// `par` (global level indices from p_first), generating each child's frames on
// the fly (fused last-level expansion, gk = g[d-1]); out[i] per MODE.
bool net_fuses_leaves(const Net &net);
// kf (nullable): fold the totals into packed keys inside the head when it supports it
// (*folded set to true); otherwise the caller runs the backup kernel.
// pf (nullable): the finalize prologue's materialised states [roots | level-1 children] ride along
// in the last leaf batch that has room for them (conv1 on the explicit states, then the batch's
// conv2+conv3 / fc / head launches); their Q rows land in pf->rows_out and pf->done is set. The
// prologue's own four launches (its latency-bound tiny batch) disappear from the step.
struct PrologueFold {
  NodeView view;
  int64_t ne = 0;
  float *rows_out = nullptr;
  bool done = false;
};
int net_eval_children(Net &net, const NodeView &par, int64_t p_first, int64_t c_begin, int64_t c_end, int A,
                      float gk, int mode, float gd, float *out, cudaStream_t st, const KeyFold *kf = nullptr,
                      bool *folded = nullptr, PrologueFold *pf = nullptr);
int net_build(Net &net, const bcts_config &cfg, std::string &err);  // 0 ok
void net_free(Net &net);

// tcgen05 layer (qnet_tc.cu); returns false if the layer shape is unsupported.
void launch_layer_simt(const Layer &L, const void *in, int64_t n_img, void *out, cudaStream_t st);

// ---------------------------------------------------------------- K3 backup
void launch_keys_init(int64_t *keys, int64_t count, cudaStream_t st);
// Fold leaf totals of global leaves [leaf_begin, leaf_begin+n) into keys by
// max; leaves_per_root = A^d, seg = A^(d-1).
void launch_segmax(const float *totals, int64_t n, int64_t leaf_begin, int64_t leaves_per_root, int64_t seg,
                   int A, int64_t *keys, cudaStream_t st, Profiler *prof = nullptr);
struct FinalizeArgs {
  int64_t n = 0;
  int A = 0, d = 0, corr = 0, clamp = 0;
  float beta = 0.f, g1 = 0.f, gd = 0.f;
  const int64_t *keys = nullptr;  // [n*A] (d >= 1)
  const float *q0 = nullptr;      // [n*A] root rows (corr or d == 0)
  const float *m1 = nullptr;      // [n*A] max_a Q_hat(s_1^a, .) (corr, d >= 1), or:
  const float *rows1 = nullptr;   // [n*A][A] the level-1 Q rows themselves (m1 taken as their row max)
  const float *r1 = nullptr;      // [n*A] R_1 of the root's children (corr, d >= 1)
  int32_t *actions = nullptr;
  float *root_q = nullptr, *vanilla = nullptr, *terms = nullptr;
  int64_t *best_leaf = nullptr;
};
void launch_finalize(const FinalizeArgs &a, cudaStream_t st, Profiler *prof = nullptr);
void launch_rowmax(const float *rows, int64_t n, int A, float *out, cudaStream_t st);
void launch_pv_targets(int64_t n, int A, int d, const int32_t *actions, const float *vanilla,
                       const int64_t *best_leaf, float *target, int32_t *path, cudaStream_t st);

// ------------------------------------------------- early pruning (prune.cu, NEXT-4)
// f = index of a node in the unpruned tree (global over the call's roots): the index array.
void launch_prune_iota(int64_t *f, int64_t first, int64_t n, cudaStream_t st);
void launch_child_index(const int64_t *pf, int64_t n_child, int A, int64_t *cf, cudaStream_t st);
struct BoundRule {            // R31; L, U, S computed on the host in the oracle's order
  double L = 0, U = 0, S = 0;
  int64_t gsz = 1;            // level-k nodes per (root, root action) group in the unpruned tree: A^(k-1)
  int64_t g0 = 0, groups = 0; // first group of the chunk, groups in the chunk
};
void launch_bound_keep(const float *cum, const int64_t *f, int64_t n, const BoundRule &b, unsigned long long *gmax,
                       uint8_t *keep, cudaStream_t st, Profiler *prof);
void launch_beam_keep(const float *m, const float *cum, float gk, int64_t n, int64_t G, int64_t beam, uint8_t *keep,
                      cudaStream_t st, Profiler *prof);
size_t compact_temp_bytes(int64_t n);
void launch_compact(const uint8_t *keep, int64_t n, int64_t *sel, int64_t *d_count, void *temp, size_t temp_bytes,
                    cudaStream_t st);
void launch_gather_level(int64_t state_bytes, const NodeView &src, const int64_t *f, const int64_t *sel, int64_t n_out,
                         const NodeOut &dst, int64_t *f_out, cudaStream_t st, Profiler *prof);
void launch_segmax_f(const float *totals, const int64_t *f, int64_t n, int64_t lpr, int64_t seg, int64_t *keys,
                     cudaStream_t st, Profiler *prof);

}  // namespace bcts
