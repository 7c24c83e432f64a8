// bcts.cu -- engine (E1) and C-ABI (A1) of the Batch-BFS + BCTS hot path.
// See include/bcts.h for the contract and DESIGN.md §4-§6 for the design.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <new>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "engine.h"

using namespace bcts;

struct bcts_handle_t {
  int dev = 0;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  int env = 0, A = 0, nS = 0;
  uint32_t flags = 0;
  int32_t *d_next = nullptr;
  float *d_envw = nullptr;   // DNN env image (dnn_repack)
  float *d_envw_tc = nullptr;   // DNN env image of the tf32 tensor-core path (dnn_tc_repack)
  std::vector<float> envw_tc_bias;   // its biases [4][112] (host: a kernel parameter)
  EnvModel em;
  float *d_rew = nullptr;
  Net net;
  int64_t ws_max = 0;
  uint8_t *ws = nullptr;      // tree workspace (library-owned, or inside the caller's memory)
  size_t ws_size = 0;
  bool ws_own = true;
  uint8_t *scratch_own = nullptr;   // library-owned net scratch (when no caller memory)
  uint8_t *ext = nullptr;           // caller-owned memory (bcts_set_workspace): [net scratch | tree ws]
  size_t ext_bytes = 0;
  // multi-GPU: the handle's NCCL communicator (world > 1)
  void *comm = nullptr;
  int rank = 0, world = 1;
  // end-to-end (host buffer) staging
  uint8_t *e2e_roots = nullptr;
  size_t e2e_roots_size = 0;
  int32_t *e2e_act = nullptr;
  float *e2e_q = nullptr;
  size_t e2e_out = 0;
  std::string err;
  int64_t launches = 0;
  Profiler prof;
  // prologue folded into a bcts_search_shard leaf batch, kept for the bcts_finalize that follows
  // (identified by roots pointer, n_roots, depth, gamma); pbuf holds its states and rows
  uint8_t *pbuf = nullptr;
  size_t pbuf_size = 0;
  PrologueFold pfs;
  bool pfs_valid = false;
  const void *pfs_roots = nullptr;
  int64_t pfs_n = 0;
  int32_t pfs_d = 0;
  float pfs_gamma = 0.f;
  // bcts_search_host replays a CUDA graph of [H2D, search, D2H] captured for its last arguments
  struct GraphKey {
    const void *rh = nullptr;
    void *ah = nullptr, *qh = nullptr;
    int64_t n = 0;
    int32_t d = 0, A = 0, corr = 0;
    float gamma = 0.f, beta = 0.f;
    uint8_t *ws = nullptr, *scratch = nullptr;
    size_t wss = 0;
    const void *dr = nullptr, *da = nullptr, *dq = nullptr;   // the device staging buffers the graph uses
    bool operator==(const GraphKey &o) const {
      return rh == o.rh && ah == o.ah && qh == o.qh && n == o.n && d == o.d && A == o.A && corr == o.corr &&
             gamma == o.gamma && beta == o.beta && ws == o.ws && wss == o.wss && scratch == o.scratch &&
             dr == o.dr && da == o.da && dq == o.dq;
    }
  } gkey;
  cudaGraphExec_t gexec = nullptr;
  bool gvalid = false;
  cudaStream_t gst = nullptr;
  // bcts_search_ex (device pointers) replays a graph of its last call's launches
  struct DevKey {
    const void *roots = nullptr;
    void *o[5] = {};
    int64_t n = 0;
    int32_t d = 0, A = 0, corr = 0;
    float gamma = 0.f, beta = 0.f;
    uint8_t *ws = nullptr, *scratch = nullptr;
    size_t wss = 0;
    bool operator==(const DevKey &k) const {
      for (int i = 0; i < 5; ++i)
        if (o[i] != k.o[i]) return false;
      return roots == k.roots && n == k.n && d == k.d && A == k.A && corr == k.corr && gamma == k.gamma &&
             beta == k.beta && ws == k.ws && scratch == k.scratch && wss == k.wss;
    }
  } dkey;
  cudaGraphExec_t dexec = nullptr;
  bool dvalid = false;
  bcts_stats dstats = {};
  bool capturing = false;   // inside a capture of ours: no nested graph logic
};

namespace bcts {
int sm_count_current() {
  static int cache[64] = {};   // per device ordinal (a benign race: every writer stores the same value)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int n = __atomic_load_n(&cache[dev], __ATOMIC_RELAXED);
  if (!n) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    __atomic_store_n(&cache[dev], n, __ATOMIC_RELAXED);
  }
  return n;
}
cudaError_t smem_optin(const void *kernel, int bytes) {
  // the attribute is an upper bound: keep the largest size any launch of (kernel, device) asked for
  // (setting a smaller one after a larger one would break the larger launches)
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, int> set_to;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  int &cur = set_to[std::make_pair(kernel, dev)];
  if (bytes <= cur) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}
}  // namespace bcts

namespace {

const int64_t kDefaultWorkspace = 16LL << 30;

int64_t state_bytes(int env) {
  return env == BCTS_ENV_TABULAR ? 4 : env == BCTS_ENV_INT_HASH ? 64 : env == BCTS_ENV_DNN ? 4 * kDnnS : kFrameBytes;
}
int64_t record_bytes(int env) {
  return env == BCTS_ENV_TABULAR ? 4 : env == BCTS_ENV_INT_HASH ? 64 : env == BCTS_ENV_DNN ? 4 * kDnnS : kAtariRecord;
}
int64_t node_bytes(int env) { return state_bytes(env) + (env == BCTS_ENV_ATARI_HASH ? 8 : 0) + 4; }
size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

struct LevelBuf {
  uint8_t *state = nullptr;
  uint64_t *key = nullptr;
  float *cum = nullptr;
  int64_t cap = 0;
};

// Bump allocator over the handle's workspace.
struct Carver {
  uint8_t *base;
  size_t off = 0;
  explicit Carver(uint8_t *b) : base(b) {}
  void *take(size_t bytes) {
    void *p = base ? base + off : nullptr;
    off = align_up(off + bytes);
    return p;
  }
  LevelBuf level(int env, int64_t cap) {
    LevelBuf b;
    b.cap = cap;
    b.state = (uint8_t *)take((size_t)cap * state_bytes(env));
    if (env == BCTS_ENV_ATARI_HASH) b.key = (uint64_t *)take((size_t)cap * 8);
    b.cum = (float *)take((size_t)cap * 4);
    return b;
  }
};

NodeView view_of(int env, const LevelBuf &b) {
  NodeView v;
  v.state = b.state;
  v.state_stride = state_bytes(env);
  v.key = b.key;
  v.key_stride = 8;
  v.cum = b.cum;
  return v;
}
NodeOut out_of(int env, const LevelBuf &b) {
  NodeOut o;
  o.state = b.state;
  o.state_stride = state_bytes(env);
  o.key = b.key;
  o.cum = b.cum;
  return o;
}
// Level-0 view straight into the caller's root records, starting at root r0.
NodeView root_view(int env, const void *roots, int64_t r0) {
  NodeView v;
  const int64_t rb = record_bytes(env);
  const uint8_t *base = (const uint8_t *)roots + r0 * rb;
  v.state = base + (env == BCTS_ENV_ATARI_HASH ? 16 : 0);
  v.state_stride = rb;
  if (env == BCTS_ENV_ATARI_HASH) {
    v.key = (const uint64_t *)base;
    v.key_stride = rb;
  }
  v.cum = nullptr;
  return v;
}

bool ipow_ok(int64_t A, int d, int64_t &out) {
  int64_t v = 1;
  for (int k = 0; k < d; ++k) {
    if (v > (INT64_MAX / 4) / A) return false;
    v *= A;
  }
  out = v;
  return true;
}

bcts_status fail(bcts_handle h, bcts_status s, const std::string &msg) {
  if (h) h->err = msg;
  return s;
}

bcts_status cuda_check(bcts_handle h, const char *where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(h, BCTS_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
  return BCTS_OK;
}

bcts_status ensure_ws(bcts_handle h, size_t bytes) {
  if (bytes <= h->ws_size) return BCTS_OK;
  if (!h->ws_own)
    return fail(h, BCTS_ERR_BUDGET, "caller workspace too small: the tree workspace needs " + std::to_string(bytes) +
                                        " bytes, " + std::to_string(h->ws_size) + " available (bcts_workspace_size)");
  h->dvalid = h->gvalid = false;   // graphs bake the workspace address in
  if (h->ws) {
    cudaStreamSynchronize(h->st);
    cudaFree(h->ws);
    h->ws = nullptr;
    h->ws_size = 0;
  }
  if (cudaMalloc(&h->ws, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(h, BCTS_ERR_OUT_OF_MEMORY, "workspace cudaMalloc of " + std::to_string(bytes) + " bytes failed");
  }
  h->ws_size = bytes;
  return BCTS_OK;
}

// The value net's scratch, bound on first use: inside the caller's memory (bcts_set_workspace) or
// one library allocation.
bcts_status ensure_net(bcts_handle h) {
  if (h->net.scratch || !net_scratch_bytes(h->net)) return BCTS_OK;
  std::string err;
  uint8_t *base = h->ext;
  if (!base) {
    if (cudaMalloc(&h->scratch_own, net_scratch_bytes(h->net)) != cudaSuccess) {
      cudaGetLastError();
      h->scratch_own = nullptr;
      return fail(h, BCTS_ERR_OUT_OF_MEMORY, "net scratch cudaMalloc of " + std::to_string(net_scratch_bytes(h->net)) +
                                                 " bytes failed");
    }
    base = h->scratch_own;
  }
  if (net_bind_scratch(h->net, base, err)) return fail(h, BCTS_ERR_CUDA, err);
  return BCTS_OK;
}

void discounts(float gamma, int d, float *g) {
  double p = 1.0;
  for (int k = 0; k <= d; ++k) {  // g[k] = (float)(product of k copies of (double)gamma)  (R3)
    g[k] = (float)p;
    p *= (double)gamma;
  }
}

bcts_status validate(bcts_handle h, const void *roots, int64_t n_roots, int32_t depth, int32_t A, float gamma) {
  if (!h) return BCTS_ERR_INVALID_ARG;
  if (A != h->A) return fail(h, BCTS_ERR_INVALID_ARG, "A != num_actions of the handle");
  if (depth < 0 || depth > kMaxDepth) return fail(h, BCTS_ERR_INVALID_ARG, "depth out of [0, 12]");
  if (n_roots < 0) return fail(h, BCTS_ERR_INVALID_ARG, "n_roots < 0");
  if (!(gamma > 0.0f && gamma < 1.0f)) return fail(h, BCTS_ERR_INVALID_ARG, "gamma must be in (0,1) (P:44)");
  if (n_roots > 0 && !roots) return fail(h, BCTS_ERR_INVALID_ARG, "roots is NULL");
  int64_t lpr;
  if (!ipow_ok(A, depth, lpr) || lpr > 0xFFFFFFFFLL)
    return fail(h, BCTS_ERR_BUDGET, "A^d exceeds 2^32-1 leaves per root");
  if (n_roots > 0 && lpr > (INT64_MAX / 8) / n_roots) return fail(h, BCTS_ERR_BUDGET, "n_roots * A^d overflows");
  if (h->env == BCTS_ENV_TABULAR && n_roots > 0) {  // root id domain check (synchronous; toy env only)
    std::vector<int32_t> ids((size_t)n_roots);
    if (cudaMemcpyAsync(ids.data(), roots, 4 * (size_t)n_roots, cudaMemcpyDeviceToHost, h->st) != cudaSuccess ||
        cudaStreamSynchronize(h->st) != cudaSuccess)
      return cuda_check(h, "root id check");
    for (int32_t s : ids)
      if (s < 0 || s >= h->nS) return fail(h, BCTS_ERR_INVALID_ARG, "TABULAR root id outside [0, nS)");
  }
  return BCTS_OK;
}

// Largest leaf chunk (multiple of A) that fits the budget. Materialised
// leaves: big level (Lc) + small level (Lc/A + 2) + leaf totals (Lc). Fused
// leaves (conv nets: the leaf level is generated inside the net): big level
// d-1 (Lc/A + 2) + small level (Lc/A^2 + 2) + totals.
// Leaf level generated inside conv1 (k_conv1_sib) unless BCTS_F_MATERIALIZE_LEAVES asks for the
// leaf states to be stored and scored like any other batch of states.
bool fused_leaves(bcts_handle h) {
  return net_fuses_leaves(h->net) && h->env == BCTS_ENV_ATARI_HASH && !(h->flags & BCTS_F_MATERIALIZE_LEAVES);
}

int64_t plan_chunk(bcts_handle h, int64_t range, size_t reserved) {
  const int64_t nb = node_bytes(h->env);
  const int64_t budget = h->ws_max - (int64_t)reserved - (1 << 20);
  if (budget <= 0) return 0;
  const double A = h->A;
  const double per_leaf = fused_leaves(h) ? nb * (1.0 / A + 1.0 / (A * A)) + 4.0 : nb * (1.0 + 1.0 / A) + 4.0;
  int64_t lc = (int64_t)((double)budget / per_leaf);
  lc -= 4 * h->A;
  lc = lc / h->A * h->A;
  const int64_t need = (range + h->A - 1) / h->A * h->A;
  return std::min(lc, need);
}

size_t chunk_bytes(bcts_handle h, int64_t lc) {
  Carver c(nullptr);
  if (fused_leaves(h)) {
    c.level(h->env, lc / h->A + 2);
    c.level(h->env, lc / h->A / h->A + 2);
  } else {
    c.level(h->env, lc);
    c.level(h->env, lc / h->A + 2);
  }
  c.take((size_t)lc * 4);
  return c.off;
}

// Workspace the shard phase needs (after `reserved` bytes).
size_t shard_ws(bcts_handle h, int64_t range, size_t reserved) {
  const int64_t lc = plan_chunk(h, range, reserved);
  return lc < h->A ? 0 : chunk_bytes(h, lc);
}
// Roots per prologue step and the workspace the finalize phase needs. A prologue step holds
// the step's roots and their A children as one batch of states ([roots | children]) plus the
// Q rows of that batch: one net evaluation serves Q_hat(s0, .) and max_a Q_hat(s1, a).
size_t prologue_root_bytes(bcts_handle h) {
  return (size_t)((h->A + 1) * node_bytes(h->env) + (int64_t)(h->A + 1) * h->A * 4);
}
int64_t prologue_per(bcts_handle h, int64_t n, size_t reserved) {
  const int64_t budget = h->ws_max - (int64_t)reserved - (2 << 20);
  int64_t per = budget > 0 ? (int64_t)((double)budget / (double)prologue_root_bytes(h)) : 1;
  return std::min(std::max<int64_t>(per, 1), n);
}
size_t prologue_ws(bcts_handle h, int64_t per) {
  Carver c(nullptr);
  c.level(h->env, per * (h->A + 1));
  c.take((size_t)per * (h->A + 1) * h->A * 4);
  return c.off;
}
size_t finalize_ws(bcts_handle h, int64_t n, size_t reserved) {
  Carver c(nullptr);
  for (int k = 0; k < 3; ++k) c.take((size_t)n * h->A * 4);   // q0, m1, r1 as finalize_impl carves them
  const size_t base = c.off;
  return base + prologue_ws(h, prologue_per(h, n, reserved + base));
}

// Leaf-range search: expand the ancestors of leaves [L0, L1), score the leaves,
// fold the totals into keys (K1 -> K2 -> K3a per chunk).
bcts_status run_shard(bcts_handle h, const void *roots, int32_t d, float gamma, int64_t L0, int64_t L1,
                      int64_t *keys, size_t reserved, bcts_stats *stats, PrologueFold *pf = nullptr) {
  const int A = h->A;
  if (L1 <= L0 || d < 1) return BCTS_OK;
  float g[kMaxDepth + 1];
  discounts(gamma, d, g);
  int64_t pw[kMaxDepth + 1];
  pw[0] = 1;
  for (int k = 1; k <= d; ++k) pw[k] = pw[k - 1] * A;
  const int64_t lc = plan_chunk(h, L1 - L0, reserved);
  if (lc < A) return fail(h, BCTS_ERR_BUDGET, "workspace budget too small for one chunk of leaves");
  if (reserved + chunk_bytes(h, lc) > h->ws_size) return fail(h, BCTS_ERR_BUDGET, "workspace not sized");
  bcts_status s = BCTS_OK;
  const bool fused = fused_leaves(h);
  const int dm = fused ? d - 1 : d;   // deepest level materialised in the workspace
  Carver c(h->ws + reserved);
  LevelBuf big = fused ? c.level(h->env, lc / A + 2) : c.level(h->env, lc);
  LevelBuf small = fused ? c.level(h->env, lc / A / A + 2) : c.level(h->env, lc / A + 2);
  float *totals = (float *)c.take((size_t)lc * 4);
  int64_t nchunks = 0, trans = 0, lvl_launch = 0;
  for (int64_t L = L0; L < L1; L += lc) {
    const int64_t Le = std::min(L1, L + lc);
    int64_t lo[kMaxDepth + 1], hi[kMaxDepth + 1];
    for (int k = 0; k <= d; ++k) {
      lo[k] = L / pw[d - k];
      hi[k] = (Le - 1) / pw[d - k] + 1;
    }
    NodeView prev = root_view(h->env, roots, lo[0]);
    int64_t vbase = lo[0];   // global level index of prev's element 0
    int expanded = 0;
    // the tf32 DNN forward model expands all of the chunk's levels in one cooperative launch
    const bool multi_level = h->env == BCTS_ENV_DNN && h->em.dnn_tc;
    DnnTcLevel mlev[kMaxDepth];
    int n_mlev = 0;
    for (int k = 1; k <= dm; ++k) {
      if (k == 1 && pf && pf->ne) {   // level 1 = the prologue front end's children (slots n .. n + nA)
        const int64_t nr = pf->ne / (A + 1);
        prev = pf->view;
        prev.state += nr * prev.state_stride;
        if (prev.key) prev.key = (const uint64_t *)((const uint8_t *)prev.key + nr * prev.key_stride);
        prev.cum += nr;
        vbase = 0;
        trans += hi[1] - lo[1];
        continue;
      }
      const LevelBuf &b = ((dm - k) % 2 == 0) ? big : small;
      if (multi_level) {   // gathered: all levels in one cooperative launch below
        DnnTcLevel &lv = mlev[n_mlev++];
        lv.par = prev;
        lv.p_first = vbase;
        lv.c_begin = lo[k];
        lv.c_end = hi[k];
        lv.gk = g[k - 1];
        lv.out = out_of(h->env, b);
      } else {
        launch_expand(h->env, prev, vbase, lo[k], hi[k], A, g[k - 1], h->em, out_of(h->env, b), h->st, &h->prof);
        ++lvl_launch;
        ++expanded;
      }
      prev = view_of(h->env, b);
      vbase = lo[k];
      trans += hi[k] - lo[k];
    }
    if (n_mlev) {
      if (launch_expand_dnn_tc_levels(mlev, n_mlev, A, h->em.dnn_tc, h->em.dnn_tc_bias, h->st, &h->prof)) {
        const cudaError_t e = cudaGetLastError();
        return fail(h, BCTS_ERR_CUDA, std::string("multi-level DNN expansion launch: ") + cudaGetErrorString(e));
      }
      ++lvl_launch;
      ++expanded;
    }
    int nl;
    bool folded = false;   // backup fused into the head's epilogue (Rainbow tcgen05 head)
    if (fused) {   // leaf level generated inside the net (s2d frames, L2-resident)
      KeyFold kf;
      kf.keys = keys;
      kf.leaf0 = L;
      kf.lpr = pw[d];
      kf.seg = pw[d - 1];
      kf.A = A;
      nl = net_eval_children(h->net, prev, vbase, L, Le, A, g[d - 1], MODE_TOTAL, g[d], totals, h->st,
                             (h->flags & BCTS_F_SEPARATE_BACKUP) ? nullptr : &kf, &folded, pf);
      trans += Le - L;
    } else {
      nl = net_eval(h->net, prev, Le - L, MODE_TOTAL, g[d], totals, h->st);
    }
    if (nl < 0) return fail(h, BCTS_ERR_CUDA, "net_eval (leaf chunk)");
    if (!folded) launch_segmax(totals, Le - L, L, pw[d], pw[d - 1], A, keys, h->st, &h->prof);
    h->launches += expanded + nl + (folded ? 0 : 1);
    ++nchunks;
    if ((s = cuda_check(h, "shard chunk"))) return s;
  }
  if (stats) {
    stats->transitions += trans;
    stats->leaves += L1 - L0;
    stats->evaluated += L1 - L0;
    stats->chunks += nchunks;
    stats->level_launches += lvl_launch;
  }
  return BCTS_OK;
}

// Depth-0/1 quantities for the BCTS terms (Prop. 1; R7):
// q0 = Q_hat(s0, .), m1[a] = max Q_hat(s1^a, .), r1[a] = R_1 of child a.
// With the level-1 terms needed, each step copies its roots' states next to their expanded
// children and evaluates the batch [roots | children] once in full-row mode (one set of net
// launches instead of two; the prologue's batches are tiny, so its cost is launch latency).
// When every root fits in one prologue step the finalize kernel reads the batch's rows and R_1
// in place (*direct set: q0 -> the root rows, *rows1 -> the level-1 rows, r1 -> R_1), which saves
// two copies and the row-max kernel; otherwise they are gathered into q0 / m1 / r1 per step.
bcts_status run_prologue(bcts_handle h, const void *roots, int64_t n, float gamma, bool need_level1, float *q0,
                         float *m1, float *r1, size_t reserved, bcts_stats *stats, const float **dq0 = nullptr,
                         const float **drows1 = nullptr, const float **dr1 = nullptr) {
  const int A = h->A;
  if (!need_level1) {
    const int nl = net_eval(h->net, root_view(h->env, roots, 0), n, MODE_ROWS, 0.0f, q0, h->st);
    h->launches += nl;
    if (stats) stats->evaluated += n;
    return cuda_check(h, "prologue");
  }
  float g[2];
  discounts(gamma, 1, g);
  const int64_t per = prologue_per(h, n, reserved);
  Carver cc(h->ws + reserved);
  LevelBuf b = cc.level(h->env, per * (A + 1));
  float *rows = (float *)cc.take((size_t)per * (A + 1) * A * 4);
  const int64_t sb = state_bytes(h->env), rb = record_bytes(h->env);
  const NodeView rv = root_view(h->env, roots, 0);
  for (int64_t r0 = 0; r0 < n; r0 += per) {
    const int64_t r1e = std::min(n, r0 + per);
    const int64_t nr = r1e - r0, cnt = nr * A;
    // slots [0, nr): the roots' states; slots [nr, nr + cnt): their children (Alg. 1 body)
    cudaMemcpy2DAsync(b.state, (size_t)sb, rv.state + r0 * rb, (size_t)rb, (size_t)sb, (size_t)nr,
                      cudaMemcpyDeviceToDevice, h->st);
    NodeOut co = out_of(h->env, b);
    co.state += nr * sb;
    if (co.key) co.key += nr;
    co.cum += nr;
    launch_expand(h->env, root_view(h->env, roots, r0), r0, r0 * A, r1e * A, A, g[0], h->em, co, h->st, &h->prof);
    const int nl = net_eval(h->net, view_of(h->env, b), nr + cnt, MODE_ROWS, 0.0f, rows, h->st);
    if (nl < 0) return fail(h, BCTS_ERR_CUDA, "net_eval (prologue)");
    if (nr == n && dq0 && drows1 && dr1) {   // one step: finalize reads the rows in place
      *dq0 = rows;
      *drows1 = rows + nr * A;
      *dr1 = b.cum + nr;
      h->launches += 1 + nl;
    } else {
      cudaMemcpyAsync(q0 + r0 * A, rows, (size_t)nr * A * 4, cudaMemcpyDeviceToDevice, h->st);
      launch_rowmax(rows + nr * A, cnt, A, m1 + r0 * A, h->st);
      cudaMemcpyAsync(r1 + r0 * A, b.cum + nr, (size_t)cnt * 4, cudaMemcpyDeviceToDevice, h->st);
      h->launches += 2 + nl;
    }
    if (stats) {
      stats->evaluated += nr + cnt;
      stats->transitions += cnt;
    }
  }
  return cuda_check(h, "prologue");
}

struct Outs {
  int32_t *actions;
  float *root_q, *vanilla, *terms;
  int64_t *best_leaf;
};

// Prologue fold (PrologueFold): bytes of the region holding [roots | level-1 children] states and
// their Q rows, and the front end that fills the states (root copy + level-1 expansion, Alg. 1
// body) -- the rows are produced later inside a leaf batch.
bool fold_wanted(bcts_handle h, int64_t n, int32_t d) {
  return d >= 1 && fused_leaves(h) && h->net.kind == BCTS_NET_RAINBOW_BF16 && n * (h->A + 1) <= (int64_t)4096 &&
         !(h->flags & BCTS_F_NO_PROLOGUE_FOLD);
}
size_t fold_bytes(bcts_handle h, int64_t n) {
  Carver pc(nullptr);
  pc.level(h->env, n * (h->A + 1));
  pc.take((size_t)n * (h->A + 1) * h->A * 4);
  return align_up(pc.off);
}
PrologueFold fold_front(bcts_handle h, const void *roots, int64_t n, float gamma, uint8_t *region) {
  const int A = h->A;
  PrologueFold pf;
  Carver pc(region);
  LevelBuf b = pc.level(h->env, n * (A + 1));
  pf.rows_out = (float *)pc.take((size_t)n * (A + 1) * A * 4);
  float g1[2];
  discounts(gamma, 1, g1);
  const int64_t sb = state_bytes(h->env), rb = record_bytes(h->env);
  const NodeView rv = root_view(h->env, roots, 0);
  // slots [0, n): the roots' states; [n, n + nA): their children
  cudaMemcpy2DAsync(b.state, (size_t)sb, rv.state, (size_t)rb, (size_t)sb, (size_t)n, cudaMemcpyDeviceToDevice, h->st);
  NodeOut co = out_of(h->env, b);
  co.state += n * sb;
  if (co.key) co.key += n;
  co.cum += n;
  launch_expand(h->env, rv, 0, 0, n * A, A, g1[0], h->em, co, h->st, &h->prof);
  h->launches += 1;
  pf.view = view_of(h->env, b);
  pf.ne = n * (A + 1);
  return pf;
}

// pre (nullable): the prologue was already evaluated (folded into a leaf batch, PrologueFold):
// pre->rows_out holds the Q rows of [roots | level-1 children] and pre->view.cum their R.
bcts_status finalize_impl(bcts_handle h, const void *roots, int64_t n, int32_t d, float gamma, float beta,
                          int32_t corr, const int64_t *keys, const Outs &o, size_t reserved, bcts_stats *stats,
                          const PrologueFold *pre = nullptr) {
  const int A = h->A;
  const bool need_q0 = corr || d == 0;
  bcts_status s = BCTS_OK;
  Carver cc(h->ws + reserved);
  float *q0 = (float *)cc.take((size_t)n * A * 4);
  float *m1 = (float *)cc.take((size_t)n * A * 4);
  float *r1 = (float *)cc.take((size_t)n * A * 4);
  const float *dq0 = nullptr, *drows1 = nullptr, *dr1 = nullptr;
  if (pre && pre->done && corr && d >= 1) {
    dq0 = pre->rows_out;
    drows1 = pre->rows_out + n * A;
    dr1 = pre->view.cum + n;
    if (stats) stats->evaluated += n * (A + 1);   // (their level-1 transitions are the shard's)
  } else if (need_q0) {
    s = run_prologue(h, roots, n, gamma, corr && d >= 1, q0, m1, r1, reserved + cc.off, stats, &dq0, &drows1, &dr1);
    if (s) return s;
  }
  float g[kMaxDepth + 1];
  discounts(gamma, d, g);
  FinalizeArgs f;
  f.n = n; f.A = A; f.d = d; f.corr = corr; f.clamp = (h->flags & BCTS_F_CLAMP_PENALTY) ? 1 : 0;
  f.beta = beta; f.g1 = d >= 1 ? g[1] : 0.0f; f.gd = g[d];
  f.keys = keys; f.q0 = q0; f.m1 = m1; f.r1 = r1;
  if (drows1) f.q0 = dq0, f.m1 = nullptr, f.rows1 = drows1, f.r1 = dr1;
  f.actions = o.actions; f.root_q = o.root_q; f.vanilla = o.vanilla; f.terms = o.terms; f.best_leaf = o.best_leaf;
  launch_finalize(f, h->st, &h->prof);
  h->launches += 1;
  return cuda_check(h, "finalize");
}

// ------------------------------------------------------------ early pruning
// NEXT-4 (R30-R33). Per-root worst-case level sizes: E[k] nodes after expanding
// level k, K[k] after its rule (BOUND: nothing pruned in the worst case; BEAM: min(beam, E/A)
// per root action). Levels 1..dm are materialised (dm = d-1 when the net generates the leaves).
struct PruneShape {
  int64_t E[kMaxDepth + 1], K[kMaxDepth + 1];
  int64_t capE = 0, leaves = 0;
};
bool prune_level(const bcts_prune &p, int k, int d) { return p.rule != BCTS_PRUNE_NONE && k >= p.first_level && k <= d - 1; }
PruneShape prune_shape(const bcts_prune &p, int A, int d, int dm) {
  PruneShape s;
  s.K[0] = s.E[0] = 1;
  for (int k = 1; k <= d; ++k) {
    s.E[k] = s.K[k - 1] * A;
    s.K[k] = s.E[k];
    if (prune_level(p, k, d) && p.rule == BCTS_PRUNE_BEAM) s.K[k] = A * std::min<int64_t>(p.beam, s.E[k] / A);
    if (k <= dm) s.capE = std::max(s.capE, s.E[k]);
  }
  s.leaves = s.E[d];
  return s;
}
// Bytes per root of one chunk: level buffers X, Y (capE each), f arrays (max(capE, leaves) each),
// flags + selection + scores (capE), totals (leaves), group maxima (A).
size_t pruned_bytes_per_root(bcts_handle h, const PruneShape &s) {
  const int64_t capF = std::max(s.capE, s.leaves);
  return (size_t)(2 * s.capE * node_bytes(h->env) + 2 * capF * 8 + s.capE * (1 + 8 + 4) + s.leaves * 4 + h->A * 8);
}
// L_k, U_k, S_k of R31 in the oracle's operation order (plain double, x86-64 host: no FMA).
void prune_bounds(const float *g, int k, int d, const bcts_prune &p, double *L, double *U, double *S) {
  double l = 0.0, u = 0.0, sa = 0.0;
  const double ra = std::max(fabs((double)p.r_lo), fabs((double)p.r_hi));
  const double qa = std::max(fabs((double)p.q_lo), fabs((double)p.q_hi));
  for (int j = k; j < d; ++j) {
    volatile double t1 = (double)g[j] * (double)p.r_lo, t2 = (double)g[j] * (double)p.r_hi, t3 = (double)g[j] * ra;
    l = l + t1;
    u = u + t2;
    sa = sa + t3;
  }
  volatile double t1 = (double)g[d] * (double)p.q_lo, t2 = (double)g[d] * (double)p.q_hi, t3 = (double)g[d] * qa;
  *L = l + t1;
  *U = u + t2;
  *S = sa + t3;
}

bcts_status run_pruned(bcts_handle h, const void *roots, int64_t n, int32_t d, float gamma, const bcts_prune &p,
                       int64_t *keys, size_t reserved, int64_t *surv, bcts_stats *stats) {
  const int A = h->A;
  const bool fused = fused_leaves(h);
  const int dm = fused ? d - 1 : d;
  const PruneShape sh = prune_shape(p, A, d, dm);
  float g[kMaxDepth + 1];
  discounts(gamma, d, g);
  int64_t pw[kMaxDepth + 1];
  pw[0] = 1;
  for (int k = 1; k <= d; ++k) pw[k] = pw[k - 1] * A;
  const size_t per_root = pruned_bytes_per_root(h, sh);
  const int64_t budget = h->ws_max - (int64_t)reserved - (8 << 20);
  int64_t per = budget > 0 ? (int64_t)((double)budget / (double)per_root) : 0;
  per = std::min<int64_t>(per, n);
  if (per < 1) return fail(h, BCTS_ERR_BUDGET, "workspace budget too small for one root of the pruned search");
  const int64_t capE = sh.capE * per, capF = std::max(sh.capE, sh.leaves) * per, capL = sh.leaves * per;
  Carver c(h->ws + reserved);
  LevelBuf X = c.level(h->env, std::max<int64_t>(capE, 1)), Y = c.level(h->env, std::max<int64_t>(capE, 1));
  int64_t *fX = (int64_t *)c.take((size_t)capF * 8), *fY = (int64_t *)c.take((size_t)capF * 8);
  uint8_t *keep = (uint8_t *)c.take((size_t)capE);
  int64_t *sel = (int64_t *)c.take((size_t)capE * 8);
  float *score = (float *)c.take((size_t)capE * 4);
  float *totals = (float *)c.take((size_t)capL * 4);
  unsigned long long *gmax = (unsigned long long *)c.take((size_t)per * A * 8);
  int64_t *d_count = (int64_t *)c.take(8);
  const size_t tbytes = compact_temp_bytes(std::max<int64_t>(capE, 1));
  void *temp = c.take(tbytes);
  if (reserved + c.off > h->ws_size) return fail(h, BCTS_ERR_BUDGET, "workspace not sized for the pruned search");
  const int64_t sb = state_bytes(h->env);
  int64_t trans = 0, evaluated = 0, leaves = 0, chunks = 0, lvl_launch = 0;
  bcts_status s = BCTS_OK;
  for (int64_t r0 = 0; r0 < n; r0 += per) {
    const int64_t nr = std::min(per, n - r0);
    // current level: view + index array; starts at the chunk's roots (f = global root index)
    NodeView cur = root_view(h->env, roots, r0);
    int64_t ncur = nr;
    int64_t *fcur = fY;
    launch_prune_iota(fcur, r0, nr, h->st);
    int inbuf = -1;   // -1: roots, 0: X, 1: Y
    h->launches += 1;
    for (int k = 1; k <= dm; ++k) {
      LevelBuf &dst = inbuf == 0 ? Y : X;
      int64_t *fdst = inbuf == 0 ? fY : fX;
      if (fdst == fcur) fdst = (fcur == fX) ? fY : fX;
      const int64_t ne = ncur * A;
      launch_expand(h->env, cur, 0, 0, ne, A, g[k - 1], h->em, out_of(h->env, dst), h->st, &h->prof);
      launch_child_index(fcur, ne, A, fdst, h->st);
      h->launches += 2;
      trans += ne;
      ++lvl_launch;
      NodeView exp = view_of(h->env, dst);
      if (!prune_level(p, k, d)) {
        cur = exp;
        fcur = fdst;
        ncur = ne;
        inbuf = (&dst == &X) ? 0 : 1;
        continue;
      }
      if (p.rule == BCTS_PRUNE_BOUND) {
        BoundRule b;
        prune_bounds(g, k, d, p, &b.L, &b.U, &b.S);
        b.gsz = pw[k - 1];
        b.g0 = r0 * A;
        b.groups = nr * A;
        launch_bound_keep(exp.cum, fdst, ne, b, gmax, keep, h->st, &h->prof);
        h->launches += 2;
      } else {
        const int nl = net_eval(h->net, exp, ne, MODE_ROWMAX, 0.0f, score, h->st);
        if (nl < 0) return fail(h, BCTS_ERR_CUDA, "net_eval (beam scores)");
        evaluated += ne;
        // every group of this level holds the same number of nodes: ne / (nr * A)
        launch_beam_keep(score, exp.cum, g[k], ne, ne / (nr * A), p.beam, keep, h->st, &h->prof);
        h->launches += nl + 1;
      }
      launch_compact(keep, ne, sel, d_count, temp, tbytes, h->st);
      int64_t kept = 0;
      cudaMemcpyAsync(&kept, d_count, 8, cudaMemcpyDeviceToHost, h->st);
      if (cudaStreamSynchronize(h->st) != cudaSuccess || (s = cuda_check(h, "prune compaction"))) return s ? s : BCTS_ERR_CUDA;
      if (kept < 1 || kept > ne) return fail(h, BCTS_ERR_NUMERIC, "prune: survivor count out of range");
      // survivors go to the other buffer (the parents' buffer is free once they are expanded)
      LevelBuf &cmp = (&dst == &X) ? Y : X;
      int64_t *fcmp = (fdst == fX) ? fY : fX;
      launch_gather_level(sb, exp, fdst, sel, kept, out_of(h->env, cmp), fcmp, h->st, &h->prof);
      h->launches += 3;
      cur = view_of(h->env, cmp);
      fcur = fcmp;
      ncur = kept;
      inbuf = (&cmp == &X) ? 0 : 1;
      if (surv) surv[k] += kept;
    }
    // leaves
    const int64_t nleaf = fused ? ncur * A : ncur;
    int64_t *fleaf = fcur;
    int nl;
    if (fused) {
      fleaf = (fcur == fX) ? fY : fX;
      launch_child_index(fcur, nleaf, A, fleaf, h->st);
      nl = net_eval_children(h->net, cur, 0, 0, nleaf, A, g[d - 1], MODE_TOTAL, g[d], totals, h->st);
      trans += nleaf;
      h->launches += 1;
    } else {
      nl = net_eval(h->net, cur, nleaf, MODE_TOTAL, g[d], totals, h->st);
    }
    if (nl < 0) return fail(h, BCTS_ERR_CUDA, "net_eval (leaves)");
    launch_segmax_f(totals, fleaf, nleaf, pw[d], pw[d - 1], keys, h->st, &h->prof);
    h->launches += nl + 1;
    evaluated += nleaf;
    leaves += nleaf;
    ++chunks;
    if ((s = cuda_check(h, "pruned chunk"))) return s;
  }
  if (stats) {
    stats->transitions += trans;
    stats->leaves += leaves;
    stats->evaluated += evaluated;
    stats->chunks += chunks;
    stats->level_launches += lvl_launch;
  }
  if (surv) surv[d] = leaves;
  return BCTS_OK;
}

// ------------------------------------------------------------ one search call
// Workspace plan of a bcts_search_ex call: [keys | folded-prologue region | phase space], the leaf
// range of this rank ([0, n A^d) on one GPU, bcts_shard_range's on rank r of a multi-GPU handle).
struct SearchPlan {
  int64_t lpr = 1, L0 = 0, L1 = 0;
  size_t kbytes0 = 0, pbytes = 0, kbytes = 0, total = 0;
  bool fold = false;
};
bcts_status plan_search(bcts_handle h, int64_t n, int32_t d, int32_t corr, SearchPlan &pl) {
  ipow_ok(h->A, d, pl.lpr);
  pl.L0 = 0;
  pl.L1 = d >= 1 ? n * pl.lpr : 0;
  if (h->world > 1 && d >= 1) bcts_shard_range(n, d, h->A, h->rank, h->world, &pl.L0, &pl.L1);
  pl.kbytes0 = align_up((size_t)n * h->A * 8);
  // with the level-1 terms needed and a conv net generating the leaves, the prologue's states
  // [roots | level-1 children] are expanded up front into a region after the keys and evaluated
  // inside this rank's last leaf batch (PrologueFold; finalize then only reads their rows)
  pl.fold = corr && fold_wanted(h, n, d) && pl.L1 > pl.L0;
  pl.pbytes = pl.fold ? fold_bytes(h, n) : 0;
  pl.kbytes = pl.kbytes0 + pl.pbytes;
  size_t need = finalize_ws(h, n, pl.kbytes);
  if (pl.L1 > pl.L0) {
    const size_t sw = shard_ws(h, pl.L1 - pl.L0, pl.kbytes);
    if (!sw) return fail(h, BCTS_ERR_BUDGET, "workspace budget too small for one chunk of leaves");
    need = std::max(need, sw);
  }
  pl.total = pl.kbytes + need;
  return BCTS_OK;
}

// Enqueue one whole search on h->st (validated arguments, sized workspace): expansion + leaf net +
// backup over this rank's leaf range, the max all-reduce of the keys on a multi-GPU handle, then
// the BCTS terms and correction (identical on every rank).
bcts_status search_body(bcts_handle h, const void *roots, int64_t n, int32_t d, float gamma, float beta, int32_t corr,
                        const Outs &o, const SearchPlan &pl, bcts_stats *stats) {
  bcts_status s = BCTS_OK;
  int64_t *keys = (int64_t *)h->ws;
  PrologueFold pf;
  if (pl.fold) pf = fold_front(h, roots, n, gamma, h->ws + pl.kbytes0);
  if (d >= 1) {
    launch_keys_init(keys, n * h->A, h->st);
    h->launches += 1;
    s = run_shard(h, roots, d, gamma, pl.L0, pl.L1, keys, pl.kbytes, stats, pl.fold ? &pf : nullptr);
    if (s) return s;
    if (h->comm) {   // the one exchange: MAX over the ranks' packed (value, ~leaf) keys
      std::string err;
      h->prof.begin(KC_COMM, 8.0 * (double)n * h->A, h->st);
      const bool ok = comm_allreduce_max_i64(h->comm, keys, n * h->A, h->st, err);
      h->prof.end(h->st);
      if (!ok) return fail(h, BCTS_ERR_NCCL, err);
    }
  }
  return finalize_impl(h, roots, n, d, gamma, beta, corr, keys, o, pl.kbytes, stats, pl.fold ? &pf : nullptr);
}

// bcts_stats.ms_*: per-phase device time of one call while profiling is on (synchronizes)
struct PhaseTimer {
  bcts_handle h;
  bool on;
  cudaEvent_t a = nullptr, b = nullptr;
  double before[KC_COUNT] = {};
  PhaseTimer(bcts_handle hh, bcts_stats *stats) : h(hh), on(stats && hh->prof.on) {
    if (!on) return;
    cudaStreamSynchronize(h->st);
    h->prof.collect();
    for (int c = 0; c < KC_COUNT; ++c) before[c] = h->prof.ms[c];
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, h->st);
  }
  void finish(bcts_stats *st) {
    if (!on) return;
    cudaEventRecord(b, h->st);
    cudaStreamSynchronize(h->st);
    h->prof.collect();
    float t = 0.f;
    cudaEventElapsedTime(&t, a, b);
    st->ms_total = t;
    auto d = [&](int c) { return (float)(h->prof.ms[c] - before[c]); };
    st->ms_expand = d(KC_EXPAND_ATARI) + d(KC_EXPAND_INT) + d(KC_EXPAND_TAB) + d(KC_EXPAND_DNN);
    st->ms_leaf = d(KC_CONV1) + d(KC_CONV2) + d(KC_CONV3) + d(KC_CONV23) + d(KC_FC_H) + d(KC_FC_OUT) + d(KC_HEAD) +
                  d(KC_MLP) + d(KC_TABLE) + d(KC_OTHER);
    st->ms_backup = d(KC_SEGMAX) + d(KC_FINALIZE) + d(KC_PRUNE);
    st->ms_comm = d(KC_COMM);
  }
  ~PhaseTimer() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
};

}  // namespace

// =================================================================== C ABI
extern "C" {

int32_t bcts_abi_version(void) { return BCTS_ABI_VERSION; }

const char *bcts_status_string(bcts_status s) {
  switch (s) {
    case BCTS_OK: return "BCTS_OK";
    case BCTS_ERR_INVALID_ARG: return "BCTS_ERR_INVALID_ARG";
    case BCTS_ERR_UNSUPPORTED: return "BCTS_ERR_UNSUPPORTED";
    case BCTS_ERR_OUT_OF_MEMORY: return "BCTS_ERR_OUT_OF_MEMORY";
    case BCTS_ERR_BUDGET: return "BCTS_ERR_BUDGET";
    case BCTS_ERR_CUDA: return "BCTS_ERR_CUDA";
    case BCTS_ERR_NCCL: return "BCTS_ERR_NCCL";
    case BCTS_ERR_NUMERIC: return "BCTS_ERR_NUMERIC";
  }
  return "BCTS_ERR_UNKNOWN";
}

const char *bcts_last_error(bcts_handle h) { return h ? h->err.c_str() : "null handle"; }

size_t bcts_root_record_bytes(bcts_handle h) { return h ? (size_t)record_bytes(h->env) : 0; }

void bcts_destroy(bcts_handle h) {
  if (!h) return;
  cudaSetDevice(h->dev);
  if (h->st) cudaStreamSynchronize(h->st);
  comm_destroy(h->comm);
  net_free(h->net);
  cudaFree(h->pbuf);
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->dexec) cudaGraphExecDestroy(h->dexec);
  if (h->gst) cudaStreamDestroy(h->gst);
  cudaFree(h->d_next);
  cudaFree(h->d_envw);
  cudaFree(h->d_envw_tc);
  cudaFree(h->d_rew);
  if (h->ws_own) cudaFree(h->ws);
  cudaFree(h->scratch_own);
  cudaFree(h->e2e_roots);
  cudaFree(h->e2e_act);
  cudaFree(h->e2e_q);
  if (h->own_stream && h->st) cudaStreamDestroy(h->st);
  delete h;
}

bcts_status bcts_create(const bcts_config *cfg, bcts_handle *out) {
  if (!cfg || !out) return BCTS_ERR_INVALID_ARG;
  *out = nullptr;
  if (cfg->abi_version != BCTS_ABI_VERSION) return BCTS_ERR_INVALID_ARG;
  if (cfg->num_actions < 2 || cfg->num_actions > kMaxA) return BCTS_ERR_INVALID_ARG;
  const bool env_ok = cfg->env == BCTS_ENV_TABULAR || cfg->env == BCTS_ENV_INT_HASH ||
                      cfg->env == BCTS_ENV_ATARI_HASH || cfg->env == BCTS_ENV_DNN;
  if (!env_ok) return BCTS_ERR_INVALID_ARG;
  const bool pair_ok = (cfg->env == BCTS_ENV_TABULAR && cfg->net == BCTS_NET_TABLE) ||
                       (cfg->env == BCTS_ENV_INT_HASH && cfg->net == BCTS_NET_MLP2_F32) ||
                       (cfg->env == BCTS_ENV_DNN && cfg->net == BCTS_NET_MLP2_F32) ||
                       (cfg->env == BCTS_ENV_ATARI_HASH &&
                        (cfg->net == BCTS_NET_NATURE_BF16 || cfg->net == BCTS_NET_RAINBOW_BF16));
  if (!pair_ok) return BCTS_ERR_UNSUPPORTED;
  if (cfg->env == BCTS_ENV_TABULAR) {
    if (cfg->num_states <= 0 || !cfg->tab_next || !cfg->tab_reward || !cfg->tab_q) return BCTS_ERR_INVALID_ARG;
    for (int64_t i = 0; i < (int64_t)cfg->num_states * cfg->num_actions; ++i)
      if (cfg->tab_next[i] < 0 || cfg->tab_next[i] >= cfg->num_states) return BCTS_ERR_INVALID_ARG;
  }
  if (cfg->env == BCTS_ENV_DNN &&
      (!cfg->env_weights || cfg->env_weights_count != dnn_env_weights_count(cfg->num_actions)))
    return BCTS_ERR_INVALID_ARG;
  if (cfg->world > 1 && !cfg->nccl_unique_id) return BCTS_ERR_INVALID_ARG;
  if (cfg->rank < 0 || cfg->rank >= std::max(cfg->world, 1)) return BCTS_ERR_INVALID_ARG;
  bcts_handle h = new (std::nothrow) bcts_handle_t();
  if (!h) return BCTS_ERR_OUT_OF_MEMORY;
  h->dev = cfg->device;
  h->env = cfg->env;
  h->A = cfg->num_actions;
  h->nS = cfg->num_states;
  h->flags = cfg->flags;
  h->ws_max = cfg->workspace_bytes_max > 0 ? cfg->workspace_bytes_max : kDefaultWorkspace;
  if (cudaSetDevice(cfg->device) != cudaSuccess) {
    cudaGetLastError();
    delete h;
    return BCTS_ERR_CUDA;
  }
  // NULL is the legacy default stream (CUDA's stream 0), which is also what
  // torch.cuda.current_stream() reports as 0: calls then order with torch's work.
  h->st = (cudaStream_t)cfg->cuda_stream;
  if (cfg->env == BCTS_ENV_TABULAR) {
    const size_t cnt = (size_t)cfg->num_states * cfg->num_actions;
    if (cudaMalloc(&h->d_next, cnt * 4) != cudaSuccess || cudaMalloc(&h->d_rew, cnt * 4) != cudaSuccess ||
        cudaMemcpy(h->d_next, cfg->tab_next, cnt * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(h->d_rew, cfg->tab_reward, cnt * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaGetLastError();
      bcts_destroy(h);
      return BCTS_ERR_CUDA;
    }
    h->em.tab_next = h->d_next;
    h->em.tab_rew = h->d_rew;
  }
  if (cfg->env == BCTS_ENV_DNN) {
    std::vector<float> img((size_t)kDnnImg + (size_t)kDnnS * cfg->num_actions);
    dnn_repack(cfg->env_weights, cfg->num_actions, img.data());
    if (cudaMalloc(&h->d_envw, img.size() * 4) != cudaSuccess ||
        cudaMemcpy(h->d_envw, img.data(), img.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaGetLastError();
      bcts_destroy(h);
      return BCTS_ERR_CUDA;
    }
    h->em.dnn = h->d_envw;
    if (cfg->flags & BCTS_F_TF32) {
      if (!dnn_tc_ok(cfg->num_actions)) {
        bcts_destroy(h);
        return BCTS_ERR_INVALID_ARG;
      }
      std::vector<float> tc(dnn_tc_image_floats(cfg->num_actions));
      dnn_tc_repack(cfg->env_weights, cfg->num_actions, tc.data());
      if (cudaMalloc(&h->d_envw_tc, tc.size() * 4) != cudaSuccess ||
          cudaMemcpy(h->d_envw_tc, tc.data(), tc.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaGetLastError();
        bcts_destroy(h);
        return BCTS_ERR_CUDA;
      }
      h->em.dnn_tc = h->d_envw_tc;
      h->envw_tc_bias.assign(tc.begin() + kDnnTcBiasOffset, tc.begin() + kDnnTcBiasOffset + 4 * 112);
      h->em.dnn_tc_bias = h->envw_tc_bias.data();
    }
  }
  std::string err;
  if (net_build(h->net, *cfg, err)) {   // weight validation and repacking (no scratch yet)
    const bool cuda = cudaGetLastError() != cudaSuccess || err.find("cuda") != std::string::npos ||
                      err.find("upload") != std::string::npos;
    bcts_destroy(h);
    return cuda ? BCTS_ERR_CUDA : BCTS_ERR_INVALID_ARG;
  }
  h->net.tc = !(cfg->flags & BCTS_F_SIMT_NET);
  h->net.sw = true;
  h->net.prof = &h->prof;
  if (cfg->world > 1 || cfg->nccl_unique_id) {   // collective: every rank creates its handle with the same id
    h->rank = cfg->rank;
    h->world = std::max(cfg->world, 1);
    if (!comm_init(&h->comm, cfg->nccl_unique_id, cfg->rank, cfg->world, err)) {
      h->comm = nullptr;
      bcts_destroy(h);
      return BCTS_ERR_NCCL;
    }
  }
  *out = h;
  return BCTS_OK;
}

bcts_status bcts_keys_init(bcts_handle h, int64_t *keys, int64_t count) {
  if (!h || count < 0 || (count > 0 && !keys)) return BCTS_ERR_INVALID_ARG;
  cudaSetDevice(h->dev);
  launch_keys_init(keys, count, h->st);
  h->launches += count > 0;
  return cuda_check(h, "keys_init");
}

bcts_status bcts_search_shard(bcts_handle h, const void *roots, int64_t n_roots, int32_t depth, int32_t A,
                              float gamma, int64_t leaf_begin, int64_t leaf_end, int64_t *keys_out,
                              bcts_stats *stats) {
  bcts_status s = validate(h, roots, n_roots, depth, A, gamma);
  if (s) return s;
  int64_t lpr;
  ipow_ok(A, depth, lpr);
  if (depth < 1) return fail(h, BCTS_ERR_INVALID_ARG, "shard search needs depth >= 1");
  if (leaf_begin < 0 || leaf_end < leaf_begin || leaf_end > n_roots * lpr)
    return fail(h, BCTS_ERR_INVALID_ARG, "leaf range outside [0, n_roots*A^d)");
  if (leaf_end > leaf_begin && !keys_out) return fail(h, BCTS_ERR_INVALID_ARG, "keys_out is NULL");
  cudaSetDevice(h->dev);
  if (stats) memset(stats, 0, sizeof(*stats));
  const int64_t l0 = h->launches;
  if ((s = ensure_net(h))) return s;
  if (leaf_end > leaf_begin) {
    const size_t need = shard_ws(h, leaf_end - leaf_begin, 0);
    if (!need) return fail(h, BCTS_ERR_BUDGET, "workspace budget too small for one chunk of leaves");
    if ((s = ensure_ws(h, need))) return s;
  }
  // the finalize prologue rides along in this shard's last leaf batch; bcts_finalize picks it up
  h->pfs_valid = false;
  PrologueFold *pf = nullptr;
  if (leaf_end > leaf_begin && fold_wanted(h, n_roots, depth)) {
    const size_t pb = fold_bytes(h, n_roots);
    if (pb > h->pbuf_size) {
      cudaFree(h->pbuf);
      h->pbuf = nullptr;
      h->pbuf_size = 0;
      if (cudaMalloc(&h->pbuf, pb) == cudaSuccess) h->pbuf_size = pb;
      cudaGetLastError();
    }
    if (h->pbuf) {
      h->pfs = fold_front(h, roots, n_roots, gamma, h->pbuf);
      pf = &h->pfs;
    }
  }
  s = run_shard(h, roots, depth, gamma, leaf_begin, leaf_end, keys_out, 0, stats, pf);
  if (!s && pf && pf->done) {
    h->pfs_valid = true;
    h->pfs_roots = roots;
    h->pfs_n = n_roots;
    h->pfs_d = depth;
    h->pfs_gamma = gamma;
  }
  if (stats) stats->kernel_launches = h->launches - l0;
  return s;
}

bcts_status bcts_finalize(bcts_handle h, const void *roots, int64_t n_roots, int32_t depth, int32_t A, float gamma,
                          float beta, int32_t correction_on, const int64_t *keys, int32_t *actions_out,
                          float *root_q_out, float *vanilla_q_out, float *terms_out, int64_t *best_leaf_out,
                          bcts_stats *stats) {
  bcts_status s = validate(h, roots, n_roots, depth, A, gamma);
  if (s) return s;
  if (!isfinite(beta) || beta < 0.0f) return fail(h, BCTS_ERR_INVALID_ARG, "beta must be finite and >= 0");
  if (correction_on < 0 || correction_on > 2) return fail(h, BCTS_ERR_INVALID_ARG, "correction_on not in {0,1,2}");
  if (n_roots == 0) return BCTS_OK;
  if (!actions_out || !root_q_out || (depth >= 1 && !keys))
    return fail(h, BCTS_ERR_INVALID_ARG, "NULL required pointer");
  cudaSetDevice(h->dev);
  const int64_t l0 = h->launches;
  Outs o{actions_out, root_q_out, vanilla_q_out, terms_out, best_leaf_out};
  if ((s = ensure_net(h))) return s;
  if ((s = ensure_ws(h, finalize_ws(h, n_roots, 0)))) return s;
  const bool pre = h->pfs_valid && h->pfs_roots == roots && h->pfs_n == n_roots && h->pfs_d == depth &&
                   h->pfs_gamma == gamma;
  h->pfs_valid = false;
  s = finalize_impl(h, roots, n_roots, depth, gamma, beta, correction_on, keys, o, 0, stats, pre ? &h->pfs : nullptr);
  if (stats) stats->kernel_launches += h->launches - l0;
  return s;
}

bcts_status bcts_search_ex(bcts_handle h, const void *roots, int64_t n_roots, int32_t depth, int32_t A, float gamma,
                           float beta, int32_t correction_on, int32_t *actions_out, float *root_q_out,
                           float *vanilla_q_out, float *terms_out, int64_t *best_leaf_out, bcts_stats *stats) {
  bcts_status s = validate(h, roots, n_roots, depth, A, gamma);
  if (s) return s;
  if (!isfinite(beta) || beta < 0.0f) return fail(h, BCTS_ERR_INVALID_ARG, "beta must be finite and >= 0");
  if (correction_on < 0 || correction_on > 2) return fail(h, BCTS_ERR_INVALID_ARG, "correction_on not in {0,1,2}");
  if (n_roots > 0 && (!actions_out || !root_q_out)) return fail(h, BCTS_ERR_INVALID_ARG, "NULL output pointer");
  if (stats) memset(stats, 0, sizeof(*stats));
  if (n_roots == 0) return BCTS_OK;
  cudaSetDevice(h->dev);
  const int64_t l0 = h->launches;
  SearchPlan pl;
  if ((s = plan_search(h, n_roots, depth, correction_on, pl))) return s;
  if ((s = ensure_net(h))) return s;
  if ((s = ensure_ws(h, pl.total))) return s;
  const Outs o{actions_out, root_q_out, vanilla_q_out, terms_out, best_leaf_out};
  // graph replay of an identical previous call (device pointers and workspace included)
  const bool graphable = !(h->flags & BCTS_F_NO_GRAPH) && !h->prof.on && !h->capturing && h->env != BCTS_ENV_TABULAR;
  bcts_handle_t::DevKey key;
  key.roots = roots, key.n = n_roots, key.d = depth, key.A = A, key.corr = correction_on;
  key.gamma = gamma, key.beta = beta, key.ws = h->ws, key.wss = h->ws_size, key.scratch = h->net.scratch;
  key.o[0] = actions_out, key.o[1] = root_q_out, key.o[2] = vanilla_q_out, key.o[3] = terms_out, key.o[4] = best_leaf_out;
  if (graphable && h->dvalid && key == h->dkey) {
    if (cudaGraphLaunch(h->dexec, h->st) == cudaSuccess) {
      if (stats) *stats = h->dstats;
      return cuda_check(h, "graph replay");
    }
    cudaGetLastError();
    h->dvalid = false;
  }
  PhaseTimer pt(h, stats);
  bcts_stats st_local;
  memset(&st_local, 0, sizeof(st_local));
  s = search_body(h, roots, n_roots, depth, gamma, beta, correction_on, o, pl, &st_local);
  if (s) return s;
  st_local.kernel_launches = h->launches - l0;
  pt.finish(&st_local);
  if (stats) *stats = st_local;
  // the same arguments twice in a row: capture this sequence for the calls that follow
  if (graphable && !h->dvalid && key == h->dkey) {
    if (!h->gst) cudaStreamCreateWithFlags(&h->gst, cudaStreamNonBlocking);
    cudaStream_t saved = h->st;
    cudaGraph_t g = nullptr;
    bool ok = h->gst && cudaStreamBeginCapture(h->gst, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      h->st = h->gst;
      h->capturing = true;
      bcts_stats scratch_stats;
      memset(&scratch_stats, 0, sizeof(scratch_stats));
      const bcts_status sc = search_body(h, roots, n_roots, depth, gamma, beta, correction_on, o, pl, &scratch_stats);
      h->capturing = false;
      h->st = saved;
      ok = cudaStreamEndCapture(h->gst, &g) == cudaSuccess && sc == BCTS_OK && g;
    }
    h->err.clear();
    cudaGraphExec_t ex = nullptr;
    if (ok && cudaGraphInstantiate(&ex, g, 0) == cudaSuccess) {
      if (h->dexec) cudaGraphExecDestroy(h->dexec);
      h->dexec = ex;
      h->dvalid = true;
      h->dstats = st_local;
      h->dstats.ms_total = h->dstats.ms_expand = h->dstats.ms_leaf = h->dstats.ms_backup = h->dstats.ms_comm = 0.f;
    }
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
  }
  if (!(key == h->dkey)) h->dvalid = false;
  h->dkey = key;
  return BCTS_OK;
}

bcts_status bcts_nccl_unique_id(void *out128) {
  if (!out128) return BCTS_ERR_INVALID_ARG;
  std::string err;
  return comm_unique_id(out128, err) ? BCTS_OK : BCTS_ERR_NCCL;
}

bcts_status bcts_workspace_size(bcts_handle h, int64_t n_roots, int32_t depth, size_t *bytes) {
  if (!h || !bytes || n_roots < 0 || depth < 0 || depth > kMaxDepth) return BCTS_ERR_INVALID_ARG;
  SearchPlan pl;
  size_t tree = 0;
  if (n_roots > 0) {
    bcts_status s = plan_search(h, n_roots, depth, 1, pl);
    if (s) return s;
    tree = pl.total;
  }
  *bytes = align_up(net_scratch_bytes(h->net)) + tree;
  return BCTS_OK;
}

bcts_status bcts_set_workspace(bcts_handle h, void *dev_ptr, size_t bytes) {
  if (!h) return BCTS_ERR_INVALID_ARG;
  if (dev_ptr && ((uintptr_t)dev_ptr % 256 != 0 || bytes < align_up(net_scratch_bytes(h->net))))
    return fail(h, BCTS_ERR_INVALID_ARG, "caller workspace misaligned or smaller than the net scratch (" +
                                             std::to_string(net_scratch_bytes(h->net)) + " bytes)");
  cudaSetDevice(h->dev);
  if (cudaStreamSynchronize(h->st) != cudaSuccess) return cuda_check(h, "set_workspace sync");
  std::string err;
  // drop the current memory (graphs bake its addresses in)
  h->dvalid = h->gvalid = false;
  if (h->ws_own) cudaFree(h->ws);
  h->ws = nullptr;
  h->ws_size = 0;
  cudaFree(h->scratch_own);
  h->scratch_own = nullptr;
  net_bind_scratch(h->net, nullptr, err);
  h->ext = (uint8_t *)dev_ptr;
  h->ext_bytes = dev_ptr ? bytes : 0;
  h->ws_own = dev_ptr == nullptr;
  if (dev_ptr) {
    const size_t ns = align_up(net_scratch_bytes(h->net));
    h->ws = h->ext + ns;
    h->ws_size = bytes - ns;
    bcts_status s = ensure_net(h);
    if (s) return s;
  }
  return cuda_check(h, "set_workspace");
}

bcts_status bcts_search_pruned(bcts_handle h, const void *roots, int64_t n_roots, int32_t depth, int32_t A,
                               float gamma, float beta, int32_t correction_on, const bcts_prune *prune,
                               int32_t *actions_out, float *root_q_out, float *vanilla_q_out, float *terms_out,
                               int64_t *best_leaf_out, int64_t *survivors_out, bcts_stats *stats) {
  bcts_status s = validate(h, roots, n_roots, depth, A, gamma);
  if (s) return s;
  if (!prune) return fail(h, BCTS_ERR_INVALID_ARG, "prune is NULL");
  if (depth < 1) return fail(h, BCTS_ERR_INVALID_ARG, "pruned search needs depth >= 1");
  bcts_prune p = *prune;
  if (p.rule < BCTS_PRUNE_NONE || p.rule > BCTS_PRUNE_BEAM) return fail(h, BCTS_ERR_INVALID_ARG, "unknown prune rule");
  if (p.rule == BCTS_PRUNE_BEAM && p.beam < 1) return fail(h, BCTS_ERR_INVALID_ARG, "beam must be >= 1");
  if (p.rule == BCTS_PRUNE_BOUND &&
      (!isfinite(p.r_lo) || !isfinite(p.r_hi) || !isfinite(p.q_lo) || !isfinite(p.q_hi) || p.r_lo > p.r_hi ||
       p.q_lo > p.q_hi))
    return fail(h, BCTS_ERR_INVALID_ARG, "BOUND needs finite r_lo <= r_hi and q_lo <= q_hi");
  if (p.first_level < 1) p.first_level = 1;
  if (!isfinite(beta) || beta < 0.0f) return fail(h, BCTS_ERR_INVALID_ARG, "beta must be finite and >= 0");
  if (correction_on < 0 || correction_on > 2) return fail(h, BCTS_ERR_INVALID_ARG, "correction_on not in {0,1,2}");
  if (n_roots > 0 && (!actions_out || !root_q_out)) return fail(h, BCTS_ERR_INVALID_ARG, "NULL output pointer");
  if (stats) memset(stats, 0, sizeof(*stats));
  if (survivors_out) {
    for (int k = 0; k <= depth; ++k) survivors_out[k] = 0;
    survivors_out[0] = n_roots;
  }
  if (n_roots == 0) return BCTS_OK;
  cudaSetDevice(h->dev);
  const int64_t l0 = h->launches;
  const size_t kbytes = align_up((size_t)n_roots * A * 8);
  const bool fused = fused_leaves(h);
  const PruneShape sh = prune_shape(p, A, depth, fused ? depth - 1 : depth);
  const size_t per_root = pruned_bytes_per_root(h, sh);
  const int64_t budget = h->ws_max - (int64_t)kbytes - (8 << 20);
  const int64_t per = budget > 0 ? std::min<int64_t>(n_roots, (int64_t)((double)budget / (double)per_root)) : 0;
  if (per < 1) return fail(h, BCTS_ERR_BUDGET, "workspace budget too small for one root of the pruned search");
  const size_t need = std::max(finalize_ws(h, n_roots, kbytes),
                               (size_t)per * per_root + compact_temp_bytes(sh.capE * per) + (4 << 20));
  if ((s = ensure_net(h))) return s;
  if ((s = ensure_ws(h, kbytes + need))) return s;
  int64_t *keys = (int64_t *)h->ws;
  launch_keys_init(keys, n_roots * A, h->st);
  h->launches += 1;
  // pruned levels accumulate their survivors over the root chunks; unpruned levels are A x the level above
  int64_t surv[kMaxDepth + 1] = {0};
  s = run_pruned(h, roots, n_roots, depth, gamma, p, keys, kbytes, surv, stats);
  if (s) return s;
  if (survivors_out) {
    int64_t cnt = n_roots;
    for (int k = 1; k < depth; ++k) {
      cnt = prune_level(p, k, depth) ? surv[k] : cnt * A;
      survivors_out[k] = cnt;
    }
    survivors_out[depth] = surv[depth];
  }
  Outs o{actions_out, root_q_out, vanilla_q_out, terms_out, best_leaf_out};
  s = finalize_impl(h, roots, n_roots, depth, gamma, beta, correction_on, keys, o, kbytes, stats);
  if (stats) stats->kernel_launches = h->launches - l0;
  return s;
}

bcts_status bcts_search(bcts_handle h, const void *roots, int64_t n_roots, int32_t depth, int32_t A, float gamma,
                        float beta, int32_t correction_on, int32_t *actions_out, float *root_q_out) {
  return bcts_search_ex(h, roots, n_roots, depth, A, gamma, beta, correction_on, actions_out, root_q_out, nullptr,
                        nullptr, nullptr, nullptr);
}

bcts_status bcts_search_host(bcts_handle h, const void *roots_host, int64_t n_roots, int32_t depth, int32_t A,
                             float gamma, float beta, int32_t correction_on, int32_t *actions_host,
                             float *root_q_host) {
  if (!h) return BCTS_ERR_INVALID_ARG;
  if (n_roots < 0 || (n_roots > 0 && (!roots_host || !actions_host || !root_q_host)))
    return fail(h, BCTS_ERR_INVALID_ARG, "NULL host pointer or n_roots < 0");
  if (n_roots == 0) return BCTS_OK;
  cudaSetDevice(h->dev);
  const size_t rb = (size_t)n_roots * record_bytes(h->env);
  if (rb > h->e2e_roots_size) {
    h->gvalid = false;   // the graph copies into the old buffer
    cudaFree(h->e2e_roots);
    h->e2e_roots = nullptr;
    h->e2e_roots_size = 0;
    if (cudaMalloc(&h->e2e_roots, rb) != cudaSuccess) {
      cudaGetLastError();
      h->e2e_roots = nullptr;
      return fail(h, BCTS_ERR_OUT_OF_MEMORY, "e2e roots buffer");
    }
    h->e2e_roots_size = rb;
  }
  if ((size_t)n_roots * A > h->e2e_out) {
    h->gvalid = false;
    cudaFree(h->e2e_act);
    cudaFree(h->e2e_q);
    h->e2e_act = nullptr;
    h->e2e_q = nullptr;
    h->e2e_out = 0;
    if (cudaMalloc(&h->e2e_act, (size_t)n_roots * 4) != cudaSuccess ||
        cudaMalloc(&h->e2e_q, (size_t)n_roots * A * 4) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(h->e2e_act);
      cudaFree(h->e2e_q);
      h->e2e_act = nullptr;
      h->e2e_q = nullptr;
      return fail(h, BCTS_ERR_OUT_OF_MEMORY, "e2e output buffers");
    }
    h->e2e_out = (size_t)n_roots * A;
  }
  // One call = H2D of the roots, the search, D2H of the outputs. With page-locked host buffers the
  // sequence is captured once as a CUDA graph (after an eager run with the same arguments, so every
  // buffer exists) and replayed: one launch instead of ~20 kernel / copy enqueues from the host.
  auto pinned = [](const void *p) {
    cudaPointerAttributes a;
    const bool ok = cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeHost;
    cudaGetLastError();
    return ok;
  };
  // TABULAR checks its root ids on the host (a synchronizing copy), which a capture cannot hold
  const bool can_graph = !h->prof.on && !(h->flags & BCTS_F_NO_GRAPH) && h->env != BCTS_ENV_TABULAR &&
                         pinned(roots_host) && pinned(actions_host) && pinned(root_q_host);
  bcts_handle_t::GraphKey key;
  key.rh = roots_host, key.ah = actions_host, key.qh = root_q_host, key.n = n_roots, key.d = depth, key.A = A;
  key.corr = correction_on, key.gamma = gamma, key.beta = beta, key.ws = h->ws, key.wss = h->ws_size;
  key.dr = h->e2e_roots, key.da = h->e2e_act, key.dq = h->e2e_q, key.scratch = h->net.scratch;
  if (can_graph && h->gvalid && key == h->gkey) {
    if (cudaGraphLaunch(h->gexec, h->st) == cudaSuccess && cudaStreamSynchronize(h->st) == cudaSuccess)
      return cuda_check(h, "e2e graph");
    cudaGetLastError();
    h->gvalid = false;
  }
  auto enqueue = [&]() -> bcts_status {
    if (cudaMemcpyAsync(h->e2e_roots, roots_host, rb, cudaMemcpyHostToDevice, h->st) != cudaSuccess)
      return cuda_check(h, "e2e H2D");
    bcts_status s2 = bcts_search(h, h->e2e_roots, n_roots, depth, A, gamma, beta, correction_on, h->e2e_act, h->e2e_q);
    if (s2) return s2;
    cudaMemcpyAsync(actions_host, h->e2e_act, (size_t)n_roots * 4, cudaMemcpyDeviceToHost, h->st);
    cudaMemcpyAsync(root_q_host, h->e2e_q, (size_t)n_roots * A * 4, cudaMemcpyDeviceToHost, h->st);
    return BCTS_OK;
  };
  bcts_status s = enqueue();
  if (s) return s;
  if (cudaStreamSynchronize(h->st) != cudaSuccess) return cuda_check(h, "e2e sync");
  if ((s = cuda_check(h, "e2e D2H"))) return s;
  if (can_graph) {   // capture the same sequence on a private stream for the next call
    h->gvalid = false;
    if (!h->gst) cudaStreamCreateWithFlags(&h->gst, cudaStreamNonBlocking);
    key.ws = h->ws, key.wss = h->ws_size, key.scratch = h->net.scratch;
    cudaStream_t saved = h->st;
    h->st = h->gst;
    cudaGraph_t g = nullptr;
    bool ok = h->gst && cudaStreamBeginCapture(h->gst, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      h->capturing = true;
      const bcts_status sc = enqueue();
      h->capturing = false;
      ok = cudaStreamEndCapture(h->gst, &g) == cudaSuccess && sc == BCTS_OK && g;
    }
    h->st = saved;
    h->err.clear();
    if (ok && h->ws == key.ws && h->ws_size == key.wss) {
      cudaGraphExec_t ex = nullptr;
      if (cudaGraphInstantiate(&ex, g, 0) == cudaSuccess) {
        if (h->gexec) cudaGraphExecDestroy(h->gexec);
        h->gexec = ex;
        h->gkey = key;
        h->gvalid = true;
      }
    }
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
  }
  return BCTS_OK;
}

bcts_status bcts_expand(bcts_handle h, const void *roots, int64_t n_roots, int32_t level, int32_t A, float gamma,
                        void *states_out, float *cum_out) {
  bcts_status s = validate(h, roots, n_roots, level, A, gamma);
  if (s) return s;
  if (n_roots == 0) return BCTS_OK;
  if (!states_out || !cum_out) return fail(h, BCTS_ERR_INVALID_ARG, "NULL output pointer");
  cudaSetDevice(h->dev);
  const int env = h->env;
  const int64_t rb = record_bytes(env);
  int64_t cnt;
  ipow_ok(A, level, cnt);
  cnt *= n_roots;
  if (level == 0) {
    cudaMemcpyAsync(states_out, roots, (size_t)(n_roots * rb), cudaMemcpyDeviceToDevice, h->st);
    cudaMemsetAsync(cum_out, 0, (size_t)n_roots * 4, h->st);
    return cuda_check(h, "expand level 0");
  }
  Carver c(nullptr);
  c.level(env, cnt);
  c.level(env, cnt / A);
  if ((int64_t)c.off > h->ws_max) return fail(h, BCTS_ERR_BUDGET, "level does not fit the workspace budget");
  if ((s = ensure_ws(h, c.off))) return s;
  Carver cc(h->ws);
  LevelBuf big = cc.level(env, cnt), small = cc.level(env, cnt / A);
  float g[kMaxDepth + 1];
  discounts(gamma, level, g);
  NodeView prev = root_view(env, roots, 0);
  int64_t n_prev = n_roots;
  for (int k = 1; k <= level; ++k) {
    const LevelBuf &b = ((level - k) % 2 == 0) ? big : small;
    launch_expand(env, prev, 0, 0, n_prev * A, A, g[k - 1], h->em, out_of(env, b), h->st);
    prev = view_of(env, b);
    n_prev *= A;
    h->launches += 1;
  }
  uint8_t *dst = (uint8_t *)states_out;
  if (env == BCTS_ENV_ATARI_HASH) {
    cudaMemcpy2DAsync(dst, rb, big.key, 8, 8, cnt, cudaMemcpyDeviceToDevice, h->st);
    cudaMemset2DAsync(dst + 8, rb, 0, 8, cnt, h->st);
    cudaMemcpy2DAsync(dst + 16, rb, big.state, kFrameBytes, kFrameBytes, cnt, cudaMemcpyDeviceToDevice, h->st);
  } else {
    cudaMemcpyAsync(dst, big.state, (size_t)(cnt * rb), cudaMemcpyDeviceToDevice, h->st);
  }
  cudaMemcpyAsync(cum_out, big.cum, (size_t)cnt * 4, cudaMemcpyDeviceToDevice, h->st);
  return cuda_check(h, "expand");
}

bcts_status bcts_q_rows(bcts_handle h, const void *states, int64_t n, float *q_out) {
  if (!h || n < 0 || (n > 0 && (!states || !q_out))) return BCTS_ERR_INVALID_ARG;
  if (n == 0) return BCTS_OK;
  cudaSetDevice(h->dev);
  bcts_status s = ensure_net(h);
  if (s) return s;
  h->launches += net_eval(h->net, root_view(h->env, states, 0), n, MODE_ROWS, 0.0f, q_out, h->st);
  return cuda_check(h, "q_rows");
}

bcts_status bcts_pv_targets(bcts_handle h, int64_t n_roots, int32_t depth, const int32_t *actions,
                            const float *vanilla_q, const int64_t *best_leaf, float *target_out,
                            int32_t *path_out) {
  if (!h || n_roots < 0 || depth < 1 || depth > kMaxDepth) return BCTS_ERR_INVALID_ARG;
  if (n_roots == 0) return BCTS_OK;
  if (!actions || !vanilla_q || !best_leaf || !target_out || !path_out) return BCTS_ERR_INVALID_ARG;
  cudaSetDevice(h->dev);
  launch_pv_targets(n_roots, h->A, depth, actions, vanilla_q, best_leaf, target_out, path_out, h->st);
  h->launches += 1;
  return cuda_check(h, "pv_targets");
}

bcts_status bcts_profile_enable(bcts_handle h, int32_t on) {
  if (!h) return BCTS_ERR_INVALID_ARG;
  cudaSetDevice(h->dev);
  cudaStreamSynchronize(h->st);
  h->prof.reset();
  h->prof.on = on != 0;
  return cuda_check(h, "profile_enable");
}

int32_t bcts_profile_read(bcts_handle h, bcts_kernel_profile *out, int32_t max) {
  static const char *names[KC_COUNT] = {"expand_atari", "expand_int", "expand_tabular", "conv1", "conv2", "conv3",
                                        "fc_hidden", "fc_out", "head", "mlp", "table", "segmax", "finalize", "other",
                                        "expand_dnn", "conv2+conv3", "prune", "comm"};
  static const int units[KC_COUNT] = {0, 0, 0, 1, 1, 1, 1, 1, 0, 1, 0, 0, 0, 0, 1, 1, 0, 0};
  if (!h || !out || max <= 0) return 0;
  cudaSetDevice(h->dev);
  cudaStreamSynchronize(h->st);
  h->prof.collect();
  int32_t k = 0;
  for (int c = 0; c < KC_COUNT && k < max; ++c) {
    if (!h->prof.launches[c]) continue;
    memset(&out[k], 0, sizeof(out[k]));
    strncpy(out[k].name, names[c], sizeof(out[k].name) - 1);
    out[k].launches = h->prof.launches[c];
    out[k].ms = h->prof.ms[c];
    out[k].work = h->prof.work[c];
    out[k].unit = units[c];
    out[k].big_launches = h->prof.big_n[c];
    out[k].big_ms = h->prof.big_ms[c];
    out[k].big_work = h->prof.big_work[c];
    ++k;
  }
  return k;
}

// Test hook (not part of the public contract): copy the head of an internal trunk buffer
// (0 = act1 planar, 1 = act2 planar, 2 = act3 dense, 3 = leaf R_d) to dst (device).
int64_t bcts_debug_net_buffer(bcts_handle h, int32_t which, void *dst, int64_t bytes) {
  if (!h || !dst || bytes <= 0) return -1;
  const void *src = which == 0 ? (const void *)h->net.act1p : which == 1 ? (const void *)h->net.act2p
                    : which == 2 ? (const void *)h->net.act3 : (const void *)h->net.leaf_cum;
  if (!src) return -1;
  cudaSetDevice(h->dev);
  cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, h->st);
  cudaStreamSynchronize(h->st);
  return cudaGetLastError() == cudaSuccess ? bytes : -1;
}

int64_t bcts_pack_key(float value, int64_t leaf_index) { return pack_key(value, leaf_index); }
float bcts_key_value(int64_t key) { return key_value(key); }
int64_t bcts_key_leaf(int64_t key) { return key_leaf(key); }

bcts_status bcts_shard_range(int64_t n_roots, int32_t depth, int32_t A, int32_t rank, int32_t world,
                             int64_t *leaf_begin, int64_t *leaf_end) {
  if (n_roots < 0 || depth < 0 || depth > kMaxDepth || A < 2 || world < 1 || rank < 0 || rank >= world ||
      !leaf_begin || !leaf_end)
    return BCTS_ERR_INVALID_ARG;
  int64_t lpr;
  if (!ipow_ok(A, depth, lpr)) return BCTS_ERR_BUDGET;
  if (n_roots > 0 && lpr > (INT64_MAX / 8) / n_roots) return BCTS_ERR_BUDGET;
  if (n_roots % world == 0) {  // whole roots per rank (C4)
    const int64_t per = n_roots / world;
    *leaf_begin = rank * per * lpr;
    *leaf_end = (rank + 1) * per * lpr;
  } else {                     // balanced contiguous leaf ranges (C5)
    const __int128 total = (__int128)n_roots * lpr;
    *leaf_begin = (int64_t)(total * rank / world);
    *leaf_end = (int64_t)(total * (rank + 1) / world);
  }
  return BCTS_OK;
}

}  // extern "C"
