/*
 * include/bcts.h -- C ABI of the B200-native Batch-BFS + BCTS hot path.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *   For each root state s_0, the exhaustive depth-d, A-ary tree is expanded
 *   one level at a time (Batch-BFS, Alg. 1): every node of a level
 *   is replicated A ways, stepped through the deterministic forward model G
 *   and the discounted reward R += gamma^k r is accumulated. The
 *   A^d leaves are scored with R + gamma^d max_a Q_theta(s_d, a), and
 *   a segmented max over each root action's A^(d-1) leaves gives the vanilla
 *   d-step Q of Eq. 1 and the greedy action of Eq. 2,
 *   i.e. Alg. 1's floor(argmax R / A^(d-1)). With correction_on, the
 *   BCTS penalty beta * gamma^d * B(delta_e, delta_o, A, d) of Eq. 5
 *    is subtracted from every root action != pi_o (Eq. 3,
 *   P:205-213; sweep constant beta), where delta_a is the root Bellman
 *   error from depths 0 and 1 (Prop. 1), delta_o = |delta_pi_o|
 *   and delta_e the mean |delta_a| over a != pi_o.
 *
 * Conventions (DESIGN.md §2 readings):
 *   - Node i of level k has children i*A + a (a = 0..A-1); leaf index within a
 *     root = sum_t a_t A^(d-1-t) (R1). Ties: lowest index everywhere (R4).
 *   - gamma^k is formed on the host as (float)(product of k copies of
 *     (double)gamma); R_{k+1} = fmaf(g[k], r, R_k); leaf = fmaf(g[d], m, R_d) (R3).
 *   - depth == 0: greedy on Q_hat(s_0, .), no correction (R11).
 *   - beta == 0 or correction_on == 0: corrected Q == vanilla Q bit for bit (R12).
 *
 * Memory and streams:
 *   - Unless stated otherwise every data pointer is a DEVICE pointer (e.g.
 *     torch.Tensor.data_ptr() on the handle's device). The caller owns roots
 *     and all outputs; the library never frees them.
 *   - Calls enqueue on the handle's stream and return; outputs are valid after
 *     a stream synchronize. bcts_search_host is the exception (synchronous).
 *   - Argument errors are detected before anything is enqueued; on ANY error
 *     the outputs are left untouched.
 *   - A handle is used by one host thread at a time; handles are independent.
 *   - No C++ exception ever crosses this boundary.
 */
#ifndef BCTS_H_
#define BCTS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BCTS_ABI_VERSION 6   /* 2: env_weights fields + BCTS_ENV_DNN; 3: bcts_search_pruned; 4: bcts_kernel_profile largest-launch fields;
                                5: NCCL (nccl_unique_id / rank / world, BCTS_ERR_NCCL), caller workspace, ms_* stats, flags 0x10-0x20;
                                6: BCTS_F_TF32 (NEXT-1 on the tensor cores) */

typedef struct bcts_handle_t *bcts_handle;

typedef enum {
  BCTS_OK = 0,
  BCTS_ERR_INVALID_ARG = 1,   /* bad argument; nothing enqueued */
  BCTS_ERR_UNSUPPORTED = 2,   /* valid request this build does not implement */
  BCTS_ERR_OUT_OF_MEMORY = 3, /* device allocation failed */
  BCTS_ERR_BUDGET = 4,        /* one root's per-call tree cannot fit the workspace, or A^d overflows */
  BCTS_ERR_CUDA = 5,          /* a CUDA runtime error (detail in bcts_last_error) */
  BCTS_ERR_NCCL = 6,          /* an NCCL error, or the communicator is in an error state (detail in bcts_last_error) */
  BCTS_ERR_NUMERIC = 7        /* non-finite value met where the contract forbids it */
} bcts_status;

/* Forward models G (DESIGN.md §3 ENV_SPEC). Root-record layouts:
 *   TABULAR    : int32 state id                                   (4 B)
 *   INT_HASH   : uint32 s[16]                                     (64 B)
 *   ATARI_HASH : uint64 key, uint64 pad, uint32 w[84*84]          (28,240 B)
 *                w[p] packs the 4-frame stack of pixel p, byte c = frame c
 *                (c = 0 oldest, 3 newest; frame stacking P:355).
 *   DNN        : float32 s[100]                                    (400 B)
 *                random-DNN learned forward model of the runtime study
 *                (P:340-341): [s; onehot(a)] -> 3 x (Linear 100, ReLU) ->
 *                Linear 101 = (s', r); fp32, each output one fixed-order
 *                fmaf chain from the bias over the inputs in index order
 *                (R27). Weights: bcts_config.env_weights. */
typedef enum {
  BCTS_ENV_TABULAR = 1,
  BCTS_ENV_INT_HASH = 2,
  BCTS_ENV_ATARI_HASH = 3,
  BCTS_ENV_DNN = 4
} bcts_env_kind;

/* Value nets Q_theta (DESIGN.md §3 NET_SPEC; random-init weights, shapes of P:83). */
typedef enum {
  BCTS_NET_TABLE = 1,        /* tabular Q_hat [nS*A] (TABULAR env only)          */
  BCTS_NET_MLP2_F32 = 2,     /* in -> hidden -> A, fp32 fixed-order FMA: INT_HASH
                              * (in = 64 state bytes / 256) or DNN (in = 100 floats) */
  BCTS_NET_NATURE_BF16 = 3,  /* Nature-DQN conv trunk + fc 512 + fc A, bf16      */
  BCTS_NET_RAINBOW_BF16 = 4  /* same trunk + dueling C51 head (51 atoms), bf16   */
} bcts_net_kind;

/* Config flags. */
#define BCTS_F_CLAMP_PENALTY 0x1u /* clamp B at 0 (opt-in; default signed, R8) */
#define BCTS_F_SIMT_NET 0x2u      /* use the SIMT reference net (no tensor cores) */
#define BCTS_F_MATERIALIZE_LEAVES 0x4u /* store the leaf level (else leaf frames are
                                        * generated inside the net's A-operand producer) */
#define BCTS_F_SEPARATE_BACKUP 0x8u /* run the segmented-max backup (Alg. 1) as its own kernel
                                     * instead of inside the Rainbow head's epilogue; same result bit
                                     * for bit (the max over packed keys is order-independent) */
#define BCTS_F_NO_PROLOGUE_FOLD 0x10u /* evaluate the depth-0/1 rows of the BCTS terms (Prop. 1) in their
                                       * own net launches instead of inside the last leaf batch; same
                                       * result bit for bit */
#define BCTS_F_NO_GRAPH 0x20u        /* never replay CUDA graphs (bcts_search_host, bcts_search_ex) */
#define BCTS_F_TF32 0x40u /* NEXT-1 on the tensor cores: the DNN forward model (BCTS_ENV_DNN) and the MLP2
                           * net run as tcgen05 kind::tf32 GEMMs (operands rounded to tf32, fp32
                           * accumulation in the MMA's order). NOT bit-exact with the fp32 default:
                           * within the tf32 tolerance of the fp64 oracle (R34). A DNN
                           * search expands each chunk's levels in one cooperative launch (one CTA
                           * per SM, all resident): if that launch cannot be made (e.g. another
                           * context holds SMs) the call fails with CUDA. Other envs / nets ignore it. */

typedef struct {
  uint32_t abi_version;     /* must be BCTS_ABI_VERSION */
  int32_t device;           /* CUDA device ordinal */
  void *cuda_stream;        /* cudaStream_t to enqueue on; NULL = the legacy default stream */
  int32_t env;              /* bcts_env_kind */
  int32_t num_actions;      /* A >= 2 (fixed per handle) */
  /* TABULAR only (HOST pointers, copied at create): */
  int32_t num_states;
  const int32_t *tab_next;  /* [nS*A] next state of (s,a) */
  const float *tab_reward;  /* [nS*A] r(s,a) */
  const float *tab_q;       /* [nS*A] Q_hat(s,a) for BCTS_NET_TABLE */
  /* Nets (HOST pointer, copied/repacked at create; caller may free after): */
  int32_t net;              /* bcts_net_kind */
  const float *weights;     /* canonical PyTorch-order fp32 blob (synth.inputs.weight_specs) */
  int64_t weights_count;    /* number of floats in weights */
  int32_t mlp_in, mlp_hidden; /* MLP2: 64 (INT_HASH) or 100 (DNN), hidden (<= 1024) */
  int32_t atoms;            /* Rainbow atoms (51) */
  float v_min, v_max;       /* Rainbow support [-10, 10] */
  int64_t workspace_bytes_max; /* per-call device workspace budget; 0 = auto (16 GiB) */
  uint32_t flags;           /* BCTS_F_* */
  /* DNN env only (HOST pointer, repacked at create; caller may free after):
   * canonical fp32 blob g1.w [100][100+A], g1.b [100], g2.w [100][100], g2.b,
   * g3.w [100][100], g3.b, g4.w [101][100], g4.b [101] (synth.inputs.env_weight_specs).
   * INVALID_ARG if null or env_weights_count != 40,501 + 100*A (the sum of
   * those sizes); ignored for the other envs. */
  const float *env_weights;
  int64_t env_weights_count;
  /* Multi-GPU (one process per GPU). world > 1: bcts_create is COLLECTIVE --
   * every rank 0..world-1 calls it with the same 128-byte id from bcts_nccl_unique_id (made on one
   * rank, shared by the caller, e.g. torch.distributed.broadcast) and its own rank; the handle owns
   * an NCCL communicator on `device` and its searches are collective. world == 1 with a non-NULL id:
   * a one-rank communicator (the collective path on one GPU, e.g. for tests). world <= 1 with a
   * NULL id: no NCCL at all. INVALID_ARG if rank is outside [0, max(world, 1)) or world > 1 with a
   * NULL id; NCCL if the communicator cannot be created. */
  const void *nccl_unique_id;  /* HOST, 128 bytes (copied at create) */
  int32_t rank, world;
} bcts_config;

typedef struct {
  int64_t transitions;     /* env steps executed (n * sum_{k=1..d} A^k on one GPU) */
  int64_t leaves;          /* leaves scored */
  int64_t evaluated;       /* net evaluations (leaves + root rows + level-1 rows) */
  int64_t kernel_launches; /* kernels this call launched */
  int64_t chunks;          /* leaf chunks the call was split into */
  int64_t level_launches;  /* expansion-kernel launches */
  /* Device time of the call by phase, in ms (CUDA events on the handle's stream). Filled only while
   * profiling is on (bcts_profile_enable(h, 1)): the call then synchronizes its stream before it
   * returns. 0 otherwise (calls stay asynchronous). expand = level expansion (Alg. 1),
   * leaf = the value net (incl. the depth-0/1 rows), backup = segmented max + BCTS
   * correction (Eq. 3/5), comm = the NCCL all-reduce (world > 1), total = the whole call. */
  float ms_total, ms_expand, ms_leaf, ms_backup, ms_comm;
} bcts_stats;

/* Create a handle: validates cfg, copies tables, repacks weights into the
 * device layouts. Device scratch is NOT allocated here: the first call that
 * needs it allocates it (library-owned), unless bcts_set_workspace gave the
 * handle caller-owned memory first. Errors: INVALID_ARG (bad kinds, A<2,
 * A>64, wrong weights_count, null required pointers, rank/world), CUDA,
 * OUT_OF_MEMORY, NCCL (world > 1). */
bcts_status bcts_create(const bcts_config *cfg, bcts_handle *out);

/* 128-byte NCCL unique id for the multi-GPU handles of one job (host memory, caller-owned);
 * call on ONE rank and give the same bytes to every rank's bcts_create. Needs no GPU.
 * Errors: INVALID_ARG (NULL), NCCL (libnccl.so.2 not loadable, or ncclGetUniqueId failed). */
bcts_status bcts_nccl_unique_id(void *out128);

/* Device memory a bcts_search / bcts_search_ex / bcts_search_host call over n_roots roots at
 * `depth` needs on this handle: the value net's scratch (conv nets: fixed, ~4-5 GB for the
 * 6-wave leaf batches) + the tree workspace (level buffers, leaf totals, packed keys, the
 * folded prologue; capped by workspace_bytes_max through chunking). *bytes is written.
 * Errors: INVALID_ARG (NULL, n_roots < 0, depth outside [0, 12]), BUDGET (one chunk does not
 * fit workspace_bytes_max). Host-only; enqueues nothing. */
bcts_status bcts_workspace_size(bcts_handle h, int64_t n_roots, int32_t depth, size_t *bytes);

/* Give the handle caller-owned device memory (e.g. a torch uint8 tensor on the handle's device):
 * [dev_ptr, dev_ptr + bytes), 256-byte aligned. From now on the handle allocates no scratch or
 * tree workspace of its own (it frees what it had); a later call that needs more than `bytes`
 * fails with BUDGET (nothing enqueued) -- size it with bcts_workspace_size. dev_ptr == NULL
 * returns to library-owned memory. The caller keeps the memory alive and untouched while the
 * handle may use it (until bcts_destroy or the next bcts_set_workspace), and must not pass it
 * to two handles whose calls can overlap. Synchronizes the handle's stream first.
 * Errors: INVALID_ARG (misaligned, or bytes smaller than the net scratch), CUDA. */
bcts_status bcts_set_workspace(bcts_handle h, void *dev_ptr, size_t bytes);

/* NULL-safe. Frees device memory owned by the handle. */
void bcts_destroy(bcts_handle h);

int32_t bcts_abi_version(void);
size_t bcts_root_record_bytes(bcts_handle h);
const char *bcts_status_string(bcts_status s);
const char *bcts_last_error(bcts_handle h); /* detail for the last failing call on h ("" if none) */

/* Batch-BFS + BCTS for n_roots independent roots (Alg. 1 per root).
 *   roots        : device, n_roots root records (layout above)
 *   depth        : d >= 0 (d = 0 -> greedy on Q_hat(s_0,.))
 *   A            : must equal cfg.num_actions
 *   gamma        : in (0,1);  beta: finite, >= 0
 *   correction_on: 0 = vanilla d-step greedy (Eq. 2); 1 = BCTS with the Bellman
 *                  penalty B of Eq. 5; 2 = BCTS with Lemma 2's exact
 *                  bias gap B_e - B_o (App. A.2) at sigma = delta/sqrt(2)
 *   actions_out  : device int32 [n_roots]      argmax of the (corrected) root Q
 *   root_q_out   : device float [n_roots * A]  corrected root Q (R14)
 * Errors: INVALID_ARG, BUDGET, CUDA. n_roots == 0 is a no-op returning OK. */
bcts_status bcts_search(bcts_handle h, const void *roots, int64_t n_roots, int32_t depth, int32_t A,
                        float gamma, float beta, int32_t correction_on, int32_t *actions_out,
                        float *root_q_out);

/* As bcts_search, plus optional (nullable) device outputs:
 *   vanilla_q_out  float [n*A]  uncorrected d-step Q (Eq. 1)
 *   terms_out      float [n*4]  (pi_o, delta_o, delta_e, B) (zeros when not computed)
 *   best_leaf_out  int64 [n*A]  lowest leaf index (within the root) attaining vanilla_q
 *   stats          HOST bcts_stats*
 * Multi-GPU handles (world > 1): the call is COLLECTIVE -- every rank passes identical arguments
 * and the full roots; rank r scores the leaf range bcts_shard_range(n, d, A, r, world), one
 * ncclAllReduce(ncclInt64, ncclMax) of the n*A packed keys runs on the handle's stream, and every
 * rank applies the identical correction: all ranks return the same outputs, bit for bit equal to
 * the single-GPU search.
 * CUDA graphs: unless BCTS_F_NO_GRAPH or profiling is on, a call whose arguments (pointers
 * included) equal the previous call's replays a graph of that call's launches captured after it
 * ran eagerly (one launch instead of ~10-20); the buffers' CURRENT contents are used. */
bcts_status bcts_search_ex(bcts_handle h, const void *roots, int64_t n_roots, int32_t depth, int32_t A,
                           float gamma, float beta, int32_t correction_on, int32_t *actions_out,
                           float *root_q_out, float *vanilla_q_out, float *terms_out,
                           int64_t *best_leaf_out, bcts_stats *stats);

/* End-to-end convenience: HOST roots in, HOST outputs out. Copies the roots
 * host->device, runs bcts_search_ex and copies actions/root_q device->host,
 * then synchronizes the stream. Same errors as bcts_search. When all three
 * host buffers are page-locked (cudaHostAlloc / torch pin_memory) the call
 * after an eager one with the same pointers and arguments replays a CUDA graph
 * of the whole sequence (captured on a private stream, launched on the
 * handle's); the buffers' CURRENT contents are copied in on every call.
 * BCTS_F_NO_GRAPH disables the graph. Collective when world > 1. */
bcts_status bcts_search_host(bcts_handle h, const void *roots_host, int64_t n_roots, int32_t depth,
                             int32_t A, float gamma, float beta, int32_t correction_on,
                             int32_t *actions_host, float *root_q_host);

/* ---- sharded search (multi-GPU) --------------------------
 * The global leaf space of a call is [0, n_roots * A^d); leaf L belongs to
 * root L / A^d. bcts_search_shard expands only the ancestors of the leaves in
 * [leaf_begin, leaf_end), scores those leaves and folds each leaf's total into
 * keys_out[root*A + a0] by max (a0 = root action of the leaf). keys_out is a
 * device int64 [n_roots * A] that the caller initialises with
 * bcts_keys_init; a key orders as (value, lowest leaf index) under SIGNED
 * int64 max, so shards combine with any max all-reduce (ncclMax over
 * ncclInt64, torch.distributed ReduceOp.MAX). bcts_finalize turns the
 * reduced keys into the outputs of bcts_search_ex, evaluating the depth-0/1
 * Bellman terms itself (the same on every rank). With a Rainbow conv net and
 * n_roots * (A + 1) <= 4096, bcts_search_shard also evaluates those depth-0/1
 * rows inside its last leaf batch and keeps them in handle-owned memory for the
 * next bcts_finalize with the same roots pointer, n_roots, depth and gamma (the
 * roots' contents must not change in between); any other finalize evaluates
 * them itself. Results are identical either way. */
bcts_status bcts_keys_init(bcts_handle h, int64_t *keys, int64_t count);
bcts_status bcts_search_shard(bcts_handle h, const void *roots, int64_t n_roots, int32_t depth, int32_t A,
                              float gamma, int64_t leaf_begin, int64_t leaf_end, int64_t *keys_out,
                              bcts_stats *stats);
bcts_status bcts_finalize(bcts_handle h, const void *roots, int64_t n_roots, int32_t depth, int32_t A,
                          float gamma, float beta, int32_t correction_on, const int64_t *keys,
                          int32_t *actions_out, float *root_q_out, float *vanilla_q_out,
                          float *terms_out, int64_t *best_leaf_out, bcts_stats *stats);

/* bcts_pv_targets: the propagated-value (PV) training target of App. B.3
 * ("use the cumulative reward and value computed during the TS")
 * and the principal variation behind it, for the actions a TS policy took.
 * For root r with executed action a_r = actions[r] (device int32 [n], each in
 * [0, A)): target_out[r] = vanilla_q[r*A + a_r] (Eq. 1's depth-d value of a_r,
 * uncorrected: the best R_d + gamma^d max_a Q over a_r's subtree; DESIGN.md
 * R29) and path_out[r*depth + t] = the t-th action of the lowest best leaf
 * best_leaf[r*A + a_r] (base-A digit t, most significant first; path[0] ==
 * a_r). vanilla_q / best_leaf are bcts_search_ex's outputs for the same
 * roots and depth (device). All pointers device; outputs caller-owned.
 * Errors: INVALID_ARG (null pointers, n < 0, depth < 1 or > 12). An action
 * outside [0, A) yields target NaN and path -1 for that root. Enqueued. */
bcts_status bcts_pv_targets(bcts_handle h, int64_t n_roots, int32_t depth, const int32_t *actions,
                            const float *vanilla_q, const int64_t *best_leaf, float *target_out,
                            int32_t *path_out);

/* ---- early pruning (NEXT-4; "future work"; R30-R33) ----
 * "Efficient pruning can be done by maintaining an index array of
 * unpruned states which are updated with each pruning step. These indices are
 * then used for tracing the optimal action at the root." bcts_search_pruned
 * runs Alg. 1 level by level; after expanding level k, for k in
 * [first_level, depth-1], a rule thins the level inside each group
 * (root, root action) and the survivors are compacted (stream compaction of
 * their states + the index array: each node's index f in the UNPRUNED tree,
 * whose base-A digits are its action path). Leaves are never pruned.
 *   BCTS_PRUNE_BOUND (exact, R31): with every one-step reward in [r_lo, r_hi]
 *     and every leaf value max_a Q_hat in [q_lo, q_hi], node i at level k is
 *     dropped iff R_i + U_k + s_i < max over its group of (R_j + L_k - s_j),
 *     L_k = sum_{j=k}^{d-1} gamma^j r_lo + gamma^d q_lo (U_k: the _hi ends),
 *     s = 2^-16 (|R| + S_k) a rounding margin. Outputs are then bit-identical
 *     to bcts_search_ex when the bounds hold (C51 nets: q in [v_min, v_max]).
 *   BCTS_PRUNE_BEAM (approximate, R32): keep the `beam` nodes of each group
 *     with the highest depth-k estimate fmaf(gamma^k, max_a Q_hat(s, a), R),
 *     ties to the lower f; costs one Q_hat evaluation per node of each
 *     pruned level.
 * Outputs as bcts_search_ex (best_leaf keeps its unpruned meaning).
 * survivors_out: HOST int64 [depth+1] (nullable): nodes kept per level over
 * all roots (survivors[0] = n_roots, survivors[depth] = leaves scored).
 * Synchronizes the stream once per pruned level (the survivor count sizes the
 * next level). Roots are processed in chunks sized for the worst case
 * (BOUND: no pruning) within workspace_bytes_max.
 * Errors: INVALID_ARG (null prune, unknown rule, beam < 1 for BEAM, r_lo >
 * r_hi or q_lo > q_hi or non-finite bounds for BOUND, depth < 1, plus those of
 * bcts_search_ex), BUDGET, CUDA. */
#define BCTS_PRUNE_NONE 0
#define BCTS_PRUNE_BOUND 1
#define BCTS_PRUNE_BEAM 2
typedef struct {
  int32_t rule;         /* BCTS_PRUNE_* */
  int32_t first_level;  /* first level pruned (values < 1 read as 1) */
  int64_t beam;         /* BEAM: nodes kept per (root, root action) group and level */
  float r_lo, r_hi;     /* BOUND: one-step reward bounds */
  float q_lo, q_hi;     /* BOUND: leaf-value (max_a Q_hat) bounds */
} bcts_prune;
bcts_status bcts_search_pruned(bcts_handle h, const void *roots, int64_t n_roots, int32_t depth, int32_t A,
                               float gamma, float beta, int32_t correction_on, const bcts_prune *prune,
                               int32_t *actions_out, float *root_q_out, float *vanilla_q_out,
                               float *terms_out, int64_t *best_leaf_out, int64_t *survivors_out,
                               bcts_stats *stats);

/* ---- inspection entry points (same kernels as the search) -------------
 * bcts_expand: expand n_roots roots to level `level` (Alg. 1 loop body,
 * P:318-321) and write the n_roots*A^level level-`level` states as root
 * records into states_out (device, record layout) and their cumulative
 * discounted rewards into cum_out (device float). */
bcts_status bcts_expand(bcts_handle h, const void *roots, int64_t n_roots, int32_t level, int32_t A,
                        float gamma, void *states_out, float *cum_out);

/* bcts_q_rows: full-row value-net evaluation Q_hat(s, .) for n states given
 * as root records (device) -> q_out device float [n*A]. */
bcts_status bcts_q_rows(bcts_handle h, const void *states, int64_t n, float *q_out);

/* ---- profiling (per kernel class, CUDA events on the handle's stream) ----
 * bcts_profile_enable(h, 1) synchronizes, clears the totals and starts
 * recording an event pair around every kernel launch; 0 stops. Each launch
 * also carries its ALGORITHMIC work (unit 0: bytes moved, unit 1: FLOPs;
 * DESIGN.md §5). bcts_profile_read synchronizes the stream and writes up to
 * max per-class totals; returns the number written. */
typedef struct {
  char name[32];
  int64_t launches;
  double ms;    /* summed event durations */
  double work;  /* summed algorithmic bytes (unit 0) or FLOPs (unit 1) */
  int32_t unit;
  /* the class's LARGEST launches (maximal work per launch, e.g. the deepest expanded level):
   * how many there were, their summed durations and the work of one */
  int64_t big_launches;
  double big_ms;
  double big_work;
} bcts_kernel_profile;
bcts_status bcts_profile_enable(bcts_handle h, int32_t on);
int32_t bcts_profile_read(bcts_handle h, bcts_kernel_profile *out, int32_t max);

/* Packed-key helpers, exposed for tests of the multi-GPU reduction:
 * bcts_pack_key(value, leaf) is the int64 key described above. Host-only. */
int64_t bcts_pack_key(float value, int64_t leaf_index);
float bcts_key_value(int64_t key);
int64_t bcts_key_leaf(int64_t key);

/* Shard plan (host-only): the [begin, end) leaf range rank `rank` of `world`
 * owns for a call over n_roots roots at depth d with A actions. Contiguous,
 * balanced to within one leaf, aligned to whole roots when n_roots is a
 * multiple of world (root sharding, C4) and to leaf ranges otherwise (C5). */
bcts_status bcts_shard_range(int64_t n_roots, int32_t depth, int32_t A, int32_t rank, int32_t world,
                             int64_t *leaf_begin, int64_t *leaf_end);

#ifdef __cplusplus
}
#endif
#endif /* BCTS_H_ */
