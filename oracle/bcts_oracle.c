/*
 * oracle/bcts_oracle.c -- TEST INFRASTRUCTURE ONLY (never on the product path).
 *
 * Plain, slow, obviously-correct CPU implementation of what the hot path
 * computes: Batch-BFS exhaustive tree search (Alg. 1),
 * i.e. the d-step Q of Eq. 1 evaluated by recursive DFS,
 * plus the BCTS correction (Eq. 3, Eq. 5, Prop. 1
 * P:264-273) and a second, structurally different brute-force enumerator
 * of all A^d action sequences (Eq. 1 written out literally).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this library. It shares no code, header,
 * table or constant generator with paper_2107_01715_b200/csrc (the CUDA path).
 *
 * Precision modes (readings R3/R17):
 *   mode 0 = fp64 reference: rewards, values and penalty in double.
 *   mode 1 = fp32 mirror   : R_{k+1} = fmaf(g[k], r, R_k), leaf = fmaf(g[d], m, R_d),
 *                            MLP as a fixed-order fmaf chain; built with
 *                            -ffp-contract=off so nothing else is fused.
 * bf16 nets (Nature / Rainbow) always emulate bf16 operands (weights and
 * hidden activations rounded RNE) with fp64 accumulation.
 *
 * Parity pins: see tests/test_oracle_pins.py (W1, W2, C1-chain, SPEC
 * examples, closed forms, brute force == DFS, torch conv2d cross-check).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <fenv.h>
#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#ifndef M_E
#define M_E 2.7182818284590452354
#endif
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_ENV_TABULAR 1
#define OR_ENV_INT_HASH 2
#define OR_ENV_ATARI_HASH 3
#define OR_ENV_DNN 4          /* random-DNN learned forward model, state = 100 floats */
#define DNN_S 100
#define OR_NET_TABLE 1
#define OR_NET_MLP2 2
#define OR_NET_NATURE 3
#define OR_NET_RAINBOW 4

#define IMG 84
#define NPIX (IMG * IMG)
#define MAXA 64
#define MAXD 12

/* ------------------------------------------------------------------ model */
typedef struct {
  int env, A, nS;
  int32_t *tab_next;      /* [nS*A] */
  double *tab_reward;     /* [nS*A] */
  int net;
  double *tab_q;          /* [nS*A] */
  /* MLP (fp32 canonical, kept as float for the mirror mode) */
  int mlp_in, mlp_hidden;
  float *l1w, *l1b, *l2w, *l2b;
  /* conv nets: weights rounded to bf16 and stored as double; biases fp32->double */
  double *c1w, *c1b, *c2w, *c2b, *c3w, *c3b;
  double *f1w, *f1b, *f2w, *f2b;          /* Nature fc1 / fc2 */
  double *hvw, *hvb, *haw, *hab;          /* Rainbow fc_h_v / fc_h_a */
  double *zvw, *zvb, *zaw, *zab;          /* Rainbow fc_z_v / fc_z_a */
  int atoms;
  double vmin, vmax;
  /* random-DNN forward model: g1 [100][100+A], g2 [100][100], g3 [100][100], g4 [101][100] (+ biases) */
  float *gw[4], *gb[4];
} oracle_model;

/* Internal state: the oracle keeps Atari frames as 4 separate planes
 * (channel, pixel) -- not the packed words of the device layout. */
typedef struct {
  int32_t id;                 /* TABULAR */
  uint32_t s[16];             /* INT_HASH */
  uint64_t key;               /* ATARI_HASH */
  uint8_t plane[4][NPIX];     /* ATARI_HASH: plane 0 oldest, 3 newest */
  float x[DNN_S];             /* DNN */
} ostate;

static uint64_t o_mix64(uint64_t z) {   /* splitmix64 finalizer (ENV_SPEC) */
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27; z *= 0x94D049BB133111EBULL;
  z ^= z >> 31; return z;
}
static uint32_t o_fmix32(uint32_t h) {  /* murmur3 finalizer (ENV_SPEC) */
  h ^= h >> 16; h *= 0x85EBCA6BU; h ^= h >> 13; h *= 0xC2B2AE35U; h ^= h >> 16; return h;
}
static uint32_t o_rotl32(uint32_t x, int r) { return (x << r) | (x >> (32 - r)); }

/* Round a double to the nearest bfloat16 value (8 significant bits), ties to
 * even, directly from the double (no intermediate fp32). Normal range only. */
static double bf16_rne(double x) {
  if (x == 0.0 || !isfinite(x)) return x;
  int e;
  double m = frexp(x, &e);           /* x = m * 2^e, 0.5 <= |m| < 1 */
  double sc = ldexp(m, 8);           /* 128 <= |sc| < 256: 8 significant bits */
  double r = nearbyint(sc);          /* current rounding mode: to nearest, ties to even */
  return ldexp(r, e - 8);
}

double oracle_bf16_round(double x) { return bf16_rne(x); }

static double *dup_bf16(const float *w, long n) {
  double *o = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  for (long i = 0; i < n; ++i) o[i] = bf16_rne((double)w[i]);
  return o;
}
static double *dup_f64(const float *w, long n) {
  double *o = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  for (long i = 0; i < n; ++i) o[i] = (double)w[i];
  return o;
}
static float *dup_f32(const float *w, long n) {
  float *o = (float *)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  memcpy(o, w, sizeof(float) * (size_t)(n > 0 ? n : 0));
  return o;
}

void oracle_destroy(oracle_model *m) {
  if (!m) return;
  for (int i = 0; i < 4; ++i) { free(m->gw[i]); free(m->gb[i]); }
  void *ptrs[] = {m->tab_next, m->tab_reward, m->tab_q, m->l1w, m->l1b, m->l2w, m->l2b,
                  m->c1w, m->c1b, m->c2w, m->c2b, m->c3w, m->c3b, m->f1w, m->f1b, m->f2w, m->f2b,
                  m->hvw, m->hvb, m->haw, m->hab, m->zvw, m->zvb, m->zaw, m->zab};
  for (size_t i = 0; i < sizeof(ptrs) / sizeof(ptrs[0]); ++i) free(ptrs[i]);
  free(m);
}

/* weights: canonical fp32 blob in synth.inputs.weight_specs order. */
oracle_model *oracle_create(int env, int A, int nS, const int32_t *tab_next, const double *tab_reward,
                            int net, const double *tab_q, const float *weights, long n_weights,
                            int mlp_in, int mlp_hidden, int atoms, double vmin, double vmax) {
  if (A < 2 || A > MAXA) return NULL;
  oracle_model *m = (oracle_model *)calloc(1, sizeof(oracle_model));
  m->env = env; m->A = A; m->nS = nS; m->net = net;
  m->mlp_in = mlp_in; m->mlp_hidden = mlp_hidden; m->atoms = atoms; m->vmin = vmin; m->vmax = vmax;
  if (env == OR_ENV_TABULAR) {
    m->tab_next = (int32_t *)malloc(sizeof(int32_t) * nS * A);
    m->tab_reward = (double *)malloc(sizeof(double) * nS * A);
    memcpy(m->tab_next, tab_next, sizeof(int32_t) * nS * A);
    memcpy(m->tab_reward, tab_reward, sizeof(double) * nS * A);
  }
  const float *w = weights;
  long need = 0;
  if (net == OR_NET_TABLE) {
    m->tab_q = (double *)malloc(sizeof(double) * nS * A);
    memcpy(m->tab_q, tab_q, sizeof(double) * nS * A);
  } else if (net == OR_NET_MLP2) {
    long H = mlp_hidden, I = mlp_in;
    need = H * I + H + A * H + A;
    if (n_weights != need) { oracle_destroy(m); return NULL; }
    m->l1w = dup_f32(w, H * I); w += H * I;
    m->l1b = dup_f32(w, H); w += H;
    m->l2w = dup_f32(w, A * H); w += A * H;
    m->l2b = dup_f32(w, A); w += A;
  } else if (net == OR_NET_NATURE || net == OR_NET_RAINBOW) {
    long sz[] = {32 * 4 * 8 * 8, 32, 64 * 32 * 4 * 4, 64, 64 * 64 * 3 * 3, 64};
    need = sz[0] + sz[1] + sz[2] + sz[3] + sz[4] + sz[5];
    if (net == OR_NET_NATURE) need += 512L * 3136 + 512 + (long)A * 512 + A;
    else need += 2 * (512L * 3136 + 512) + (long)atoms * 512 + atoms + (long)A * atoms * 512 + (long)A * atoms;
    if (n_weights != need) { oracle_destroy(m); return NULL; }
    m->c1w = dup_bf16(w, sz[0]); w += sz[0];
    m->c1b = dup_f64(w, sz[1]); w += sz[1];
    m->c2w = dup_bf16(w, sz[2]); w += sz[2];
    m->c2b = dup_f64(w, sz[3]); w += sz[3];
    m->c3w = dup_bf16(w, sz[4]); w += sz[4];
    m->c3b = dup_f64(w, sz[5]); w += sz[5];
    if (net == OR_NET_NATURE) {
      m->f1w = dup_bf16(w, 512L * 3136); w += 512L * 3136;
      m->f1b = dup_f64(w, 512); w += 512;
      m->f2w = dup_bf16(w, (long)A * 512); w += (long)A * 512;
      m->f2b = dup_f64(w, A); w += A;
    } else {
      m->hvw = dup_bf16(w, 512L * 3136); w += 512L * 3136;
      m->hvb = dup_f64(w, 512); w += 512;
      m->haw = dup_bf16(w, 512L * 3136); w += 512L * 3136;
      m->hab = dup_f64(w, 512); w += 512;
      m->zvw = dup_bf16(w, (long)atoms * 512); w += (long)atoms * 512;
      m->zvb = dup_f64(w, atoms); w += atoms;
      m->zaw = dup_bf16(w, (long)A * atoms * 512); w += (long)A * atoms * 512;
      m->zab = dup_f64(w, (long)A * atoms); w += (long)A * atoms;
    }
  } else {
    oracle_destroy(m);
    return NULL;
  }
  return m;
}

/* random-DNN forward-model weights (canonical fp32 blob: g1.w, g1.b, g2.w, g2.b, g3.w, g3.b, g4.w, g4.b) */
int oracle_set_env_weights(oracle_model *m, const float *w, long count) {
  const int A = m->A;
  const long sz[8] = {100L * (100 + A), 100, 100L * 100, 100, 100L * 100, 100, 101L * 100, 101};
  long need = 0;
  for (int i = 0; i < 8; ++i) need += sz[i];
  if (m->env != OR_ENV_DNN || count != need) return -1;
  for (int i = 0; i < 4; ++i) {
    m->gw[i] = dup_f32(w, sz[2 * i]);
    w += sz[2 * i];
    m->gb[i] = dup_f32(w, sz[2 * i + 1]);
    w += sz[2 * i + 1];
  }
  return 0;
}

/* ------------------------------------------------------- record <-> state */
long oracle_record_bytes(const oracle_model *m) {
  if (m->env == OR_ENV_TABULAR) return 4;
  if (m->env == OR_ENV_INT_HASH) return 64;
  if (m->env == OR_ENV_DNN) return 4 * DNN_S;
  return 16 + 4L * NPIX;
}

static void from_record(const oracle_model *m, const uint8_t *rec, ostate *s) {
  if (m->env == OR_ENV_TABULAR) {
    memcpy(&s->id, rec, 4);
  } else if (m->env == OR_ENV_INT_HASH) {
    memcpy(s->s, rec, 64);
  } else if (m->env == OR_ENV_DNN) {
    memcpy(s->x, rec, 4 * DNN_S);
  } else {
    memcpy(&s->key, rec, 8);
    const uint8_t *px = rec + 16;
    for (int p = 0; p < NPIX; ++p)
      for (int c = 0; c < 4; ++c) {
        uint32_t word;
        memcpy(&word, px + 4 * p, 4);
        s->plane[c][p] = (uint8_t)((word >> (8 * c)) & 0xFFu);
      }
  }
}

static void to_record(const oracle_model *m, const ostate *s, uint8_t *rec) {
  if (m->env == OR_ENV_TABULAR) {
    memcpy(rec, &s->id, 4);
  } else if (m->env == OR_ENV_INT_HASH) {
    memcpy(rec, s->s, 64);
  } else if (m->env == OR_ENV_DNN) {
    memcpy(rec, s->x, 4 * DNN_S);
  } else {
    uint64_t pad = 0;
    memcpy(rec, &s->key, 8);
    memcpy(rec + 8, &pad, 8);
    for (int p = 0; p < NPIX; ++p) {
      uint32_t word = 0;
      for (int c = 0; c < 4; ++c) word |= (uint32_t)s->plane[c][p] << (8 * c);
      memcpy(rec + 16 + 4 * p, &word, 4);
    }
  }
}

/* ------------------------------------------------------------- env step G */
/* Deterministic forward model (P:44 deterministic transitions; ENV_SPEC in
 * DESIGN.md §3). Returns 0 on success, -1 on a domain error. */
static int env_step(const oracle_model *m, const ostate *s, int a, ostate *out, double *r, int mode) {
  if (a < 0 || a >= m->A) return -1;
  if (m->env == OR_ENV_TABULAR) {
    if (s->id < 0 || s->id >= m->nS) return -1;
    out->id = m->tab_next[s->id * m->A + a];
    *r = m->tab_reward[s->id * m->A + a];
    return 0;
  }
  if (m->env == OR_ENV_INT_HASH) {
    for (int w = 0; w < 16; ++w) {
      uint32_t v = s->s[w] ^ o_rotl32(s->s[(w + 1) & 15], 13) ^ (0x9E3779B9U * (uint32_t)(a + 1)) ^
                   (0x85EBCA6BU * (uint32_t)w);
      out->s[w] = o_fmix32(v);
    }
    uint32_t t = out->s[0] >> 30;
    *r = (t == 3) ? 1.0 : (t == 0) ? -1.0 : 0.0;
    return 0;
  }
  if (m->env == OR_ENV_DNN) {
    /* random-DNN learned model: x = [s; onehot(a)] -> 3 ReLU layers of
     * width 100 -> linear 101 = (next state, reward) (R27). fp32 mirror: fixed-order
     * fmaf chains from the bias over the inputs in index order; fp64 mode: doubles. */
    const int A = m->A, I1 = DNN_S + A;
    if (mode) {
      float in[DNN_S + MAXA], h[2][DNN_S];
      for (int j = 0; j < I1; ++j) in[j] = j < DNN_S ? s->x[j] : (j - DNN_S == a ? 1.0f : 0.0f);
      const float *src = in;
      int nin = I1;
      for (int L = 0; L < 3; ++L) {
        float *dst = h[L & 1];
        for (int u = 0; u < DNN_S; ++u) {
          float acc = m->gb[L][u];
          for (int i = 0; i < nin; ++i) acc = fmaf(m->gw[L][(long)u * nin + i], src[i], acc);
          dst[u] = acc > 0.0f ? acc : 0.0f;
        }
        src = dst;
        nin = DNN_S;
      }
      for (int u = 0; u <= DNN_S; ++u) {
        float acc = m->gb[3][u];
        for (int i = 0; i < DNN_S; ++i) acc = fmaf(m->gw[3][(long)u * DNN_S + i], src[i], acc);
        if (u < DNN_S) out->x[u] = acc;
        else *r = (double)acc;
      }
    } else {
      double in[DNN_S + MAXA], h[2][DNN_S];
      for (int j = 0; j < I1; ++j) in[j] = j < DNN_S ? (double)s->x[j] : (j - DNN_S == a ? 1.0 : 0.0);
      const double *src = in;
      int nin = I1;
      for (int L = 0; L < 3; ++L) {
        double *dst = h[L & 1];
        for (int u = 0; u < DNN_S; ++u) {
          double acc = (double)m->gb[L][u];
          for (int i = 0; i < nin; ++i) acc += (double)m->gw[L][(long)u * nin + i] * src[i];
          dst[u] = acc > 0.0 ? acc : 0.0;
        }
        src = dst;
        nin = DNN_S;
      }
      for (int u = 0; u <= DNN_S; ++u) {
        double acc = (double)m->gb[3][u];
        for (int i = 0; i < DNN_S; ++i) acc += (double)m->gw[3][(long)u * DNN_S + i] * src[i];
        if (u < DNN_S) out->x[u] = (float)acc;   /* states are stored as fp32 in both modes */
        else *r = acc;
      }
    }
    return 0;
  }
  /* ATARI_HASH: shift the frame stack by one frame; the new newest frame is
   * the old newest XOR a key-derived noise byte per pixel. */
  uint64_t k2 = o_mix64(s->key ^ (0x9E3779B97F4A7C15ULL * (uint64_t)(a + 1)));
  out->key = k2;
  memcpy(out->plane[0], s->plane[1], NPIX);
  memcpy(out->plane[1], s->plane[2], NPIX);
  memcpy(out->plane[2], s->plane[3], NPIX);
  for (int p = 0; p < NPIX; ++p) {
    uint8_t noise = (uint8_t)((o_mix64(k2 + (uint64_t)(p / 8)) >> (8 * (p % 8))) & 0xFFu);
    out->plane[3][p] = s->plane[3][p] ^ noise;
  }
  uint64_t t = k2 >> 61;
  *r = (t == 7) ? 1.0 : (t == 0) ? -1.0 : 0.0;
  return 0;
}

int oracle_step(const oracle_model *m, const void *rec_in, int a, void *rec_out, double *r) {
  ostate *s = (ostate *)malloc(sizeof(ostate)), *o = (ostate *)malloc(sizeof(ostate));
  from_record(m, (const uint8_t *)rec_in, s);
  int rc = env_step(m, s, a, o, r, 1);   /* fp32 mirror for the DNN model */
  if (rc == 0) to_record(m, o, (uint8_t *)rec_out);
  free(s); free(o);
  return rc;
}

/* -------------------------------------------------------------- value net */
/* Conv layer, plain definition: out[o][oy][ox] = b[o] + sum_{c,ky,kx}
 * W[o][c][ky][kx] * in[c][oy*st+ky][ox*st+kx]; then ReLU, then bf16 RNE. */
static void conv_relu_bf16(const double *in, int C, int H, const double *W, const double *b,
                           int O, int K, int st, double *out, int OH) {
  for (int o = 0; o < O; ++o)
    for (int oy = 0; oy < OH; ++oy)
      for (int ox = 0; ox < OH; ++ox) {
        double acc = 0.0;
        for (int c = 0; c < C; ++c)
          for (int ky = 0; ky < K; ++ky)
            for (int kx = 0; kx < K; ++kx)
              acc += W[((o * C + c) * K + ky) * K + kx] * in[(c * H + oy * st + ky) * H + ox * st + kx];
        acc += b[o];
        out[(o * OH + oy) * OH + ox] = bf16_rne(acc > 0.0 ? acc : 0.0);
      }
}

/* Linear: y[j] = b[j] + sum_i W[j][i] x[i]; optionally ReLU + bf16 RNE. */
static void linear(const double *x, int I, const double *W, const double *b, int J, double *y, int relu_bf16) {
  for (int j = 0; j < J; ++j) {
    double acc = 0.0;
    for (int i = 0; i < I; ++i) acc += W[(long)j * I + i] * x[i];
    acc += b[j];
    y[j] = relu_bf16 ? bf16_rne(acc > 0.0 ? acc : 0.0) : acc;
  }
}

/* Q-hat(s, .) row. Returns 0, or -1 on a domain error. */
static int qrow(const oracle_model *m, const ostate *s, int mode, double *q) {
  const int A = m->A;
  if (m->net == OR_NET_TABLE) {
    if (s->id < 0 || s->id >= m->nS) return -1;
    for (int a = 0; a < A; ++a) {
      double v = m->tab_q[s->id * A + a];
      q[a] = mode ? (double)(float)v : v;
    }
    return 0;
  }
  if (m->net == OR_NET_MLP2) {
    const int I = m->mlp_in, H = m->mlp_hidden;
    double x[256];
    float xf[256];
    for (int j = 0; j < I; ++j) {
      if (m->env == OR_ENV_DNN) {          /* DNN env: the 100 state floats are the features */
        xf[j] = s->x[j];
        x[j] = (double)s->x[j];
      } else {                             /* INT_HASH: byte j / 256 (exact) */
        uint32_t byte = (s->s[(j / 4) & 15] >> (8 * (j % 4))) & 0xFFu;
        x[j] = (double)byte / 256.0;
        xf[j] = (float)byte / 256.0f;
      }
    }
    if (mode) { /* fp32 mirror: fixed-order fmaf chains starting from the bias */
      float h[1024];
      for (int j = 0; j < H; ++j) {
        float acc = m->l1b[j];
        for (int i = 0; i < I; ++i) acc = fmaf(m->l1w[(long)j * I + i], xf[i], acc);
        h[j] = acc > 0.0f ? acc : 0.0f;
      }
      for (int a = 0; a < A; ++a) {
        float acc = m->l2b[a];
        for (int j = 0; j < H; ++j) acc = fmaf(m->l2w[(long)a * H + j], h[j], acc);
        q[a] = (double)acc;
      }
    } else {
      double h[1024];
      for (int j = 0; j < H; ++j) {
        double acc = (double)m->l1b[j];
        for (int i = 0; i < I; ++i) acc += (double)m->l1w[(long)j * I + i] * x[i];
        h[j] = acc > 0.0 ? acc : 0.0;
      }
      for (int a = 0; a < A; ++a) {
        double acc = (double)m->l2b[a];
        for (int j = 0; j < H; ++j) acc += (double)m->l2w[(long)a * H + j] * h[j];
        q[a] = acc;
      }
    }
    return 0;
  }
  /* Nature-DQN / Rainbow trunk (R15/R17): input bytes, unscaled
   * (1/255 is folded into conv1 weights). */
  double *in = (double *)malloc(sizeof(double) * 4 * NPIX);
  double *h1 = (double *)malloc(sizeof(double) * 32 * 20 * 20);
  double *h2 = (double *)malloc(sizeof(double) * 64 * 9 * 9);
  double *h3 = (double *)malloc(sizeof(double) * 64 * 7 * 7);
  for (int c = 0; c < 4; ++c)
    for (int p = 0; p < NPIX; ++p) in[c * NPIX + p] = (double)s->plane[c][p];
  conv_relu_bf16(in, 4, 84, m->c1w, m->c1b, 32, 8, 4, h1, 20);
  conv_relu_bf16(h1, 32, 20, m->c2w, m->c2b, 64, 4, 2, h2, 9);
  conv_relu_bf16(h2, 64, 9, m->c3w, m->c3b, 64, 3, 1, h3, 7);
  /* h3 is already in PyTorch NCHW flatten order: index c*49 + y*7 + x. */
  if (m->net == OR_NET_NATURE) {
    double h4[512];
    linear(h3, 3136, m->f1w, m->f1b, 512, h4, 1);
    linear(h4, 512, m->f2w, m->f2b, A, q, 0);
  } else {
    const int NA = m->atoms;
    double hv[512], ha[512];
    double *v = (double *)malloc(sizeof(double) * NA);
    double *adv = (double *)malloc(sizeof(double) * A * NA);
    linear(h3, 3136, m->hvw, m->hvb, 512, hv, 1);
    linear(h3, 3136, m->haw, m->hab, 512, ha, 1);
    linear(hv, 512, m->zvw, m->zvb, NA, v, 0);
    linear(ha, 512, m->zaw, m->zab, A * NA, adv, 0);
    for (int i = 0; i < NA; ++i) {
      double mean = 0.0;
      for (int a = 0; a < A; ++a) mean += adv[a * NA + i];
      mean /= A;
      for (int a = 0; a < A; ++a) adv[a * NA + i] = v[i] + adv[a * NA + i] - mean;   /* logits */
    }
    for (int a = 0; a < A; ++a) {
      double mx = adv[a * NA];
      for (int i = 1; i < NA; ++i) mx = adv[a * NA + i] > mx ? adv[a * NA + i] : mx;
      double den = 0.0, num = 0.0;
      for (int i = 0; i < NA; ++i) {
        double e = exp(adv[a * NA + i] - mx);
        double z = m->vmin + i * (m->vmax - m->vmin) / (NA - 1);
        den += e;
        num += z * e;
      }
      q[a] = num / den;   /* sum_i z_i softmax_i */
    }
    free(v); free(adv);
  }
  free(in); free(h1); free(h2); free(h3);
  if (mode) for (int a = 0; a < A; ++a) q[a] = (double)(float)q[a];
  return 0;
}

int oracle_qrow(const oracle_model *m, const void *rec, int mode, double *q_out) {
  ostate *s = (ostate *)malloc(sizeof(ostate));
  from_record(m, (const uint8_t *)rec, s);
  int rc = qrow(m, s, mode, q_out);
  free(s);
  return rc;
}

/* ---------------------------------------------------- discount + accumulate */
static void discounts(double gamma, int d, double *g) {
  g[0] = 1.0;
  for (int k = 1; k <= d; ++k) g[k] = g[k - 1] * gamma;   /* product of k copies of gamma */
}
/* R_{k+1} = R_k + gamma^k r_k  (Alg. 1 "Accumulate discounted reward") */
static double acc_reward(int mode, const double *g, int k, double r, double R) {
  if (mode) return (double)fmaf((float)g[k], (float)r, (float)R);
  return R + g[k] * r;
}
/* R_d + gamma^d max_a Q(s_d, a)  (Alg. 1 leaf line) */
static double leaf_total(int mode, const double *g, int d, double mq, double R) {
  if (mode) return (double)fmaf((float)g[d], (float)mq, (float)R);
  return R + g[d] * mq;
}
static double rowmax(const double *q, int A) {
  double mx = q[0];
  for (int a = 1; a < A; ++a) if (q[a] > mx) mx = q[a];
  return mx;
}
static int argmax_low(const double *q, int A) {   /* lowest index attaining the max */
  int b = 0;
  for (int a = 1; a < A; ++a) if (q[a] > q[b]) b = a;
  return b;
}

/* ----------------------------------------------------------- Eq. 4 / Eq. 5 */
/* Eq. 5: B = sqrt(log A)(de sqrt(d) - do sqrt(d-1)) - (de - do)/sqrt(8); log = ln (R5). */
double oracle_penalty_eq5(double de, double dob, int A, int d) {
  return sqrt(log((double)A)) * (de * sqrt((double)d) - dob * sqrt((double)(d - 1))) - (de - dob) / sqrt(8.0);
}
/* Eq. 4: sqrt(2 log A)(se sqrt(d) - so sqrt(d-1)) - (se - so)/2. */
double oracle_bias_gap_eq4(double so, double se, int A, int d) {
  return sqrt(2.0 * log((double)A)) * (se * sqrt((double)d) - so * sqrt((double)(d - 1))) - (se - so) / 2.0;
}

/* ------------------------------------------------- Lemma 2 exact biases */
/* Inverse standard normal CDF: Acklam's rational approximation refined by one
 * Halley step on erfc (|Phi(z) - p| ~ 1e-15). Independent of the CUDA path,
 * which uses the CUDA math library's normcdfinv. */
double oracle_inv_norm_cdf(double p) {
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                             1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                             6.680131188771972e+01, -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                             -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00};
  static const double dd[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                              3.754408661907416e+00};
  if (!(p > 0.0 && p < 1.0)) return NAN;
  const double plow = 0.02425, phigh = 1 - plow;
  double x;
  if (p < plow) {
    double q = sqrt(-2 * log(p));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((dd[0] * q + dd[1]) * q + dd[2]) * q + dd[3]) * q + 1);
  } else if (p <= phigh) {
    double q = p - 0.5, r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1);
  } else {
    double q = sqrt(-2 * log(1 - p));
    x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((dd[0] * q + dd[1]) * q + dd[2]) * q + dd[3]) * q + 1);
  }
  /* Halley refinement: e = Phi(x) - p, u = e * sqrt(2 pi) exp(x^2/2) */
  double e = 0.5 * erfc(-x / sqrt(2.0)) - p;
  double u = e * sqrt(2 * M_PI) * exp(x * x / 2);
  return x - u / (1 + x * u / 2);
}

/* B(n) of App. A.2: 0 if n = 1, else
 * gamma_EM * Phi^-1(1 - 1/(e n)) + (1 - gamma_EM) * Phi^-1(1 - 1/n). */
double oracle_B_n(double n) {
  const double gem = 0.57721566490153286; /* Euler-Mascheroni */
  if (n <= 1.0) return 0.0;
  return gem * oracle_inv_norm_cdf(1.0 - 1.0 / (M_E * n)) + (1.0 - gem) * oracle_inv_norm_cdf(1.0 - 1.0 / n);
}

/* Lemma 2: B_o = sigma_o B(A^(d-1)), B_e = sigma_e B(A^d - A^(d-1));
 * returns the exact gap B_e - B_o (Eq. 3's subtrahend before gamma^d). */
double oracle_bias_exact(double sigma_o, double sigma_e, int A, int d) {
  double ad1 = pow((double)A, (double)(d - 1)), ad = pow((double)A, (double)d);
  return sigma_e * oracle_B_n(ad - ad1) - sigma_o * oracle_B_n(ad1);
}

/* --------------------------------------------------------------- the DFS */
typedef struct {
  const oracle_model *m;
  int d, mode;
  double g[MAXD + 1];
  ostate *buf;          /* [d+1] per-depth scratch states */
  double q[MAXA];
} dfs_ctx;

/* dfs(s, t, R): if t = d: leaf total; else max over a of dfs(s'_a, t+1, R + g[t] r).
 * Returns the max value and, through *leaf, the lowest leaf index (within the
 * subtree, base-A digits a_t..a_{d-1}) attaining it. */
static int dfs(dfs_ctx *c, int t, double R, double *best, long *leaf) {
  const oracle_model *m = c->m;
  ostate *s = &c->buf[t];
  if (t == c->d) {
    if (qrow(m, s, c->mode, c->q)) return -1;
    *best = leaf_total(c->mode, c->g, c->d, rowmax(c->q, m->A), R);
    *leaf = 0;
    return 0;
  }
  double bv = -INFINITY;
  long bl = 0, span = 1;
  for (int k = t + 1; k < c->d; ++k) span *= m->A;
  for (int a = 0; a < m->A; ++a) {
    double r, v;
    long lf;
    if (env_step(m, s, a, &c->buf[t + 1], &r, c->mode)) return -1;
    if (dfs(c, t + 1, acc_reward(c->mode, c->g, t, r, R), &v, &lf)) return -1;
    if (v > bv) { bv = v; bl = (long)a * span + lf; }
  }
  *best = bv;
  *leaf = bl;
  return 0;
}

/* BCTS terms at one root: pi_o, delta_o, delta_e, B (Prop. 1, Eq. 5).
 * delta_a = r(s0,a) + gamma max Q(s1^a, .) - Q(s0, a) with depth-0/1 samples. */
static int bcts_terms(const oracle_model *m, const ostate *root, int d, int mode, const double *g,
                      double *terms, double *q0, int corr) {
  const int A = m->A;
  ostate *s1 = (ostate *)malloc(sizeof(ostate));
  double q1[MAXA], delta[MAXA];
  int rc = qrow(m, root, mode, q0);
  int pio = argmax_low(q0, A);
  for (int a = 0; a < A && !rc; ++a) {
    double r;
    rc = env_step(m, root, a, s1, &r, mode);
    if (!rc) rc = qrow(m, s1, mode, q1);
    if (rc) break;
    double R1 = acc_reward(mode, g, 0, r, 0.0);
    double one_step = leaf_total(mode, g, 1, rowmax(q1, A), R1);   /* Q-hat_1(s0, a) */
    delta[a] = mode ? (double)((float)one_step - (float)q0[a]) : one_step - q0[a];
  }
  free(s1);
  if (rc) return rc;
  double dob = fabs(delta[pio]), sum = 0.0;
  for (int a = 0; a < A; ++a) if (a != pio) sum += fabs(delta[a]);
  double de = sum / (A - 1);
  terms[0] = pio;
  terms[1] = dob;
  terms[2] = de;
  /* corr == 2: Lemma 2's exact gap with sigma = delta / sqrt(2) (Prop. 1); else Eq. 5 */
  terms[3] = corr == 2 ? oracle_bias_exact(dob / sqrt(2.0), de / sqrt(2.0), A, d) : oracle_penalty_eq5(de, dob, A, d);
  return 0;
}

/* Eq. 3 with the sweep constant beta: subtract beta*g[d]*B
 * from every root action != pi_o; beta == 0 or correction off -> vanilla exactly. */
static void apply_correction(int A, int d, int mode, const double *g, double beta, int corr,
                             const double *vanilla, const double *terms, double *q) {
  for (int a = 0; a < A; ++a) q[a] = vanilla[a];
  if (!corr || beta == 0.0 || d == 0) return;
  int pio = (int)terms[0];
  double gd = mode ? (double)(float)g[d] : g[d];
  double pen = beta * gd * terms[3];
  for (int a = 0; a < A; ++a)
    if (a != pio) q[a] = mode ? (double)(float)(vanilla[a] - pen) : vanilla[a] - pen;
}

/* Full search over n roots (records in ABI format). Outputs (nullable except
 * actions/root_q): vanilla_q [n*A], terms [n*4] (pi_o, delta_o, delta_e, B),
 * best_leaf [n*A] (lowest leaf index attaining each vanilla_q entry). */
int oracle_search(const oracle_model *m, const void *roots, long n_roots, int depth, double gamma,
                  double beta, int corr, int mode, int threads, int32_t *actions, double *root_q,
                  double *vanilla_q, double *terms_out, int64_t *best_leaf) {
  const int A = m->A;
  if (depth < 0 || depth > MAXD || n_roots < 0) return -1;
  const long rb = oracle_record_bytes(m);
  double g[MAXD + 1];
  discounts(gamma, depth, g);
  double *van = (double *)malloc(sizeof(double) * (n_roots * A + 1));
  int64_t *bl = (int64_t *)malloc(sizeof(int64_t) * (n_roots * A + 1));
  int err = 0;
  long ntask = n_roots * A;
  if (threads < 1) threads = 1;
  if (depth >= 1) {
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
    for (long task = 0; task < ntask; ++task) {
      long r = task / A;
      int a0 = (int)(task % A);
      dfs_ctx c;
      c.m = m; c.d = depth; c.mode = mode;
      memcpy(c.g, g, sizeof(g));
      c.buf = (ostate *)malloc(sizeof(ostate) * (depth + 1));
      from_record(m, (const uint8_t *)roots + r * rb, &c.buf[0]);
      double rr, v = 0.0;
      long lf = 0;
      int rc = env_step(m, &c.buf[0], a0, &c.buf[1], &rr, mode);
      if (!rc) rc = dfs(&c, 1, acc_reward(mode, g, 0, rr, 0.0), &v, &lf);
      long span = 1;
      for (int k = 1; k < depth; ++k) span *= A;
      van[task] = v;
      bl[task] = (int64_t)a0 * span + lf;
      if (rc) {
#pragma omp atomic write
        err = 1;
      }
      free(c.buf);
    }
  }
  if (err) { free(van); free(bl); return -1; }
  ostate *root = (ostate *)malloc(sizeof(ostate));
  for (long r = 0; r < n_roots && !err; ++r) {
    from_record(m, (const uint8_t *)roots + r * rb, root);
    double q0[MAXA], terms[4] = {0, 0, 0, 0}, q[MAXA];
    double *vr = van + r * A;
    if (depth == 0) {          /* d = 0: greedy on Q-hat(s0, .) (R11) */
      if (qrow(m, root, mode, q0)) { err = 1; break; }
      for (int a = 0; a < A; ++a) { vr[a] = q0[a]; q[a] = q0[a]; bl[r * A + a] = 0; }
      terms[0] = argmax_low(q0, A);
    } else {
      if (corr && bcts_terms(m, root, depth, mode, g, terms, q0, corr)) { err = 1; break; }
      apply_correction(A, depth, mode, g, beta, corr, vr, terms, q);
    }
    actions[r] = argmax_low(q, A);
    for (int a = 0; a < A; ++a) root_q[r * A + a] = q[a];
    if (vanilla_q) for (int a = 0; a < A; ++a) vanilla_q[r * A + a] = vr[a];
    if (terms_out) for (int k = 0; k < 4; ++k) terms_out[r * 4 + k] = terms[k];
    if (best_leaf) for (int a = 0; a < A; ++a) best_leaf[r * A + a] = bl[r * A + a];
  }
  free(root); free(van); free(bl);
  return err ? -1 : 0;
}

/* Node `index` of level `level` below one root: the state reached by the
 * action sequence given by the base-A digits of index (a_0 most significant,
 * R1 reading), and its cumulative discounted reward R_level. */
int oracle_node(const oracle_model *m, const void *root_rec, int level, int64_t index, double gamma,
                int mode, void *rec_out, double *R_out) {
  const int A = m->A;
  if (level < 0 || level > MAXD) return -1;
  double g[MAXD + 1];
  discounts(gamma, level, g);
  ostate *a = (ostate *)malloc(sizeof(ostate)), *b = (ostate *)malloc(sizeof(ostate));
  from_record(m, (const uint8_t *)root_rec, a);
  double R = 0.0;
  int rc = 0;
  for (int t = 0; t < level && !rc; ++t) {
    int64_t div = 1;
    for (int k = t + 1; k < level; ++k) div *= A;
    int act = (int)((index / div) % A);
    double r;
    rc = env_step(m, a, act, b, &r, mode);
    R = acc_reward(mode, g, t, r, R);
    ostate *tmp = a; a = b; b = tmp;
  }
  if (!rc) { to_record(m, a, (uint8_t *)rec_out); *R_out = R; }
  free(a); free(b);
  return rc;
}

/* Brute force: Eq. 1 literally -- enumerate all A^d action sequences in
 * lexicographic order (leaf index base A), roll each out from the root, and
 * take the max over each a_0 block. Same outputs as oracle_search. */
int oracle_search_bruteforce(const oracle_model *m, const void *roots, long n_roots, int depth,
                             double gamma, double beta, int corr, int mode, int32_t *actions,
                             double *root_q, double *vanilla_q, double *terms_out, int64_t *best_leaf) {
  const int A = m->A;
  if (depth < 1 || depth > MAXD) return -1;
  const long rb = oracle_record_bytes(m);
  double g[MAXD + 1];
  discounts(gamma, depth, g);
  int64_t nleaf = 1;
  for (int k = 0; k < depth; ++k) nleaf *= A;
  int64_t seg = nleaf / A;
  uint8_t *rec = (uint8_t *)malloc(rb);
  ostate *leaf = (ostate *)malloc(sizeof(ostate)), *root = (ostate *)malloc(sizeof(ostate));
  double q[MAXA], van[MAXA], qq[MAXA], q0[MAXA], terms[4] = {0, 0, 0, 0};
  int64_t bl[MAXA];
  int rc = 0;
  for (long r = 0; r < n_roots && !rc; ++r) {
    const uint8_t *rr = (const uint8_t *)roots + r * rb;
    for (int a = 0; a < A; ++a) { van[a] = -INFINITY; bl[a] = 0; }
    for (int64_t i = 0; i < nleaf && !rc; ++i) {
      double R;
      rc = oracle_node(m, rr, depth, i, gamma, mode, rec, &R);
      if (rc) break;
      from_record(m, rec, leaf);
      rc = qrow(m, leaf, mode, q);
      double tot = leaf_total(mode, g, depth, rowmax(q, A), R);
      int a0 = (int)(i / seg);
      if (tot > van[a0]) { van[a0] = tot; bl[a0] = i; }
    }
    if (rc) break;
    from_record(m, rr, root);
    if (corr) rc = bcts_terms(m, root, depth, mode, g, terms, q0, corr);
    if (rc) break;
    apply_correction(A, depth, mode, g, beta, corr, van, terms, qq);
    actions[r] = argmax_low(qq, A);
    for (int a = 0; a < A; ++a) root_q[r * A + a] = qq[a];
    if (vanilla_q) for (int a = 0; a < A; ++a) vanilla_q[r * A + a] = van[a];
    if (terms_out) for (int k = 0; k < 4; ++k) terms_out[r * 4 + k] = terms[k];
    if (best_leaf) for (int a = 0; a < A; ++a) best_leaf[r * A + a] = bl[a];
  }
  free(rec); free(leaf); free(root);
  return rc ? -1 : 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* BCTS terms only (pi_o, delta_o, delta_e, B at depth d) for n roots: needs
 * just the root row and the A level-1 rows (Prop. 1), so it runs at
 * full-size configs where the complete DFS would not finish in a test. */
int oracle_terms(const oracle_model *m, const void *roots, long n_roots, int depth, double gamma, int mode,
                 double *terms_out, double *q0_out) {
  const long rb = oracle_record_bytes(m);
  double g[MAXD + 1];
  if (depth < 1 || depth > MAXD) return -1;
  discounts(gamma, depth, g);
  ostate *root = (ostate *)malloc(sizeof(ostate));
  int rc = 0;
  for (long r = 0; r < n_roots && !rc; ++r) {
    from_record(m, (const uint8_t *)roots + r * rb, root);
    rc = bcts_terms(m, root, depth, mode, g, terms_out + 4 * r, q0_out + (long)m->A * r, 1);
  }
  free(root);
  return rc;
}

/* Bounded CPU-baseline sample: the same DFS, restricted to the depth-2
 * subtrees t in [t_begin, t_end) of one root (t = a0*A + a1), one OpenMP task
 * per subtree. out[t - t_begin] = max over the subtree's leaves of the leaf
 * total. Used only to time the oracle on a bounded sample (bench.py). */
int oracle_search_subtrees(const oracle_model *m, const void *root_rec, int depth, double gamma, int mode,
                           int threads, long t_begin, long t_end, double *out) {
  const int A = m->A;
  if (depth < 2 || depth > MAXD || t_begin < 0 || t_end > (long)A * A || t_end < t_begin) return -1;
  double g[MAXD + 1];
  discounts(gamma, depth, g);
  int err = 0;
  if (threads < 1) threads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
  for (long t = t_begin; t < t_end; ++t) {
    dfs_ctx c;
    c.m = m; c.d = depth; c.mode = mode;
    memcpy(c.g, g, sizeof(g));
    c.buf = (ostate *)malloc(sizeof(ostate) * (depth + 1));
    ostate *mid = (ostate *)malloc(sizeof(ostate));
    from_record(m, (const uint8_t *)root_rec, &c.buf[0]);
    double r0, r1, v = 0.0;
    long lf = 0;
    int rc = env_step(m, &c.buf[0], (int)(t / A), mid, &r0, mode);
    if (!rc) rc = env_step(m, mid, (int)(t % A), &c.buf[2], &r1, mode);
    if (!rc) rc = dfs(&c, 2, acc_reward(mode, g, 1, r1, acc_reward(mode, g, 0, r0, 0.0)), &v, &lf);
    out[t - t_begin] = v;
    if (rc) {
#pragma omp atomic write
      err = 1;
    }
    free(mid);
    free(c.buf);
  }
  return err ? -1 : 0;
}

/* Leaf total of leaf `index` below one root: R_d + gamma^d max_a Q(s_d, a)
 * with the oracle's own arithmetic (fmaf in the fp32-mirror mode, R3). */
int oracle_leaf_total(const oracle_model *m, const void *root_rec, int depth, int64_t index, double gamma,
                      int mode, double *total) {
  if (depth < 1 || depth > MAXD) return -1;
  double g[MAXD + 1], q[MAXA], R;
  discounts(gamma, depth, g);
  uint8_t *rec = (uint8_t *)malloc(oracle_record_bytes(m));
  ostate *s = (ostate *)malloc(sizeof(ostate));
  int rc = oracle_node(m, root_rec, depth, index, gamma, mode, rec, &R);
  if (!rc) {
    from_record(m, rec, s);
    rc = qrow(m, s, mode, q);
  }
  if (!rc) *total = leaf_total(mode, g, depth, rowmax(q, m->A), R);
  free(rec);
  free(s);
  return rc;
}

/* ------------------------------------------------ early pruning (NEXT-4) */
/* Early pruning with an index array of unpruned states ("future work";
 * DESIGN.md R30-R33). Alg. 1 run level by level over explicit node
 * lists; every node carries its implicit index f in the UNPRUNED tree below its
 * root (base-A digits = the action path, R1), so the root action of a node is
 * its leading digit and the best leaf is traced through f ("These indices
 * are then used for tracing the optimal action at the root"). After level k is
 * expanded, for k in [first, d-1], one rule thins it within each group
 * (root, root action a_0) = f / A^(k-1):
 *   rule 1 (BOUND, exact; R31): with one-step rewards in [r_lo, r_hi] and leaf
 *     values max_a Q in [q_lo, q_hi], every leaf below node i totals within
 *     [R_i + L_k, R_i + U_k], L_k = sum_{j=k}^{d-1} g[j] r_lo + g[d] q_lo (U_k with
 *     the _hi ends). Node i is pruned iff R_i + U_k + s_i < max over its group of
 *     (R_j + L_k - s_j), s = 2^-16 (|R| + S_k) a rounding margin, S_k the same
 *     sum over max(|lo|, |hi|). Such a node holds no leaf that can reach its
 *     group's max, so the search result is unchanged (only work is saved).
 *   rule 2 (BEAM; R32): keep the `beam` nodes of each group with the highest
 *     depth-k estimate v_i = R_i + g[k] max_a Q(s_i, a) (the "estimated value
 *     over all the tree nodes" of P:299), ties to the lower f.
 * Leaves (level d) are never pruned. survivors[k] (nullable) = nodes kept at
 * level k summed over roots (survivors[0] = n_roots, survivors[d] = leaves scored). Other outputs as
 * oracle_search. The bound arithmetic is plain double, the discounts g[j]
 * rounded to fp32 in mode 1 (the values the search itself uses). */
typedef struct {
  ostate s;
  double R;
  int64_t f;
} pnode;

static void prune_bounds(const double *g, int k, int d, double r_lo, double r_hi, double q_lo, double q_hi,
                         double *L, double *U, double *S) {
  double l = 0.0, u = 0.0, sa = 0.0;
  const double ra = fabs(r_lo) > fabs(r_hi) ? fabs(r_lo) : fabs(r_hi);
  const double qa = fabs(q_lo) > fabs(q_hi) ? fabs(q_lo) : fabs(q_hi);
  for (int j = k; j < d; ++j) {
    l = l + g[j] * r_lo;
    u = u + g[j] * r_hi;
    sa = sa + g[j] * ra;
  }
  *L = l + g[d] * q_lo;
  *U = u + g[d] * q_hi;
  *S = sa + g[d] * qa;
}

int oracle_search_pruned(const oracle_model *m, const void *roots, long n_roots, int depth, double gamma,
                         double beta, int corr, int mode, int rule, int first, long beam, double r_lo,
                         double r_hi, double q_lo, double q_hi, int32_t *actions, double *root_q,
                         double *vanilla_q, double *terms_out, int64_t *best_leaf, int64_t *survivors) {
  const int A = m->A;
  if (depth < 1 || depth > MAXD || n_roots < 0 || rule < 0 || rule > 2) return -1;
  if (rule == 2 && beam < 1) return -1;
  if (rule == 1 && !(r_lo <= r_hi && q_lo <= q_hi)) return -1;
  if (first < 1) first = 1;
  const long rb = oracle_record_bytes(m);
  double g[MAXD + 1], gu[MAXD + 1];
  discounts(gamma, depth, g);
  for (int k = 0; k <= depth; ++k) gu[k] = mode ? (double)(float)g[k] : g[k];
  if (survivors) {
    for (int k = 0; k <= depth; ++k) survivors[k] = 0;
    survivors[0] = n_roots;
  }
  int64_t span = 1;                       /* A^(d-1) leaves per root action */
  for (int k = 1; k < depth; ++k) span *= A;
  int rc = 0;
  for (long r = 0; r < n_roots && !rc; ++r) {
    pnode *cur = (pnode *)malloc(sizeof(pnode));
    long ncur = 1;
    from_record(m, (const uint8_t *)roots + r * rb, &cur[0].s);
    cur[0].R = 0.0;
    cur[0].f = 0;
    double van[MAXA], q[MAXA];
    int64_t bl[MAXA];
    for (int a = 0; a < A; ++a) { van[a] = -INFINITY; bl[a] = 0; }
    for (int k = 1; k <= depth && !rc; ++k) {
      if (k == depth) {                   /* leaves: R_d + g[d] max_a Q, max per root action */
        ostate *leaf = (ostate *)malloc(sizeof(ostate));
        if (survivors) survivors[depth] += ncur * A;
        for (long i = 0; i < ncur && !rc; ++i)
          for (int a = 0; a < A && !rc; ++a) {
            double rr;
            rc = env_step(m, &cur[i].s, a, leaf, &rr, mode);
            if (!rc) rc = qrow(m, leaf, mode, q);
            if (rc) break;
            const double tot = leaf_total(mode, g, depth, rowmax(q, A), acc_reward(mode, g, k - 1, rr, cur[i].R));
            const int64_t f = cur[i].f * A + a;
            const int a0 = (int)(f / span);
            if (tot > van[a0] || (tot == van[a0] && f < bl[a0])) { van[a0] = tot; bl[a0] = f; }
          }
        free(leaf);
        break;
      }
      /* expand: children of node i in action order (Alg. 1) */
      pnode *nxt = (pnode *)malloc(sizeof(pnode) * (size_t)(ncur * A));
      long nn = 0;
      for (long i = 0; i < ncur && !rc; ++i)
        for (int a = 0; a < A && !rc; ++a) {
          double rr;
          rc = env_step(m, &cur[i].s, a, &nxt[nn].s, &rr, mode);
          nxt[nn].R = acc_reward(mode, g, k - 1, rr, cur[i].R);
          nxt[nn].f = cur[i].f * A + a;
          ++nn;
        }
      free(cur);
      cur = nxt;
      ncur = nn;
      if (rc) break;
      if (rule != 0 && k >= first && k <= depth - 1) {
        int64_t gsz = 1;                  /* A^(k-1) level-k nodes per root action */
        for (int j = 1; j < k; ++j) gsz *= A;
        char *keep = (char *)calloc((size_t)ncur, 1);
        if (rule == 1) {
          double L, U, S, best[MAXA];
          prune_bounds(gu, k, depth, r_lo, r_hi, q_lo, q_hi, &L, &U, &S);
          for (int a = 0; a < A; ++a) best[a] = -INFINITY;
          for (long i = 0; i < ncur; ++i) {
            const double s = ldexp(fabs(cur[i].R) + S, -16);
            const double lb = (cur[i].R + L) - s;
            const int a0 = (int)(cur[i].f / gsz);
            if (lb > best[a0]) best[a0] = lb;
          }
          for (long i = 0; i < ncur; ++i) {
            const double s = ldexp(fabs(cur[i].R) + S, -16);
            const double ub = (cur[i].R + U) + s;
            keep[i] = !(ub < best[cur[i].f / gsz]);
          }
        } else {
          double *v = (double *)malloc(sizeof(double) * (size_t)ncur);
          for (long i = 0; i < ncur && !rc; ++i) {
            rc = qrow(m, &cur[i].s, mode, q);
            v[i] = leaf_total(mode, g, k, rowmax(q, A), cur[i].R);   /* depth-k estimate */
          }
          for (long i = 0; i < ncur; ++i) {   /* rank within the group: better = higher v, then lower f */
            long rank = 0;
            for (long j = 0; j < ncur; ++j)
              if (j != i && cur[j].f / gsz == cur[i].f / gsz &&
                  (v[j] > v[i] || (v[j] == v[i] && cur[j].f < cur[i].f)))
                ++rank;
            keep[i] = rank < beam;
          }
          free(v);
        }
        long w = 0;
        for (long i = 0; i < ncur; ++i)
          if (keep[i]) cur[w++] = cur[i];
        ncur = w;
        free(keep);
      }
      if (survivors) survivors[k] += ncur;
    }
    free(cur);
    if (rc) break;
    ostate *root = (ostate *)malloc(sizeof(ostate));
    from_record(m, (const uint8_t *)roots + r * rb, root);
    double q0[MAXA], terms[4] = {0, 0, 0, 0}, qq[MAXA];
    if (corr) rc = bcts_terms(m, root, depth, mode, g, terms, q0, corr);
    free(root);
    if (rc) break;
    apply_correction(A, depth, mode, g, beta, corr, van, terms, qq);
    actions[r] = argmax_low(qq, A);
    for (int a = 0; a < A; ++a) root_q[r * A + a] = qq[a];
    if (vanilla_q) for (int a = 0; a < A; ++a) vanilla_q[r * A + a] = van[a];
    if (terms_out) for (int k = 0; k < 4; ++k) terms_out[r * 4 + k] = terms[k];
    if (best_leaf) for (int a = 0; a < A; ++a) best_leaf[r * A + a] = bl[a];
  }
  return rc ? -1 : 0;
}
