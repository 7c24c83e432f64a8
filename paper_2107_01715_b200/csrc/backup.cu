// backup.cu -- K3: segmented max/argmax backup (Alg. 1 return line P:324,
// Eq. 1) and the BCTS correction + action (Eq. 3, Eq. 5
// P:276-280, Prop. 1, sweep constant P:371).
//
// The backup folds each leaf total into the key of its (root, root action)
// segment: key = (orderable(total), lowest leaf index). Max over packed keys is
// exact and associative, so the warp-shuffle reduction + one atomicMax per warp
// equals the level-by-level max over each node's A children,
// independent of chunking, launch order and sharding (bit-identical results).
#include <math.h>

#include "engine.h"

namespace bcts {

__global__ void k_keys_init(int64_t *keys, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) keys[i] = kKeyEmpty;
}

void launch_keys_init(int64_t *keys, int64_t count, cudaStream_t st) {
  if (count > 0) k_keys_init<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(keys, count);
}

__global__ void k_segmax(const float *__restrict__ totals, int64_t n, int64_t leaf_begin, int64_t lpr, int64_t seg,
                         int A, int64_t *__restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x % 32;
  int64_t key = kKeyEmpty, slot = -1;
  if (i < n) {
    const int64_t L = leaf_begin + i;
    const int64_t root = L / lpr;
    const int64_t within = L - root * lpr;
    slot = root * A + within / seg;
    key = pack_key(totals[i], within);
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

void launch_segmax(const float *totals, int64_t n, int64_t leaf_begin, int64_t leaves_per_root, int64_t seg, int A,
                   int64_t *keys, cudaStream_t st, Profiler *prof) {
  if (n <= 0) return;
  if (prof) prof->begin(KC_SEGMAX, 4.0 * (double)n, st);   // algorithmic bytes: one fp32 total per leaf
  k_segmax<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(totals, n, leaf_begin, leaves_per_root, seg, A, keys);
  if (prof) prof->end(st);
}

// out[i] = max_a rows[i*A + a] (the level-1 maxima of the prologue, from full rows).
__global__ void k_rowmax(const float *__restrict__ rows, int64_t n, int A, float *__restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float m = rows[i * A];
  for (int a = 1; a < A; ++a) m = fmaxf(m, rows[i * A + a]);
  out[i] = m;
}

void launch_rowmax(const float *rows, int64_t n, int A, float *out, cudaStream_t st) {
  if (n > 0) k_rowmax<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(rows, n, A, out);
}

// B(n) of App. A.2 with the CUDA math library's inverse normal CDF.
__device__ double B_of_n(double n) {
  const double gem = 0.57721566490153286;   // Euler-Mascheroni
  if (n <= 1.0) return 0.0;
  return gem * normcdfinv(1.0 - 1.0 / (2.718281828459045 * n)) + (1.0 - gem) * normcdfinv(1.0 - 1.0 / n);
}

// One warp per root, lane a (and a + 32) owns action a: the loads and the level-1 row maxima run
// in parallel across the lanes; the order-sensitive double sum of |delta_a| (R6: increasing a) and
// the Eq. 5 arithmetic run on lane 0 in exactly the sequential order of the single-thread form.
__global__ void k_finalize(FinalizeArgs f) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (r >= f.n) return;   // warp-uniform
  const int A = f.A;
  float van[2], q0v[2], dl[2];
  for (int h = 0; h < 2; ++h) {
    const int a = lane + 32 * h;
    van[h] = q0v[h] = dl[h] = 0.0f;
    if (a >= A) continue;
    if (f.d == 0) {
      van[h] = f.q0[r * A + a];
      if (f.best_leaf) f.best_leaf[r * A + a] = 0;
    } else {
      const int64_t k = f.keys[r * A + a];
      van[h] = key_value(k);
      if (f.best_leaf) f.best_leaf[r * A + a] = key_leaf(k);
    }
    if (f.d == 0 || f.corr) {
      q0v[h] = f.q0[r * A + a];
      if (f.d >= 1) {   // delta_a = fmaf(g1, max_a' Q(s1^a, a'), R1_a) - Q(s0, a)   (Prop. 1; R7)
        float m1;
        if (f.rows1) {  // max over the level-1 row (fmaxf is exact)
          const float *row = f.rows1 + (r * A + a) * A;
          m1 = row[0];
          for (int b = 1; b < A; ++b) m1 = fmaxf(m1, row[b]);
        } else {
          m1 = f.m1[r * A + a];
        }
        dl[h] = fmaf(f.g1, m1, f.r1[r * A + a]) - q0v[h];
      }
    }
  }
  float terms[4] = {0.f, 0.f, 0.f, 0.f};
  double pen = 0.0;
  int pio = 0;
  if (f.d == 0 || f.corr) {
    // pi_o = lowest argmax of Q_hat(s0, .) (R23), gathered in increasing a on every lane
    float best = -INFINITY;
    for (int a = 0; a < A; ++a) {
      const float v = __shfl_sync(0xffffffffu, q0v[a >> 5], a & 31);
      if (a == 0 || v > best) best = v, pio = a;
    }
    terms[0] = (float)pio;
    if (f.d >= 1) {
      double dob = 0.0, sum = 0.0;
      for (int a = 0; a < A; ++a) {
        const float delta = __shfl_sync(0xffffffffu, dl[a >> 5], a & 31);
        if (a == pio) dob = fabs((double)delta);
        else sum += fabs((double)delta);
      }
      const double de = sum / (double)(A - 1);
      double B;
      if (f.corr == 2) {   // Lemma 2 exact gap B_e - B_o with sigma = delta / sqrt(2)
        const double ad1 = pow((double)A, (double)(f.d - 1)), ad = ad1 * (double)A;
        B = (de / sqrt(2.0)) * B_of_n(ad - ad1) - (dob / sqrt(2.0)) * B_of_n(ad1);
      } else {             // Eq. 5 (natural log, R5)
        B = sqrt(log((double)A)) * (de * sqrt((double)f.d) - dob * sqrt((double)(f.d - 1))) - (de - dob) / sqrt(8.0);
      }
      if (f.clamp && B < 0.0) B = 0.0;
      terms[1] = (float)dob;
      terms[2] = (float)de;
      terms[3] = (float)B;
      if (f.beta != 0.0f) pen = (double)f.beta * (double)f.gd * B;   // Eq. 3 (R9, R12)
    }
  }
  float q[2];
  for (int h = 0; h < 2; ++h) {
    const int a = lane + 32 * h;
    q[h] = (pen != 0.0 && a != pio) ? (float)((double)van[h] - pen) : van[h];
    if (a < A) {
      f.root_q[r * A + a] = q[h];
      if (f.vanilla) f.vanilla[r * A + a] = van[h];
    }
  }
  // lowest index attaining the max of q (R4), gathered in increasing a
  int best = 0;
  float bq = 0.0f;
  for (int a = 0; a < A; ++a) {
    const float v = __shfl_sync(0xffffffffu, q[a >> 5], a & 31);
    if (a == 0 || v > bq) bq = v, best = a;
  }
  if (lane == 0) {
    f.actions[r] = best;
    if (f.terms)
      for (int k = 0; k < 4; ++k) f.terms[r * 4 + k] = terms[k];
  }
}

void launch_finalize(const FinalizeArgs &a, cudaStream_t st, Profiler *prof) {
  if (a.n <= 0) return;
  if (prof) prof->begin(KC_FINALIZE, (double)a.n * a.A * 28.0, st);
  k_finalize<<<(unsigned)((a.n + 3) / 4), 128, 0, st>>>(a);   // one warp per root
  if (prof) prof->end(st);
}

// PV target (App. B.3; R29): gather the executed action's Eq. 1
// value and decode its best leaf into base-A digits (one thread per root).
__global__ void k_pv_targets(int64_t n, int A, int d, const int32_t *__restrict__ actions,
                             const float *__restrict__ vanilla, const int64_t *__restrict__ best_leaf,
                             float *__restrict__ target, int32_t *__restrict__ path) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int a = actions[r];
  if (a < 0 || a >= A) {
    target[r] = __int_as_float(0x7fc00000);
    for (int t = 0; t < d; ++t) path[r * d + t] = -1;
    return;
  }
  target[r] = vanilla[r * A + a];
  int64_t leaf = best_leaf[r * A + a];
  for (int t = d - 1; t >= 0; --t) {
    path[r * d + t] = (int32_t)(leaf % A);
    leaf /= A;
  }
}

void launch_pv_targets(int64_t n, int A, int d, const int32_t *actions, const float *vanilla,
                       const int64_t *best_leaf, float *target, int32_t *path, cudaStream_t st) {
  if (n <= 0) return;
  k_pv_targets<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(n, A, d, actions, vanilla, best_leaf, target, path);
}

}  // namespace bcts
