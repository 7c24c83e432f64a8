/* bcts_example.c -- the C ABI used from plain C99 (no Python, no torch): one Batch-BFS + BCTS search
 * (Alg. 1; Eq. 3/5) on the synthetic INT_HASH env with an MLP2 64-256-4 value net whose
 * weights come from a fixed linear congruential generator.
 *
 *   gcc -std=c99 -I include examples/bcts_example.c -L paper_2107_01715_b200 -lbcts \
 *       -Wl,-rpath,paper_2107_01715_b200 -o bcts_example
 *   ./bcts_example [inputs.bin]      # prints one line per root: action, corrected Q[0..A-1]
 *
 * With an argument it also writes its inputs (weights, then root records, as raw little-endian
 * fp32 / uint32) so a test can replay the same search through the oracle. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "bcts.h"

enum { A = 4, IN = 64, HID = 256, N_ROOTS = 8, DEPTH = 3 };

static uint64_t lcg_state = 0x2107017150ull;
static uint32_t lcg(void) {
  lcg_state = lcg_state * 6364136223846793005ull + 1442695040888963407ull;
  return (uint32_t)(lcg_state >> 32);
}
static float uniform_pm(float bound) { return bound * (2.0f * (float)(lcg() >> 8) / 16777216.0f - 1.0f); }

int main(int argc, char **argv) {
  /* MLP2 weights in the canonical order: w1 [HID][IN], b1 [HID], w2 [A][HID], b2 [A] */
  const int64_t nw = (int64_t)HID * IN + HID + (int64_t)A * HID + A;
  float *w = (float *)malloc((size_t)nw * sizeof(float));
  int64_t k = 0;
  for (int64_t i = 0; i < (int64_t)HID * IN + HID; ++i) w[k++] = uniform_pm(1.0f / sqrtf((float)IN));
  for (int64_t i = 0; i < (int64_t)A * HID + A; ++i) w[k++] = uniform_pm(1.0f / sqrtf((float)HID));
  uint32_t roots[N_ROOTS][16];
  for (int r = 0; r < N_ROOTS; ++r)
    for (int j = 0; j < 16; ++j) roots[r][j] = lcg();

  bcts_config cfg = {0};
  cfg.abi_version = BCTS_ABI_VERSION;
  cfg.device = 0;
  cfg.env = BCTS_ENV_INT_HASH;
  cfg.num_actions = A;
  cfg.net = BCTS_NET_MLP2_F32;
  cfg.weights = w;
  cfg.weights_count = nw;
  cfg.mlp_in = IN;
  cfg.mlp_hidden = HID;
  bcts_handle h = NULL;
  bcts_status s = bcts_create(&cfg, &h);
  if (s != BCTS_OK) {
    fprintf(stderr, "bcts_create: %s\n", bcts_status_string(s));
    return 1;
  }
  int32_t actions[N_ROOTS];
  float q[N_ROOTS * A];
  s = bcts_search_host(h, roots, N_ROOTS, DEPTH, A, 0.99f, 1.0f, 1, actions, q);
  if (s != BCTS_OK) {
    fprintf(stderr, "bcts_search_host: %s (%s)\n", bcts_status_string(s), bcts_last_error(h));
    bcts_destroy(h);
    return 1;
  }
  for (int r = 0; r < N_ROOTS; ++r) {
    printf("%d", actions[r]);
    for (int a = 0; a < A; ++a) printf(" %.9g", q[r * A + a]);
    printf("\n");
  }
  if (argc > 1) {
    FILE *f = fopen(argv[1], "wb");
    if (!f || fwrite(w, sizeof(float), (size_t)nw, f) != (size_t)nw ||
        fwrite(roots, sizeof(roots), 1, f) != 1) {
      fprintf(stderr, "cannot write %s\n", argv[1]);
      return 1;
    }
    fclose(f);
  }
  bcts_destroy(h);
  free(w);
  return 0;
}
