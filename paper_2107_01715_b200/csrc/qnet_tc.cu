// qnet_tc.cu -- tcgen05/TMEM implicit-GEMM layer (placeholder until the
// tensor-core kernel lands; every layer falls back to the SIMT reference).
#include "engine.h"

namespace bcts {
bool tc_supported(const Layer &) { return false; }
void launch_layer_tc(const Layer &L, const void *in, int64_t n_img, void *out, cudaStream_t st) {
  launch_layer_simt(L, in, n_img, out, st);
}
}  // namespace bcts
