// qnet_conv.cu -- K2 conv trunk on the tensor cores by SHIFTED WINDOWS.
//
// Every conv of the trunk is written as a stride-1 conv (conv1 on the
// space-to-depth(4) frame, conv2 on space-to-depth(2) of act1, conv3 as is):
//   out[q] = sum_taps sum_c W[tap][c] * in[q + off(tap)][c],   q = oy*W_in + ox
// with "full-width" output rows q (ox in [0, W_in); the ox >= OW columns are
// discarded). For a fixed tap the A operand of the GEMM is then a contiguous
// window of input rows starting at (tile_row0 + off(tap)). Activations are
// stored per image in a chunk-planar K-major layout
//     byte(row r, channel chunk j of 8 bf16) = j * PLANE + r * 16
// which is the tcgen05 K-major SWIZZLE_NONE canonical layout (8-row core
// matrices of 16-byte rows: SBO = 128 B between row groups, LBO = PLANE
// between K chunks) for ANY starting row -- so each tap's A operand is just a
// descriptor at a shifted address. One bulk copy brings an image into shared
// memory once; no im2col duplication crosses L2 (TMA im2col re-read every
// input 4-9x). The epilogue writes the next layer's planar input directly.
//
// Warp roles (192 threads, persistent over images):
//   warp 0    : bulk-copy producer, double-buffered input image
//   warp 1    : TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5 : epilogue (TMEM -> bias/ReLU/bf16 -> next layer's layout),
//               double-buffered accumulators (one set per image)
#include <algorithm>

#include "engine.h"

namespace bcts {
namespace {

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(saddr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(saddr(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major SWIZZLE_NONE descriptor: LBO = K-chunk stride, SBO = 8-row-group stride.
__device__ __forceinline__ uint64_t desc_planar(uint32_t addr, uint32_t plane_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((plane_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)(128 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;                                   // layout type 0 = SWIZZLE_NONE
}
// K-major SWIZZLE_128B descriptor for a window starting at any 128-byte row;
// base_offset (bits 49-51) carries the window's swizzle phase when requested.
__device__ __forceinline__ uint64_t desc_sw128_win(uint32_t addr, bool phase) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  if (phase) d |= (uint64_t)((addr >> 7) & 7u) << 49;
  d |= (uint64_t)2 << 61;
  return d;
}
// K-major SWIZZLE_128B descriptor (resident weights, 8 rows x 128 B atoms).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// Warp-uniform issue: the whole MMA warp runs the (fully unrolled) loop with
// descriptors in uniform registers; only the elected lane's predicate is set.
// (A lane-0-only loop costs ~150 cycles of R2UR / ELECT overhead per MMA,
// measured in tools/mma_bench.cu; this form reaches the SMEM-operand floor.)
__device__ __forceinline__ uint32_t elect_one() {
  uint32_t e;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(e));
  return e;
}
__device__ __forceinline__ void mma_pred(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc,
                                         uint32_t issue) {
  asm volatile(
      "{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nsetp.ne.b32 q, %5, 0;\n"
      "@q tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(issue));
}
__device__ __forceinline__ void commit_pred(uint64_t *bar, uint32_t issue) {
  asm volatile(
      "{\n.reg .pred q;\nsetp.ne.b32 q, %1, 0;\n"
      "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(saddr(bar)),
      "r"(issue)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

constexpr int kThreads = 192;

// Debug phase timestamps (CTA 0 only; BCTS_CONV_TRACE=1): [img][4] =
// copy issued, input ready (MMA side), MMAs issued, epilogue done.
__device__ unsigned long long *g_trace = nullptr;
__device__ int g_trace_sel = -1;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Compile-time trunk geometry (stride-1 convs after space-to-depth).
struct G1 { static constexpr int N = 32, CIN = 64, KH = 2, KW = 2, W_IN = 21, N_MT = 4; static constexpr uint32_t BPLANE = kPlane1 * 8; };
struct G2 { static constexpr int N = 64, CIN = 128, KH = 2, KW = 2, W_IN = 10, N_MT = 1; static constexpr uint32_t BPLANE = kPlane2 * 8; };
struct G3 { static constexpr int N = 64, CIN = 64, KH = 3, KW = 3, W_IN = 9, N_MT = 1; static constexpr uint32_t BPLANE = kPlane3 * 8; };

template <class G>
__global__ void __launch_bounds__(kThreads, 1)
    k_conv_sw(ConvSW P, const uint8_t *__restrict__ Wsw, const float *__restrict__ bias,
              const uint8_t *__restrict__ in, int64_t n_img, uint8_t *__restrict__ out) {
  constexpr int N = G::N;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *sW = smem;                                   // K/64 blocks of [N x 128 B], SW128
  const int nkb = P.K / 64;
  uint8_t *sIn0 = smem + (size_t)nkb * N * 128;         // two input-image buffers
  const uint32_t in_stride = (P.in_img_bytes + 1023u) & ~1023u;
  __shared__ __align__(8) uint64_t in_full[2], in_empty[2], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const uint32_t tcols_img = (uint32_t)(P.n_mt * N);
  uint32_t tcols = 32;
  while (tcols < 2 * tcols_img) tcols <<= 1;

  __shared__ float sbias[64];
  __shared__ __align__(8) uint64_t wbar;
  if (threadIdx.x < N) sbias[threadIdx.x] = bias[threadIdx.x];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&in_full[i], 1);
      mbar_init(&in_empty[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    mbar_init(&wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // resident weights: one bulk copy of their pre-swizzled SW128 shared-memory image
    mbar_expect_tx(&wbar, (uint32_t)(nkb * N * 128));
    bulk_g2s(saddr(sW), Wsw, (uint32_t)(nkb * N * 128), &wbar);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_slot)),
                 "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t i = 0;
      for (int64_t img = blockIdx.x; img < n_img; img += gridDim.x, ++i) {
        const uint32_t b = i & 1u, ph = (i >> 1) & 1u;
        mbar_wait(&in_empty[b], ph ^ 1u);
        if (g_trace && P.out_mode == g_trace_sel && blockIdx.x == 0 && i < 64) g_trace[i * 4 + 0] = gtime();
        mbar_expect_tx(&in_full[b], P.in_img_bytes);
        bulk_g2s(saddr(sIn0 + b * in_stride), in + img * (int64_t)P.in_img_bytes, P.in_img_bytes, &in_full[b]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------- MMA issuer (whole warp, one elected lane issues)
    constexpr uint32_t idesc = idesc_bf16(128, N);
    constexpr int TAPS = G::KH * G::KW, KSTEPS = G::CIN / 16;
    const uint32_t elected = elect_one();
    mbar_wait(&wbar, 0);
    const uint64_t wdesc = desc_sw128(saddr(sW));
    uint32_t i = 0;
    for (int64_t img = blockIdx.x; img < n_img; img += gridDim.x, ++i) {
      const uint32_t b = i & 1u, ph = (i >> 1) & 1u;
      mbar_wait(&in_full[b], ph);
      if (g_trace && P.out_mode == g_trace_sel && blockIdx.x == 0 && i < 64 && elected) g_trace[i * 4 + 1] = gtime();
      mbar_wait(&tempty[b], ph ^ 1u);
      tc_fence_after();
      const uint32_t a_base = saddr(sIn0 + b * in_stride);
      const uint64_t adesc0 = desc_sw128_win(a_base, false);
      const uint32_t d0 = tmem + b * tcols_img;
#pragma unroll
      for (int mt = 0; mt < G::N_MT; ++mt)
#pragma unroll
        for (int tap = 0; tap < TAPS; ++tap)
#pragma unroll
          for (int kk = 0; kk < KSTEPS; ++kk) {
            // A: SW128 row block kk/4, window row mt*128 + ty*W_IN + tx, +32 B per 16 channels
            constexpr int dummy = 0;
            (void)dummy;
            const uint32_t a_off = (uint32_t)(kk >> 2) * G::BPLANE +
                                   (uint32_t)(mt * 128 + (tap / G::KW) * G::W_IN + (tap % G::KW)) * 128u +
                                   (uint32_t)((kk & 3) * 32);
            const int k = tap * G::CIN + 16 * kk;   // weight K index, (tap, c) order
            const uint32_t w_off = (uint32_t)(k >> 6) * (N * 128) + (uint32_t)((k & 63) * 2);
            mma_pred(d0 + (uint32_t)(mt * N), adesc0 + (a_off >> 4), wdesc + (w_off >> 4), idesc,
                     (tap | kk) != 0, elected);
          }
      if (g_trace && P.out_mode == g_trace_sel && blockIdx.x == 0 && i < 64 && elected) g_trace[i * 4 + 2] = gtime();
      commit_pred(&in_empty[b], elected);   // input buffer free once these MMAs retire
      commit_pred(&tfull[b], elected);      // accumulators of this image complete
      __syncwarp();
    }
  } else {
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    uint32_t i = 0;
    for (int64_t img = blockIdx.x; img < n_img; img += gridDim.x, ++i) {
      const uint32_t b = i & 1u, ph = (i >> 1) & 1u;
      mbar_wait(&tfull[b], ph);
      tc_fence_after();
      uint8_t *oimg = out + img * P.out_img_bytes;
      for (int mt = 0; mt < P.n_mt; ++mt) {
        const int q = mt * 128 + r;
        const int oy = q / P.W_in, ox = q - oy * P.W_in;
        const bool valid = oy < P.OH && ox < P.OW;
        const uint32_t trow = tmem + b * tcols_img + (uint32_t)(mt * N) + ((uint32_t)(q4 * 32) << 16);
#pragma unroll
        for (int c = 0; c < N; c += 16) {
          uint32_t v[16];
          tmem_ld16(trow + (uint32_t)c, v);
          if (!valid) continue;
          uint32_t pk[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float x = __uint_as_float(v[2 * e]) + sbias[c + 2 * e];
            const float y = __uint_as_float(v[2 * e + 1]) + sbias[c + 2 * e + 1];
            __nv_bfloat162 hh = __floats2bfloat162_rn(x > 0.0f ? x : 0.0f, y > 0.0f ? y : 0.0f);
            pk[e] = *(uint32_t *)&hh;
          }
          // channels c..c+15 = two 8-channel chunks
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint4 val = make_uint4(pk[4 * h], pk[4 * h + 1], pk[4 * h + 2], pk[4 * h + 3]);
            const int ch = c + 8 * h;           // first channel of this chunk
            uint8_t *dst;
            if (P.out_mode == 0) {              // conv2's s2d(2) input (32 ch -> chunk sub*4 + ch/8)
              const int sub = ((oy & 1) << 1) | (ox & 1);
              const int row = (oy >> 1) * P.out_w + (ox >> 1);
              dst = oimg + act_off(P.layout, P.out_plane, row, sub * 4 + (ch >> 3));
            } else if (P.out_mode == 1) {       // conv3's input
              const int row = oy * P.out_w + ox;
              dst = oimg + act_off(P.layout, P.out_plane, row, ch >> 3);
            } else {                            // fc input: dense [(y, x)][64]
              dst = oimg + ((size_t)(oy * P.out_w + ox) * N + ch) * 2;
            }
            *(uint4 *)dst = val;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[b]);
      if (g_trace && P.out_mode == g_trace_sel && blockIdx.x == 0 && i < 64 && r == 0) g_trace[i * 4 + 3] = gtime();
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols));
  }
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <class G>
void launch_n(const ConvSW &P, const Layer &L, const void *in, int64_t n_img, void *out, cudaStream_t st) {
  constexpr int N = G::N;
  const int smem = (P.K / 64) * N * 128 + 2 * (int)((P.in_img_bytes + 1023u) & ~1023u) + 1024;
  static int attr_for = 0;
  if (attr_for < smem) {
    cudaFuncSetAttribute(k_conv_sw<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_for = smem;
  }
  const int grid = (int)std::min<int64_t>(n_img, num_sms());
  k_conv_sw<G><<<grid, kThreads, smem, st>>>(P, P.wsw, L.bias, (const uint8_t *)in, n_img, (uint8_t *)out);
}

}  // namespace

void conv_trace_set(unsigned long long *p, int sel) {
  cudaMemcpyToSymbol(g_trace, &p, sizeof(p));
  cudaMemcpyToSymbol(g_trace_sel, &sel, sizeof(sel));
}

void launch_conv_sw(const ConvSW &P, const Layer &L, const void *in, int64_t n_img, void *out, cudaStream_t st) {
  if (n_img <= 0) return;
  // the MMA loop is compile-time unrolled per trunk layer (SW128 activations)
  if (P.N == 32) launch_n<G1>(P, L, in, n_img, out, st);
  else if (P.Cin == 128) launch_n<G2>(P, L, in, n_img, out, st);
  else launch_n<G3>(P, L, in, n_img, out, st);
}

}  // namespace bcts
