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

template <int N>
__global__ void __launch_bounds__(kThreads, 1)
    k_conv_sw(ConvSW P, const __nv_bfloat16 *__restrict__ Wt, const float *__restrict__ bias,
              const uint8_t *__restrict__ in, int64_t n_img, uint8_t *__restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *sW = smem;                                   // K/64 blocks of [N x 128 B], SW128
  const int nkb = P.K / 64;
  uint8_t *sIn0 = smem + (size_t)nkb * N * 128;         // two input-image buffers
  const uint32_t in_stride = (P.in_img_bytes + 1023u) & ~1023u;
  __shared__ __align__(8) uint64_t in_full[2], in_empty[2], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t tcols_img = (uint32_t)(P.n_mt * N);
  uint32_t tcols = 32;
  while (tcols < 2 * tcols_img) tcols <<= 1;

  // resident weights -> SW128 smem (all threads)
  for (int e = threadIdx.x; e < N * nkb * 8; e += kThreads) {
    const int j = e & 7, kb = (e >> 3) % nkb, n = (e >> 3) / nkb;
    const uint4 w = __ldg((const uint4 *)(Wt + (int64_t)n * P.K + (int64_t)kb * 64) + j);
    *(uint4 *)(sW + (size_t)kb * N * 128 + (uint32_t)(n >> 3) * 1024u + (uint32_t)(n & 7) * 128u +
               (uint32_t)((j ^ (n & 7)) << 4)) = w;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&in_full[i], 1);
      mbar_init(&in_empty[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
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
        mbar_expect_tx(&in_full[b], P.in_img_bytes);
        bulk_g2s(saddr(sIn0 + b * in_stride), in + img * (int64_t)P.in_img_bytes, P.in_img_bytes, &in_full[b]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(128, N);
      const int ksteps = P.Cin / 16;
      uint32_t i = 0;
      for (int64_t img = blockIdx.x; img < n_img; img += gridDim.x, ++i) {
        const uint32_t b = i & 1u, ph = (i >> 1) & 1u;
        mbar_wait(&in_full[b], ph);
        mbar_wait(&tempty[b], ph ^ 1u);
        tc_fence_after();
        const uint32_t a_base = saddr(sIn0 + b * in_stride), w_base = saddr(sW);
        for (int mt = 0; mt < P.n_mt; ++mt) {
          const uint32_t d = tmem + b * tcols_img + (uint32_t)(mt * N);
          for (int tap = 0; tap < P.KH * P.KW; ++tap) {
            const int ty = tap / P.KW, tx = tap - ty * P.KW;
            const uint32_t row0 = (uint32_t)(mt * 128 + ty * P.W_in + tx);
            for (int kk = 0; kk < ksteps; ++kk) {
              const uint32_t a = a_base + (uint32_t)(2 * kk) * P.plane + row0 * 16u;
              const int k = tap * P.Cin + 16 * kk;   // weight K index, (tap, c) order
              const uint32_t w = w_base + (uint32_t)(k >> 6) * (N * 128) + (uint32_t)((k & 63) * 2);
              mma_bf16(d, desc_planar(a, P.plane), desc_sw128(w), idesc, (tap | kk) != 0);
            }
          }
        }
        mma_commit(&in_empty[b]);   // input buffer free once these MMAs retire
        mma_commit(&tfull[b]);      // accumulators of this image complete
      }
    }
    __syncwarp();
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
            const float x = __uint_as_float(v[2 * e]) + __ldg(bias + c + 2 * e);
            const float y = __uint_as_float(v[2 * e + 1]) + __ldg(bias + c + 2 * e + 1);
            __nv_bfloat162 hh = __floats2bfloat162_rn(x > 0.0f ? x : 0.0f, y > 0.0f ? y : 0.0f);
            pk[e] = *(uint32_t *)&hh;
          }
          // channels c..c+15 = two 8-channel chunks
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint4 val = make_uint4(pk[4 * h], pk[4 * h + 1], pk[4 * h + 2], pk[4 * h + 3]);
            const int ch = c + 8 * h;           // first channel of this chunk
            uint8_t *dst;
            if (P.out_mode == 0) {              // conv2's s2d(2) planar input (32 ch -> sub*4 + ch/8)
              const int sub = ((oy & 1) << 1) | (ox & 1);
              const int row = (oy >> 1) * P.out_w + (ox >> 1);
              dst = oimg + (size_t)(sub * 4 + (ch >> 3)) * P.out_plane + (size_t)row * 16;
            } else if (P.out_mode == 1) {       // conv3's planar input
              const int row = oy * P.out_w + ox;
              dst = oimg + (size_t)(ch >> 3) * P.out_plane + (size_t)row * 16;
            } else {                            // fc input: dense [(y, x)][64]
              dst = oimg + ((size_t)(oy * P.out_w + ox) * N + ch) * 2;
            }
            *(uint4 *)dst = val;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[b]);
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

template <int N>
void launch_n(const ConvSW &P, const Layer &L, const void *in, int64_t n_img, void *out, cudaStream_t st) {
  const int smem = (P.K / 64) * N * 128 + 2 * (int)((P.in_img_bytes + 1023u) & ~1023u) + 1024;
  static int attr_for = 0;
  if (attr_for < smem) {
    cudaFuncSetAttribute(k_conv_sw<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_for = smem;
  }
  const int grid = (int)std::min<int64_t>(n_img, num_sms());
  k_conv_sw<N><<<grid, kThreads, smem, st>>>(P, L.Wt, L.bias, (const uint8_t *)in, n_img, (uint8_t *)out);
}

}  // namespace

void launch_conv_sw(const ConvSW &P, const Layer &L, const void *in, int64_t n_img, void *out, cudaStream_t st) {
  if (n_img <= 0) return;
  if (P.N == 32) launch_n<32>(P, L, in, n_img, out, st);
  else launch_n<64>(P, L, in, n_img, out, st);
}

}  // namespace bcts
