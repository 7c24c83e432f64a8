// qnet_tma.cu -- K2 layers whose A operand is a plain TMA load:
//   * fc layers: A = activations [M][K] (2-D tiled TMA, 128 rows x 64 bf16);
//   * conv2 / conv3: A = im2col of an NHWC activation tensor (4-D im2col TMA:
//     one load per (M tile, filter tap) brings 128 output pixels x C channels;
//     the filter tap is the TMA im2col offset), i.e. implicit GEMM with the
//     gather done by the TMA engine instead of by threads.
// B (weights [Npad][K], K-major) streams per k-block with 2-D tiled TMA.
//
// Warp roles (192 threads, persistent over tiles):
//   warp 0     : TMA producer (one elected thread), kStages-deep smem ring
//   warp 1     : TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5  : epilogue (TMEM -> registers -> bias/ReLU/bf16 -> global),
//                double-buffered TMEM accumulator so it overlaps the next tile.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "engine.h"
#include "ptx.cuh"

namespace bcts {
namespace {


__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(dst),
      "l"(map), "r"(x), "r"(y), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ void tma_im2col_4d(uint32_t dst, const CUtensorMap *map, int c, int w, int h, int n,
                                              uint16_t off_w, uint16_t off_h, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(map), "r"(saddr(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(off_w), "h"(off_h)
      : "memory");
}

// tcgen05 shared-memory descriptor, K-major with 128B (KB=64) or 64B (KB=32) swizzle.
template <int KB>
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8 * KB * 2) >> 4) << 32;      // SBO: 8 rows x row bytes
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(KB == 64 ? 2 : 4) << 61;       // SWIZZLE_128B / SWIZZLE_64B
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// warp-uniform issue, elected lane predicated (see qnet_conv.cu / tools/mma_bench.cu)

constexpr int kBM = 128;
constexpr int kThreads = 192;

template <int BN, int KB>
struct TmaCfg {
  static constexpr int A_BYTES = kBM * KB * 2;
  static constexpr int B_BYTES = BN * KB * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE > 8 ? 8 : (200 * 1024) / STAGE;
  static constexpr uint32_t TCOLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int SMEM = STAGES * STAGE + 1024;
};

// Geometry the producer needs per layer (passed by value).
struct TmaGeom {
  int im2col;      // 0: 2-D tiled A, 1: 4-D im2col A
  int OH, OW, S;   // conv output geometry and stride (im2col)
  int KW, C;       // filter width and channels (im2col k-block -> (ky, kx, c0))
};

template <int BN, int KB>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_tma(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, Layer L,
               TmaGeom G, int64_t M, void *__restrict__ out, int n_m, int n_n, uint32_t a_bytes) {
  // a_bytes: bytes of A one k-block brings (C::A_BYTES; less for the small-M maps, whose
  // 32-row boxes fill only the first rows of the 128-row tile -- the other rows' outputs
  // are never stored, and every output row depends only on its own A row)
  using C = TmaCfg<BN, KB>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base, derived from smem_raw by an OFFSET so the compiler keeps the
  // shared address space (a uintptr_t round trip turns every access into a generic LD/ST)
  uint8_t *smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[C::STAGES], empty[C::STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const int nk = L.K / KB;
  const int n_tiles = n_m * n_n;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_slot)),
                 "r"(C::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();      // A operand = the previous kernel's output (PDL)
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      const int rows = G.OH * G.OW;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int mt = tile / n_n, ntile = tile - mt * n_n;
        const int64_t m0 = (int64_t)mt * kBM;
        int img = 0, oy = 0, ox = 0;
        if (G.im2col) {
          img = (int)(m0 / rows);
          const int pos = (int)(m0 - (int64_t)img * rows);
          oy = pos / G.OW;
          ox = pos - oy * G.OW;
        }
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % C::STAGES;
          const uint32_t ph = (it / C::STAGES) & 1u;
          mbar_wait_spin(&empty[s], ph ^ 1u);
          const uint32_t sa = saddr(smem + s * C::STAGE);
          mbar_expect_tx(&full[s], a_bytes + C::B_BYTES);
          if (G.im2col) {
            const int k0 = kb * KB;
            const int kwc = G.KW * G.C;
            const int ky = k0 / kwc, r = k0 - ky * kwc;
            const int kx = r / G.C, c0 = r - kx * G.C;
            tma_im2col_4d(sa, &mapA, c0, ox * G.S, oy * G.S, img, (uint16_t)kx, (uint16_t)ky, &full[s]);
          } else {
            tma_2d(sa, &mapA, kb * KB, (int)m0, &full[s]);
          }
          tma_2d(sa + C::A_BYTES, &mapB, kb * KB, ntile * BN, &full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // MMA issuer: whole warp runs the loop, the elected lane's MMAs are predicated on
    const uint32_t elected = elect_one();
    uint32_t it = 0, acc_it = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++acc_it) {
      const int ntile = tile % n_n;
      const int nt = min(BN, L.Npad - ntile * BN);
      const uint32_t idesc = idesc_bf16(kBM, nt);
      const uint32_t a = acc_it & 1u, aph = (acc_it >> 1) & 1u;
      mbar_wait_spin(&tempty[a], aph ^ 1u);
      tc_fence_after();
      const uint32_t d = tmem + a * BN;
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = it % C::STAGES;
        const uint32_t ph = (it / C::STAGES) & 1u;
        mbar_wait_spin(&full[s], ph);
        tc_fence_after();
        const uint32_t a0 = saddr(smem + s * C::STAGE), b0 = a0 + C::A_BYTES;
        const uint64_t ad = sdesc<KB>(a0), bd = sdesc<KB>(b0);
#pragma unroll
        for (int kk = 0; kk < KB / 16; ++kk)   // +32 B per 16 elements inside the swizzle row
          mma_pred(d, ad + (uint64_t)(2 * kk), bd + (uint64_t)(2 * kk), idesc, (kb | kk) != 0, elected);
        commit_pred(&empty[s], elected);
      }
      commit_pred(&tfull[a], elected);
      __syncwarp();
    }
  } else {
    const int q = warp & 3;
    const int r = q * 32 + lane;
    uint32_t acc_it = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++acc_it) {
      const int mt = tile / n_n, ntile = tile - mt * n_n;
      const int64_t m = (int64_t)mt * kBM + r;
      const int n0 = ntile * BN;
      const int nt = min(BN, L.Npad - n0);
      const uint32_t a = acc_it & 1u, aph = (acc_it >> 1) & 1u;
      mbar_wait_spin(&tfull[a], aph);
      tc_fence_after();
      const uint32_t trow = tmem + a * BN + ((uint32_t)(q * 32) << 16);
      for (int c = 0; c < nt; c += 16) {
        uint32_t v[16];
        tmem_ld16(trow + (uint32_t)c, v);
        if (m >= M) continue;
        const float *bias = L.bias + n0 + c;
        if (L.relu_bf16) {
          uint32_t pk[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float x = __uint_as_float(v[2 * i]) + __ldg(bias + 2 * i);
            const float y = __uint_as_float(v[2 * i + 1]) + __ldg(bias + 2 * i + 1);
            __nv_bfloat162 hh = __floats2bfloat162_rn(x > 0.0f ? x : 0.0f, y > 0.0f ? y : 0.0f);
            pk[i] = *(uint32_t *)&hh;
          }
          uint4 *dst = (uint4 *)((__nv_bfloat16 *)out + m * L.out_ld + n0 + c);
          dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        } else {
          float4 *dst = (float4 *)((float *)out + m * L.out_ld + n0 + c);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_float4(__uint_as_float(v[4 * i]) + __ldg(bias + 4 * i),
                                 __uint_as_float(v[4 * i + 1]) + __ldg(bias + 4 * i + 1),
                                 __uint_as_float(v[4 * i + 2]) + __ldg(bias + 4 * i + 2),
                                 __uint_as_float(v[4 * i + 3]) + __ldg(bias + 4 * i + 3));
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[a]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TCOLS));
  }
}

// ============================================== fc GEMM with B multicast over a CTA pair
// out[m][n] = act(A[m][:] . W[n][:] + b[n]) for the fc layers (2-D TMA A), persistent over
// pair-tiles (M-tiles 2pm, 2pm+1) x (N-tile nt): the two CTAs of a cluster take the two
// M-tiles and the SAME N-tile, so each weight k-block is fetched from L2 once and
// TMA-multicast into both CTAs' shared memory (the fc GEMMs are L2-bandwidth bound on
// re-reading W for every M-tile). MMAs stay cta_group::1. Slot reuse needs both CTAs'
// consumers: each MMA commit is multicast to the empty barrier of both CTAs (count 2).
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_2d_mc(uint32_t dst, const CUtensorMap *map, int x, int y, uint64_t *bar,
                                          uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(map), "r"(x), "r"(y), "r"(saddr(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void commit_mc_pred(uint64_t *bar, uint16_t mask, uint32_t issue) {
  asm volatile(
      "{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n"
      "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::
          "r"(saddr(bar)),
      "h"(mask), "r"(issue)
      : "memory");
}

template <int BN, int KB>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_mc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, Layer L,
              int64_t M, void *__restrict__ out, int n_pm, int n_n) {
  using C = TmaCfg<BN, KB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[C::STAGES], empty[C::STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int nk = L.K / KB;
  const int n_tiles = n_pm * n_n;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);   // both CTAs' MMAs must release a slot (B lands in both)
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_slot)),
                 "r"(C::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();          // barriers of both CTAs initialised before any multicast
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {   // ------------------------------------------------ producer
      uint32_t it = 0;
      for (int tile = cl; tile < n_tiles; tile += ncl) {
        const int pm = tile / n_n, nt = tile - pm * n_n;
        const int m0 = (2 * pm + (int)rank) * kBM;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % C::STAGES;
          mbar_wait_spin(&empty[s], ((it / C::STAGES) & 1u) ^ 1u);
          const uint32_t sa = saddr(smem + s * C::STAGE);
          mbar_expect_tx(&full[s], C::STAGE);             // own A + the multicast B
          tma_2d(sa, &mapA, kb * KB, m0, &full[s]);
          if (rank == 0) tma_2d_mc(sa + C::A_BYTES, &mapB, kb * KB, nt * BN, &full[s], (uint16_t)3);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {   // ------------------------------------------ MMA issuer
    const uint32_t elected = elect_one();
    uint32_t it = 0, acc_it = 0;
    for (int tile = cl; tile < n_tiles; tile += ncl, ++acc_it) {
      const int nt = tile % n_n;
      const int ntn = min(BN, L.Npad - nt * BN);
      const uint32_t idesc = idesc_bf16(kBM, ntn);
      const uint32_t a = acc_it & 1u, aph = (acc_it >> 1) & 1u;
      mbar_wait_spin(&tempty[a], aph ^ 1u);
      tc_fence_after();
      const uint32_t d = tmem + a * BN;
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = it % C::STAGES;
        mbar_wait_spin(&full[s], (it / C::STAGES) & 1u);
        tc_fence_after();
        const uint32_t a0 = saddr(smem + s * C::STAGE), b0 = a0 + C::A_BYTES;
        const uint64_t ad = sdesc<KB>(a0), bd = sdesc<KB>(b0);
#pragma unroll
        for (int kk = 0; kk < KB / 16; ++kk)
          mma_pred(d, ad + (uint64_t)(2 * kk), bd + (uint64_t)(2 * kk), idesc, (kb | kk) != 0, elected);
        commit_mc_pred(&empty[s], (uint16_t)3, elected);   // release the slot in both CTAs
      }
      commit_pred(&tfull[a], elected);
      __syncwarp();
    }
  } else {   // ---------------------------------------------------------- epilogue
    const int q = warp & 3;
    const int r = q * 32 + lane;
    uint32_t acc_it = 0;
    for (int tile = cl; tile < n_tiles; tile += ncl, ++acc_it) {
      const int pm = tile / n_n, nt = tile - pm * n_n;
      const int64_t m = (int64_t)(2 * pm + (int)rank) * kBM + r;
      const int n0 = nt * BN;
      const int ntn = min(BN, L.Npad - n0);
      const uint32_t a = acc_it & 1u, aph = (acc_it >> 1) & 1u;
      mbar_wait_spin(&tfull[a], aph);
      tc_fence_after();
      const uint32_t trow = tmem + a * BN + ((uint32_t)(q * 32) << 16);
      for (int c = 0; c < ntn; c += 16) {
        uint32_t v[16];
        tmem_ld16(trow + (uint32_t)c, v);
        if (m >= M) continue;
        const float *bias = L.bias + n0 + c;
        uint32_t pk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float x = __uint_as_float(v[2 * i]) + __ldg(bias + 2 * i);
          const float y = __uint_as_float(v[2 * i + 1]) + __ldg(bias + 2 * i + 1);
          __nv_bfloat162 hh = __floats2bfloat162_rn(x > 0.0f ? x : 0.0f, y > 0.0f ? y : 0.0f);
          pk[i] = *(uint32_t *)&hh;
        }
        uint4 *dst = (uint4 *)((__nv_bfloat16 *)out + m * L.out_ld + n0 + c);
        dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
      tc_fence_before();
      mbar_arrive(&tempty[a]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TCOLS));
  }
  cluster_sync_all();          // no CTA leaves while its peer may still multicast into it
}

// =========================================== fc GEMM on a CTA pair with the 2-SM MMA
// tcgen05.mma.cta_group::2, M = 256 (128 rows per CTA) x N = 256 (B split along N: CTA r holds
// weight rows nt*256 + 128r .. +127), issued by the leader (cluster rank 0); each CTA's TMEM
// receives its own 128 rows x all 256 columns (semantics checked in tools/mma2sm_test.cu).
// Per SM a k-block brings A 16 KB + B 16 KB instead of 16 + 32 KB: the fc GEMM is bound by
// per-SM operand ingest, which this halves for B. Cross-CTA signalling: both CTAs' TMA loads
// (the .cta_group::2 form) complete on the LEADER's full barrier, armed by the leader with both
// halves' bytes; the leader's commits multicast to both CTAs' empty / tfull barriers; the
// peer's epilogue threads arrive remotely on the leader's tempty barrier. (A first version that
// forwarded the peer's fills through its idle MMA warp ran 2.5x slower: that hop sat on the
// critical path of every stage.)
constexpr int k2smStages = 6, k2smStage = 32768;
constexpr int k2smSmem = k2smStages * k2smStage + 1024;
__device__ __forceinline__ uint32_t mapa_rank0(uint32_t local_saddr) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(local_saddr));
  return r;
}
// 2-D TMA load into this CTA's smem whose completion is counted on a barrier of the CTA pair
// (here: the leader's), the .cta_group::2 form (SASS UTMALDG.2D.2CTA)
__device__ __forceinline__ void tma_2d_2cta(uint32_t dst, const CUtensorMap *map, int x, int y, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(x), "r"(y), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_2sm(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, Layer L,
               int64_t M, void *__restrict__ out, int n_pm, int n_n) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[k2smStages], empty[k2smStages], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int nk = L.K / 64;
  const int n_tiles = n_pm * n_n;
  if (threadIdx.x == 0) {
    for (int s = 0; s < k2smStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 256);   // both CTAs' epilogue threads (leader's barrier is the one used)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {   // -------------------- producer: own halves, completing on the LEADER's barrier
      uint32_t it = 0;
      const uint32_t full0 = mapa_rank0(saddr(&full[0]));
      for (int tile = cl; tile < n_tiles; tile += ncl) {
        const int pm = tile / n_n, nt = tile - pm * n_n;
        const int m0 = pm * 256 + (int)rank * kBM, n0 = nt * 256 + (int)rank * 128;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % k2smStages;
          mbar_wait_spin(&empty[s], ((it / k2smStages) & 1u) ^ 1u);
          const uint32_t sa = saddr(smem + s * k2smStage);
          if (rank == 0) mbar_expect_tx(&full[s], 2 * k2smStage);   // both CTAs' bytes land on this barrier
          tma_2d_2cta(sa, &mapA, kb * 64, m0, full0 + (uint32_t)s * 8u);
          tma_2d_2cta(sa + 16384, &mapB, kb * 64, n0, full0 + (uint32_t)s * 8u);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (rank == 0) {   // --------------------------------------------- MMA issuer (leader)
      const uint32_t elected = elect_one();
      const uint32_t idesc = idesc_bf16(256, 256);
      uint32_t it = 0, acc_it = 0;
      for (int tile = cl; tile < n_tiles; tile += ncl, ++acc_it) {
        const uint32_t a = acc_it & 1u, aph = (acc_it >> 1) & 1u;
        mbar_wait_spin(&tempty[a], aph ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + a * 256;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % k2smStages;
          const uint32_t ph = (it / k2smStages) & 1u;
          mbar_wait_spin(&full[s], ph);
          tc_fence_after();
          const uint32_t a0 = saddr(smem + s * k2smStage), b0 = a0 + 16384;
          const uint64_t ad = sdesc<64>(a0), bd = sdesc<64>(b0);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            asm volatile(
                "{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nsetp.ne.b32 q, %5, 0;\n"
                "@q tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                "l"(ad + (uint64_t)(2 * kk)), "l"(bd + (uint64_t)(2 * kk)), "r"(idesc), "r"((kb | kk) != 0 ? 1u : 0u),
                "r"(elected));
          }
          asm volatile(
              "{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n"
              "@q tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::
                  "r"(saddr(&empty[s])),
              "h"((uint16_t)3), "r"(elected)
              : "memory");
        }
        asm volatile(
            "{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n"
            "@q tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::
                "r"(saddr(&tfull[a])),
            "h"((uint16_t)3), "r"(elected)
            : "memory");
        __syncwarp();
      }
    }
    __syncwarp();
  } else {   // ---------------------------------------------------------- epilogue (own 128 rows)
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t tempty0 = mapa_rank0(saddr(&tempty[0]));
    uint32_t acc_it = 0;
    for (int tile = cl; tile < n_tiles; tile += ncl, ++acc_it) {
      const int pm = tile / n_n, nt = tile - pm * n_n;
      const int64_t m = (int64_t)pm * 256 + (int64_t)rank * kBM + r;
      const int n0 = nt * 256;
      const uint32_t a = acc_it & 1u, aph = (acc_it >> 1) & 1u;
      mbar_wait_spin(&tfull[a], aph);
      tc_fence_after();
      const uint32_t trow = tmem + a * 256 + ((uint32_t)(q * 32) << 16);
      for (int c = 0; c < 256; c += 16) {
        uint32_t v[16];
        tmem_ld16(trow + (uint32_t)c, v);
        if (m >= M) continue;
        const float *bias = L.bias + n0 + c;
        uint32_t pk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float x = __uint_as_float(v[2 * i]) + __ldg(bias + 2 * i);
          const float y = __uint_as_float(v[2 * i + 1]) + __ldg(bias + 2 * i + 1);
          __nv_bfloat162 hh = __floats2bfloat162_rn(x > 0.0f ? x : 0.0f, y > 0.0f ? y : 0.0f);
          pk[i] = *(uint32_t *)&hh;
        }
        uint4 *dst = (uint4 *)((__nv_bfloat16 *)out + m * L.out_ld + n0 + c);
        dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
      tc_fence_before();
      mbar_arrive_remote(tempty0 + a * 8u);   // the leader's accumulator may be reused
    }
  }
  __syncthreads();
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// =============================================================== fused Rainbow head
// z_v, z_a and the dueling C51 head in ONE kernel (the 4-byte logits never reach
// HBM). Per 128-leaf tile, jobs (each a K = 512 GEMM into a 256-column TMEM buffer):
//   job v     : z_v = h_v W_v^T + b_v (N = 64, 51 atoms)
//   job mean  : S = h_a (sum_a W_a)^T (N = 64): the action-sum of the advantage logits
//               by linearity; sum_a W_a is carried as a bf16 hi + lo pair (K = 1024
//               over [h_a; h_a]), i.e. to ~2^-16 relative, and sum_a b_a is added in
//               fp32 -> mean_t = (S_t + sum_a b_a,t) / A.
//   chunk c   : z_a for actions 4c..4c+3 (51 TMEM columns per action, packed: N = 208 for
//               4 actions, the weights streamed as kHeadChunkRows-row boxes) -> logits =
//               (v - mean) + z_a -> softmax expectation -> max_a.
// h_a (128 KB) stays resident in SMEM; h_v and the weight k-blocks stream through a
// 3-stage ring. TMEM: two 256-column accumulators, alternating by job parity.
constexpr int kHeadStages = 3, kHeadSlot = 32768, kHeadA = 8 * 16384;
constexpr int kHeadThreads = 320;   // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue (2 groups)
constexpr int kHeadSmem = kHeadA + kHeadStages * kHeadSlot + 1024;

__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, uint32_t *r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// 64 columns (one action, z_v or S) of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t (&r)[64]) {
  tmem_ld32_nw(taddr, r);
  tmem_ld32_nw(taddr + 32, r + 32);
  tmem_wait_ld();
}

// (Round-1 timing experiments: with every part switched off but the TMA ring the
// C5 52K-leaf launch still took ~70 of ~80 us, T(stages) = 37 + 102 / stages us -- the weight ring
// beside the 128 KB resident h_a bounds it.)
template <int ATOMS>
__global__ void __launch_bounds__(kHeadThreads, 1)
    k_zhead(const __grid_constant__ CUtensorMap mapAv, const __grid_constant__ CUtensorMap mapAa,
            const __grid_constant__ CUtensorMap mapBv, const __grid_constant__ CUtensorMap mapBa,
            const __grid_constant__ CUtensorMap mapBs, const __grid_constant__ HeadBias hb, int A, int64_t M, float vmin,
            float dz, int mode, float gd, const float *__restrict__ cum, float *__restrict__ out, int ns,
            const KeyFold kf, int64_t mrow0, float *__restrict__ rows_out) {
  // rows m >= mrow0 (MODE_TOTAL / ROWMAX batches only) are full-row rows appended to the batch
  // (the finalize prologue's [roots | level-1 children]): Q rows -> rows_out
  // ns: work items per 128-row tile, each taking a contiguous slice of the action chunks
  // (MODE_ROWS only: tiny batches spread their z_a weight stream over ns CTAs; ns = 1 otherwise)
  static_assert(ATOMS * 4 <= kHeadChunkRows && kHeadChunkRows <= 256, "4 actions per z_a chunk");
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  uint8_t *sA = smem, *sRing = smem + kHeadA;
  __shared__ __align__(8) uint64_t full[kHeadStages], empty[kHeadStages], tfull[2], tempty[2], a_full, a_empty;
  __shared__ uint32_t tmem_slot;
  __shared__ float s_best[2][kBM];                   // group 1's max_a, per tile parity
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const int n_m = (int)((M + kBM - 1) / kBM);
  const int nch = (A + 3) / 4;                       // z_a chunks of 4 actions (256 columns)
  const int cpc = (nch + ns - 1) / ns, n_work = n_m * ns;
  constexpr int nst = kHeadStages;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kHeadStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 256);
    }
    mbar_init(&a_full, 1);
    mbar_init(&a_empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();      // A operand = the previous kernel's output (PDL)
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {   // ------------------------------------------------ TMA producer
      uint32_t it = 0, tl = 0;
      auto slot_wait = [&](uint32_t bytes) {
        const int st = it % nst;
        mbar_wait_spin(&empty[st], ((it / nst) & 1u) ^ 1u);
        mbar_expect_tx(&full[st], bytes);
        return st;
      };
      for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++tl) {
        const int tile = w / ns, c_lo = (w - tile * ns) * cpc, c_hi = min(nch, c_lo + cpc);
        const int m0 = tile * kBM;
        for (int kb = 0; kb < 8; ++kb, ++it) {     // job v: h_v and W_v k-blocks through the ring
          const int st = slot_wait(16384 + 8192);
          const uint32_t slot = saddr(sRing + st * kHeadSlot);
          tma_2d(slot, &mapAv, kb * 64, m0, &full[st]);
          tma_2d(slot + 16384, &mapBv, kb * 64, 0, &full[st]);
        }
        mbar_wait_spin(&a_empty, (tl & 1u) ^ 1u);      // previous tile's MMAs are done with sA
        mbar_expect_tx(&a_full, kHeadA);
        for (int kb = 0; kb < 8; ++kb) tma_2d(saddr(sA + kb * 16384), &mapAa, kb * 64, m0, &a_full);
        for (int kb = 0; kb < 16; ++kb, ++it) {    // job mean: hi (rows 0..63) then lo (64..127)
          const int st = slot_wait(8192);
          tma_2d(saddr(sRing + st * kHeadSlot), &mapBs, (kb & 7) * 64, (kb >> 3) * 64, &full[st]);
        }
        for (int c = c_lo; c < c_hi; ++c)
          for (int kb = 0; kb < 8; ++kb, ++it) {
            const int st = slot_wait(kHeadChunkRows * 128);
            tma_2d(saddr(sRing + st * kHeadSlot), &mapBa, kb * 64, c * kHeadChunkRows, &full[st]);
          }
      }
    }
    __syncwarp();
  } else if (warp == 1) {   // ------------------------------------------ MMA issuer
    const uint32_t elected = elect_one();
    uint32_t it = 0, job = 0, tl = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++tl) {
      const int tile = w / ns, c_lo = (w - tile * ns) * cpc, c_hi = min(nch, c_lo + cpc);
      (void)tile;
      for (int j = 0; j < c_hi - c_lo + 2; ++j, ++job) {   // v, mean, chunks
        const uint32_t b = job & 1u;
        mbar_wait_spin(&tempty[b], ((job >> 1) & 1u) ^ 1u);
        tc_fence_after();
        if (j == 1) {
          mbar_wait_spin(&a_full, tl & 1u);
          tc_fence_after();
        }
        const int c = c_lo + j - 2;
        const int nt = j < 2 ? 64 : (min(4, A - 4 * c) * ATOMS + 15) / 16 * 16;   // 208 for 4 actions
        const uint32_t idesc = idesc_bf16(kBM, nt);
        const int nkb = j == 1 ? 16 : 8;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int st = it % nst;
          mbar_wait_spin(&full[st], (it / nst) & 1u);
          tc_fence_after();
          const uint32_t slot = saddr(sRing + st * kHeadSlot);
          const uint64_t ad = sdesc<64>(j == 0 ? slot : saddr(sA + (kb & 7) * 16384));
          const uint64_t bd = sdesc<64>(j == 0 ? slot + 16384 : slot);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_pred(tmem + b * 256, ad + (uint64_t)(2 * kk), bd + (uint64_t)(2 * kk), idesc, (kb | kk) != 0,
                     elected);
          commit_pred(&empty[st], elected);
        }
        commit_pred(&tfull[b], elected);
        __syncwarp();
      }
      commit_pred(&a_empty, elected);   // sA free once this tile's MMAs have completed
      __syncwarp();
    }
  } else {   // ------------------------------- epilogue: 2 groups x 4 warps (lane quarter q = rows)
    // Both groups read v and the action mean; the softmax work is split by action parity
    // (group g takes actions 4c + s with s % 2 == g) and max_a is combined through SMEM.
    const int q = warp & 3, grp = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const uint32_t lanes = (uint32_t)(q * 32) << 16;
    uint32_t job = 0, tl = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++tl) {
      const int tile = w / ns, c_lo = (w - tile * ns) * cpc, c_hi = min(nch, c_lo + cpc);
      const int64_t m = (int64_t)tile * kBM + r;
      float v[ATOMS];
      uint32_t x[64];
      {   // job v
        const uint32_t b = job & 1u;
        mbar_wait_spin(&tfull[b], (job >> 1) & 1u);
        tc_fence_after();
        tmem_ld64(tmem + b * 256 + lanes, x);
        tc_fence_before();
        mbar_arrive(&tempty[b]);
        ++job;
#pragma unroll
        for (int t = 0; t < ATOMS; ++t) v[t] = __uint_as_float(x[t]) + hb.v[t];
      }
      {   // job mean: v_t - mean_a adv[a][t]
        const uint32_t b = job & 1u;
        mbar_wait_spin(&tfull[b], (job >> 1) & 1u);
        tc_fence_after();
        tmem_ld64(tmem + b * 256 + lanes, x);
        tc_fence_before();
        mbar_arrive(&tempty[b]);
        ++job;
#pragma unroll
        for (int t = 0; t < ATOMS; ++t) v[t] = v[t] - (__uint_as_float(x[t]) + hb.sum[t]) / (float)A;
      }
      float best = -INFINITY;
      for (int c = c_lo; c < c_hi; ++c, ++job) {   // softmax expectation per action
        const uint32_t b = job & 1u;
        mbar_wait_spin(&tfull[b], (job >> 1) & 1u);
        tc_fence_after();
        const int na = min(4, A - 4 * c);
        for (int s = grp; s < na; s += 2) {
          tmem_ld64(tmem + b * 256 + lanes + (uint32_t)(s * ATOMS), x);   // action s: columns 51 s ..
          const int a = 4 * c + s;
          float mx = -INFINITY;
#pragma unroll
          for (int t = 0; t < ATOMS; ++t) {
            x[t] = __float_as_uint(v[t] + (__uint_as_float(x[t]) + hb.a64[a * 64 + t]));   // logit
            mx = fmaxf(mx, __uint_as_float(x[t]));
          }
          // exp(l - max) = 2^(l log2e - max log2e): one FFMA + MUFU.EX2 per atom (expf's range
          // reduction is ~5 more instructions; the epilogue's issue rate bounds this kernel)
          const float mxs = mx * 1.4426950408889634f;
          float den = 0.0f, num = 0.0f;
#pragma unroll
          for (int t = 0; t < ATOMS; ++t) {
            float ex;
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ex) : "f"(fmaf(__uint_as_float(x[t]), 1.4426950408889634f, -mxs)));
            den += ex;
            num = fmaf(hb.z[t], ex, num);   // support z_t = v_min + t dz (constant bank)
          }
          const float qa = num / den;
          if (mode == MODE_ROWS && m < M) out[m * A + a] = qa;
          else if (m >= mrow0 && m < M) rows_out[(m - mrow0) * A + a] = qa;
          best = fmaxf(best, qa);
        }
        tc_fence_before();
        mbar_arrive(&tempty[b]);
      }
      if (mode != MODE_ROWS) {   // max_a over both groups (max is order-independent)
        if (grp == 1) s_best[tl & 1u][r] = best;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (grp == 0) {
          int64_t key = kKeyEmpty, slot = -1;
          if (m < M && m < mrow0) {
            best = fmaxf(best, s_best[tl & 1u][r]);
            const float tot = mode == MODE_ROWMAX ? best : fmaf(gd, best, cum ? cum[m] : 0.0f);
            out[m] = tot;
            if (kf.keys) {   // fused backup (same fold as k_segmax)
              const int64_t L = kf.leaf0 + m, root = L / kf.lpr, within = L - root * kf.lpr;
              slot = root * kf.A + within / kf.seg;
              key = pack_key(tot, within);
            }
          }
          if (kf.keys) {
            const int64_t s0 = __shfl_sync(0xffffffffu, slot, 0);
            if (__all_sync(0xffffffffu, slot == s0 || slot < 0)) {
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) {
                const int64_t other = __shfl_xor_sync(0xffffffffu, key, o);
                key = other > key ? other : key;
              }
              if (lane == 0 && s0 >= 0) atomicMax((long long *)&kf.keys[s0], (long long)key);
            } else if (slot >= 0) {
              atomicMax((long long *)&kf.keys[slot], (long long)key);
            }
          }
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode_tiled = nullptr;
PFN_cuTensorMapEncodeIm2col_v12000 g_encode_im2col = nullptr;

bool load_driver() {
  if (g_encode_tiled && g_encode_im2col) return true;
  cudaDriverEntryPointQueryResult q;
  void *f = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess || !f) return false;
  g_encode_tiled = (PFN_cuTensorMapEncodeTiled_v12000)f;
  f = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &q) != cudaSuccess || !f)
    return false;
  g_encode_im2col = (PFN_cuTensorMapEncodeIm2col_v12000)f;
  return true;
}

int num_sms() { return sm_count_current(); }

// fc layer with ReLU + bf16 output (fc_hidden): the B-multicast pair kernel
template <int BN, int KB>
bool launch_gemm_mc(const TmaPlan &P, const Layer &L, int64_t M, void *out, cudaStream_t st) {
  using C = TmaCfg<BN, KB>;
  smem_optin((const void *)k_gemm_mc<BN, KB>, C::SMEM);
  const int n_m = (int)((M + kBM - 1) / kBM), n_pm = (n_m + 1) / 2, n_n = (L.Npad + BN - 1) / BN;
  const int n_cl = std::min(n_pm * n_n, num_sms() / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * n_cl);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k_gemm_mc<BN, KB>, *(const CUtensorMap *)P.mapA, *(const CUtensorMap *)P.mapB, L, M,
                            out, n_pm, n_n) == cudaSuccess;
}

// fc layer (ReLU + bf16) on CTA pairs with the 2-SM MMA; needs B tensor map boxes of 128 rows
bool launch_gemm_2sm(const TmaPlan &P, const Layer &L, int64_t M, void *out, cudaStream_t st) {
  if (!P.ok2sm) return false;
  smem_optin((const void *)k_gemm_2sm, k2smSmem);
  const int n_m = (int)((M + kBM - 1) / kBM), n_pm = (n_m + 1) / 2, n_n = L.Npad / 256;
  const int n_cl = std::min(n_pm * n_n, num_sms() / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * n_cl);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = k2smSmem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k_gemm_2sm, *(const CUtensorMap *)P.mapA, *(const CUtensorMap *)P.mapB2, L, M, out,
                            n_pm, n_n) == cudaSuccess;
}

void launch_gemm_small(const TmaPlan &P, const Layer &L, int64_t M, void *out, cudaStream_t st);

template <int BN, int KB>
void launch_gemm(const TmaPlan &P, const Layer &L, int64_t M, void *out, cudaStream_t st) {
  if (P.ok_small && M <= kSmallM && KB == 64 && !P.im2col) {
    launch_gemm_small(P, L, M, out, st);
    return;
  }
  // one kernel per shape, chosen by eligibility (a failed launch stays pending for the caller's
  // cuda_check; nothing falls back silently): CTA pairs for the wide fc_hidden, otherwise the
  // cluster-multicast kernel for N-multiple-of-256 layers, otherwise the plain TMA GEMM
  if (!P.im2col && L.relu_bf16 && BN == 256 && KB == 64 && L.Npad % 256 == 0) {
    launch_gemm_2sm(P, L, M, out, st);
    return;
  }
  if (!P.im2col && L.relu_bf16 && BN == 256 && L.Npad % BN == 0) {
    launch_gemm_mc<BN, KB>(P, L, M, out, st);
    return;
  }
  using C = TmaCfg<BN, KB>;
  smem_optin((const void *)k_gemm_tma<BN, KB>, C::SMEM);
  const int n_m = (int)((M + kBM - 1) / kBM), n_n = (L.Npad + BN - 1) / BN;
  const int grid = (int)std::min<int64_t>((int64_t)n_m * n_n, num_sms());
  TmaGeom G{P.im2col, L.OH, L.OW, L.S, L.KW, L.C};
  launch_pdl(k_gemm_tma<BN, KB>, dim3(grid), dim3(kThreads), (size_t)C::SMEM, st, *(const CUtensorMap *)P.mapA,
             *(const CUtensorMap *)P.mapB, L, G, M, out, n_m, n_n, (uint32_t)C::A_BYTES);
}

// Tiny fc batches (M <= 32 rows: the prologue's [roots | level-1 children] at one root) are
// latency-bound streams of the weights: 32-column N tiles put them on Npad/32 SMs and 32-row
// A boxes stop every CTA from fetching 128 rows of A (~4 KB + 4 KB per k-block and CTA).
void launch_gemm_small(const TmaPlan &P, const Layer &L, int64_t M, void *out, cudaStream_t st) {
  using C = TmaCfg<32, 64>;
  smem_optin((const void *)k_gemm_tma<32, 64>, C::SMEM);
  const int n_n = L.Npad / 32;
  const int grid = std::min(n_n, num_sms());
  TmaGeom G{0, L.OH, L.OW, L.S, L.KW, L.C};
  launch_pdl(k_gemm_tma<32, 64>, dim3(grid), dim3(kThreads), (size_t)C::SMEM, st, *(const CUtensorMap *)P.mapAs,
             *(const CUtensorMap *)P.mapBs, L, G, M, out, 1, n_n, (uint32_t)(kSmallM * 64 * 2));
}

}  // namespace

// Build the A / B tensor maps of a layer whose input is the fixed buffer `in`
// holding up to `cap_img` images. Returns false if the layer cannot use TMA.
bool tma_plan(TmaPlan &P, const Layer &L, const void *in, int64_t cap_img) {
  P.ok = false;
  if (L.in_u8 || L.K % 32 || L.Npad % 16 || !load_driver()) return false;
  const bool conv = !(L.OH == 1 && L.OW == 1 && L.KH == L.H && L.KW == L.W);
  int KB;
  if (conv) {
    if (L.C != 32 && L.C != 64) return false;
    KB = L.C;
  } else {
    KB = 64;
    if (L.K % 64) return false;
  }
  P.kb = KB;
  P.im2col = conv ? 1 : 0;
  P.bn = L.Npad <= 32 ? 32 : L.Npad <= 64 ? 64 : 256;
  const CUtensorMapSwizzle sw = KB == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  CUtensorMap *ma = (CUtensorMap *)P.mapA, *mb = (CUtensorMap *)P.mapB;
  CUresult r;
  if (conv) {
    cuuint64_t dims[4] = {(cuuint64_t)L.C, (cuuint64_t)L.W, (cuuint64_t)L.H, (cuuint64_t)cap_img};
    cuuint64_t strides[3] = {(cuuint64_t)L.C * 2, (cuuint64_t)L.W * L.C * 2, (cuuint64_t)L.in_img_stride * 2};
    int lower[2] = {0, 0};
    int upper[2] = {-(L.KW - 1), -(L.KH - 1)};
    cuuint32_t estr[4] = {1, (cuuint32_t)L.S, (cuuint32_t)L.S, 1};
    r = g_encode_im2col(ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(in), dims, strides, lower, upper,
                        (cuuint32_t)L.C, (cuuint32_t)kBM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[2] = {(cuuint64_t)L.K, (cuuint64_t)cap_img};
    cuuint64_t strides[1] = {(cuuint64_t)L.in_img_stride * 2};
    cuuint32_t box[2] = {(cuuint32_t)KB, (cuuint32_t)kBM};
    cuuint32_t estr[2] = {1, 1};
    r = g_encode_tiled(ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                       const_cast<__nv_bfloat16 *>((const __nv_bfloat16 *)in) + L.in_col_off, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) return false;
  {
    cuuint64_t dims[2] = {(cuuint64_t)L.K, (cuuint64_t)L.Npad};
    cuuint64_t strides[1] = {(cuuint64_t)L.K * 2};
    cuuint32_t box[2] = {(cuuint32_t)KB, (cuuint32_t)P.bn};
    cuuint32_t estr[2] = {1, 1};
    r = g_encode_tiled(mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16 *>(L.Wt), dims, strides, box,
                       estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    P.ok_small = false;
    if (r == CUDA_SUCCESS && !conv && KB == 64 && L.Npad % 32 == 0) {
      // small-M maps: 32-row A boxes (kSmallM) and 32-row B boxes (N tiles of 32)
      cuuint64_t adims[2] = {(cuuint64_t)L.K, (cuuint64_t)cap_img};
      cuuint64_t astr[1] = {(cuuint64_t)L.in_img_stride * 2};
      cuuint32_t abox[2] = {64u, (cuuint32_t)kSmallM}, bbox[2] = {64u, 32u};
      P.ok_small = g_encode_tiled((CUtensorMap *)P.mapAs, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                  const_cast<__nv_bfloat16 *>((const __nv_bfloat16 *)in) + L.in_col_off, adims, astr,
                                  abox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS &&
                   g_encode_tiled((CUtensorMap *)P.mapBs, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                  const_cast<__nv_bfloat16 *>(L.Wt), dims, strides, bbox, estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    P.ok2sm = false;
    if (r == CUDA_SUCCESS && !conv && KB == 64 && L.Npad % 256 == 0) {   // 2-SM GEMM: half-tile B boxes
      cuuint32_t box2[2] = {(cuuint32_t)KB, 128u};
      P.ok2sm = g_encode_tiled((CUtensorMap *)P.mapB2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                               const_cast<__nv_bfloat16 *>(L.Wt), dims, strides, box2, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
  }
  if (r != CUDA_SUCCESS) return false;
  P.ok = true;
  return true;
}

// Fused Rainbow head (k_zhead): maps over the hidden activations (h_v = columns
// 0..511, h_a = 512..1023 of [cap][1024] bf16) and the head weights.
bool head_plan(HeadPlan &H, const __nv_bfloat16 *hid, int64_t cap, const __nv_bfloat16 *wv64,
               const __nv_bfloat16 *wa64, const __nv_bfloat16 *wsum, int A) {
  H.ok = false;
  if (!load_driver()) return false;
  auto enc = [](void *map, const void *base, uint64_t cols, uint64_t rows, uint64_t ld_elems, uint32_t box_rows) {
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld_elems * 2};
    cuuint32_t box[2] = {64u, box_rows};
    cuuint32_t estr[2] = {1, 1};
    return g_encode_tiled((CUtensorMap *)map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  if (!enc(H.mapAv, hid, 512, (uint64_t)cap, 1024, 128) || !enc(H.mapAa, hid + 512, 512, (uint64_t)cap, 1024, 128) ||
      !enc(H.mapBv, wv64, 512, 64, 512, 64) ||
      !enc(H.mapBa, wa64, 512, (uint64_t)((A + 3) / 4) * kHeadChunkRows, 512, kHeadChunkRows) ||
      !enc(H.mapBs, wsum, 512, 128, 512, 64))
    return false;

  H.ok = true;
  return true;
}

void launch_zhead(const HeadPlan &H, int A, int atoms, int64_t M, float vmin, float dz, int mode, float gd,
                  const float *cum, float *out, cudaStream_t st, KeyFold kf, int64_t mrow0, float *rows_out) {
  if (M <= 0 || atoms != 51) return;
  smem_optin((const void *)k_zhead<51>, kHeadSmem);
  const int n_m = (int)((M + kBM - 1) / kBM), nch = (A + 3) / 4;
  // full-row batches smaller than the GPU: split each tile's action chunks over several CTAs
  const int ns = mode == MODE_ROWS ? std::max(1, std::min(nch, num_sms() / n_m)) : 1;
  const int grid = std::min(n_m * ns, num_sms());
  launch_pdl(k_zhead<51>, dim3(grid), dim3(kHeadThreads), (size_t)kHeadSmem, st, *(const CUtensorMap *)H.mapAv,
             *(const CUtensorMap *)H.mapAa, *(const CUtensorMap *)H.mapBv, *(const CUtensorMap *)H.mapBa,
             *(const CUtensorMap *)H.mapBs, H.bias, A, M, vmin, dz, mode, gd, cum, out, ns, kf,
             rows_out ? mrow0 : INT64_MAX, rows_out);
}

void launch_layer_tma(const TmaPlan &P, const Layer &L, int64_t n_img, void *out, cudaStream_t st) {
  const int64_t M = n_img * L.rows_per_img();
  if (M <= 0) return;
  if (P.kb == 32) {
    if (P.bn == 64) launch_gemm<64, 32>(P, L, M, out, st);
    else if (P.bn == 32) launch_gemm<32, 32>(P, L, M, out, st);
    else launch_gemm<256, 32>(P, L, M, out, st);
  } else {
    if (P.bn == 64) launch_gemm<64, 64>(P, L, M, out, st);
    else if (P.bn == 32) launch_gemm<32, 64>(P, L, M, out, st);
    else launch_gemm<256, 64>(P, L, M, out, st);
  }
}

}  // namespace bcts
