// K8 on the 5th-generation tensor cores: S = Q X^T with tcgen05.mma
// (kind::tf32, accumulators in TMEM), operands staged by TMA
// (cp.async.bulk.tensor, 128-byte swizzle) through a 4-stage mbarrier ring,
// and the candidate filter fused into the TMEM epilogue, so the nq x n score
// matrix never reaches HBM (north_star item 5; the contraction of
// index.py:67-72 / kernels.py:41-62's exact keys, SURVEY §8(d) C4 batch 1024).
//
// Warp roles of the persistent CTA (one per SM, 320 threads):
//   warp 0      TMA producer (one elected lane): A = 128 queries x 32 dims,
//               B = 256 vectors x 32 dims per stage (48 KB)
//   warp 1      TMEM allocator + MMA issuer (one lane): 4 x
//               tcgen05.mma.cta_group::1.kind::tf32 M128 N256 K8 per stage,
//               tcgen05.commit frees the stage / publishes the accumulator
//   warps 2-9   epilogue: tcgen05.ld 32x32b.x32 (thread = query row, two
//               warps per TMEM lane quarter, 128 columns each), the
//               interval [lb, ub] of every (query, vector) pair around the
//               reference key (pair_bounds, tested as a threshold on s), then
//                 MODE 0: S written densely (the first chunk, whose k-th
//                         upper bound seeds tau via pdx_k8_filter),
//                 MODE 1: pairs with lb <= tau[q] appended to q's candidates.
// Two accumulator stages (2 x 256 TMEM columns) let the epilogue of tile i
// overlap the MMAs of tile i+1.  Tiles: m fastest, so the 8 query tiles of a
// 256-vector slice run back to back and the slice is read from HBM once.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "pdx_common.cuh"

namespace pdx {
namespace {

// Tile M (queries) x N (vectors) x one 128-byte swizzle row of K per stage:
// 32 tf32 or 64 bf16 elements.
constexpr int kTM = 128, kTN = 256, kRowBytes = 128;
constexpr int kMaxStages = 6;
constexpr int kABytes = kTM * kRowBytes, kBBytes = kTN * kRowBytes;
constexpr int kEpiWarps = 8;  // two per TMEM lane quarter, each half the columns
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kSmem = 4 * (kABytes + kBBytes) + 1024 /*align*/ + 16 * kMaxStages + 64;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(b), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
// CTA-pair (cta_group::2) helpers: the cluster address of a CTA's variable,
// remote arrives, the pair's TMA load (bytes counted on the leader's
// barrier), the pair MMA and its multicast commit, the cluster barrier.
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int c0,
                                                 int c1, uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
template <bool BF16>
__device__ __forceinline__ void tc_mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  if (BF16)
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

template <bool BF16>
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  if (BF16)
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// K-major operand tile in 128-byte swizzle (rows of 32 floats, 8-row groups
// 1024 B apart): start address, LBO 16 B (unused for swizzled K-major), SBO
// 1024 B, descriptor version 1, layout SWIZZLE_128B (2).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor: D f32, A/B tf32 (format 2) or bf16 (format 1),
// both K-major, N = 256, M = 128
template <bool BF16, int M = kTM>
__host__ __device__ constexpr uint32_t idesc_of() {
  return (1u << 4) | ((BF16 ? 1u : 2u) << 7) | ((BF16 ? 1u : 2u) << 10) |
         ((uint32_t)(kTN >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

#define PDX_TMEM_LD32(taddr, r)                                                                   \
  asm volatile(                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"             \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),       \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),   \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),            \
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),            \
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])             \
      : "r"(taddr))

struct K8Args {
  int64_t nq, r0, r1;  // queries; vector rows [r0, r1) of X
  int nk;              // K blocks of one 128-byte row (32 tf32 / 64 bf16 elements)
  int metric;
  float c, e2;         // pdx_k8_margin and the L2 expansion's relative term
  const float* qn2;    // [nq]
  const float* xn2;    // [n] (indexed by absolute row)
  const float* tau;    // [nq] (MODE 1)
  int64_t* cand;       // [nq][C]
  float* cand_lb;      // [nq][C]
  float* cand_ub;      // [nq][C]
  int32_t* ccount;     // [nq]
  int C;
  float* S;            // MODE 0: [nq][ldS], column j = row r0 + j
  int64_t ldS;
};

// PAIR: a CTA pair (cluster of 2) shares each MMA (tcgen05.mma.cta_group::2,
// M = 256): CTA r loads queries [m*256 + r*128, +128) and vectors
// [n*256 + r*128, +128) of the tile, the leader (rank 0) issues the MMAs,
// each CTA's TMEM holds its 128 query rows x 256 columns and its epilogue
// filters them.  B operand bytes per CTA halve for the same FLOPs.
template <int MODE, bool BF16, bool PAIR>
__global__ void __launch_bounds__(kThreads, 1) k8_tc_kernel(const __grid_constant__ CUtensorMap tq,
                                                            const __grid_constant__ CUtensorMap tx,
                                                            const K8Args a) {
  constexpr int BROWS = PAIR ? kTN / 2 : kTN;  // B rows this CTA stages
  constexpr int BBYTES = BROWS * kRowBytes;
  constexpr int MQ = PAIR ? 2 * kTM : kTM;  // queries per tile
  constexpr int kStages = PAIR ? 6 : 4;     // (the same shared-memory budget)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sA = base, sB = base + kStages * kABytes;
  const uint32_t bars = sB + kStages * BBYTES;  // full[S] empty[S] tfull[2] tempty[2] tmem_ptr
  const uint32_t full0 = bars, empty0 = bars + 8 * kStages, tfull0 = bars + 16 * kStages,
                 tempty0 = tfull0 + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + (bars + 16 * kStages + 32 - raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cta_rank() : 0u;
  const int64_t unit = PAIR ? blockIdx.x / 2 : blockIdx.x;
  const int64_t nunits = PAIR ? gridDim.x / 2 : gridDim.x;

  const int64_t num_m = (a.nq + MQ - 1) / MQ;
  const int64_t num_n = (a.r1 - a.r0 + kTN - 1) / kTN;
  const int64_t ntiles = num_m * num_n;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full0 + 8 * s, PAIR ? 2 : 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tfull0 + 8 * s, 1);
      mbar_init(tempty0 + 8 * s, PAIR ? 2 * kEpiWarps : kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tq)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tx)) : "memory");
  }
  if (warp == 1) {  // TMEM: 2 accumulator stages x 256 columns
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       su32(tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       su32(tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // the peer's barriers are initialised before any remote use
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (in each CTA of a pair: its halves)
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = unit; t < ntiles; t += nunits) {
        const int m = (int)(t % num_m);
        const int64_t n = t / num_m;
        const int qrow = m * MQ + (int)rank * kTM;
        const int xrow = (int)(a.r0 + n * kTN) + (int)rank * BROWS;
        for (int kb = 0; kb < a.nk; ++kb) {
          mbar_wait(empty0 + 8 * stage, phase ^ 1);
          const int kel = kb * (BF16 ? 64 : 32);  // element column of this K block
          if (PAIR) {
            const uint32_t lb = mapa(full0 + 8 * stage, 0);  // the leader's barrier
            if (rank == 0)
              mbar_expect_tx(full0 + 8 * stage, 2 * (kABytes + BBYTES));
            else
              mbar_arrive_cluster(lb);
            tma_load_2d_pair(sA + stage * kABytes, &tq, kel, qrow, lb);
            tma_load_2d_pair(sB + stage * BBYTES, &tx, kel, xrow, lb);
          } else {
            const uint32_t fb = full0 + 8 * stage;
            mbar_expect_tx(fb, kABytes + BBYTES);
            tma_load_2d(sA + stage * kABytes, &tq, kel, qrow, fb);
            tma_load_2d(sB + stage * BBYTES, &tx, kel, xrow, fb);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---- MMA issuer (the leader of a pair)
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int64_t t = unit; t < ntiles; t += nunits, ++it) {
        const int acc = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        mbar_wait(tempty0 + 8 * acc, aphase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem + acc * kTN;
        for (int kb = 0; kb < a.nk; ++kb) {
          mbar_wait(full0 + 8 * stage, phase);
          tc_fence_after();
          const uint64_t ad = smem_desc(sA + stage * kABytes);
          const uint64_t bd = smem_desc(sB + stage * BBYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // 32 bytes per MMA: K = 8 tf32 / 16 bf16
            if (PAIR)
              tc_mma_pair<BF16>(tmem_d, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k),
                                idesc_of<BF16, 2 * kTM>(), (kb | k) != 0);
            else
              tc_mma<BF16>(tmem_d, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k),
                           idesc_of<BF16>(), (kb | k) != 0);
          }
          // the stage is free (in both CTAs) once these MMAs finish
          if (PAIR) tc_commit_pair(empty0 + 8 * stage); else tc_commit(empty0 + 8 * stage);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        // the accumulator is complete (in both CTAs)
        if (PAIR) tc_commit_pair(tfull0 + 8 * acc); else tc_commit(tfull0 + 8 * acc);
      }
    }
  } else {  // ---- epilogue: warps 2..9; TMEM lane quarter = warp % 4, column half = (warp-2)/4
    __shared__ float col_u[2][kTN], col_xn[2][kTN];
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const int et = threadIdx.x - 64;  // 0..255: this thread's column for the per-tile constants
    // the filter as a threshold on s (the interval test of pair_bounds
    // rearranged; e2t adds slack for the rearrangement's own rounding)
    const float e2t = a.e2 + 32.f / 16777216.f;
    int it = 0;
    for (int64_t t = unit; t < ntiles; t += nunits, ++it) {
      const int m = (int)(t % num_m);
      const int64_t n = t / num_m;
      const int acc = it & 1;
      const int64_t x0 = a.r0 + n * kTN;
      if (MODE == 1) {  // per-column constants, shared by every query row
        const int64_t x = x0 + et;
        const float xx = x < a.r1 ? __ldg(a.xn2 + x) : 0.f;
        col_xn[acc][et] = a.c * (sqrtf(xx) * 1.000001f);
        col_u[acc][et] = a.metric == PDX_METRIC_IP ? 0.f : 0.5f * (1.f - e2t) * xx;
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      }
      mbar_wait(tfull0 + 8 * acc, (it >> 1) & 1);
      tc_fence_after();
      const int64_t q = (int64_t)m * MQ + (int64_t)rank * kTM + row;
      const bool qok = q < a.nq;
      const float qq = qok ? a.qn2[q] : 0.f;
      const float qn = sqrtf(qq) * 1.000001f;
      const float tau = (MODE == 1 && qok) ? a.tau[q] : -INFINITY;
      // keep (q, x) iff s >= base + u[x] - qn * xn[x]
      const float base = a.metric == PDX_METRIC_IP ? -tau : 0.5f * ((1.f - e2t) * qq - tau);
      for (int ch = half * (kTN / 64); ch < (half + 1) * (kTN / 64); ++ch) {
        uint32_t r[32];
        const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + acc * kTN + ch * 32;
        PDX_TMEM_LD32(taddr, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (!qok) continue;
        const int64_t xb = x0 + ch * 32;
        if (MODE == 0) {
          float* srow = a.S + q * a.ldS + (xb - a.r0);
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            if (xb + j + 3 < a.r1) {
              *reinterpret_cast<float4*>(srow + j) =
                  make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                              __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (xb + j + u < a.r1) srow[j + u] = __uint_as_float(r[j + u]);
            }
          }
        } else {
          const float4* u4 = reinterpret_cast<const float4*>(&col_u[acc][ch * 32]);
          const float4* n4 = reinterpret_cast<const float4*>(&col_xn[acc][ch * 32]);
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float4 uu = u4[j4], nn = n4[j4];
            const float us[4] = {uu.x, uu.y, uu.z, uu.w}, ns[4] = {nn.x, nn.y, nn.z, nn.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int j = j4 * 4 + e;
              const float sv = __uint_as_float(r[j]);
              if (sv >= fmaf(-qn, ns[e], base + us[e]) && xb + j < a.r1) {
                const int64_t x = xb + j;
                const float xx = __ldg(a.xn2 + x);
                const float ed = a.c * qn * (sqrtf(xx) * 1.000001f);
                float lb, ub;
                if (a.metric == PDX_METRIC_IP) {
                  lb = -sv - ed;
                  ub = -sv + ed;
                } else {
                  const float dt = qq + xx - 2.f * sv;
                  const float del = 2.f * ed + a.e2 * (qq + xx);
                  lb = dt - del;
                  ub = dt + del;
                }
                const int at = atomicAdd(a.ccount + q, 1);
                if (at < a.C) {
                  a.cand[q * a.C + at] = x;
                  a.cand_lb[q * a.C + at] = lb;
                  a.cand_ub[q * a.C + at] = ub;
                }
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR)
          mbar_arrive_cluster(mapa(tempty0 + 8 * acc, 0));  // the leader's MMA waits on it
        else
          mbar_arrive(tempty0 + 8 * acc);
      }
    }
  }
  __syncthreads();
  if (PAIR) cluster_sync();  // both CTAs are done with TMEM and the leader's barriers
  if (warp == 1) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem)
                   : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// rows x ld elements (float32 or bf16), row-major; box = one 128-byte
// swizzle row of elements x box_rows
int make_map(CUtensorMap* m, const void* p, int64_t rows, int64_t ld, int box_rows, bool bf16) {
  auto fn = encode_fn();
  PDX_REQUIRE(fn, "cuTensorMapEncodeTiled is unavailable (driver too old)");
  const int es_bytes = bf16 ? 2 : 4;
  const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * es_bytes};
  const cuuint32_t box[2] = {(cuuint32_t)(kRowBytes / es_bytes), (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        2, const_cast<void*>(p), dims, strides,
                        box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  PDX_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return PDX_OK;
}

// float32 rows (ld floats apart) -> bf16 rows (ld16 elements apart, zero padded), RN
__global__ void __launch_bounds__(256) to_bf16_kernel(const float* __restrict__ x, int64_t n, int d,
                                                      int64_t ld, int64_t ld16,
                                                      __nv_bfloat16* __restrict__ y) {
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= n) return;
  for (int j = threadIdx.x & 31; j < ld16; j += 32)
    y[r * ld16 + j] = __float2bfloat16_rn(j < d ? x[r * ld + j] : 0.f);
}

}  // namespace

int k8_to_bf16(const float* d_x, int64_t n, int d, int64_t ld, int64_t ld16, void* d_y,
               cudaStream_t st) {
  if (n == 0) return PDX_OK;
  to_bf16_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(d_x, n, d, ld, ld16,
                                                          static_cast<__nv_bfloat16*>(d_y));
  PDX_LAUNCH_CHECK();
  return PDX_OK;
}

// The tensor-core pass over X rows [r0, r1) (mode 0: dense S; mode 1: fused
// candidate filter).  Shared by pdx_k8_candidates (pdx_k8.cu).
int k8_tc_pass(int mode, bool bf16, const void* d_x, int64_t n, int64_t ld, const void* d_q,
               int64_t nq, int64_t r0, int64_t r1, int d, int metric, float c, float e2,
               const float* qn2, const float* xn2, const float* tau, int64_t* cand,
               float* cand_lb, float* cand_ub, int32_t* ccount, int C, float* S, int64_t ldS,
               cudaStream_t st) {
  PDX_REQUIRE(ld % (bf16 ? 8 : 4) == 0 && ld >= d, "row stride must be 16-byte aligned and >= d");
  PDX_REQUIRE(((uintptr_t)d_x & 15) == 0 && ((uintptr_t)d_q & 15) == 0, "rows must be 16-B aligned");
  if (r1 <= r0 || nq == 0) return PDX_OK;
  CUtensorMap tq, tx;
  // CTA pairs (cta_group::2) with PDX_K8_PAIR=1 (exact, but measured at C4:
  // 16.4 ms against 9.2-10.8 ms for single-CTA tiles per candidate pass, so
  // off by default); a pair CTA stages half of the tile's vectors
  static const bool pair = [] {
    const char* e = getenv("PDX_K8_PAIR");
    return e && atoi(e) == 1;
  }();
  PDX_TRY(make_map(&tq, d_q, nq, ld, kTM, bf16));
  PDX_TRY(make_map(&tx, d_x, n, ld, pair ? kTN / 2 : kTN, bf16));
  K8Args a;
  a.nq = nq;
  a.r0 = r0;
  a.r1 = r1;
  const int kel = bf16 ? 64 : 32;
  a.nk = (int)((d + kel - 1) / kel);
  a.metric = metric;
  a.c = c;
  a.e2 = e2;
  a.qn2 = qn2;
  a.xn2 = xn2;
  a.tau = tau;
  a.cand = cand;
  a.cand_lb = cand_lb;
  a.cand_ub = cand_ub;
  a.ccount = ccount;
  a.C = C;
  a.S = S;
  a.ldS = ldS;
  int dev = 0, nsm = 148;
  PDX_CUDA_CHECK(cudaGetDevice(&dev));
  PDX_CUDA_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int mq = pair ? 2 * kTM : kTM;
  const int64_t tiles = ((nq + mq - 1) / mq) * ((r1 - r0 + kTN - 1) / kTN);
  const unsigned grid = pair ? (unsigned)(2 * std::min<int64_t>(tiles, nsm / 2))
                             : (unsigned)std::min<int64_t>(tiles, nsm);
  auto launch = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = pair ? 2 : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, tq, tx, a);
  };
  cudaError_t e;
  if (pair)
    e = mode == 0 ? (bf16 ? launch(k8_tc_kernel<0, true, true>) : launch(k8_tc_kernel<0, false, true>))
                  : (bf16 ? launch(k8_tc_kernel<1, true, true>) : launch(k8_tc_kernel<1, false, true>));
  else
    e = mode == 0 ? (bf16 ? launch(k8_tc_kernel<0, true, false>) : launch(k8_tc_kernel<0, false, false>))
                  : (bf16 ? launch(k8_tc_kernel<1, true, false>) : launch(k8_tc_kernel<1, false, false>));
  PDX_CUDA_CHECK(e);
  PDX_LAUNCH_CHECK();
  return PDX_OK;
}

}  // namespace pdx
