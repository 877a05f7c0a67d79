// Bucket-major batched IVF search: the reference's ivf_search (index.py:130-156)
// for a whole query batch, with results, every prune decision and the stats
// of the reference (search.py:125-205), bit for bit.
//
// Why: at IVF scale a probed bucket is shared by many queries of a batch
// (C2: ~31 queries per probed bucket), but the per-query scan
// (pdx_scan_kernel) re-reads and re-evaluates each tile once per query along
// a latency-bound chain.  Here each tile's head dimensions are loaded into
// registers ONCE per work item and evaluated for every query probing it.
//
// The reference's threshold chain is sequential per query (T_b = the k-th
// best distance when block b starts, search.py:159).  Exactness comes from
// three facts: partial sums do not depend on T, the ADS / BOND / BSA bounds
// are monotone in T, and the top-k after a set of pushes does not depend on
// their order (TopK keeps the k smallest (dist, id) pairs, search.py:44-51).
//
//  Phase 1  each query's first selected bucket that has blocks (at most its
//           first kP1Cap tiles), exactly: bdense_kernel records every
//           slot's partial at every step end (prune-free), and
//           bchain1_kernel (one warp per query; for results-only searches
//           running underneath the dense pass, tile by tile) replays the
//           reference chain over those partials.  Heap H, T' =
//           its k-th distance; every later block has T_b <= T'.  The rest of
//           the selected blocks (the bucket's tail first) form the window.
//  Phase 2  (bscan_kernel MODE 0) every (query, tile) pair of the window,
//           tile-major (work items: a bucket's tile range x up to 32 of the
//           queries probing it), under the fixed bound B_s(T'): per-step
//           survivor counts, the
//           pair's certainty margin rho = max over (slot, step) surviving
//           under T' of v_s / beta_s (beta_s: the bound's factor, B_s(T) ~
//           T beta_s), and the T'-survivors with their distances.
//  Chain    (bchain_kernel) per query: T^_p = the k-th smallest of H and the
//           T'-survivors of pairs before p — the reference's T_b provided
//           every T'-survivor is a real survivor.  A pair whose decisions
//           could differ between T^_p and T' (T^_p < T' and rho_p >= T^_p,
//           with slack) is listed as uncertain.
//  Recompute (bscan_kernel MODE 1) re-evaluates each uncertain pair exactly
//           under T^_p, tile-major like phase 2, overwriting its stats and
//           confirming its real survivors.  A T'-survivor it does not
//           confirm is dropped; if its distance is below T^_p (an ADS prune
//           of the exact chain that T' did not make) the assumption behind
//           T^ broke and the query is flagged.
//  Final    (bfinal_kernel) top-k = k smallest of H and all T'-survivors,
//           values_touched / values_total / survivor traces summed per pair.
//  Fallback flagged queries (and any whose phase-1 heap is not full, or
//           whose buffers overflowed) are re-run by the per-query scan.
//  The work-list kernels (bucket histogram, scans, entries, items) run on a
//  side stream while phase 1 runs.
//
// Certain pairs: for T in [T^_p, T'] a slot pruned under T' is pruned under
// T (monotone), and a slot surviving step s under T' has v_s < B_s(T^_p) <=
// B_s(T), so the decisions, counts and survivors are T'-s.  By induction
// over the pairs the chain's T_b equals T^_p everywhere when no query is
// flagged.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "pdx_batch.cuh"
#include "pdx_common.cuh"
#include "pdx_scan_kernel.cuh"

#ifndef PDX_BSCAN_MIN_BLOCKS
#define PDX_BSCAN_MIN_BLOCKS 3  // work-item CTAs per SM (80 registers)
#endif

namespace pdx {
namespace {

constexpr int kBW = 8;          // warps per work-item CTA
constexpr int kBWD = 4;         // warps per work-item CTA of the dense variant (d > 256)
constexpr int kQC = 32;         // queries per work item
constexpr int kTC = 32;         // tiles per work item (long buckets are split: load balance)
constexpr int kP1Cap = 64;      // phase 1 covers at most this many tiles of the first bucket
__constant__ int c_p1cap = kP1Cap;  // (PDX_P1CAP lowers it, for measurements)
constexpr int kHeadDims = 16;   // dims every pair evaluates for all 64 slots
constexpr int kMaxHead = 5;     // steps inside the head (initial_step 1: 1,3,7,15)
constexpr int kDeepCap = 64;    // deep items per warp queue
constexpr int kMaxBatchK = 256;
constexpr float kRhoSlack = 1.00001f;
constexpr int kTodoCap = 256;   // recompute pass: per-tile masks for buckets up to this many tiles

struct BEntry {  // a query probing a bucket
  int32_t q;
  int32_t base;  // query-local pair index of the bucket's first tile
};
struct BItem {  // a work item: bucket, its entries [e0, e0 + ne), tiles [t0, t0 + kTC)
  int32_t bucket, e0, ne, t0;
};
// A T'-survivor (phase 2).  The chain kernel sorts a query's list by pair and
// sets tafter = T^ after the pushes of that pair; the recompute pass sets
// real = 1 on the survivors it confirms under T^.
struct BSurv {
  float dist;
  int32_t pair;  // query-local pair index
  int64_t id;
  int32_t slot;
  float tafter;
  int32_t real;
  int32_t tile;  // the store tile holding the slot (bverify_kernel)
  float tbefore;  // T^ before the pushes of its pair (= that_of(pair)): no search in verify / final
};
struct DeepItem {
  float acc;
  int16_t j, slot;
  float that;     // recompute pass: the pair's T^
  int16_t s, pos;  // where the item resumes: next step, next dim
};

// Per-call constants (kernel parameter; copied to shared memory where they
// are indexed at run time).
struct BParams {
  int32_t d, d_pad, nsteps, hsteps, hdims, k, pruner, nseg;
  int32_t nq, surv_cap;
  int32_t p1max;   // phase-1 tiles per query (stride of part1 and of the ready flags)
  int32_t dbg;     // PDX_BATCH_DEBUG: MODE 1 counts its work in nitems[4..6]
  int32_t norho;   // results only: no rho; every pair with T^ < T' counts as uncertain
  uint32_t hmask;  // bit e: a head step ends after dim e
  int32_t ends[kMaxSteps];
  double ratio[kMaxSteps], band[kMaxSteps];
  float invb[kMaxSteps];
  int32_t wmin[kTile + 1];
};

struct BArgs {
  const float* tiles;
  const int64_t* tile_ids;
  int64_t tile_stride;
  const int64_t* bucket_block;
  const int64_t* block_tile;
  const int32_t* block_m;
  const float* queries;
  const int32_t* sel;   // [nq][nseg]
  const int32_t* fseg;  // [nq] first selected segment with blocks (phase 1's bucket)
  const float* resid;  // BSA [ntiles][nsteps][64]
  const float* coef;   // BSA [nsteps]
  // per query
  float* tprime;
  float* bounds;        // [nq][nsteps]  B_s(T')
  float* bsaq;          // BSA [nq][2][nsteps]  rq_s, sqrt(rq_s)
  const int64_t* qoff;  // [nq+1]
  int32_t* flags;
  int32_t* nsurv;
  BSurv* surv;  // [nq][surv_cap]
  // per pair
  uint32_t* ptouched;
  float* prho;
  uint8_t* pcnt;  // [P][nsteps] (survivor traces only)
  // work
  const BItem* items;
  const int32_t* nitems;
  int32_t* wctr;  // [2]: work items handed out by MODE 0 / MODE 1
  const BEntry* entries;
  const int64_t* bnvec;  // vectors per bucket
  // outputs
  float* out_dist;
  int64_t* out_ids;
  int32_t* out_count;
  int64_t* out_touched;
  int64_t* out_total;
  int32_t* trace;
  int64_t trace_cap;
  int64_t* trace_len;
};

__device__ __forceinline__ float l2upd(float acc, float q, float x) {
  const float t = __fsub_rn(q, x);
  return __fadd_rn(acc, __fmul_rn(t, t));
}

// (q - x0)^2 and (q - x1)^2 for a slot pair held as one 64-bit register:
// FADD2 with q broadcast, FMUL2 — each lane of the pair rounded on its own,
// exactly like __fsub_rn / __fmul_rn.  The accumulation stays scalar: ptxas
// contracts an f32x2 multiply followed by an f32x2 add into FFMA2.
__device__ __forceinline__ unsigned long long pack2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 sqdiff2(float q, unsigned long long xx) {
  unsigned long long qq, t, p;
  asm("mov.b64 %0, {%1, %1};" : "=l"(qq) : "f"(q));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(qq), "l"(xx));
  asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(p) : "l"(t));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(p));
  return r;
}

// acc + (q - x)^2 for a slot pair, all three steps f32x2: FADD2 (q
// broadcast), the square as FFMA2 with a +0 addend — the exact square
// rounded once, bit-identical to mul.rn (a square is never -0) — and FADD2.
// ptxas does not contract FFMA2 + FADD2, so each op stays separately rounded
// (the reference's per-op rounding) at 3 instructions per dim per pair.
__device__ __forceinline__ unsigned long long sqacc2(unsigned long long acc, float q,
                                                     unsigned long long xx) {
  unsigned long long qq, z, t, p, r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(qq) : "f"(q));
  asm("mov.b64 %0, {%1, %1};" : "=l"(z) : "f"(0.0f));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(qq), "l"(xx));
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(p) : "l"(t), "l"(z));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(acc), "l"(p));
  return r;
}
// (a, b) as a register pair computed once: x + (-0) is exact for every x
// (-0 included), and as a real FADD2 ptxas keeps the pair instead of
// rebuilding it from the two loads' registers at every use.
__device__ __forceinline__ unsigned long long pack2_hold(float a, float b) {
  unsigned long long r, nz;
  asm("mov.b64 %0, {%1, %1};" : "=l"(nz) : "f"(-0.0f));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pack2(a, b)), "l"(nz));
  return r;
}
__device__ __forceinline__ float2 unpack2(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}

// Plain f32x2 helpers of the results-only head filter (bscan0_kernel): no
// per-op-rounding contract — its results only discard slots under a
// certainty margin.
__device__ __forceinline__ unsigned long long bcast2(float a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(a));
  return r;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b,
                                                   unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long mul2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// (asm volatile: the load stays where it is written — ptxas otherwise hoists
// these out of the pair loop and spills them)
__device__ __forceinline__ unsigned long long lds64(const unsigned long long* p) {
  unsigned long long r;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(r) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return r;
}
// position of the r-th (0-based) set bit of m (r < popc(m))
__device__ __forceinline__ int nth_bit(uint32_t m, int r) {
  int pos = 0;
#pragma unroll
  for (int wd = 16; wd >= 1; wd >>= 1) {
    const int c = __popc(m & ((1u << wd) - 1u));
    if (r >= c) {
      r -= c;
      pos += wd;
      m >>= wd;
    }
  }
  return pos;
}

// BSA estimate (bsa_est in pdx_scan_spec.cuh, same association).
__device__ __forceinline__ float bsa_est2(float acc, float rx, float rq, float sq, float coef) {
  const float cx = __fmul_rn(coef, __fsqrt_rn(rx));
  return __fsub_rn(__fadd_rn(__fadd_rn(acc, rx), rq), __fmul_rn(cx, sq));
}

// --------------------------------------------------------------- planning
// One warp per query: first bucket, query-local pair bases of the other
// selected buckets, the window's pair count, and the bucket histogram.
__global__ void bprep_kernel(const int32_t* __restrict__ sel, int nq, int nseg,
                             const int64_t* __restrict__ bucket_block,
                             const int64_t* __restrict__ block_tile,
                             int64_t* __restrict__ wcount, int32_t* __restrict__ pbase,
                             int32_t* __restrict__ bcnt, int32_t* __restrict__ fseg) {
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= nq) return;
  const int32_t* sq = sel + (int64_t)q * nseg;
  // phase 1 takes the first min(nt0, kP1Cap) tiles of the first bucket; its
  // tail (if any) opens the speculative window, pair indices from 0
  // (the reference's block list skips empty buckets: phase 1 takes the first
  // selected bucket that has blocks — on a bucket shard, often not segment 0)
  int f = 0;
  auto ntiles = [&](int c) {
    return (int)(block_tile[bucket_block[c + 1]] - block_tile[bucket_block[c]]);
  };
  while (f < nseg - 1 && ntiles(sq[f]) == 0) ++f;
  const int nt0 = ntiles(sq[f]);
  const int p1 = min(nt0, c_p1cap);
  if (lane == 0) {
    fseg[q] = f;
    if (q == 0) wcount[nq] = 0;
    pbase[(int64_t)q * nseg + f] = -p1;
    if (nt0 > p1) atomicAdd(&bcnt[sq[f]], 1);
  }
  int run = nt0 - p1;
  for (int s0 = f + 1; s0 < nseg; s0 += 32) {
    const int s = s0 + lane;
    int nt = 0;
    if (s < nseg) {
      const int c = sq[s];
      nt = (int)(block_tile[bucket_block[c + 1]] - block_tile[bucket_block[c]]);
      if (nt > 0) atomicAdd(&bcnt[c], 1);
    }
    int incl = nt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
    if (s < nseg) pbase[(int64_t)q * nseg + s] = run + incl - nt;
    run += __shfl_sync(kFull, incl, 31);
  }
  if (lane == 0) wcount[q] = run;
}

// Per bucket: work-item count and vector count.
__global__ void bchunks_kernel(const int32_t* __restrict__ bcnt, int nb,
                               const int64_t* __restrict__ bucket_block,
                               const int32_t* __restrict__ block_m, int32_t* __restrict__ nch,
                               int64_t* __restrict__ bnvec) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > nb) return;
  if (c == nb) {
    nch[c] = 0;
    return;
  }
  const int ntc = (int)(bucket_block[c + 1] - bucket_block[c]);
  nch[c] = ((bcnt[c] + kQC - 1) / kQC) * ((ntc + kTC - 1) / kTC);
  int64_t v = 0;
  for (int64_t b = bucket_block[c]; b < bucket_block[c + 1]; ++b) v += block_m[b];
  bnvec[c] = v;
}

__global__ void bfill_kernel(const int32_t* __restrict__ sel, int nq, int nseg,
                             const int64_t* __restrict__ bucket_block,
                             const int64_t* __restrict__ block_tile,
                             const int32_t* __restrict__ pbase, const int32_t* __restrict__ boff,
                             int32_t* __restrict__ bcur, BEntry* __restrict__ entries,
                             const int32_t* __restrict__ fseg) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)nq * nseg) return;
  const int q = (int)(i / nseg), s = (int)(i % nseg);
  const int c = sel[(int64_t)q * nseg + s];
  const int64_t ntc = block_tile[bucket_block[c + 1]] - block_tile[bucket_block[c]];
  const int f = fseg[q];
  if (s < f || (s == f ? ntc <= c_p1cap : ntc == 0)) return;  // before / no tail of the first bucket
  const int pos = atomicAdd(&bcur[c], 1);
  entries[boff[c] + pos] = BEntry{q, pbase[(int64_t)q * nseg + s]};
}

__global__ void bitems_kernel(const int32_t* __restrict__ bcnt, int nb,
                              const int32_t* __restrict__ boff, const int32_t* __restrict__ choff,
                              const int64_t* __restrict__ bucket_block, BItem* __restrict__ items,
                              int32_t* __restrict__ nitems) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c == 0) *nitems = choff[nb];
  if (c >= nb) return;
  const int n = bcnt[c];
  const int ntc = (int)(bucket_block[c + 1] - bucket_block[c]);
  int j = choff[c];
  for (int t = 0; t < ntc; t += kTC)
    for (int i = 0; i < n; i += kQC) items[j++] = BItem{c, boff[c] + i, min(kQC, n - i), t};
}

// T' of a query (the phase-1 heap's k-th distance, +inf while the heap is not
// full: the query is flagged for the per-query scan), the bounds B_s(T'), and
// the BSA query residual energies (the scan kernel's prologue order); called
// by the query's chain warp once its heap is final.
__device__ __forceinline__ void btprime_query(const BParams& P, const BArgs& A, const int q,
                                              const float T, const int lane) {
  if (lane == 0) {
    const_cast<float*>(A.tprime)[q] = T;
    A.flags[q] = T == INFINITY ? 1 : 0;
    A.nsurv[q] = 0;
  }
  if (lane < P.nsteps) {
    const int s = lane;
    const_cast<float*>(A.bounds)[(int64_t)q * P.nsteps + s] =
        T == INFINITY ? -INFINITY
                      : (P.pruner == PDX_PRUNER_BSA ? T : ads_or_bond_bound(T, P.ratio[s], P.band[s]));
    if (P.pruner == PDX_PRUNER_BSA) {
      const float* qg = A.queries + (int64_t)q * P.d;
      float* bq = const_cast<float*>(A.bsaq) + (int64_t)q * 2 * P.nsteps;
      float r = 0.f;
      for (int j = P.ends[s]; j < P.d; ++j) r = __fadd_rn(r, __fmul_rn(qg[j], qg[j]));
      bq[s] = r;
      bq[P.nsteps + s] = __fsqrt_rn(r);
    }
  }
}

__device__ __forceinline__ void record_survivor(const BParams& P, const BArgs& A, int q,
                                                int32_t pair, float dist, int64_t tile, int slot) {
  const int i = atomicAdd(&A.nsurv[q], 1);
  if (i < P.surv_cap)
    A.surv[(int64_t)q * P.surv_cap + i] =
        BSurv{dist, pair, __ldg(A.tile_ids + tile * kTile + slot), slot, 0.f, 0, (int32_t)tile, 0.f};
  else
    A.flags[q] = 1;
}

__device__ __forceinline__ float bound_at(const BParams& P, float T, int s, const double* ratio,
                                          const double* band) {
  return P.pruner == PDX_PRUNER_BSA ? T : ads_or_bond_bound(T, ratio[s], band[s]);
}

// Phase 1's bucket of query q: the first selected bucket that has tiles (the
// last selected one if none has) — bprep_kernel's fseg, recomputed here so
// that phase 1 does not wait for the planning kernels.  Its partials and
// ready flags live at a fixed stride: tile ti of query q is entry q * p1max + ti.
__device__ __forceinline__ int first_bucket(const BParams& P, const BArgs& A, const int q) {
  const int32_t* sq = A.sel + (int64_t)q * P.nseg;
  int f = 0;
  for (;;) {
    const int c = sq[f];
    const int64_t nt = A.block_tile[A.bucket_block[c + 1]] - A.block_tile[A.bucket_block[c]];
    if (nt > 0 || f >= P.nseg - 1) return c;
    ++f;
  }
}

// ---------------------------------------------------------------- phase 1
// The reference chain over each query's first selected bucket, in two
// kernels.  bdense_kernel: every slot's partial (the BSA estimate for bsa)
// at every step end, prune-free, one warp per (query, tile) — a dense,
// throughput-bound pass with no dependence between tiles.  bchain1_kernel:
// one warp per query walks the bucket's blocks in order with the exact
// threshold chain (search.py:193-205), reading the recorded partials — the
// linear first block, every prune decision, the top-k pushes, values_touched
// and the survivor traces.  (A query's first bucket is where its threshold
// moves at almost every block, so pruned speculation would be replayed
// anyway after chasing long survivor tails one L2 round trip at a time.)
// (Pruning the dense pass under T_0, the threshold after the first block, was
// measured and removed: in a query's own bucket T_0 prunes little, the
// conditional loads and the extra first-block kernel cost more than the
// bytes they save — dense pass 85 -> 79 us, and 14 us of first-block kernel
// gone from the critical path.)
// st.release / ld.acquire at gpu scope: the per-tile ready flags between the
// dense kernel and the chain kernel running next to it.
__device__ __forceinline__ void st_release(int32_t* p, int32_t v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int32_t ld_acquire(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// One CTA of the dense pass: query q, warp w takes tile tile0 + w of the
// query's first bucket.  ready (overlapped phase 1): flag per phase-1 tile,
// set once the tile's partials are written.
template <bool BSA>
__device__ __forceinline__ void bdense_cta(const BParams& P, const BArgs& A,
                                           float* __restrict__ part1, const int q, const int tile0,
                                           int32_t* ready) {
  extern __shared__ __align__(16) float s_q[];  // [d_pad] query, then [2][nsteps] BSA rq, sqrt
  __shared__ int32_t s_ends[kMaxSteps];
  __shared__ float s_coef[kMaxSteps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = first_bucket(P, A, q);
  const int64_t b0 = A.bucket_block[c];
  const int nt = (int)(A.bucket_block[c + 1] - b0);
  if (tile0 >= min(nt, c_p1cap)) return;
  const int nsteps = P.nsteps;
  const float* qg = A.queries + (int64_t)q * P.d;
  for (int j = threadIdx.x; j < P.d_pad; j += blockDim.x) s_q[j] = j < P.d ? qg[j] : 0.f;
  for (int i = threadIdx.x; i < kMaxSteps; i += blockDim.x) {
    s_ends[i] = P.ends[i];
    s_coef[i] = (BSA && i < nsteps) ? A.coef[i] : 0.f;
  }
  __syncthreads();
  float* s_bq = s_q + P.d_pad;
  if (BSA) {  // the query's residual energies (pdx_scan_kernel's prologue order)
    if (threadIdx.x < nsteps) {
      float r = 0.f;
      for (int j = s_ends[threadIdx.x]; j < P.d; ++j) r = __fadd_rn(r, __fmul_rn(s_q[j], s_q[j]));
      s_bq[threadIdx.x] = r;
      s_bq[nsteps + threadIdx.x] = __fsqrt_rn(r);
    }
    __syncthreads();
  }
  // one tile per warp (latency-bound: many tiles in flight)
  const int ti = tile0 + w;
  if (ti >= min(nt, c_p1cap)) return;
  const int64_t tile = A.block_tile[b0] + ti;
  const int m = A.block_m[b0 + ti];
  const float* __restrict__ tb = A.tiles + tile * A.tile_stride;
  float* __restrict__ out = part1 + ((int64_t)q * P.p1max + ti) * nsteps * kTile;
  const int ng = P.d_pad >> 3;
  float acc0 = 0.f, acc1 = 0.f;
  const bool in0 = lane < m, in1 = lane + 32 < m;
  int nend = s_ends[0];  // end of the current step
  int s = 0;
  float n0[8], n1[8];  // the next group loads while the current one is evaluated
  ldg8(tb + lane * 8, n0);
  ldg8(tb + (32 + lane) * 8, n1);
  for (int g = 0; g < ng && s < nsteps; ++g) {
    float x0[8], x1[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      x0[e] = n0[e];
      x1[e] = n1[e];
    }
    if (g + 1 < ng) {
      ldg8(tb + ((size_t)(g + 1) * kTile + lane) * 8, n0);
      ldg8(tb + ((size_t)(g + 1) * kTile + 32 + lane) * 8, n1);
    }
    const float4 qa = *reinterpret_cast<const float4*>(s_q + g * 8);
    const float4 qb = *reinterpret_cast<const float4*>(s_q + g * 8 + 4);
    const float qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
    if (g * 8 + 8 < nend) {  // no step ends in this group: straight-line arithmetic
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        acc0 = l2upd(acc0, qv[e], x0[e]);
        acc1 = l2upd(acc1, qv[e], x1[e]);
      }
      continue;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int dim = g * 8 + e;
      if (s < nsteps) {  // (dims past d are never reached: the last step ends at d)
        const float qe = qv[e];
        acc0 = l2upd(acc0, qe, x0[e]);
        acc1 = l2upd(acc1, qe, x1[e]);
        if (dim + 1 == nend) {
          float v0 = acc0, v1 = acc1;
          if (BSA) {
            const float* rs = A.resid + ((size_t)tile * nsteps + s) * kTile;
            v0 = bsa_est2(acc0, __ldg(rs + lane), s_bq[s], s_bq[nsteps + s], s_coef[s]);
            v1 = bsa_est2(acc1, __ldg(rs + lane + 32), s_bq[s], s_bq[nsteps + s], s_coef[s]);
          }
          out[s * kTile + lane] = in0 ? v0 : INFINITY;  // (slots past the block's m vectors)
          out[s * kTile + 32 + lane] = in1 ? v1 : INFINITY;
          ++s;
          nend = s < nsteps ? s_ends[s] : 0x7fffffff;
        }
      }
    }
  }
  if (ready) {  // the tile's partials are complete: publish
    __threadfence();
    __syncwarp();
    if (lane == 0)
      st_release(ready + (int64_t)q * P.p1max + ti, P.dbg ? (int32_t)(gtimer_ns() >> 7) | 1 : 1);
  }
}

// (9 CTAs per SM: 56 registers — the pass is occupancy bound: -6 us per step
// against 64 registers / 8 CTAs; 10 CTAs / 48 registers spill in the loop)
template <bool BSA>
__global__ void __launch_bounds__(128, BSA ? 7 : 9) bdense_kernel(const BParams P, const BArgs A,
                                                     float* __restrict__ part1,
                                                     int32_t* __restrict__ ready) {
  bdense_cta<BSA>(P, A, part1, blockIdx.x, (int)blockIdx.y * 4, ready);
}


// NSM >= nsteps: register arrays sized to the schedule.  RK (k <= 32): the
// heap lives in registers, lane i holding the i-th smallest (dist, id).
// A chain CTA: 8 warps, warp wq walks query oct * 8 + wq for oct = oct0, oct0 +
// oct_stride, ...  ready (overlapped phase 1): the dense CTAs' per-tile flags —
// a tile's partials are read (at L2) only after its flag has been observed.
template <int NSM, bool RK, bool ST>
__device__ __forceinline__ void bchain1_cta(const BParams& P, const BArgs& A,
                                            const float* __restrict__ part1, const int oct0,
                                            const int oct_stride, const int32_t* ready) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  __shared__ Control s_ctl[8];
  __shared__ int32_t s_cnt[8][kMaxSteps];
  __shared__ int32_t s_ends[kMaxSteps], s_wmin[kTile + 1];
  __shared__ double s_ratio[kMaxSteps], s_band[kMaxSteps];
  for (int i = threadIdx.x; i < kMaxSteps; i += blockDim.x) {
    s_ends[i] = P.ends[i];
    s_ratio[i] = P.ratio[i];
    s_band[i] = P.band[i];
  }
  for (int i = threadIdx.x; i <= kTile; i += blockDim.x) s_wmin[i] = P.wmin[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  for (int oct = oct0; oct * 8 < P.nq; oct += oct_stride) {
  const int q = oct * 8 + wq;
  if (q >= P.nq) return;
  const int k = P.k, nsteps = P.nsteps;
  float* tkd = reinterpret_cast<float*>(s_raw) + (size_t)wq * k;
  int64_t* tki = reinterpret_cast<int64_t*>(s_raw + (size_t)8 * k * sizeof(float)) + (size_t)wq * k;
  Control& ctl = s_ctl[wq];
  if (lane == 0) ctl.n = 0;
  __syncwarp();
  float rd = INFINITY;  // RK heap
  int64_t ri = INT64_MAX;
  int rn = 0;
  // TopK.push (search.py:44-51) of the lanes' candidates, in lane order
  auto rk_push = [&](bool cand, float dv, int64_t iv) {
    unsigned mask = __ballot_sync(kFull, cand);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const float d = __shfl_sync(kFull, dv, src);
      const int64_t i = __shfl_sync(kFull, iv, src);
      if (rn == k && !pair_less(d, i, __shfl_sync(kFull, rd, k - 1), __shfl_sync(kFull, ri, k - 1)))
        continue;
      const int pos = __popc(__ballot_sync(kFull, lane < rn && pair_less(rd, ri, d, i)));
      const float pd = __shfl_up_sync(kFull, rd, 1);
      const int64_t pi = __shfl_up_sync(kFull, ri, 1);
      if (lane > pos) {
        rd = pd;
        ri = pi;
      } else if (lane == pos) {
        rd = d;
        ri = i;
      }
      rn = rn < k ? rn + 1 : k;
    }
  };
  auto rk_threshold = [&]() { return rn < k ? INFINITY : __shfl_sync(kFull, rd, k - 1); };
  const int c = first_bucket(P, A, q);
  const int64_t b0 = A.bucket_block[c];
  const int nt = min((int)(A.bucket_block[c + 1] - b0), c_p1cap);
  const int64_t t0 = A.block_tile[b0];
  int32_t* tr = A.trace ? A.trace + (int64_t)q * A.trace_cap : nullptr;
  int64_t touched = 0, total = 0, tlen = 0;  // lane 0
  float T = INFINITY, Tb = -1.f, bl = 0.f;
  float bs[NSM];  // B_s(T) of every step, in every lane
  // software pipeline: the next tile's partials, ids and size load while the
  // current tile is decided (one L2 round trip per tile, hidden)
  float u0[NSM], u1[NSM], n0[NSM], n1[NSM];
  int64_t id0 = 0, id1 = 0, nid0 = 0, nid1 = 0;
  int m = 0, nm = 0;
  const float* __restrict__ pq = part1 + (int64_t)q * P.p1max * nsteps * kTile;
  const int32_t* rdy = ready ? ready + (int64_t)q * P.p1max : nullptr;
  if (P.dbg && ready && lane == 0) A.ptouched[2 * q] = (uint32_t)(gtimer_ns() >> 7);
  auto fetch = [&](int ti) {
    if (ti >= nt) return;
    const float* __restrict__ pp = pq + (int64_t)ti * nsteps * kTile;
#pragma unroll
    for (int s = 0; s < NSM; ++s) {  // (L2 reads: the partials may come from a concurrent CTA)
      n0[s] = s < nsteps ? __ldcg(pp + s * kTile + lane) : 0.f;
      n1[s] = s < nsteps ? __ldcg(pp + s * kTile + 32 + lane) : 0.f;
    }
    const int64_t* gid = A.tile_ids + (t0 + ti) * kTile;
    nid0 = __ldg(gid + lane);
    nid1 = __ldg(gid + lane + 32);
    nm = A.block_m[b0 + ti];
  };
  // nready: tiles [0, nready) are known to be published.  A refresh reads the flags of the next 32 tiles in one
  // go (flags only ever go up), so the chain pays an L2 round trip for flags
  // only while it runs ahead of the dense pass.
  int nready = rdy ? 0 : nt;
  auto refresh = [&]() {
    const int t = nready + lane;
    const int f = t < nt ? ld_acquire(rdy + t) : 0;
    const unsigned mk = __ballot_sync(kFull, f != 0);
    __syncwarp();
    nready += mk == 0xffffffffu ? 32 : __ffs(~mk) - 1;  // consecutive published tiles
  };
  bool have = false;  // n0 / n1 hold tile ti's partials
  bool dead = false;  // a tile never arrived (cannot happen while the dense CTAs run): give up
  for (int ti = 0; ti < nt; ++ti) {
    if (!have) {
      if (ti >= nready) {
        const long long t_start = clock64();
        for (;;) {
          refresh();
          if (ti < nready) break;
          __nanosleep(64);
          if (clock64() - t_start > (1ll << 22)) {  // ~2 ms: no heap -> T' = +inf -> the per-query scan
            dead = true;
            break;
          }
        }
        if (dead) break;
      }
      fetch(ti);
    }
#pragma unroll
    for (int s = 0; s < NSM; ++s) {
      u0[s] = n0[s];
      u1[s] = n1[s];
    }
    id0 = nid0;
    id1 = nid1;
    m = nm;
    if (ti + 1 >= nready && ti + 1 < nt) refresh();  // (one poll; the wait is at the top)
    have = ti + 1 < nready || ti + 1 >= nt;
    if (have) fetch(ti + 1);
    const bool linear = ti == 0 || T == INFINITY;  // search.py:201
    bool c0 = lane < m, c1 = lane + 32 < m;
    if (linear) {
      if (ST && lane == 0) {
        touched += (int64_t)m * P.d;
        if (tr) {
          if (tlen >= 0 && tlen + 2 <= A.trace_cap) {
            tr[tlen] = 1;
            tr[tlen + 1] = m;
            tlen += 2;
          } else {
            tlen = -1;
          }
        }
      }
    } else {
      if (T != Tb) {  // the bounds move only with the threshold
        bl = lane < nsteps ? bound_at(P, T, lane, s_ratio, s_band) : 0.f;
#pragma unroll
        for (int s = 0; s < NSM; ++s) bs[s] = __shfl_sync(kFull, bl, s);
        Tb = T;
      }
      // per step independently: bit s = partial below B_s; a slot survives
      // steps 0 .. d-1 where d = the number of trailing ones (its chain)
      uint32_t ok0 = 0, ok1 = 0;
#pragma unroll
      for (int s = 0; s < NSM; ++s) {
        if (s >= nsteps) break;
        const float B = bs[s];
        ok0 |= (u0[s] < B ? 1u : 0u) << s;
        ok1 |= (u1[s] < B ? 1u : 0u) << s;
      }
      const int d0 = c0 ? __ffs(~ok0) - 1 : 0, d1 = c1 ? __ffs(~ok1) - 1 : 0;
      // survivors after step s = #slots with d > s: byte s of a unary code
      // (one byte per step, <= 64 per byte), summed over the warp per 4 steps
      int mycnt = 0;
#pragma unroll
      for (int g = 0; g < (ST ? (NSM + 3) / 4 : 0); ++g) {
        if (4 * g >= nsteps) break;
        auto unary = [&](int dd) -> unsigned {
          const int u = min(max(dd - 4 * g, 0), 4);
          return u == 4 ? 0x01010101u : ((1u << (8 * u)) - 1u) & 0x01010101u;
        };
        const unsigned w = __reduce_add_sync(kFull, unary(d0) + unary(d1));
        if ((lane >> 2) == g) mycnt = (int)((w >> (8 * (lane & 3))) & 0xffu);
      }
      c0 = d0 >= nsteps;
      c1 = d1 >= nsteps;
      if (ST) {
      // values_touched (search.py:148-169): step s counts m * w_s while the
      // entering count stays >= the WARMUP minimum (counts only fall, so the
      // flag is just that test), entering * w_s after; one lane per step
      const int enter = __shfl_up_sync(kFull, mycnt, 1);
      int64_t tv = 0;
      if (lane < nsteps) {
        const int e_s = lane == 0 ? m : enter;
        const int w_s = s_ends[lane] - (lane ? s_ends[lane - 1] : 0);
        tv = (int64_t)(e_s >= s_wmin[m] ? m : e_s) * w_s;
      }
      const unsigned tsum = __reduce_add_sync(kFull, (unsigned)tv);  // <= 64 * d per block
      if (tr && lane < nsteps) s_cnt[wq][lane] = mycnt;
      __syncwarp();
      if (lane == 0) {
        touched += tsum;
        if (tr) {
          if (tlen >= 0 && tlen + 1 + nsteps <= A.trace_cap) {
            tr[tlen] = nsteps;
            for (int s = 0; s < nsteps; ++s) tr[tlen + 1 + s] = s_cnt[wq][s];
            tlen += 1 + nsteps;
          } else {
            tlen = -1;
          }
        }
      }
      }
    }
    if (ST && lane == 0) total += (int64_t)m * P.d;
    if (ti == 0 && k <= kTile) {
      // the linear first block into an empty heap: the k smallest (dist, id)
      // of its m vectors, by a warp bitonic sort of the 64 slots
      float f0 = INFINITY, f1 = INFINITY;
#pragma unroll
      for (int s = 0; s < NSM; ++s)
        if (s == nsteps - 1) {
          f0 = c0 ? u0[s] : INFINITY;
          f1 = c1 ? u1[s] : INFINITY;
        }
      int64_t i0 = c0 ? id0 : INT64_MAX, i1 = c1 ? id1 : INT64_MAX;
      // element e = lane (f0) and e = lane + 32 (f1); ascending (dist, id)
      for (int size = 2; size <= 64; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          if (stride == 32) {  // partners are f0/f1 of the same lane
            const bool asc = true;  // size == 64: one ascending sequence
            const bool sw = pair_less(f1, i1, f0, i0) == asc;
            if (sw) {
              const float tf = f0; f0 = f1; f1 = tf;
              const int64_t tt = i0; i0 = i1; i1 = tt;
            }
          } else {
            auto cx = [&](float& f, int64_t& id, int e) {
              const float of = __shfl_xor_sync(kFull, f, stride);
              const int64_t oi = __shfl_xor_sync(kFull, id, stride);
              const bool lower = (e & stride) == 0;
              const bool asc = (e & size) == 0;
              const bool mine_less = pair_less(f, id, of, oi);
              const bool keep = (lower == asc) ? mine_less : !mine_less;
              if (!keep) { f = of; id = oi; }
            };
            cx(f0, i0, lane);
            cx(f1, i1, lane + 32);
          }
        }
      }
      const int n = min(k, m);
      if (RK) {
        rd = f0;
        ri = i0;
        rn = n;
        T = rk_threshold();
      } else {
        if (lane < n) { tkd[lane] = f0; tki[lane] = i0; }
        if (lane + 32 < n) { tkd[lane + 32] = f1; tki[lane + 32] = i1; }
        if (lane == 0) ctl.n = n;
        __syncwarp();
        T = topk_threshold(ctl, k, tkd);
      }
      c0 = c1 = false;
    }
    if (__any_sync(kFull, c0 || c1)) {  // push the block's survivors (search.py:173-174)
      float f0 = 0.f, f1 = 0.f;  // the partial at the last step is the distance
#pragma unroll
      for (int s = 0; s < NSM; ++s)
        if (s == nsteps - 1) {
          f0 = u0[s];
          f1 = u1[s];
        }
      if (RK) {
        rk_push(c0, f0, id0);
        rk_push(c1, f1, id1);
        T = rk_threshold();
      } else {
        topk_push_lanes(ctl, k, tkd, tki, c0, f0, id0, lane);
        topk_push_lanes(ctl, k, tkd, tki, c1, f1, id1, lane);
        __syncwarp();
        T = topk_threshold(ctl, k, tkd);
      }
    }
  }
  __syncwarp();
  if (RK) {
    if (dead) rn = 0;
    if (lane < k) {
      A.out_dist[(int64_t)q * k + lane] = lane < rn ? rd : INFINITY;
      A.out_ids[(int64_t)q * k + lane] = lane < rn ? ri : -1;
    }
    if (lane == 0) {
      A.out_count[q] = rn;
      if (A.out_touched) A.out_touched[q] = touched;
      if (A.out_total) A.out_total[q] = total;
      if (A.trace_len) A.trace_len[q] = tlen;
    }
    btprime_query(P, A, q, rk_threshold(), lane);
    if (P.dbg && ready && lane == 0) A.ptouched[2 * q + 1] = (uint32_t)(gtimer_ns() >> 7);
    continue;
  }
  const int n = dead ? 0 : ctl.n;
  for (int i = lane; i < k; i += 32) {
    A.out_dist[(int64_t)q * k + i] = i < n ? tkd[i] : INFINITY;
    A.out_ids[(int64_t)q * k + i] = i < n ? tki[i] : -1;
  }
  if (lane == 0) {
    A.out_count[q] = n;
    if (A.out_touched) A.out_touched[q] = touched;
    if (A.out_total) A.out_total[q] = total;
    if (A.trace_len) A.trace_len[q] = tlen;
  }
  btprime_query(P, A, q, n >= k ? tkd[k - 1] : INFINITY, lane);
  __syncwarp();
  }  // queries of this warp
}

template <int NSM, bool RK, bool ST = true>
__global__ void __launch_bounds__(256) bchain1_kernel(const BParams P, const BArgs A,
                                                      const float* __restrict__ part1,
                                                      const int32_t* __restrict__ ready) {
  bchain1_cta<NSM, RK, ST>(P, A, part1, blockIdx.x, gridDim.x, ready);
}

// ------------------------------------------------------------ phase 2 scan
// Head schedule known at compile time: initial_step IS, step s ends after
// dim IS * (2^(s+1) - 1) (step_schedule, search.py:106-117) while <= 16.
// IS = 0 is the run-time version (any schedule, d < 16).
template <int IS>
struct HeadSched {
  static constexpr int n = IS == 0 ? 0
                           : (15 * IS <= kHeadDims) ? 4
                           : (7 * IS <= kHeadDims)  ? 3
                           : (3 * IS <= kHeadDims)  ? 2
                           : (IS <= kHeadDims)      ? 1
                                                    : 0;
  static constexpr int dims = n > 0 ? ((2 << (n - 1)) - 1) * IS : 0;
  __host__ __device__ static constexpr int step_at(int e) {  // step ending after dim e
    return (n >= 1 && e + 1 == IS)       ? 0
           : (n >= 2 && e + 1 == 3 * IS) ? 1
           : (n >= 3 && e + 1 == 7 * IS) ? 2
           : (n >= 4 && e + 1 == 15 * IS) ? 3
                                          : -1;
  }
};

// A pair is uncertain (its decisions may differ between T' and T^) unless
// T^ == T' or every (slot, step) surviving under T' has v_s < B_s(T^): rho
// bounds v_s / beta_s and kRhoSlack covers the rounding of rho, beta_s and
// B_s.
__device__ __forceinline__ bool pair_uncertain(float that, float tp, float rho) {
  return that < tp && !(that >= 1e-30f && __fmul_rn(rho, kRhoSlack) < that);
}

// T^ before pair `pl` of query q: tafter of the last survivor of an earlier
// pair in the query's pair-sorted list, else T'.
__device__ __forceinline__ float that_of(const BSurv* sv, int n, int pl, float tp) {
  int lo = 0, hi = n;  // first entry with pair >= pl
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sv[mid].pair < pl) lo = mid + 1; else hi = mid;
  }
  return lo > 0 ? sv[lo - 1].tafter : tp;
}

__device__ __forceinline__ void confirm_survivor(const BParams& P, const BArgs& A, int q, int pl,
                                                 int slot) {
  BSurv* sv = A.surv + (int64_t)q * P.surv_cap;
  const int n = min(A.nsurv[q], P.surv_cap);
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sv[mid].pair < pl) lo = mid + 1; else hi = mid;
  }
  for (; lo < n && sv[lo].pair == pl; ++lo)
    if (sv[lo].slot == slot) {
      sv[lo].real = 1;
      return;
    }
  A.flags[q] = 1;  // not a T'-survivor: cannot happen (T^ <= T'); fall back
}

// One CTA per work item (a bucket and up to kQC queries probing it).  Warp w
// takes tiles w, w + kBW, ... of the bucket; per tile, lane l holds the head
// dims of slots l and l + 32 in registers and loops over the queries.
// Slots alive after the head become deep items, finished one per lane.
// MODE 0: every pair under B_s(T').  MODE 1: only the uncertain pairs, under
// B_s(T^_p) — their stats are overwritten and their real survivors confirmed.
// DENSE (d > 256): after the head, every live query of a tile advances
// together group by group (the group loaded once per warp, per-query
// accumulators in shared memory) until few live slots remain; otherwise
// the head's survivors go straight to the one-lane-per-survivor queue.
// ST: the pairs' statistics (survivor counts per step, values_touched,
// traces) are kept; a results-only search (MODE 0 before bverify_kernel)
// needs only rho and the T'-survivors.
template <int IS, bool BSA, int MODE, bool DENSE, bool ST = true>
__global__ void __launch_bounds__((DENSE ? kBWD : kBW) * 32, DENSE ? 4 : PDX_BSCAN_MIN_BLOCKS)
    bscan_kernel(const BParams P, const BArgs A) {
  constexpr int BW = DENSE ? kBWD : kBW;  // warps per CTA
  __shared__ __align__(16) float s_qh[kQC][kHeadDims];
  __shared__ __align__(16) float s_bnd[kQC][kMaxSteps];
  __shared__ float s_bq[BSA ? kQC : 1][2][kMaxHead];  // BSA head: rq_s, sqrt(rq_s)
  __shared__ int32_t s_qid[kQC], s_base[kQC];
  __shared__ int64_t s_qo[kQC];
  __shared__ float s_tp[kQC];
  __shared__ uint32_t s_hcnt[BW][kQC];             // head-step counts, one byte per step
  __shared__ uint32_t s_dcnt[BW][kQC][kMaxSteps];  // deep-step counts
  __shared__ uint32_t s_rho[BW][kQC];
  __shared__ float s_that[BW][kQC];                // MODE 1: T^ of this tile's pairs
  __shared__ float s_that0[kQC];                     // MODE 1: T^ at the bucket's first pair
  __shared__ uint32_t s_jvar, s_jmay;                // MODE 1: T^ varies in the bucket / may be < T'
  __shared__ uint32_t s_todo[MODE == 1 ? kTodoCap : 1];  // MODE 1: uncertain queries per tile
  __shared__ DeepItem s_deep[BW][kDeepCap];
  extern __shared__ __align__(16) float s_accd[];  // DENSE: [BW][kQC][kTile] partials of live slots
  __shared__ uint32_t s_alm[DENSE ? BW : 1][kQC][2];  // DENSE: their alive masks (slot l, l + 32)
  __shared__ float s_rx[BSA ? BW : 1][kMaxHead][kTile];
  __shared__ int32_t s_ends[kMaxSteps], s_wmin[kTile + 1];
  __shared__ float s_invb[kMaxSteps], s_coef[kMaxSteps];
  __shared__ double s_ratio[kMaxSteps], s_band[kMaxSteps];

  __shared__ int s_itx;
  // one work item (the body returns early for an item with nothing to do)
  auto run_item = [&](const int itx) {
  const BItem it = A.items[itx];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ne = it.ne, nsteps = P.nsteps;
  const int64_t bk0 = A.bucket_block[it.bucket];
  const int tbeg = it.t0;  // this item's tiles of the bucket: [tbeg, tend); ti below is local
  const int tend = min((int)(A.bucket_block[it.bucket + 1] - bk0), tbeg + kTC);
  const int nt = tend - tbeg;
  const int64_t b0 = bk0 + tbeg;  // block (= tile, 64-blocks) of local tile 0
  const int64_t t0 = A.block_tile[b0];
  if (MODE == 1) {
    if (threadIdx.x < 32) {
      const int j = threadIdx.x;
      bool may = false, var = false;
      if (j < ne) {
        const BEntry en = A.entries[it.e0 + j];
        if (!A.flags[en.q]) {
          const BSurv* sv = A.surv + (int64_t)en.q * P.surv_cap;
          const int n = min(A.nsurv[en.q], P.surv_cap);
          const float tp = A.tprime[en.q];
          const float t0 = that_of(sv, n, en.base + tbeg, tp);
          const float t1 = that_of(sv, n, en.base + tbeg + nt - 1, tp);
          s_that0[j] = t0;
          var = t1 != t0;
          may = t0 < tp || t1 < tp;
        }
      }
      const unsigned mm = __ballot_sync(kFull, may), vv = __ballot_sync(kFull, var);
      if (j == 0) {
        s_jmay = mm;
        s_jvar = vv;
      }
    }
    __syncthreads();
    if (s_jmay == 0) return;  // every pair of this item is certain
    if (P.dbg && threadIdx.x == 0) atomicAdd(const_cast<int32_t*>(A.nitems) + 4, 1);
  }
  for (int i = threadIdx.x; i < ne * kHeadDims; i += blockDim.x) {
    const int j = i / kHeadDims, e = i % kHeadDims;
    const int q = A.entries[it.e0 + j].q;
    s_qh[j][e] = e < P.d ? A.queries[(int64_t)q * P.d + e] : 0.f;
  }
  if (MODE == 0)
    for (int i = threadIdx.x; i < ne * nsteps; i += blockDim.x) {
      const int j = i / nsteps, s = i % nsteps;
      s_bnd[j][s] = A.bounds[(int64_t)A.entries[it.e0 + j].q * nsteps + s];
    }
  if (BSA)
    for (int i = threadIdx.x; i < ne * P.hsteps; i += blockDim.x) {
      const int j = i / P.hsteps, s = i % P.hsteps;
      const float* bq = A.bsaq + (int64_t)A.entries[it.e0 + j].q * 2 * nsteps;
      s_bq[j][0][s] = bq[s];
      s_bq[j][1][s] = bq[nsteps + s];
    }
  for (int j = threadIdx.x; j < ne; j += blockDim.x) {
    const BEntry en = A.entries[it.e0 + j];
    s_qid[j] = en.q;
    s_base[j] = en.base + tbeg;  // pair index of local tile 0
    s_qo[j] = A.qoff[en.q];
    s_tp[j] = A.tprime[en.q];
  }
  for (int i = threadIdx.x; i < kMaxSteps; i += blockDim.x) {
    s_ends[i] = P.ends[i];
    s_invb[i] = P.invb[i];
    s_ratio[i] = P.ratio[i];
    s_band[i] = P.band[i];
    s_coef[i] = (BSA && i < nsteps) ? A.coef[i] : 0.f;
  }
  for (int i = threadIdx.x; i <= kTile; i += blockDim.x) s_wmin[i] = P.wmin[i];
  __syncthreads();

  if (MODE == 1 && nt <= kTodoCap) {  // which (query, tile) pairs are uncertain, all at once
    for (int i = threadIdx.x; i < nt; i += blockDim.x) s_todo[i] = 0u;
    __syncthreads();
    for (int i = threadIdx.x; i < ne * nt; i += blockDim.x) {
      const int j = i / nt, ti = i - j * nt;
      if (!((s_jmay >> j) & 1u)) continue;
      const int pl = s_base[j] + ti;
      if (pl < 0) continue;
      float that = s_that0[j];
      if ((s_jvar >> j) & 1u) {
        const int q = s_qid[j];
        that = that_of(A.surv + (int64_t)q * P.surv_cap, min(A.nsurv[q], P.surv_cap), pl, s_tp[j]);
      }
      if (pair_uncertain(that, s_tp[j], A.prho[s_qo[j] + pl])) atomicOr(&s_todo[ti], 1u << j);
    }
    __syncthreads();
  }
  constexpr int HS = HeadSched<IS>::n, HD = HeadSched<IS>::dims;
  const int hs = IS ? HS : P.hsteps, hd = IS ? HD : P.hdims;
  const float ib0 = s_invb[0], ib1 = s_invb[1], ib2 = s_invb[2], ib3 = s_invb[3];
  for (int ti = w; ti < nt; ti += BW) {
    const int64_t tile = t0 + ti;
    // MODE 1: which queries of this tile are uncertain (bit j)
    uint32_t todo = __ballot_sync(kFull, lane < ne && s_base[lane] + ti >= 0);
    if (!todo) continue;  // (tiles of a first bucket that phase 1 covered)
    if (MODE == 1 && nt <= kTodoCap) {
      todo = s_todo[ti];
      if (!todo) continue;
      if (P.dbg && lane == 0) {
        atomicAdd(const_cast<int32_t*>(A.nitems) + 5, 1);
        atomicAdd(const_cast<int32_t*>(A.nitems) + 6, __popc(todo));
      }
      if ((todo >> lane) & 1u) {
        float that = s_that0[lane];
        if ((s_jvar >> lane) & 1u) {
          const int q = s_qid[lane];
          that = that_of(A.surv + (int64_t)q * P.surv_cap, min(A.nsurv[q], P.surv_cap),
                         s_base[lane] + ti, s_tp[lane]);
        }
        s_that[w][lane] = that;
      }
      __syncwarp();
    } else if (MODE == 1) {
      bool unc = false;
      if (((s_jmay >> lane) & 1u) && s_base[lane] + ti >= 0) {
        const int q = s_qid[lane], pl = s_base[lane] + ti;
        float that = s_that0[lane];
        if ((s_jvar >> lane) & 1u) {
          const BSurv* sv = A.surv + (int64_t)q * P.surv_cap;
          that = that_of(sv, min(A.nsurv[q], P.surv_cap), pl, s_tp[lane]);
        }
        unc = pair_uncertain(that, s_tp[lane], A.prho[s_qo[lane] + pl]);
        if (unc) s_that[w][lane] = that;
      }
      todo = __ballot_sync(kFull, unc);
      if (!todo) continue;
      __syncwarp();
    }
    const int m = A.block_m[b0 + ti];
    const float* __restrict__ tb = A.tiles + tile * A.tile_stride;
    float x0[kHeadDims], x1[kHeadDims];
    ldg8(tb + lane * 8, *reinterpret_cast<float(*)[8]>(x0));
    ldg8(tb + (32 + lane) * 8, *reinterpret_cast<float(*)[8]>(x1));
    if ((IS ? HD : kHeadDims) > 8 && P.d_pad > 8) {
      ldg8(tb + (kTile + lane) * 8, *reinterpret_cast<float(*)[8]>(x0 + 8));
      ldg8(tb + (kTile + 32 + lane) * 8, *reinterpret_cast<float(*)[8]>(x1 + 8));
    } else {
#pragma unroll
      for (int e = 8; e < kHeadDims; ++e) x0[e] = x1[e] = 0.f;
    }
    if (BSA) {
      for (int s = 0; s < hs; ++s) {
        s_rx[w][s][lane] = __ldg(A.resid + ((size_t)tile * nsteps + s) * kTile + lane);
        s_rx[w][s][lane + 32] = __ldg(A.resid + ((size_t)tile * nsteps + s) * kTile + lane + 32);
      }
      __syncwarp();
    }
    unsigned long long xx[IS > 0 ? HD : 1];
    if (IS > 0) {
#pragma unroll
      for (int e = 0; e < (IS > 0 ? HD : 1); ++e) xx[e] = pack2_hold(x0[e], x1[e]);
    }
    const bool in0 = lane < m, in1 = lane + 32 < m;
    int qn = 0;  // deep items queued by this warp for this tile
    uint32_t live = 0;  // DENSE: queries with live slots after the head
    int nlive = 0;      // DENSE: live (query, slot) pairs

    // finish the queued deep items, one per lane (all belong to this tile and
    // sit at the same schedule position: they were queued together after the
    // head or the dense continuation).  Step by step: a pass over the queue
    // accumulates the step's dims for 32 items per warp iteration and takes
    // the step's decision; the survivors are compacted to the front of the
    // queue for the next step, so dead items stop costing lanes.
    auto flush = [&]() {
      __syncwarp();
      if (qn == 0) return;
      int n = qn;
      int s = s_deep[w][0].s, pos = s_deep[w][0].pos;
      const bool q4 = (P.d & 3) == 0;
      while (n > 0 && s < nsteps) {
        const int a = pos, bend = s_ends[s];
        int nn = 0;
        for (int base = 0; base < n; base += 32) {
          const bool act = base + lane < n;
          const DeepItem di = act ? s_deep[w][base + lane] : DeepItem{0.f, 0, 0, 0.f, 0, 0};
          const int j = di.j, slot = di.slot;
          const int q = s_qid[j];
          const float* __restrict__ qg = A.queries + (int64_t)q * P.d;
          float acc = di.acc;
          if (act) {
            for (int g = a >> 3; g * 8 < bend; ++g) {
              float x[8], qv[8];
              ldg8(tb + ((size_t)g * kTile + slot) * 8, x);
              if (q4 && g * 8 + 8 <= P.d) {
                const float4 u = ldg4(qg + g * 8), c = ldg4(qg + g * 8 + 4);
                qv[0] = u.x; qv[1] = u.y; qv[2] = u.z; qv[3] = u.w;
                qv[4] = c.x; qv[5] = c.y; qv[6] = c.z; qv[7] = c.w;
              } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) qv[e] = g * 8 + e < P.d ? __ldg(qg + g * 8 + e) : 0.f;
              }
              if (g * 8 >= a && g * 8 + 8 <= bend) {  // a whole group inside the step
#pragma unroll
                for (int e = 0; e < 8; ++e) acc = l2upd(acc, qv[e], x[e]);
              } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  const int dim = g * 8 + e;
                  if (dim >= a && dim < bend) acc = l2upd(acc, qv[e], x[e]);
                }
              }
            }
          }
          bool ok = false;
          if (act) {
            float v = acc;
            if (BSA) {
              const float* bq = A.bsaq + (int64_t)q * 2 * nsteps;
              v = bsa_est2(acc, __ldg(A.resid + ((size_t)tile * nsteps + s) * kTile + slot), bq[s],
                           bq[nsteps + s], s_coef[s]);
            }
            const float B = MODE == 0 ? s_bnd[j][s] : bound_at(P, di.that, s, s_ratio, s_band);
            ok = v < B;
            if (ok) {
              if (ST) atomicAdd(&s_dcnt[w][j][s], 1u);
              if (MODE == 0 && ST)
                atomicMax(&s_rho[w][j], __float_as_uint(fmaxf(__fmul_rn(v, s_invb[s]), 0.f)));
              if (s + 1 == nsteps) {
                if (MODE == 0)
                  record_survivor(P, A, q, s_base[j] + ti, acc, tile, slot);
                else
                  confirm_survivor(P, A, q, s_base[j] + ti, slot);
                ok = false;
              }
            }
          }
          // compact the survivors to the front (positions < base + 32: this
          // batch has been read by every lane, later batches are not touched)
          const unsigned keep = __ballot_sync(kFull, ok);
          __syncwarp();
          if (ok)
            s_deep[w][nn + __popc(keep & ((1u << lane) - 1u))] =
                DeepItem{acc, (int16_t)j, (int16_t)slot, di.that, (int16_t)(s + 1), (int16_t)bend};
          nn += __popc(keep);
          __syncwarp();
        }
        n = nn;
        pos = bend;
        ++s;
      }
      __syncwarp();
      qn = 0;
    };

    for (int j = lane; j < ne; j += 32)  // deep-step counters of this tile's pairs
      if ((todo >> j) & 1u)
        if (ST)
          for (int t = hs; t < nsteps; ++t) s_dcnt[w][j][t] = 0u;
    __syncwarp();
    for (uint32_t tm = todo; tm; tm &= tm - 1) {
      const int j = __ffs(tm) - 1;
      float bnd[kMaxHead];
      float that = 0.f;
      if (MODE == 0) {
        const float4 b4 = *reinterpret_cast<const float4*>(s_bnd[j]);
        bnd[0] = b4.x; bnd[1] = b4.y; bnd[2] = b4.z; bnd[3] = b4.w;
        bnd[4] = IS > 0 ? 0.f : s_bnd[j][4];
      } else {
        that = s_that[w][j];
        const float bl = lane < nsteps ? bound_at(P, that, lane, s_ratio, s_band) : 0.f;
#pragma unroll
        for (int s = 0; s < kMaxHead; ++s) bnd[s] = __shfl_sync(kFull, bl, s);
      }
      float acc0 = 0.f, acc1 = 0.f, rho = 0.f;
      float mx[kMaxHead] = {0.f, 0.f, 0.f, 0.f, 0.f};  // per head step: max surviving partial
      bool al0 = in0, al1 = in1;
      uint32_t cntl = 0;  // this lane's survivors per head step, one byte per step
      auto step = [&](int s, float ib) {
        float v0 = acc0, v1 = acc1;
        if (BSA) {
          v0 = bsa_est2(acc0, s_rx[w][s][lane], s_bq[j][0][s], s_bq[j][1][s], s_coef[s]);
          v1 = bsa_est2(acc1, s_rx[w][s][lane + 32], s_bq[j][0][s], s_bq[j][1][s], s_coef[s]);
        }
        const float B = bnd[s];
        al0 = al0 && v0 < B;
        al1 = al1 && v1 < B;
        if (MODE == 0 && ST) {
          if (IS > 0) {  // s is a compile-time constant here: v * ib is folded in once per pair
            if (al0) mx[s] = fmaxf(mx[s], v0);
            if (al1) mx[s] = fmaxf(mx[s], v1);
          } else {
            if (al0) rho = fmaxf(rho, __fmul_rn(v0, ib));
            if (al1) rho = fmaxf(rho, __fmul_rn(v1, ib));
          }
        }
        if (ST) cntl += (al0 ? 1u << (8 * s) : 0u) + (al1 ? 1u << (8 * s) : 0u);
      };
      if (IS > 0) {
        float qv[HD > 0 ? HD : 1];
#pragma unroll
        for (int i = 0; i < (HD + 3) / 4; ++i) {
          const float4 t = *reinterpret_cast<const float4*>(&s_qh[j][4 * i]);
          if (4 * i < HD) qv[4 * i] = t.x;
          if (4 * i + 1 < HD) qv[4 * i + 1] = t.y;
          if (4 * i + 2 < HD) qv[4 * i + 2] = t.z;
          if (4 * i + 3 < HD) qv[4 * i + 3] = t.w;
        }
        unsigned long long acc2 = pack2(0.f, 0.f);
#pragma unroll
        for (int e = 0; e < HD; ++e) {
          acc2 = sqacc2(acc2, qv[e], xx[e]);
          const int s = HeadSched<IS>::step_at(e);
          if (s >= 0) {
            const float2 a = unpack2(acc2);
            acc0 = a.x;
            acc1 = a.y;
            step(s, s == 0 ? ib0 : s == 1 ? ib1 : s == 2 ? ib2 : ib3);
            // every slot of the pair already pruned: the rest of the head
            // would only add dead dims (its counts stay 0, no deep items)
            if (s >= 1 && s + 1 < HS && !__any_sync(kFull, al0 || al1)) break;
          }
        }
      } else {
        int s = 0;
        const uint32_t hmask = P.hmask;
#pragma unroll
        for (int e = 0; e < kHeadDims; ++e) {
          if (e < hd) {
            const float qe = s_qh[j][e];
            acc0 = l2upd(acc0, qe, x0[e]);
            acc1 = l2upd(acc1, qe, x1[e]);
            if ((hmask >> e) & 1u) {
              step(s, s_invb[s]);
              ++s;
            }
          }
        }
      }
      if (ST) {
        const uint32_t packed = __reduce_add_sync(kFull, cntl);  // counts <= 64: no carries
        if (lane == 0) s_hcnt[w][j] = packed;
      }
      if (MODE == 0 && ST) {
        if (IS > 0) {  // max_s(max v_s * ib_s) = max over (slot, s) of v * ib: rounding is monotone
#pragma unroll
          for (int s = 0; s < HS; ++s)
            rho = fmaxf(rho, __fmul_rn(mx[s], s == 0 ? ib0 : s == 1 ? ib1 : s == 2 ? ib2 : ib3));
        }
        const uint32_t r = __reduce_max_sync(kFull, __float_as_uint(rho));
        if (lane == 0) s_rho[w][j] = r;
      }
      const int pl = s_base[j] + ti;
      if (hs == nsteps) {  // the whole schedule fits in the head (d <= 16)
        if (MODE == 0) {
          if (al0) record_survivor(P, A, s_qid[j], pl, acc0, tile, lane);
          if (al1) record_survivor(P, A, s_qid[j], pl, acc1, tile, lane + 32);
        } else {
          if (al0) confirm_survivor(P, A, s_qid[j], pl, lane);
          if (al1) confirm_survivor(P, A, s_qid[j], pl, lane + 32);
        }
      } else if (DENSE) {
        const unsigned m0 = __ballot_sync(kFull, al0), m1 = __ballot_sync(kFull, al1);
        s_accd[(w * kQC + j) * kTile + lane] = acc0;
        s_accd[(w * kQC + j) * kTile + lane + 32] = acc1;
        if (lane == 0) {
          s_alm[w][j][0] = m0;
          s_alm[w][j][1] = m1;
        }
        if (m0 | m1) live |= 1u << j;
        nlive += __popc(m0) + __popc(m1);
      } else {
        const unsigned m0 = __ballot_sync(kFull, al0), m1 = __ballot_sync(kFull, al1);
        const int n = __popc(m0) + __popc(m1);
        if (n) {
          if (qn + n > kDeepCap) flush();
          const unsigned lt = (1u << lane) - 1u;
          const int pre = qn + __popc(m0 & lt) + __popc(m1 & lt);
          if (al0)
            s_deep[w][pre] = DeepItem{acc0, (int16_t)j, (int16_t)lane, that, (int16_t)hs, (int16_t)hd};
          if (al1)
            s_deep[w][pre + (al0 ? 1 : 0)] =
                DeepItem{acc1, (int16_t)j, (int16_t)(lane + 32), that, (int16_t)hs, (int16_t)hd};
          qn += n;
        }
      }
    }
    if constexpr (DENSE) {
      // ---- dense continuation: every live query advances together, group by
      // group (all share the schedule position), the tile's group loaded once
      {
        int s = hs, pos = hd;
        const int ngr = P.d_pad >> 3;
        __syncwarp();
        while (live) {
          if (nlive <= 32) {  // few left: one lane per survivor from here (flush)
            if (qn + nlive > kDeepCap) flush();
            for (uint32_t tm = live; tm; tm &= tm - 1) {
              const int j = __ffs(tm) - 1;
              const unsigned m0 = s_alm[w][j][0], m1 = s_alm[w][j][1];
              const bool a0 = (m0 >> lane) & 1u, a1 = (m1 >> lane) & 1u;
              const unsigned lt = (1u << lane) - 1u;
              const int pre = qn + __popc(m0 & lt) + __popc(m1 & lt);
              const float th = MODE == 1 ? s_that[w][j] : 0.f;
              if (a0)
                s_deep[w][pre] = DeepItem{s_accd[(w * kQC + j) * kTile + lane], (int16_t)j,
                                          (int16_t)lane, th, (int16_t)s, (int16_t)pos};
              if (a1)
                s_deep[w][pre + (a0 ? 1 : 0)] =
                    DeepItem{s_accd[(w * kQC + j) * kTile + lane + 32], (int16_t)j,
                             (int16_t)(lane + 32), th, (int16_t)s, (int16_t)pos};
              qn += __popc(m0) + __popc(m1);
            }
            flush();
            live = 0;
            break;
          }
          const int g = pos >> 3;
          if (g >= ngr) break;
          float xa[8], xb[8];
          ldg8(tb + ((size_t)g * kTile + lane) * 8, xa);
          ldg8(tb + ((size_t)g * kTile + 32 + lane) * 8, xb);
          unsigned long long xx2[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) xx2[e] = pack2_hold(xa[e], xb[e]);
          // step ends inside this group (the same for every query)
          uint32_t bm = 0;
          const int sg = s;
          for (int ss = s; ss < nsteps && s_ends[ss] <= g * 8 + 8; ++ss)
            bm |= 1u << (s_ends[ss] - 1 - g * 8);
          const int e0 = pos - g * 8;
          for (uint32_t tm = live; tm; tm &= tm - 1) {
            const int j = __ffs(tm) - 1;
            const int q = s_qid[j];
            const float* __restrict__ qg = A.queries + (int64_t)q * P.d + g * 8;
            float qv[8];
            if ((P.d & 3) == 0 && g * 8 + 8 <= P.d) {
              const float4 u = ldg4(qg), v = ldg4(qg + 4);
              qv[0] = u.x; qv[1] = u.y; qv[2] = u.z; qv[3] = u.w;
              qv[4] = v.x; qv[5] = v.y; qv[6] = v.z; qv[7] = v.w;
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) qv[e] = g * 8 + e < P.d ? __ldg(qg + e) : 0.f;
            }
            float a0 = s_accd[(w * kQC + j) * kTile + lane], a1 = s_accd[(w * kQC + j) * kTile + lane + 32];
            if (bm == 0) {  // no step ends in this group: the alive masks stay
              unsigned long long a2 = pack2(a0, a1);
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (e >= e0) a2 = sqacc2(a2, qv[e], xx2[e]);
              const float2 af = unpack2(a2);
              a0 = af.x;
              a1 = af.y;
              s_accd[(w * kQC + j) * kTile + lane] = a0;
              s_accd[(w * kQC + j) * kTile + lane + 32] = a1;
              continue;
            }
            const unsigned o0 = s_alm[w][j][0], o1 = s_alm[w][j][1];
            bool l0 = (o0 >> lane) & 1u, l1 = (o1 >> lane) & 1u;
            int se = sg;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              if (e >= e0) {
                const float2 d2 = sqdiff2(qv[e], xx2[e]);
                a0 = __fadd_rn(a0, d2.x);
                a1 = __fadd_rn(a1, d2.y);
                if ((bm >> e) & 1u) {  // step se ends after this dim (warp-uniform)
                  float v0 = a0, v1 = a1;
                  if (BSA) {
                    const float* rs = A.resid + ((size_t)tile * nsteps + se) * kTile;
                    const float* bq = A.bsaq + (int64_t)q * 2 * nsteps;
                    v0 = bsa_est2(a0, l0 ? __ldg(rs + lane) : 0.f, bq[se], bq[nsteps + se],
                                  s_coef[se]);
                    v1 = bsa_est2(a1, l1 ? __ldg(rs + lane + 32) : 0.f, bq[se], bq[nsteps + se],
                                  s_coef[se]);
                  }
                  const float B =
                      MODE == 0 ? s_bnd[j][se] : bound_at(P, s_that[w][j], se, s_ratio, s_band);
                  l0 = l0 && v0 < B;
                  l1 = l1 && v1 < B;
                  const int c = __popc(__ballot_sync(kFull, l0)) + __popc(__ballot_sync(kFull, l1));
                  if (MODE == 0 && ST) {
                    float r = 0.f;
                    if (l0) r = fmaxf(r, __fmul_rn(v0, s_invb[se]));
                    if (l1) r = fmaxf(r, __fmul_rn(v1, s_invb[se]));
                    const uint32_t rm = __reduce_max_sync(kFull, __float_as_uint(r));
                    if (lane == 0 && rm > s_rho[w][j]) s_rho[w][j] = rm;
                  }
                  if (ST && lane == 0) s_dcnt[w][j][se] = (uint32_t)c;
                  if (se == nsteps - 1) {  // the last step: survivors
                    if (MODE == 0) {
                      if (l0) record_survivor(P, A, q, s_base[j] + ti, a0, tile, lane);
                      if (l1) record_survivor(P, A, q, s_base[j] + ti, a1, tile, lane + 32);
                    } else {
                      if (l0) confirm_survivor(P, A, q, s_base[j] + ti, lane);
                      if (l1) confirm_survivor(P, A, q, s_base[j] + ti, lane + 32);
                    }
                    l0 = l1 = false;
                  }
                  ++se;
                }
              }
            }
            const unsigned m0 = __ballot_sync(kFull, l0), m1 = __ballot_sync(kFull, l1);
            nlive += (int)(__popc(m0) + __popc(m1)) - (int)(__popc(o0) + __popc(o1));
            __syncwarp();
            s_accd[(w * kQC + j) * kTile + lane] = a0;
            s_accd[(w * kQC + j) * kTile + lane + 32] = a1;
            if (lane == 0) {
              s_alm[w][j][0] = m0;
              s_alm[w][j][1] = m1;
            }
            if (!(m0 | m1)) live &= ~(1u << j);
            __syncwarp();
          }
          s = sg + __popc(bm);
          pos = (g + 1) * 8;
        }
        if (qn) flush();
      }
    } else {
      flush();
    }
    // the pairs' stats: values_touched (search.py:148-169) and trace counts
    for (int j = lane; j < ne; j += 32) {
      if (!((todo >> j) & 1u)) continue;
      const int64_t p = s_qo[j] + s_base[j] + ti;
      if (!ST) continue;  // (results only: every pair with T^ < T' is verified, no rho)
      const uint32_t hp = s_hcnt[w][j];
      int64_t touched = 0, prev = m;
      bool warm = true;
      int a = 0;
      for (int s = 0; s < nsteps; ++s) {
        const int w_s = s_ends[s] - a;
        a = s_ends[s];
        if (warm && prev >= s_wmin[m]) {
          touched += (int64_t)m * w_s;
        } else {
          warm = false;
          touched += prev * w_s;
        }
        prev = s < hs ? (int)((hp >> (8 * s)) & 0xffu) : (int)s_dcnt[w][j][s];
        if (A.pcnt) A.pcnt[p * nsteps + s] = (uint8_t)prev;
      }
      A.ptouched[p] = (uint32_t)touched;
      if (MODE == 0) A.prho[p] = __uint_as_float(s_rho[w][j]);
    }
    __syncwarp();
  }
  };
  if constexpr (MODE == 0) {  // one item per CTA: CTAs retire independently (no item barrier)
    if ((int)blockIdx.x < *A.nitems) run_item(blockIdx.x);
  } else {
    // MODE 1 (most items need little work): persistent CTAs pull work items
    // from a counter instead of launching the item-count upper bound
    for (;;) {
      __syncthreads();
      if (threadIdx.x == 0) s_itx = atomicAdd(A.wctr + MODE, 1);
      __syncthreads();
      const int itx = s_itx;
      if (itx >= *A.nitems) return;
      run_item(itx);
    }
  }
}

// ------------------------------------------- phase 2, results-only searches
// bscan0_kernel: MODE 0 of bscan_kernel for searches that output only ids and
// distances (ADS / BOND with a compile-time head schedule; d <= 256, and
// wider vectors under ADS): same work items, same T'-survivors with the same
// float32 distances — no pair statistics.  Two things differ from bscan_kernel's head:
//
// 1. The head is a FILTER.  Per (query, tile) pair it only discards slots
//    that the reference prunes at some head step for certain; everything
//    else is a candidate whose exact chain is evaluated later.  Slot x is
//    pruned at step s iff v_s >= B_s (v_s the per-op-rounded partial,
//    search.py:165).  In exact arithmetic V_s - B_s = XX_s + QQ_s - B_s -
//    2 DOT_s, so with h = (1 - c) / 2, c = 2^-17 = 128 u (u = 2^-24):
//        dot_s <= fl(h xx_s) + G_s,   G_s = fl(h (qq_s - B_s)) - (c |B_s| + floor)
//    implies v_s - B_s >= c (W + |B_s|) - (72.5 W + 4.04 |B_s|) u + floor > 0
//    (W = QQ_s + XX_s, n <= 16 head dims: |v - V| <= 2 (n + 2) u W; the dot
//    product, the norms and the threshold sum contribute ((2n + 4) W + 4 |B|)
//    u).  One FFMA2 per dim and slot pair (the dot products of two queries
//    interleaved), one FADD2 and two compares per step; the slots' prefix
//    norms are computed once per tile, G once per work item.  A tile or a
//    query with a non-finite or huge (>= 1e30) norm or bound skips the
//    filter: every slot is a candidate.
// 2. The candidates of a tile are expanded from the per-query ballot masks
//    (lane j keeps query j's masks) 32 at a time — one lane per candidate —
//    and each lane runs the reference's chain for its (query, slot) from dim
//    0 with __fsub_rn / __fmul_rn / __fadd_rn: the head dims and the rest of
//    the first 16 dims from shared memory (the tile's two first groups and
//    the queries' first 32 dims are staged there), every head decision and
//    the first deep step exactly as bscan_kernel takes them.  Survivors go to
//    the warp's queue and finish step by step with compaction, as there.
// Every decision that reaches the output is therefore taken on the
// per-op-rounded partials; the filter only saves evaluating slots whose
// pruning is certain.
constexpr float kFiltC = 7.62939453125e-06f;       // c = 2^-17
constexpr float kFiltH = 0.49999618530273438f;     // (1 - c) / 2, exact in float32
constexpr float kFiltFloor = 1e-30f;
constexpr float kFiltHuge = 1e30f;
#ifndef PDX_FILT_LAST_ONLY
#define PDX_FILT_LAST_ONLY 1
#endif
// The filter tests only the LAST head step: a slot pruned at an earlier head
// step almost always fails the last one too (the bounds tighten relative to
// the partials as dims accumulate), and the few that do not are discarded by
// their exact chains' head decisions — fewer filter instructions per pair
// for a few more candidates.
constexpr bool kFiltLastOnly = PDX_FILT_LAST_ONLY != 0;
#ifndef PDX_BSCAN0_MIN_BLOCKS
#define PDX_BSCAN0_MIN_BLOCKS 3
#endif
#ifndef PDX_FILT_NQ
#define PDX_FILT_NQ 2  // (4 measured: +5 us, register pressure)
#endif
constexpr int kFiltNQ = PDX_FILT_NQ;  // queries per filter call of the counted loop (2 or 4)
constexpr int kQRow = 36;  // floats per staged query row: 32 dims + 4 (rows of distinct queries in distinct banks)
constexpr int kXRow = 18;  // floats per staged slot row: 16 dims + 2 (9 8-byte words: consecutive slots in distinct banks)
constexpr int kBscan0Smem = kBW * kTile * kXRow * (int)sizeof(float);

template <int IS>
__global__ void __launch_bounds__(kBW * 32, PDX_BSCAN0_MIN_BLOCKS)
    bscan0_kernel(const BParams P, const BArgs A) {
  constexpr int HS = HeadSched<IS>::n, HD = HeadSched<IS>::dims;
  static_assert(HS >= 1 && HD <= 16, "compile-time head schedule");
  __shared__ __align__(16) float s_q[kQC][kQRow];
  __shared__ __align__(16) float s_bnd[kQC][kMaxSteps];
  __shared__ __align__(16) float s_g[kQC][4];
  __shared__ int32_t s_qid[kQC], s_base[kQC];
  __shared__ uint32_t s_qex;
  __shared__ unsigned long long s_hn[kBW][HS][32];
  __shared__ uint2 s_mm[kBW][kQC];  // candidate masks (slots l, l + 32) per query of the warp's tile
  __shared__ uint16_t s_dkey[kBW][kDeepCap];
  __shared__ float s_dacc[kBW][kDeepCap];
  __shared__ int32_t s_ends[kMaxSteps];
  extern __shared__ __align__(16) float s_xh[];  // [kBW][kTile][kXRow]

  if ((int)blockIdx.x >= *A.nitems) return;
  const BItem it = A.items[blockIdx.x];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ne = it.ne, nsteps = P.nsteps;
  const int64_t bk0 = A.bucket_block[it.bucket];
  const int tbeg = it.t0;
  const int tend = min((int)(A.bucket_block[it.bucket + 1] - bk0), tbeg + kTC);
  const int nt = tend - tbeg;
  const int64_t b0 = bk0 + tbeg;
  const int64_t t0 = A.block_tile[b0];

  // ---- stage the item's queries: first 32 dims, bounds, filter thresholds
  for (int i = threadIdx.x; i < ne * 32; i += blockDim.x) {
    const int j = i >> 5, e = i & 31;
    const int q = A.entries[it.e0 + j].q;
    s_q[j][e] = e < P.d ? A.queries[(int64_t)q * P.d + e] : 0.f;
  }
  for (int i = threadIdx.x; i < ne * nsteps; i += blockDim.x) {
    const int j = i / nsteps, s = i % nsteps;
    s_bnd[j][s] = A.bounds[(int64_t)A.entries[it.e0 + j].q * nsteps + s];
  }
  for (int i = threadIdx.x; i < kMaxSteps; i += blockDim.x) s_ends[i] = P.ends[i];
  if (threadIdx.x < 32) {  // (ne <= kQC = 32: one lane per query)
    bool ex = false;
    if ((int)threadIdx.x < ne) {
      const BEntry en = A.entries[it.e0 + threadIdx.x];
      s_qid[threadIdx.x] = en.q;
      s_base[threadIdx.x] = en.base + tbeg;  // pair index of local tile 0
      const float* __restrict__ qg = A.queries + (int64_t)en.q * P.d;
      float qq = 0.f;
#pragma unroll
      for (int e = 0; e < HD; ++e) {
        const float qe = __ldg(qg + e);
        qq = fmaf(qe, qe, qq);
        const int s = HeadSched<IS>::step_at(e);
        if (s >= 0) {
          const float B = A.bounds[(int64_t)en.q * nsteps + s];
          s_g[threadIdx.x][s] = kFiltH * (qq - B) - fmaf(kFiltC, fabsf(B), kFiltFloor);
          if (!(fabsf(B) < kFiltHuge)) ex = true;
        }
      }
      if (!(qq < kFiltHuge)) ex = true;
    }
    const unsigned mex = __ballot_sync(kFull, ex);
    if (threadIdx.x == 0) s_qex = mex;
  }
  __syncthreads();
  const uint32_t qex = s_qex;
  const int hs = HS;
  constexpr int E1C = IS * ((2 << HS) - 1);  // the first deep step's end when d reaches it
  static_assert(E1C > 16 && E1C <= 32, "first deep step inside the staged 32 dims");
  const int e1 = s_ends[hs];  // end of the first deep step: 16 <= e1 <= 32

  for (int ti = w; ti < nt; ti += kBW) {
    const int64_t tile = t0 + ti;
    const uint32_t todo = __ballot_sync(kFull, lane < ne && s_base[lane] + ti >= 0);
    if (!todo) continue;  // (tiles of a first bucket that phase 1 covered)
    const int m = A.block_m[b0 + ti];
    const float* __restrict__ tb = A.tiles + tile * A.tile_stride;
    unsigned long long xx[HD];
    bool tile_all = false;
    {
      float x0[16], x1[16];
      ldg8(tb + lane * 8, *reinterpret_cast<float(*)[8]>(x0));
      ldg8(tb + (32 + lane) * 8, *reinterpret_cast<float(*)[8]>(x1));
      ldg8(tb + (kTile + lane) * 8, *reinterpret_cast<float(*)[8]>(x0 + 8));
      ldg8(tb + (kTile + 32 + lane) * 8, *reinterpret_cast<float(*)[8]>(x1 + 8));
      // the first 16 dims of both slots, for the exact chains
      float* xa = s_xh + (size_t)(w * kTile + lane) * kXRow;
      float* xb = s_xh + (size_t)(w * kTile + 32 + lane) * kXRow;
#pragma unroll
      for (int e = 0; e < 16; e += 2) {
        *reinterpret_cast<float2*>(xa + e) = make_float2(x0[e], x0[e + 1]);
        *reinterpret_cast<float2*>(xb + e) = make_float2(x1[e], x1[e + 1]);
      }
#pragma unroll
      for (int e = 0; e < HD; ++e) xx[e] = pack2_hold(x0[e], x1[e]);
      // h * (prefix norms at the head step ends) of the slot pair
      unsigned long long n2 = pack2(0.f, 0.f);
#pragma unroll
      for (int e = 0; e < HD; ++e) {
        n2 = fma2(xx[e], xx[e], n2);
        const int s = HeadSched<IS>::step_at(e);
        if (s >= 0) {
          const float2 hn = unpack2(mul2(n2, bcast2(kFiltH)));
          s_hn[w][s][lane] = pack2(lane < m ? hn.x : INFINITY, lane + 32 < m ? hn.y : INFINITY);
        }
      }
      const float2 nl = unpack2(n2);
      tile_all = __any_sync(kFull, !(nl.x < kFiltHuge) || !(nl.y < kFiltHuge));
    }
    const uint32_t fex = tile_all ? 0xffffffffu : qex;
    __syncwarp();

    // ---- the filter: two queries per iteration; lane j keeps query j's masks
    // (slots past the block's m vectors carry a +inf norm: never candidates)
    // NQ queries per call: their dot-product chains are independent (ILP), the
    // tile's norms are read once
    auto filter = [&](auto nqc, const int (&jj)[4]) {
      constexpr int NQ = decltype(nqc)::value;
      unsigned long long dt[NQ];
      const float* __restrict__ qp[NQ];
#pragma unroll
      for (int u = 0; u < NQ; ++u) {
        dt[u] = pack2(0.f, 0.f);
        qp[u] = s_q[jj[u]];
      }
      bool a0[NQ], a1[NQ];
#pragma unroll
      for (int u = 0; u < NQ; ++u) a0[u] = a1[u] = true;
#pragma unroll
      for (int e = 0; e < HD; ++e) {
#pragma unroll
        for (int u = 0; u < NQ; ++u) dt[u] = fma2(xx[e], bcast2(qp[u][e]), dt[u]);
        const int s = HeadSched<IS>::step_at(e) == HS - 1 || !kFiltLastOnly ? HeadSched<IS>::step_at(e) : -1;
        if (s >= 0) {
          const unsigned long long hn = lds64(&s_hn[w][s][lane]);
#pragma unroll
          for (int u = 0; u < NQ; ++u) {
            const float2 th = unpack2(add2(hn, bcast2(s_g[jj[u]][s])));
            const float2 v = unpack2(dt[u]);
            a0[u] = a0[u] && v.x > th.x;
            a1[u] = a1[u] && v.y > th.y;
          }
        }
      }
      uint32_t m0[NQ], m1[NQ];
#pragma unroll
      for (int u = 0; u < NQ; ++u) {
        m0[u] = __ballot_sync(kFull, a0[u]);
        m1[u] = __ballot_sync(kFull, a1[u]);
      }
      if (fex) {  // a forced query (non-finite / huge norms) keeps every slot of the block
        const uint32_t inm0 = m >= 32 ? 0xffffffffu : (1u << m) - 1u;
        const uint32_t inm1 = m >= 64 ? 0xffffffffu : m > 32 ? (1u << (m - 32)) - 1u : 0u;
#pragma unroll
        for (int u = 0; u < NQ; ++u)
          if ((fex >> jj[u]) & 1u) {
            m0[u] = inm0;
            m1[u] = inm1;
          }
      }
      // (every lane stores the same words: no divergence; repeated queries of
      // a ragged last group store the same masks)
#pragma unroll
      for (int u = 0; u < NQ; ++u) s_mm[w][jj[u]] = make_uint2(m0[u], m1[u]);
    };
    if (todo == (ne >= 32 ? 0xffffffffu : (1u << ne) - 1u)) {  // every query of the item: a counted loop
      for (int j = 0; j < ne; j += kFiltNQ) {
        const int jj[4] = {j, min(j + 1, ne - 1), min(j + 2, ne - 1), min(j + 3, ne - 1)};
        filter(std::integral_constant<int, kFiltNQ>{}, jj);
      }
    } else {
      for (uint32_t tm = todo; tm;) {
        const int ja = __ffs(tm) - 1;
        tm &= tm - 1;
        const int jb = tm ? __ffs(tm) - 1 : ja;
        tm &= tm - 1;
        const int jj[4] = {ja, jb, jb, jb};
        filter(std::integral_constant<int, 2>{}, jj);
      }
    }
    __syncwarp();
    uint32_t mm0 = 0u, mm1 = 0u;  // lane j: query j's candidate masks
    if ((todo >> lane) & 1u) {
      const uint2 mm = s_mm[w][lane];
      mm0 = mm.x;
      mm1 = mm.y;
    }

    // ---- the candidates' exact chains
    int qn = 0;  // survivors of the first deep step queued by this warp
    const bool q4 = (P.d & 3) == 0;
    // finish the queued survivors step by step (all sit after step hs)
    auto drain = [&]() {
      __syncwarp();
      int n = qn, s = hs + 1, pos = e1;
      while (n > 0 && s < nsteps) {
        const int a = pos, bend = s_ends[s];
        int nn = 0;
        for (int base = 0; base < n; base += 32) {
          const bool act = base + lane < n;
          const uint32_t key = act ? s_dkey[w][base + lane] : 0u;
          const int j = key >> 8, slot = key & 0xffu;
          float acc = act ? s_dacc[w][base + lane] : 0.f;
          const float* __restrict__ qg = A.queries + (int64_t)s_qid[j] * P.d;
          if (act) {
            for (int g0 = a >> 3; g0 * 8 < bend; g0 += 2) {  // two groups in flight
              float x[2][8];
              ldg8(tb + ((size_t)g0 * kTile + slot) * 8, x[0]);
              const bool two = (g0 + 1) * 8 < bend;
              if (two) ldg8(tb + ((size_t)(g0 + 1) * kTile + slot) * 8, x[1]);
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                if (u == 1 && !two) break;
                const int g = g0 + u;
                float qv[8];
                if (q4 && g * 8 + 8 <= P.d) {
                  const float4 v0 = ldg4(qg + g * 8), v1 = ldg4(qg + g * 8 + 4);
                  qv[0] = v0.x; qv[1] = v0.y; qv[2] = v0.z; qv[3] = v0.w;
                  qv[4] = v1.x; qv[5] = v1.y; qv[6] = v1.z; qv[7] = v1.w;
                } else {
#pragma unroll
                  for (int e = 0; e < 8; ++e) qv[e] = g * 8 + e < P.d ? __ldg(qg + g * 8 + e) : 0.f;
                }
                if (g * 8 >= a && g * 8 + 8 <= bend) {  // a whole group inside the step
#pragma unroll
                  for (int e = 0; e < 8; ++e) acc = l2upd(acc, qv[e], x[u][e]);
                } else {
#pragma unroll
                  for (int e = 0; e < 8; ++e) {
                    const int dim = g * 8 + e;
                    if (dim >= a && dim < bend) acc = l2upd(acc, qv[e], x[u][e]);
                  }
                }
              }
            }
          }
          bool ok = act && acc < s_bnd[j][s];
          if (ok && s + 1 == nsteps) {
            record_survivor(P, A, s_qid[j], s_base[j] + ti, acc, tile, slot);
            ok = false;
          }
          const unsigned keep = __ballot_sync(kFull, ok);
          __syncwarp();
          if (ok) {
            const int at = nn + __popc(keep & ((1u << lane) - 1u));
            s_dkey[w][at] = (uint16_t)key;
            s_dacc[w][at] = acc;
          }
          nn += __popc(keep);
          __syncwarp();
        }
        n = nn;
        pos = bend;
        ++s;
      }
      __syncwarp();
      qn = 0;
    };

    const int cnt = __popc(mm0) + __popc(mm1);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
    const int ntot = __shfl_sync(kFull, incl, 31);
    for (int base = 0; base < ntot; base += 32) {
      const int idx = base + lane;
      const bool act = idx < ntot;
      int j = 0;  // the first query whose inclusive count exceeds idx
#pragma unroll
      for (int st = 16; st >= 1; st >>= 1) {
        const int v = __shfl_sync(kFull, incl, j + st - 1);
        if (v <= idx) j += st;
      }
      const int excl = __shfl_sync(kFull, incl - cnt, j);
      const uint32_t m0 = __shfl_sync(kFull, mm0, j), m1 = __shfl_sync(kFull, mm1, j);
      int slot = 0;
      if (act) {
        const int r = idx - excl, p0 = __popc(m0);
        const bool hi = r >= p0;  // (one n-th-bit search, over the half that holds it)
        slot = nth_bit(hi ? m1 : m0, hi ? r - p0 : r) + (hi ? 32 : 0);
      } else {
        j = 0;
      }
      // dims 16 .. e1 of the slot come from HBM / L2: issue the loads first
      float xg[2][8];
      if (act && e1 > 16) ldg8(tb + ((size_t)2 * kTile + slot) * 8, xg[0]);
      if (act && e1 > 24) ldg8(tb + ((size_t)3 * kTile + slot) * 8, xg[1]);
      const float* __restrict__ xr = s_xh + (size_t)(w * kTile + slot) * kXRow;
      const float* __restrict__ qr = s_q[j];
      float acc = 0.f;
      bool ok = act;
#pragma unroll
      for (int e = 0; e < 16; e += 4) {  // the reference's chain, per-op rounded; every head decision
        const float2 xa = *reinterpret_cast<const float2*>(xr + e);
        const float2 xb = *reinterpret_cast<const float2*>(xr + e + 2);
        const float4 qv = *reinterpret_cast<const float4*>(qr + e);
        const float xs[4] = {xa.x, xa.y, xb.x, xb.y}, qs[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc = l2upd(acc, qs[u], xs[u]);
          if (HeadSched<IS>::step_at(e + u) >= 0) ok = ok && acc < s_bnd[j][HeadSched<IS>::step_at(e + u)];
        }
      }
      if (e1 == E1C) {  // (d >= the schedule's step end: compile-time bounds, no per-dim tests)
        if (ok) {
#pragma unroll
          for (int e = 16; e < E1C; e += 4) {
            const float4 qv = *reinterpret_cast<const float4*>(qr + e);
            const float qs[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (e + u < E1C) acc = l2upd(acc, qs[u], xg[(e + u - 16) >> 3][(e + u) & 7]);
          }
        }
      } else if (e1 > 16) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (16 + u * 8 >= e1) break;
          if (ok) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (16 + u * 8 + e < e1) acc = l2upd(acc, qr[16 + u * 8 + e], xg[u][e]);
          }
        }
      }
      ok = ok && acc < s_bnd[j][hs];
      if (ok && hs + 1 == nsteps) {
        record_survivor(P, A, s_qid[j], s_base[j] + ti, acc, tile, slot);
        ok = false;
      }
      const unsigned keep = __ballot_sync(kFull, ok);
      if (ok) {
        const int at = qn + __popc(keep & ((1u << lane) - 1u));
        s_dkey[w][at] = (uint16_t)((j << 8) | slot);
        s_dacc[w][at] = acc;
      }
      qn += __popc(keep);
      if (qn > kDeepCap - 32) drain();
    }
    drain();
  }
}

// ------------------------------------------------------------------ chain
// One warp per query: sort its T'-survivors by pair and record, per entry,
// T^ after the pushes of its pair (the k-th smallest of H and the survivors
// of pairs up to it).  Pushing a T'-survivor the exact chain prunes leaves
// the k-th distance unchanged when its distance is >= T^ (bfinal_kernel
// checks that every such survivor is), so this is the reference's chain.
__device__ __forceinline__ void bchain_query(const BParams& P, const BArgs& A, const int q,
                                             const int lane, float* top, BSurv* ls) {
  const int n = min(A.nsurv[q], P.surv_cap);
  if (n == 0) return;
  const int k = P.k;
  BSurv* sv = A.surv + (int64_t)q * P.surv_cap;
  for (int i = lane; i < k; i += 32) top[i] = A.out_dist[(int64_t)q * k + i];
  // rank sort by (pair, list position), lane-parallel: O(n^2 / 32)
  for (int i = lane; i < n; i += 32) {
    const int pi = sv[i].pair;
    int r = 0;
    for (int j = 0; j < n; ++j) {
      const int pj = sv[j].pair;
      r += pj < pi || (pj == pi && j < i);
    }
    ls[r] = sv[i];
  }
  __syncwarp();
  if (k <= 32) {
    // the heap's distances in registers (lane l: the l-th smallest); a push
    // lands after the elements <= it, the rest shift up by one lane
    float t = lane < k ? top[lane] : INFINITY;
    for (int i = 0; i < n;) {
      const int pi = ls[i].pair;
      const float Tb = __shfl_sync(kFull, t, k - 1);
      int e = i;
      for (; e < n && ls[e].pair == pi; ++e) {
        const float dv = ls[e].dist;
        if (dv < __shfl_sync(kFull, t, k - 1)) {  // TopK.push, threshold value only
          const int pos = __popc(__ballot_sync(kFull, lane < k && t <= dv));
          const float up = __shfl_up_sync(kFull, t, 1);
          if (lane == pos) t = dv;
          else if (lane > pos && lane < k) t = up;
        }
      }
      const float T = __shfl_sync(kFull, t, k - 1);
      for (int j = i + lane; j < e; j += 32) {
        ls[j].tafter = T;
        ls[j].tbefore = Tb;
      }
      i = e;
    }
  } else if (lane == 0) {
    for (int i = 0; i < n;) {
      int e = i;
      const float Tb = top[k - 1];
      for (; e < n && ls[e].pair == ls[i].pair; ++e) {
        const float dv = ls[e].dist;
        if (dv < top[k - 1]) {  // TopK.push, threshold value only
          int j = k - 1;
          while (j > 0 && top[j - 1] > dv) {
            top[j] = top[j - 1];
            --j;
          }
          top[j] = dv;
        }
      }
      for (int j = i; j < e; ++j) {
        ls[j].tafter = top[k - 1];
        ls[j].tbefore = Tb;
      }
      i = e;
    }
  }
  __syncwarp();
  for (int i = lane; i < n; i += 32) sv[i] = ls[i];
}

__global__ void bchain_kernel(const BParams P, const BArgs A) {
  extern __shared__ float s_top[];  // [warps][k] then [warps][surv_cap] BSurv
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int q = blockIdx.x * nw + wq;
  if (q >= P.nq || A.flags[q]) return;
  bchain_query(P, A, q, lane, s_top + (size_t)wq * P.k,
               reinterpret_cast<BSurv*>(s_top + (size_t)nw * P.k + 4) + (size_t)wq * P.surv_cap);
}

// Results-only searches (no values_touched / traces requested): the only
// thing MODE 1 contributes to the ids and distances is which T'-survivors of
// uncertain pairs the exact chain keeps.  One thread per T'-survivor of such
// a pair recomputes that slot's chain — the same per-op-rounded partials at
// every step end and the same bounds B_s(T^_p) MODE 1 would use — and
// confirms it when it survives every step (bfinal drops the rest, and
// flags a query whose dropped survivor lies below T^_p, exactly as after
// MODE 1).  Pair statistics are not recomputed: they are not output.
template <bool BSA>
__device__ __forceinline__ void bverify_entry(const BParams& P, const BArgs& A, const int q,
                                              const int i, const int n) {
  BSurv* sv = A.surv + (int64_t)q * P.surv_cap;  // pair-sorted (bchain_kernel)
  const BSurv e = sv[i];
  const float tp = A.tprime[q];
  const float that = e.tbefore;  // (= that_of(sv, n, e.pair, tp))
  (void)n;
  if (!(P.norho ? that < tp : pair_uncertain(that, tp, A.prho[A.qoff[q] + e.pair]))) return;
  const float* __restrict__ tb = A.tiles + (int64_t)e.tile * A.tile_stride;
  const float* __restrict__ qg = A.queries + (int64_t)q * P.d;
  const float* bq = BSA ? A.bsaq + (int64_t)q * 2 * P.nsteps : nullptr;
  float acc = 0.f;
  int s = 0;
  int nend = P.ends[0];
  const int ng = (P.d + 7) >> 3;
  for (int g0 = 0; g0 < ng; g0 += 4) {  // four 8-dim groups in flight at a time
    float x[4][8], qv[4][8];
    const bool q4 = (P.d & 3) == 0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (g0 + u < ng) {
        ldg8(tb + ((size_t)(g0 + u) * kTile + e.slot) * 8, x[u]);
        const int g = g0 + u;
        if (q4 && g * 8 + 8 <= P.d) {  // the query's group with the slot's: all loads in flight together
          const float4 a = ldg4(qg + g * 8), b = ldg4(qg + g * 8 + 4);
          qv[u][0] = a.x; qv[u][1] = a.y; qv[u][2] = a.z; qv[u][3] = a.w;
          qv[u][4] = b.x; qv[u][5] = b.y; qv[u][6] = b.z; qv[u][7] = b.w;
        } else {
#pragma unroll
          for (int v8 = 0; v8 < 8; ++v8) qv[u][v8] = g * 8 + v8 < P.d ? __ldg(qg + g * 8 + v8) : 0.f;
        }
      }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (g0 + u >= ng) break;
#pragma unroll
      for (int v8 = 0; v8 < 8; ++v8) {
        const int dim = (g0 + u) * 8 + v8;
        if (dim >= P.d) break;
        acc = l2upd(acc, qv[u][v8], x[u][v8]);
        if (dim + 1 == nend) {
          float v = acc;
          if (BSA)
            v = bsa_est2(acc, __ldg(A.resid + ((size_t)e.tile * P.nsteps + s) * kTile + e.slot),
                         bq[s], bq[P.nsteps + s], A.coef[s]);
          if (!(v < bound_at(P, that, s, P.ratio, P.band))) return;  // the exact chain prunes it
          ++s;
          nend = s < P.nsteps ? P.ends[s] : 0x7fffffff;
        }
      }
    }
  }
  sv[i].real = 1;
}

template <bool BSA>
__global__ void __launch_bounds__(256) bverify_kernel(const BParams P, const BArgs A) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int q = (int)(gid / P.surv_cap), i = (int)(gid % P.surv_cap);
  if (q >= P.nq || A.flags[q]) return;
  const int n = min(A.nsurv[q], P.surv_cap);
  if (i >= n) return;
  bverify_entry<BSA>(P, A, q, i, n);
}

// ------------------------------------------------------------------ final
// One warp per unflagged query: survivors of uncertain pairs that the
// recompute pass did not confirm are dropped (or, below T^, flag the query);
// top-k of H and the real survivors; the stats.
__device__ __forceinline__ void bfinal_query(const BParams& P, const BArgs& A, const int q,
                                             const int lane, const int wq, unsigned char* s_raw) {
  const int k = P.k;
  const int nwb = blockDim.x >> 5;  // smem: td, hd | ti | hi | tsi | ts, each 16-byte aligned
  const size_t o_ti = ((size_t)nwb * 2 * k * 4 + 15) & ~(size_t)15;
  const size_t o_hi = o_ti + (size_t)nwb * k * 8;
  const size_t o_tsi = o_hi + (size_t)nwb * k * 8;
  const size_t o_ts = o_tsi + (size_t)nwb * P.surv_cap * 8;
  float* td = reinterpret_cast<float*>(s_raw) + (size_t)wq * 2 * k;
  float* hd = td + k;  // the heap (H) staged for the merge
  int64_t* ti = reinterpret_cast<int64_t*>(s_raw + o_ti) + (size_t)wq * k;
  int64_t* hid = reinterpret_cast<int64_t*>(s_raw + o_hi) + (size_t)wq * k;
  int64_t* tsi = reinterpret_cast<int64_t*>(s_raw + o_tsi) + (size_t)wq * P.surv_cap;
  float* ts = reinterpret_cast<float*>(s_raw + o_ts) + (size_t)wq * P.surv_cap;
  const int n = min(A.nsurv[q], P.surv_cap);
  BSurv* sv = A.surv + (int64_t)q * P.surv_cap;
  float* od = A.out_dist + (int64_t)q * k;
  int64_t* oi = A.out_ids + (int64_t)q * k;
  const int64_t p0 = A.qoff[q], p1 = A.qoff[q + 1];
  const float tp = A.tprime[q];
  // drop unconfirmed survivors of uncertain pairs (the list is pair-sorted)
  bool bad = false;
  for (int i = lane; i < n; i += 32) {
    const float that = sv[i].tbefore;  // (= that_of(sv, n, sv[i].pair, tp))
    const bool unc = P.norho ? that < tp : pair_uncertain(that, tp, A.prho[p0 + sv[i].pair]);
    if (unc && !sv[i].real) {
      if (sv[i].dist < that) bad = true;
      sv[i].real = -1;
    }
  }
  if (__any_sync(kFull, bad)) {
    if (lane == 0) A.flags[q] = 1;
    return;
  }
  __syncwarp();
  if (n > 0) {
    // real survivors ascending by (dist, id): lane-parallel rank sort (ids are
    // distinct), into the first nr entries of this warp's smem buffers
    int nr = 0;
    for (int i = lane; i < n; i += 32) {
      if (sv[i].real < 0) continue;
      const float di = sv[i].dist;
      const int64_t ii = sv[i].id;
      int r = 0;
      for (int j = 0; j < n; ++j)
        r += sv[j].real >= 0 && pair_less(sv[j].dist, sv[j].id, di, ii);
      ts[r] = di;
      tsi[r] = ii;
    }
    for (int i = lane; i < n; i += 32) nr += sv[i].real >= 0;
    nr = __reduce_add_sync(kFull, nr);
    __syncwarp();
    // merge of the heap (k entries, ascending) and the nr real survivors by
    // rank: the ids of the two lists are distinct (the heap holds vectors of
    // the first bucket), so an entry's output position is its own index plus
    // the number of entries of the other list below it
    for (int a = lane; a < k; a += 32) {
      hd[a] = od[a];
      hid[a] = oi[a];
    }
    __syncwarp();
    for (int a = lane; a < k; a += 32) {
      const float da = hd[a];
      const int64_t ia = hid[a];
      int lo = 0, hi = nr;  // survivors below (da, ia)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (pair_less(ts[mid], tsi[mid], da, ia)) lo = mid + 1; else hi = mid;
      }
      if (a + lo < k) {
        td[a + lo] = da;
        ti[a + lo] = ia;
      }
    }
    for (int b = lane; b < nr && b < k; b += 32) {
      const float db = ts[b];
      const int64_t ib = tsi[b];
      int lo = 0, hi = k;  // heap entries below (db, ib)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (pair_less(hd[mid], hid[mid], db, ib)) lo = mid + 1; else hi = mid;
      }
      if (b + lo < k) {
        td[b + lo] = db;
        ti[b + lo] = ib;
      }
    }
    __syncwarp();
    for (int r = lane; r < k; r += 32) {
      od[r] = td[r];
      oi[r] = ti[r];
    }
  }
  if (lane == 0 && A.out_count) A.out_count[q] = k;
  if (A.out_touched) {
    unsigned long long t = 0;
    for (int64_t p = p0 + lane; p < p1; p += 32) t += A.ptouched[p];
    t = __reduce_add_sync(kFull, (unsigned)(t & 0xffffffffu)) +
        ((unsigned long long)__reduce_add_sync(kFull, (unsigned)(t >> 32)) << 32);
    if (lane == 0) A.out_touched[q] += (int64_t)t;
  }
  if (A.out_total) {
    int64_t v = 0;
    const int fs = A.fseg[q];
    for (int s = fs + 1 + lane; s < P.nseg; s += 32) v += A.bnvec[A.sel[(int64_t)q * P.nseg + s]];
    const int64_t f0 = A.bucket_block[A.sel[(int64_t)q * P.nseg + fs]];
    const int nt0 = (int)(A.bucket_block[A.sel[(int64_t)q * P.nseg + fs] + 1] - f0);
    for (int ti = c_p1cap + lane; ti < nt0; ti += 32) v += A.block_m[f0 + ti];  // first-bucket tail
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    if (lane == 0) A.out_total[q] += v * P.d;
  }
  if (A.trace) {
    const int64_t tl = A.trace_len[q];
    const int64_t np = p1 - p0, rec = 1 + P.nsteps;
    const bool fits = tl >= 0 && tl + np * rec <= A.trace_cap;
    if (fits) {
      int32_t* tr = A.trace + (int64_t)q * A.trace_cap + tl;
      for (int64_t p = lane; p < np; p += 32) {
        tr[p * rec] = P.nsteps;
        for (int s = 0; s < P.nsteps; ++s) tr[p * rec + 1 + s] = A.pcnt[(p0 + p) * P.nsteps + s];
      }
    }
    if (lane == 0) A.trace_len[q] = fits ? tl + np * rec : -1;
  }
}

__global__ void bfinal_kernel(const BParams P, const BArgs A) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int q = blockIdx.x * (blockDim.x >> 5) + wq;
  if (q >= P.nq || A.flags[q]) return;
  bfinal_query(P, A, q, lane, wq, s_raw);
}

int schedule(int d, int initial_step, int32_t* ends) {
  int n = 0;
  int64_t start = 0, width = initial_step;
  while (start < d && n < kMaxSteps) {
    start = start + width < d ? start + width : d;
    ends[n++] = (int32_t)start;
    width *= 2;
  }
  return start < d ? -1 : n;
}

int host_warm_min(int m, double sf) {  // warm_min_count (pdx_scan_kernel.cuh)
  int p = (int)ceil(sf * (double)m);
  p = p < 0 ? 0 : (p > m ? m : p);
  while (p > 0 && (double)(p - 1) / (double)m >= sf) --p;
  while (p < m && (double)p / (double)m < sf) ++p;
  return p;
}

// A side stream and fork/join events for the planning kernels, per host
// thread and device: a call's record-then-wait on its fork event must not
// interleave with another thread's (the ABI allows concurrent calls on
// different streams); calls of one thread are ordered by the thread itself.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
// slot 0..3: the work-list stream of one pipeline instance; slots 4..7: the
// streams the query chunks of an overlapped batch run on; slots 8..11: the
// phase-1 chain stream of one pipeline instance
SideStream& side_stream(int slot = 0) {
  thread_local SideStream per_dev[16][16];
  int dev = 0;
  cudaGetDevice(&dev);
  SideStream& ss = per_dev[dev & 15][slot & 15];
  if (!ss.s) {
    // (a high-priority chain stream was measured: the overlap becomes
    // reliable for direct launches, but the replayed graph loses 17 us)
    cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming);
  }
  return ss;
}

// Phase timing of the batched pipeline (pdx_batch_profile): plan, phase 1,
// T', MODE 0, chain, MODE 1, final, fallback.
struct BatchProfile {
  static constexpr int kEv = 9;
  bool enabled = false;
  cudaEvent_t ev[kEv] = {};
  double ms[kEv] = {};
  int64_t calls = 0;
};
BatchProfile& batch_profile() {
  static BatchProfile p;
  return p;
}

// Device scratch one batched call may take (PDX_BATCH_SCRATCH_MB overrides;
// default 4 GiB, well inside 180 GB next to the largest store).
int64_t batch_scratch_budget() {
  static const int64_t b = [] {
    const char* e = getenv("PDX_BATCH_SCRATCH_MB");
    const long long mb = e ? atoll(e) : 0;
    return mb > 0 ? (int64_t)mb << 20 : (int64_t)4 << 30;
  }();
  return b;
}

template <typename T>
T* carve(unsigned char*& at, int64_t count) {
  T* p = reinterpret_cast<T*>(at);
  at += ((count * (int64_t)sizeof(T) + 255) / 256) * 256;
  return p;
}

}  // namespace

bool batched_eligible(const pdx_store* store, const pdx_search_params* prm, int64_t nq,
                      const int32_t* d_seg_bucket, int32_t nseg, const uint16_t* d_orders,
                      const pdx_search_out* out) {
  if (prm->batched == 1) return false;
  if (!d_seg_bucket || nseg < 2 || d_orders || store->group != 8) return false;
  if (store->ntiles != store->nblocks) return false;  // every block one tile (64-blocks)
  if (prm->pruner == PDX_PRUNER_NONE || prm->metric != PDX_METRIC_L2) return false;
  if (prm->splits > 1 || out->d_debug || prm->k > kMaxBatchK) return false;
  if (prm->initial_step > kHeadDims || store->d_pad > 8192) return false;
  // auto: batches of 32+ queries (C2 d = 128: 2.2x the per-query scan; with
  // the dense continuation for d > 256, C3 d = 960: 1.2-1.5x, C5-scaled
  // d = 768: BOND 1.34x, ADS 0.97x)
  if (prm->batched == 0 && nq < 32) return false;
  if (nq > (1 << 24)) return false;
  const int64_t pairs = nq * (int64_t)(nseg - 1) * store->max_bucket_tiles;
  return pairs <= (int64_t)1 << 31;
}

// One pipeline instance over queries [0, nq64) of the given arrays.  With
// flags_out the flagged queries are copied there (the caller runs the
// fallback once for all instances) instead of answered here; side_slot picks
// the work-list stream.
int search_batched_core(const pdx_store* store, const pdx_search_params* prm,
                        const float* d_queries, int64_t nq64, const int32_t* d_seg_bucket,
                        int32_t nseg, const pdx_search_out* out, void* d_work, int64_t work_bytes,
                        void* stream, int32_t* flags_out, int side_slot) {
  cudaStream_t st = as_stream(stream);
  const int nq = (int)nq64, k = prm->k, nb = store->nbuckets;
  BParams P;
  memset(&P, 0, sizeof(P));
  P.d = store->d;
  P.d_pad = store->d_pad;
  P.k = k;
  P.pruner = prm->pruner;
  P.nseg = nseg;
  P.nq = nq;
  P.nsteps = schedule(store->d, prm->initial_step, P.ends);
  PDX_REQUIRE(P.nsteps > 0, "step schedule too long");
  for (int s = P.nsteps; s < kMaxSteps; ++s) P.ends[s] = 0x7fffffff;
  const int ads_d = (prm->ads_d >= 1 && prm->pruner != PDX_PRUNER_BSA) ? prm->ads_d : store->d;
  for (int s = 0; s < P.nsteps; ++s) {  // bound_factors (pdx_scan.cu)
    double ratio = 1.0, band = 1.0;
    if (prm->pruner == PDX_PRUNER_ADS && P.ends[s] < ads_d) {
      ratio = (double)P.ends[s] / (double)ads_d;
      band = 1.0 + prm->ads_epsilon0 / sqrt((double)P.ends[s]);
    }
    P.ratio[s] = ratio;
    P.band[s] = band;
    P.invb[s] = (float)(1.0 / (ratio * band * band));
    if (P.ends[s] <= kHeadDims && P.hsteps < kMaxHead) {
      P.hsteps = s + 1;
      P.hdims = P.ends[s];
      P.hmask |= 1u << (P.ends[s] - 1);
    }
  }
  PDX_REQUIRE(P.hsteps >= 1, "batched search needs initial_step <= %d", kHeadDims);
  for (int m = 0; m <= kTile; ++m) P.wmin[m] = m > 0 ? host_warm_min(m, prm->selection_fraction) : 0;
  static const int p1cap = [] {
    const char* e = getenv("PDX_P1CAP");
    const int v = e ? atoi(e) : kP1Cap;
    const int c = v < 1 ? 1 : (v > kP1Cap ? kP1Cap : v);
    if (c != kP1Cap) cudaMemcpyToSymbol(c_p1cap, &c, sizeof(int));
    return c;
  }();
  static const int surv_extra = [] {
    const char* e = getenv("PDX_SURV_EXTRA");
    return e ? atoi(e) : 64;
  }();
  P.surv_cap = 4 * k + surv_extra;
  P.p1max = std::min(store->max_bucket_tiles, p1cap);
  P.dbg = getenv("PDX_BATCH_DEBUG") != nullptr;
  P.norho = !(out->d_touched || out->d_total || out->d_trace || getenv("PDX_FULL_MODE1"));
  const int64_t pmax = nq64 * nseg * store->max_bucket_tiles;
  const bool trace = out->d_trace != nullptr;
  // results only (no values_touched / traces requested): phase 1 and MODE 0
  // keep no pair statistics and bverify_kernel replaces the MODE 1 recompute
  const bool stats_wanted = out->d_touched || out->d_total || trace || getenv("PDX_FULL_MODE1");
  const int64_t nitems_max = (nb + (nq64 * nseg + kQC - 1) / kQC + 1) *
                             ((store->max_bucket_tiles + kTC - 1) / kTC);

  // cub scratch (three exclusive sums)
  size_t cub1 = 0, cub2 = 0;
  PDX_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, cub1, (int64_t*)nullptr, (int64_t*)nullptr,
                                                nq + 1, st));
  PDX_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, cub2, (int32_t*)nullptr, (int32_t*)nullptr,
                                                nb + 1, st));
  const size_t cubb = std::max(cub1, cub2);

  int64_t bytes = 0;
  {
    unsigned char* z = nullptr;
    unsigned char* at = z;
    carve<int32_t>(at, nq);                    // fseg
    carve<int64_t>(at, nq + 1);                // wcount
    carve<int64_t>(at, nq + 1);                // qoff
    carve<float>(at, nq64 * std::min(store->max_bucket_tiles, p1cap) * P.nsteps * kTile);  // part1
    carve<int32_t>(at, nq64 * nseg);           // pbase
    carve<int32_t>(at, nb + 1);                // bcnt     } zeroed by one memset
    carve<int32_t>(at, nb + 1);                // bcur     }
    carve<int32_t>(at, 8);                     // counters }
    carve<int32_t>(at, nq64 * std::min(store->max_bucket_tiles, p1cap) + 1);  // p1ready }
    carve<int32_t>(at, nb + 1);                // boff
    carve<int32_t>(at, nb + 1);                // nch
    carve<int32_t>(at, nb + 1);                // choff
    carve<int64_t>(at, nb + 1);                // bnvec
    carve<BEntry>(at, nq64 * nseg + 1);        // entries
    carve<BItem>(at, nitems_max);              // items
    carve<int32_t>(at, nq);                    // count scratch
    carve<float>(at, nq);                      // tprime
    carve<float>(at, nq64 * P.nsteps);         // bounds
    carve<float>(at, nq64 * 2 * P.nsteps);     // bsaq
    carve<int32_t>(at, nq);                    // flags
    carve<int32_t>(at, nq);                    // nsurv
    carve<BSurv>(at, nq64 * P.surv_cap);       // surv
    carve<uint32_t>(at, pmax + 1);             // ptouched
    carve<float>(at, pmax + 1);                // prho
    carve<uint8_t>(at, trace ? pmax * P.nsteps + 1 : 1);  // pcnt
    carve<unsigned char>(at, (int64_t)cubb + 16);
    bytes = at - z;
  }
  // Scratch grows linearly with the batch (part1 alone is nq x 64 tiles x
  // nsteps x 64 floats): a batch whose scratch exceeds the budget is answered
  // as two halves, each its own pipeline over the same store (results are
  // per query, so the split is invisible).  Traces index one flat buffer per
  // call and are not split.
  if (bytes > batch_scratch_budget() && nq64 >= 64 && !trace) {
    const int64_t h = nq64 / 2;
    pdx_search_out lo = *out, hi = *out;
    hi.d_dist = out->d_dist + h * k;
    hi.d_ids = out->d_ids + h * k;
    if (out->d_count) hi.d_count = out->d_count + h;
    if (out->d_touched) hi.d_touched = out->d_touched + h;
    if (out->d_total) hi.d_total = out->d_total + h;
    const int r0 = search_batched_core(store, prm, d_queries, h, d_seg_bucket, nseg, &lo, d_work,
                                       work_bytes, stream, flags_out, side_slot);
    if (r0 != PDX_OK) return r0;
    return search_batched_core(store, prm, d_queries + h * store->d, nq64 - h,
                               d_seg_bucket + h * nseg, nseg, &hi, d_work, work_bytes, stream,
                               flags_out ? flags_out + h : nullptr, side_slot);
  }
  unsigned char* base = nullptr;
  PDX_CUDA_CHECK(cudaMallocAsync(&base, bytes, st));
  unsigned char* at = base;
  int32_t* fseg = carve<int32_t>(at, nq);
  int64_t* wcount = carve<int64_t>(at, nq + 1);
  int64_t* qoff = carve<int64_t>(at, nq + 1);
  float* part1 = carve<float>(at, nq64 * std::min(store->max_bucket_tiles, p1cap) * P.nsteps * kTile);
  int32_t* pbase = carve<int32_t>(at, nq64 * nseg);
  int32_t* bcnt = carve<int32_t>(at, nb + 1);  // bcnt .. p1ready: zeroed by one memset
  int32_t* bcur = carve<int32_t>(at, nb + 1);
  int32_t* ctr = carve<int32_t>(at, 8);
  const int64_t p1ready_n = nq64 * std::min(store->max_bucket_tiles, p1cap) + 1;
  int32_t* p1ready = carve<int32_t>(at, p1ready_n);
  const unsigned char* zero_end = at;
  int32_t* boff = carve<int32_t>(at, nb + 1);
  int32_t* nch = carve<int32_t>(at, nb + 1);
  int32_t* choff = carve<int32_t>(at, nb + 1);
  int64_t* bnvec = carve<int64_t>(at, nb + 1);
  BEntry* entries = carve<BEntry>(at, nq64 * nseg + 1);
  BItem* items = carve<BItem>(at, nitems_max);
  int32_t* cnt_scratch = carve<int32_t>(at, nq);
  float* tprime = carve<float>(at, nq);
  float* bounds = carve<float>(at, nq64 * P.nsteps);
  float* bsaq = carve<float>(at, nq64 * 2 * P.nsteps);
  int32_t* flags = carve<int32_t>(at, nq);
  int32_t* nsurv = carve<int32_t>(at, nq);
  BSurv* surv = carve<BSurv>(at, nq64 * P.surv_cap);
  uint32_t* ptouched = carve<uint32_t>(at, pmax + 1);
  float* prho = carve<float>(at, pmax + 1);
  uint8_t* pcnt = carve<uint8_t>(at, trace ? pmax * P.nsteps + 1 : 1);
  void* cubtmp = carve<unsigned char>(at, (int64_t)cubb + 16);

  int rc = PDX_OK;
  const bool dbg_sync = getenv("PDX_BATCH_SYNC") != nullptr;
  // live phase timing (pdx_batch_profile): events on the main stream at
  // each phase boundary; not while the stream is being captured
  BatchProfile& prof = batch_profile();
  cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cap_st);
  // (while the stream is being captured the phase events become external
  // event-record nodes of the graph: pdx_batch_profile(2) reads them after a
  // replay)
  const bool capturing = cap_st != cudaStreamCaptureStatusNone;
  const bool timing = prof.enabled && !flags_out;
  int nev = 0;
  auto mark = [&]() {
    if (capturing)
      cudaEventRecordWithFlags(prof.ev[nev++], st, cudaEventRecordExternal);
    else
      cudaEventRecord(prof.ev[nev++], st);
  };
  if (timing) mark();
  auto phase = [&](const char* name) {
    if (timing && nev < BatchProfile::kEv) mark();
    if (!dbg_sync) return;
    const cudaError_t e = cudaStreamSynchronize(st);
    fprintf(stderr, "[pdx batched] %s done: %s\n", name, cudaGetErrorString(e));
  };
  // after the fork the side stream may still write into base: join it
  // before the free
  SideStream* forked = nullptr;
  SideStream* forked2 = nullptr;  // the phase-1 chain stream
  auto fail = [&](int r) {
    if (forked && cudaEventRecord(forked->join, forked->s) == cudaSuccess)
      cudaStreamWaitEvent(st, forked->join, 0);
    if (forked2 && cudaEventRecord(forked2->join, forked2->s) == cudaSuccess)
      cudaStreamWaitEvent(st, forked2->join, 0);
    cudaFreeAsync(base, st);
    return r;
  };
#define PDX_B_CHECK(expr)                                                                    \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess) {                                                                 \
      ::pdx::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e));   \
      return fail(PDX_ECUDA);                                                                \
    }                                                                                        \
  } while (0)

  // ---- plan: per-query windows, bucket-major entries, work items.  Phase 1
  // needs none of it (its kernels find each query's first bucket themselves,
  // its buffers have a fixed stride): the whole plan runs on a side stream
  // while phase 1 runs; the main stream only clears phase 1's ready flags and
  // joins before phase 2.
  SideStream& side = side_stream(side_slot);
  cudaStream_t st2 = side.s;
  PDX_B_CHECK(cudaEventRecord(side.fork, st));
  PDX_B_CHECK(cudaStreamWaitEvent(st2, side.fork, 0));
  forked = &side;
  PDX_B_CHECK(cudaMemsetAsync(bcnt, 0, reinterpret_cast<unsigned char*>(p1ready) -
                                           reinterpret_cast<unsigned char*>(bcnt), st2));
  PDX_B_CHECK(cudaMemsetAsync(p1ready, 0, zero_end - reinterpret_cast<unsigned char*>(p1ready), st));
  bprep_kernel<<<(nq + 7) / 8, 256, 0, st2>>>(d_seg_bucket, nq, nseg, store->d_bucket_block,
                                              store->d_block_tile, wcount, pbase, bcnt, fseg);
  PDX_B_CHECK(cudaGetLastError());
  size_t cb = cubb;
  PDX_B_CHECK(cub::DeviceScan::ExclusiveSum(cubtmp, cb, wcount, qoff, nq + 1, st2));
  cb = cubb;
  PDX_B_CHECK(cub::DeviceScan::ExclusiveSum(cubtmp, cb, bcnt, boff, nb + 1, st2));
  bchunks_kernel<<<(nb + 256) / 256, 256, 0, st2>>>(bcnt, nb, store->d_bucket_block,
                                                    store->d_block_m, nch, bnvec);
  PDX_B_CHECK(cudaGetLastError());
  cb = cubb;
  PDX_B_CHECK(cub::DeviceScan::ExclusiveSum(cubtmp, cb, nch, choff, nb + 1, st2));
  if (nq64 * nseg > 0) {
    bfill_kernel<<<(unsigned)((nq64 * nseg + 255) / 256), 256, 0, st2>>>(
        d_seg_bucket, nq, nseg, store->d_bucket_block, store->d_block_tile, pbase, boff, bcur,
        entries, fseg);
    PDX_B_CHECK(cudaGetLastError());
  }
  bitems_kernel<<<(nb + 256) / 256, 256, 0, st2>>>(bcnt, nb, boff, choff, store->d_bucket_block,
                                                   items, ctr);
  PDX_B_CHECK(cudaGetLastError());
  PDX_B_CHECK(cudaEventRecord(side.join, st2));
  phase("plan");

  pdx_search_out o1 = *out;
  if (!o1.d_count) o1.d_count = cnt_scratch;
  BArgs A;
  memset(&A, 0, sizeof(A));
  A.tiles = store->d_tiles;
  A.tile_ids = store->d_tile_ids;
  A.tile_stride = (int64_t)store->d_pad * kTile;
  A.bucket_block = store->d_bucket_block;
  A.block_tile = store->d_block_tile;
  A.block_m = store->d_block_m;
  A.queries = d_queries;
  A.sel = d_seg_bucket;
  A.fseg = fseg;
  A.resid = store->d_resid;
  A.coef = prm->bsa_coef;
  A.tprime = tprime;
  A.bounds = bounds;
  A.bsaq = bsaq;
  A.qoff = qoff;
  A.flags = flags;
  A.nsurv = nsurv;
  A.surv = surv;
  A.ptouched = ptouched;
  A.prho = prho;
  A.pcnt = trace ? pcnt : nullptr;
  A.items = items;
  A.nitems = ctr;
  A.wctr = ctr + 2;
  A.entries = entries;
  A.bnvec = bnvec;
  A.out_dist = out->d_dist;
  A.out_ids = out->d_ids;
  A.out_count = o1.d_count;
  A.out_touched = out->d_touched;
  A.out_total = out->d_total;
  A.trace = out->d_trace;
  A.trace_cap = out->trace_cap;
  A.trace_len = out->d_trace_len;

  const bool bsa = prm->pruner == PDX_PRUNER_BSA;
  // ---- phase 1: the first selected bucket of every query (exact chain)
  {
    const int p1max = std::min(store->max_bucket_tiles, p1cap);
    const dim3 g((unsigned)nq, (unsigned)((p1max + 3) / 4));
    const size_t sm = sizeof(float) * (store->d_pad + 2 * kMaxSteps);
    if (sm > 48 * 1024) {
      PDX_B_CHECK(cudaFuncSetAttribute(bdense_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      PDX_B_CHECK(cudaFuncSetAttribute(bdense_kernel<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    }
    // results only, k <= 32: the threshold chain (latency-bound, one warp per
    // query) runs underneath the dense pass — its kernel goes first, on a
    // second stream, with at most one persistent CTA per SM, and consumes a
    // tile as soon as the dense kernel has raised the tile's ready flag.  The
    // dense CTAs never wait, so there is no circular wait; a chain warp that
    // still waits after ~2 ms gives its query up to the per-query scan.
    // (PDX_P1_OVERLAP=0: the two kernels one after the other.)
    static const bool overlap_env = [] {
      const char* e = getenv("PDX_P1_OVERLAP");
      return e ? atoi(e) != 0 : true;
    }();
    int nsm = 148, dv = 0;
    cudaGetDevice(&dv);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dv);
    // (larger batches: the chain CTAs would have to take turns — the chain
    // kernel after the dense one, all its CTAs at once, is faster there)
    const bool overlap = overlap_env && !stats_wanted && k <= 32 && P.nsteps <= 12 && p1max > 0 &&
                         (nq + 7) / 8 <= nsm;
    const int nchain = (nq + 7) / 8;  // at most one chain CTA per SM
    const size_t hsm = (size_t)8 * k * (sizeof(float) + sizeof(int64_t));
    auto chain1 = [&](auto kern, cudaStream_t cs, int nblk, const int32_t* rdy) -> cudaError_t {
      if (hsm > 48 * 1024) {
        const cudaError_t e =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
        if (e != cudaSuccess) return e;
      }
      kern<<<nblk, 256, hsm, cs>>>(P, A, part1, rdy);
      return cudaGetLastError();
    };
    SideStream& cside = side_stream(8 + side_slot);
    if (p1max > 0) {
      if (overlap) {  // the chain first (its CTAs become resident), then the dense pass
        PDX_B_CHECK(cudaEventRecord(cside.fork, st));
        PDX_B_CHECK(cudaStreamWaitEvent(cside.s, cside.fork, 0));
        forked2 = &cside;
        if (P.nsteps <= 8)
          PDX_B_CHECK(chain1(bchain1_kernel<8, true, false>, cside.s, nchain, p1ready));
        else
          PDX_B_CHECK(chain1(bchain1_kernel<12, true, false>, cside.s, nchain, p1ready));
        PDX_B_CHECK(cudaEventRecord(cside.join, cside.s));
      }
      {
        int32_t* rdy = overlap ? p1ready : nullptr;
        if (bsa)
          bdense_kernel<true><<<g, 128, sm, st>>>(P, A, part1, rdy);
        else
          bdense_kernel<false><<<g, 128, sm, st>>>(P, A, part1, rdy);
        PDX_B_CHECK(cudaGetLastError());
      }
      if (overlap) {
        PDX_B_CHECK(cudaStreamWaitEvent(st, cside.join, 0));
        forked2 = nullptr;
      }
    }
    const bool rk = k <= 32;  // the heap in registers
    const int nq8 = (nq + 7) / 8;
    if (overlap && p1max > 0) {
      // (the chain ran underneath the dense pass)
    } else if (!stats_wanted && rk && P.nsteps <= 8)  // results only: no chain statistics
      PDX_B_CHECK(chain1(bchain1_kernel<8, true, false>, st, nq8, nullptr));
    else if (!stats_wanted && rk && P.nsteps <= 12)
      PDX_B_CHECK(chain1(bchain1_kernel<12, true, false>, st, nq8, nullptr));
    else if (P.nsteps <= 8)
      PDX_B_CHECK(rk ? chain1(bchain1_kernel<8, true>, st, nq8, nullptr)
                     : chain1(bchain1_kernel<8, false>, st, nq8, nullptr));
    else if (P.nsteps <= 12)
      PDX_B_CHECK(rk ? chain1(bchain1_kernel<12, true>, st, nq8, nullptr)
                     : chain1(bchain1_kernel<12, false>, st, nq8, nullptr));
    else
      PDX_B_CHECK(rk ? chain1(bchain1_kernel<kMaxSteps, true>, st, nq8, nullptr)
                     : chain1(bchain1_kernel<kMaxSteps, false>, st, nq8, nullptr));
  }
  if (P.dbg && getenv("PDX_P1_TIMING")) {  // development aid: the overlapped phase 1's timeline
    cudaStreamSynchronize(st);
    const int p1m = std::min(store->max_bucket_tiles, p1cap);
    std::vector<int32_t> fl((size_t)nq * p1m);
    std::vector<uint32_t> cs(2 * (size_t)nq);
    cudaMemcpy(fl.data(), p1ready, fl.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(cs.data(), ptouched, cs.size() * 4, cudaMemcpyDeviceToHost);
    uint32_t t0 = 0xffffffffu, dend = 0, cend = 0;
    for (int q = 0; q < nq; ++q) t0 = std::min(t0, cs[2 * q]);
    double lag = 0;
    for (int q = 0; q < nq; ++q) {
      uint32_t last = 0;
      for (int t = 0; t < p1m; ++t)
        if (fl[(size_t)q * p1m + t]) last = std::max(last, (uint32_t)fl[(size_t)q * p1m + t] - t0);
      dend = std::max(dend, last);
      cend = std::max(cend, cs[2 * q + 1] - t0);
      lag += (double)(cs[2 * q + 1] - t0) - last;
    }
    fprintf(stderr, "[pdx p1] dense end %.1f us, chain end %.1f us, mean chain lag after its last tile %.1f us\n",
            dend * 0.128, cend * 0.128, lag / nq * 0.128);
  }
  phase("phase1");
  PDX_B_CHECK(cudaStreamWaitEvent(st, side.join, 0));  // the work lists are ready
  forked = nullptr;
  phase("tprime");
  // ---- phase 2: every (query, tile) pair of the other buckets under T';
  // chain; recompute of the uncertain pairs under T^ (same kernel, MODE 1)
  const int is = (store->d >= kHeadDims) ? prm->initial_step : 0;
  auto scan = [&](int mode) -> cudaError_t {
    // wide vectors: survivors of the head are many and long — the dense
    // continuation variant (all live queries of a tile advance together)
    static const int dense_env = [] {
      const char* e = getenv("PDX_BSCAN_DENSE");
      return e ? atoi(e) : -1;
    }();
    const bool dense = dense_env >= 0 ? dense_env != 0 : store->d > 256;
    // results-only MODE 0 through the filtered head (PDX_BSCAN_FILTER=0: bscan_kernel)
    static const bool filt_env = [] {
      const char* e = getenv("PDX_BSCAN_FILTER");
      return e ? atoi(e) != 0 : true;
    }();
    // ... also for wide vectors (d > 256) under ADS, whose head leaves few
    // survivors (C3, d = 960: 620K -> 774K q/s); BOND on unrotated-energy data
    // prunes late, and the dense continuation stays faster there (C3: 151K
    // vs 131K q/s).  PDX_BSCAN_FILTER_WIDE=0/1 forces either.
    static const int filt_wide_env = [] {
      const char* e = getenv("PDX_BSCAN_FILTER_WIDE");
      return e ? atoi(e) : -1;
    }();
    const bool filt_wide =
        filt_wide_env >= 0 ? filt_wide_env != 0 : prm->pruner == PDX_PRUNER_ADS;
    int nsm = 148, dv = 0;
    cudaGetDevice(&dv);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dv);
    // MODE 0: one CTA per work item (upper bound; the extra CTAs exit);
    // MODE 1: persistent, about two CTAs per SM slot pull the items
    const dim3 g(mode == 0 ? (unsigned)nitems_max
                           : (unsigned)std::min<int64_t>(nitems_max, (int64_t)nsm * (dense ? 8 : 6)));
    const dim3 b(kBW * 32), bd(kBWD * 32);
    const int dsm = (int)(sizeof(float) * kBWD * kQC * kTile);
#define PDX_B_DENSE(IS, B, M, S)                                                       \
  {                                                                                    \
    auto fn = bscan_kernel<IS, B, M, true, S>;                                         \
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dsm);        \
    fn<<<g, bd, dsm, st>>>(P, A);                                                      \
  }
#define PDX_B_MODE0(IS, B, D)                                                          \
  {                                                                                    \
    if (D && !(filt_wide && !stats_wanted && !B && IS > 0 && filt_env)) {              \
      if (stats_wanted) PDX_B_DENSE(IS, B, 0, true) else PDX_B_DENSE(IS, B, 0, false)  \
    } else if (stats_wanted) {                                                         \
      bscan_kernel<IS, B, 0, false, true><<<g, b, 0, st>>>(P, A);                      \
    } else if (!B && IS > 0 && filt_env) {                                             \
      auto fn = bscan0_kernel<(IS > 0 ? IS : 1)>;                                      \
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kBscan0Smem); \
      fn<<<g, b, kBscan0Smem, st>>>(P, A);                                             \
    } else {                                                                           \
      bscan_kernel<IS, B, 0, false, false><<<g, b, 0, st>>>(P, A);                     \
    }                                                                                  \
  }
#define PDX_B_LAUNCH(IS)                                                               \
  if (mode == 0) {                                                                     \
    if (bsa) PDX_B_MODE0(IS, true, dense) else PDX_B_MODE0(IS, false, dense)           \
  } else if (dense) {                                                                  \
    if (bsa) PDX_B_DENSE(IS, true, 1, true) else PDX_B_DENSE(IS, false, 1, true)       \
  } else if (bsa) {                                                                    \
    bscan_kernel<IS, true, 1, false><<<g, b, 0, st>>>(P, A);                           \
  } else {                                                                             \
    bscan_kernel<IS, false, 1, false><<<g, b, 0, st>>>(P, A);                          \
  }
    switch (is) {
      case 1: PDX_B_LAUNCH(1) break;
      case 2: PDX_B_LAUNCH(2) break;
      case 4: PDX_B_LAUNCH(4) break;
      case 8: PDX_B_LAUNCH(8) break;
      default: PDX_B_LAUNCH(0) break;
    }
#undef PDX_B_LAUNCH
#undef PDX_B_MODE0
#undef PDX_B_DENSE
    return cudaGetLastError();
  };
  if (nitems_max > 0) PDX_B_CHECK(scan(0));
  phase("scan");
  const size_t fper = (size_t)2 * k * (sizeof(float) + sizeof(int64_t)) +
                      (size_t)P.surv_cap * (sizeof(float) + sizeof(int64_t));
  // one warp per query; its heap threshold and survivor list live in shared memory
  const size_t cper = (size_t)k * sizeof(float) + (size_t)P.surv_cap * sizeof(BSurv);
  const int cw = (int)std::max<size_t>(1, std::min<size_t>(8, (160u << 10) / cper));
  const size_t csm = cw * cper + 16;
  if (csm > 48 * 1024)
    PDX_B_CHECK(cudaFuncSetAttribute(bchain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)csm));
  bchain_kernel<<<(nq + cw - 1) / cw, cw * 32, csm, st>>>(P, A);
  PDX_B_CHECK(cudaGetLastError());
  phase("chain");
  if (!stats_wanted) {  // results only: verify the uncertain pairs' survivors
    const int64_t nt = nq64 * P.surv_cap;
    if (bsa)
      bverify_kernel<true><<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(P, A);
    else
      bverify_kernel<false><<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(P, A);
    PDX_B_CHECK(cudaGetLastError());
  } else if (nitems_max > 0) {
    PDX_B_CHECK(scan(1));
  }
  phase("recompute");
  const int fw = (int)std::max<size_t>(1, std::min<size_t>(8, (160u << 10) / fper));
  const size_t fsm = fw * fper + 32;
  if (fsm > 48 * 1024)
    PDX_B_CHECK(cudaFuncSetAttribute(bfinal_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)fsm));
  bfinal_kernel<<<(nq + fw - 1) / fw, fw * 32, fsm, st>>>(P, A);
  PDX_B_CHECK(cudaGetLastError());
  phase("final");
  // ---- fallback: flagged queries through the per-query scan
  if (flags_out) {
    PDX_B_CHECK(cudaMemcpyAsync(flags_out, flags, sizeof(int32_t) * nq, cudaMemcpyDeviceToDevice,
                                st));
  } else {
    rc = search_classic(store, prm, d_queries, nq64, d_seg_bucket, nseg, out, d_work, work_bytes,
                        stream, flags);
    if (rc != PDX_OK) return fail(rc);
  }
  phase("fallback");
  if (getenv("PDX_BATCH_DEBUG")) {  // development aid: work items, uncertain pairs, fallbacks
    int32_t h[8] = {0};
    std::vector<int32_t> fl(nq);
    cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(fl.data(), flags, sizeof(int32_t) * nq, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    int nf = 0;
    for (int32_t f : fl) nf += f != 0;
    fprintf(stderr,
            "[pdx batched] nq=%d items=%d fallback=%d mode1: active items %d, tiles %d, "
            "uncertain pairs %d\n",
            nq, h[0], nf, h[4], h[5], h[6]);
  }
  PDX_B_CHECK(cudaFreeAsync(base, st));
  if (timing && !capturing) {
    PDX_CUDA_CHECK(cudaEventSynchronize(prof.ev[nev - 1]));
    for (int i = 1; i < nev; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, prof.ev[i - 1], prof.ev[i]);
      prof.ms[i - 1] += ms;
    }
    prof.calls += 1;
  }
  return PDX_OK;
#undef PDX_B_CHECK
}


// The batch as `parts` query chunks, each its own pipeline instance on its
// own stream, forked from and joined back to the caller's: one chunk's
// latency-bound phases (phase 1, the chain) overlap another's issue-bound
// scan.  The fallback for every flagged query runs once after the join.
// PDX_BATCH_SPLIT=n sets the number of chunks (default 1: one instance).
int search_batched(const pdx_store* store, const pdx_search_params* prm, const float* d_queries,
                   int64_t nq64, const int32_t* d_seg_bucket, int32_t nseg,
                   const pdx_search_out* out, void* d_work, int64_t work_bytes, void* stream) {
  static const int split = [] {
    const char* e = getenv("PDX_BATCH_SPLIT");
    const int v = e ? atoi(e) : 1;
    return v < 1 ? 1 : (v > 4 ? 4 : v);
  }();
  const int parts = (int)std::min<int64_t>(split, nq64 / 128);
  if (parts <= 1 || out->d_trace || !out->d_count)
    return search_batched_core(store, prm, d_queries, nq64, d_seg_bucket, nseg, out, d_work,
                               work_bytes, stream, nullptr, 0);
  cudaStream_t st = as_stream(stream);
  const int k = prm->k;
  int32_t* flags_all = nullptr;
  PDX_CUDA_CHECK(cudaMallocAsync(&flags_all, sizeof(int32_t) * nq64, st));
  SideStream& root = side_stream(4);
  PDX_CUDA_CHECK(cudaEventRecord(root.fork, st));
  int rc = PDX_OK;
  for (int pi = 0; pi < parts && rc == PDX_OK; ++pi) {
    const int64_t q0 = nq64 * pi / parts, q1 = nq64 * (pi + 1) / parts;
    SideStream& ps = side_stream(4 + pi);
    PDX_CUDA_CHECK(cudaStreamWaitEvent(ps.s, root.fork, 0));
    pdx_search_out o = *out;
    o.d_dist = out->d_dist + q0 * k;
    o.d_ids = out->d_ids + q0 * k;
    o.d_count = out->d_count + q0;
    if (out->d_touched) o.d_touched = out->d_touched + q0;
    if (out->d_total) o.d_total = out->d_total + q0;
    rc = search_batched_core(store, prm, d_queries + q0 * store->d, q1 - q0,
                             d_seg_bucket + q0 * nseg, nseg, &o, d_work, work_bytes, ps.s,
                             flags_all + q0, pi);
    PDX_CUDA_CHECK(cudaEventRecord(ps.join, ps.s));
  }
  for (int pi = 0; pi < parts; ++pi) PDX_CUDA_CHECK(cudaStreamWaitEvent(st, side_stream(4 + pi).join, 0));
  if (rc != PDX_OK) {
    cudaFreeAsync(flags_all, st);
    return rc;
  }
  rc = search_classic(store, prm, d_queries, nq64, d_seg_bucket, nseg, out, d_work, work_bytes,
                      stream, flags_all);
  cudaFreeAsync(flags_all, st);
  return rc;
}

}  // namespace pdx

// Accumulated per-phase device time of batched searches since the last
// enable (CUDA events on the search stream; see include/pdx_b200.h).
extern "C" int pdx_batch_profile(int32_t enable, double* out_ms, int32_t cap, int64_t* out_calls) {
  pdx::BatchProfile& p = pdx::batch_profile();
  if (out_ms)
    for (int i = 0; i < cap && i < pdx::BatchProfile::kEv - 1; ++i) out_ms[i] = p.ms[i];
  if (out_calls) *out_calls = p.calls;
  if (enable == 2) {  // a replayed graph's phase events (the caller has synchronised)
    for (int i = 1; i < pdx::BatchProfile::kEv; ++i) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, p.ev[i - 1], p.ev[i]) == cudaSuccess) p.ms[i - 1] += ms;
    }
    cudaGetLastError();
    p.calls += 1;
    return PDX_OK;
  }
  if (enable >= 0) {
    if (enable && !p.ev[0])
      for (auto& e : p.ev) PDX_CUDA_CHECK(cudaEventCreate(&e));
    p.enabled = enable != 0;
    for (double& v : p.ms) v = 0.0;
    p.calls = 0;
  }
  return PDX_OK;
}