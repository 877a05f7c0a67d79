// Speculative tile scan for the compute warps of pdx_scan_kernel.
//
// A compute warp owns `tpw` consecutive tiles of a round.  For each tile it
// runs the DENSE phase — lane l owns slots l and l+32, the whole warp
// reads the live slots' dims group by group — until at most sparse_max of
// the tile's 64 slots survive.  Those survivors are parked in a
// warp-private list; after the warp's last tile the SPARSE phase finishes
// them one survivor per lane, so the long tail of the schedule (where a few
// of 64 slots live) runs on full warps instead of nearly empty ones.
// Either way the tile reports, in shared memory, each slot's partial sum
// after every step it reached, its per-step survivor counts under tspec,
// its final survivor mask and the ids of its final survivors — the commit
// warp consumes exactly that.
//
// Record contract (TileSum): part[s][slot] is valid for every slot for
// s < dense_steps (+inf once the slot is pruned under tspec); for
// s >= dense_steps only for slots in items0/items1 (the parked survivors),
// up to the step where they are pruned.
#pragma once
#include "pdx_common.cuh"

namespace pdx {

// a tile goes sparse once <= A.sparse_max (= 32 / tiles per claim) slots survive
constexpr int kMaxTpw = 8;  // tiles per compute-warp claim
#ifndef PDX_ITEMS_PER_WARP
#define PDX_ITEMS_PER_WARP 32
#endif
// sparse items a compute warp parks per claim (sparse_max * tpw); the sparse
// phase finishes them 32 at a time
constexpr int kItemsPerWarp = PDX_ITEMS_PER_WARP;
constexpr unsigned kFull = 0xffffffffu;

// One tile of a query's visit list (built by build_visits_kernel).
struct TileEntry {
  int64_t tile;     // tile index in the store
  int32_t m_tile;   // valid slots in this tile
  int32_t block_m;  // vectors in its logical block
  int32_t seg;      // visit segment (selected bucket) — picks the visit order
  int32_t vis;      // ordinal of its block in the query's block sequence
  int32_t tib;      // tile index within its block
  int32_t flags;    // bit1 first tile of block, bit2 last tile of block
};
static_assert(sizeof(TileEntry) == 32, "tile entry is 32 bytes");

struct TileDesc {
  int64_t tile;
  int32_t m_tile;
  int32_t seg;
  int32_t block_m;
  int32_t vis;
  float tspec;
  int32_t flags;  // bit1 first tile of block, bit2 last tile of block
};

// What a compute warp reports about a tile besides the partials.
struct TileSum {
  int32_t cnt[kMaxSteps];   // survivors after each step under tspec
  uint32_t alive0, alive1;  // final speculative survivors: bit l = slot 2l / 2l+1
  uint32_t items0, items1;  // slots parked for the sparse phase
  int32_t dense_steps;      // steps recorded for every slot
  int32_t _pad;
  int64_t touched_spec;     // values_touched of the block if the speculation is exact
};

struct SparseItem {
  int16_t tj;    // tile index within the warp's slice of the round
  int16_t slot;  // slot within the tile
  int16_t step;  // next schedule step
  int16_t pos;   // next dimension
  float acc;     // partial sum so far
};

struct ScanArgs {
  const float* tiles;
  const int64_t* tile_ids;
  int32_t d, d_pad;
  int64_t tile_stride;
  const TileEntry* vis;
  int64_t vis_qstride;
  const int32_t* vis_count;
  int32_t vis_count_qstride;
  const float* queries;
  const uint16_t* orders;
  int64_t oqs, oss;
  int32_t k, pruner, initial_step, nsteps;
  double sf;
  int32_t ads_d;
  double eps0;
  float* out_dist;
  int64_t* out_ids;
  int32_t* out_count;
  int64_t* out_touched;
  int64_t* out_total;
  int32_t* trace;
  int64_t trace_cap;
  int64_t* trace_len;
  int64_t* debug;  // optional [nq][8] counters (see pdx_search_out)
  int32_t sparse_max;  // a tile goes sparse once at most this many slots survive
  double factors[2 * kMaxSteps];  // per-step bound ratio, then band (bound_factors, pdx_scan.cu)
  int32_t nq, nsplit;     // split mode: CTA b scans range b / nq of query b % nq
  const float* resid;     // BSA: [ntiles][nsteps][64] residual energy per slot and step
  const float* bsa_coef;  // BSA: [nsteps]
  const int32_t* only;    // optional [nq]: scan only queries with only[q] != 0
  int32_t dense_spec;     // compute warps speculate with T' = +inf (prune-free scans; the
                          // commit warp replays every decision from the partials)
};

// Shared-memory views of one round slice (the tiles of one compute warp).
struct SliceRefs {
  const TileDesc* desc;  // [tpw]
  float* part;           // [tpw][nsteps][64]
  TileSum* sum;          // [tpw]
  float* bnd;            // [tpw][kMaxSteps] speculative bound per step
  SparseItem* items;     // [kItemsPerWarp]
  uint16_t* ordc;        // this warp's staged visit order (ORD), d entries
  int32_t* ordseg;       // the segment it belongs to (-1: none)
};

// Per-query constants shared by all warps.
struct QueryRefs {
  const float* q;        // [d_pad] query, zero padded
  const int32_t* ends;   // [nsteps] step ends
  const double* ratio;   // [nsteps] dims_seen / ads_d
  const double* band;    // [nsteps] 1 + eps0 / sqrt(dims_seen)
  const float* bsa;      // BSA: [3][kMaxSteps] query residual energy, its sqrt, coef
  const uint8_t* bmask;  // [d_pad/8] bit e of group g: a step ends after dim 8g+e
};

// A slot survives step s iff acc < bound(T).  pruning.py:88: threshold *
// (dims_seen / d) * band * band, in float64, left to right; the comparison
// then happens in float32 (numpy casts the Python float to the array's
// float32).  The host sets ratio = band = 1 wherever the reference compares
// against T itself (BOND, none, ADS once dims_seen >= d): T * 1 * 1 * 1
// rounds back to T exactly, so one branch-free formula serves every pruner.
__device__ __forceinline__ float ads_or_bond_bound(float T, double ratio, double band) {
  // bound_factors never pairs ratio 1 with band != 1: same value as the
  // formula, fewer live registers
  if (ratio == 1.0) return T;
  const double t = __dmul_rn(__dmul_rn(__dmul_rn((double)T, ratio), band), band);
  return __double2float_rn(t);
}

// BSA estimate after step s (PDX_PRUNER_BSA in pdx_b200.h), float32 per-op
// rounding: ((acc + rx) + rq) - (coef * sqrt(rx)) * sqrt(rq).  At the last
// step rx = rq = 0 and the estimate is acc itself.
__device__ __forceinline__ float bsa_est(const QueryRefs& Q, int s, float acc, float rx) {
  const float cx = __fmul_rn(Q.bsa[2 * kMaxSteps + s], __fsqrt_rn(rx));
  return __fsub_rn(__fadd_rn(__fadd_rn(acc, rx), Q.bsa[s]), __fmul_rn(cx, Q.bsa[kMaxSteps + s]));
}

// Residual energy of slot `slot` of tile `tile` after step s.
__device__ __forceinline__ float bsa_resid(const ScanArgs& A, int64_t tile, int s, int slot) {
  return __ldg(A.resid + ((size_t)tile * A.nsteps + s) * kTile + slot);
}

__device__ __forceinline__ const uint16_t* order_of(const ScanArgs& A, int q, int seg) {
  return A.orders + ((int64_t)q * A.oqs + (int64_t)seg * A.oss) * A.d;
}

// The warp's visit order for segment `seg` (warp-uniform), staged in shared
// memory once per segment: the per-dim index reads then cost no L2 trip.
__device__ __forceinline__ const uint16_t* warp_order(const ScanArgs& A, int q, int seg,
                                                      const SliceRefs& R, int lane) {
  if (*R.ordseg != seg) {
    __syncwarp();
    const uint16_t* g = order_of(A, q, seg);
    for (int j = lane; j < A.d; j += 32) R.ordc[j] = __ldg(g + j);
    __syncwarp();
    if (lane == 0) *R.ordseg = seg;
    __syncwarp();
  }
  return R.ordc;
}

// Lane `lane` < nsteps holds the tile's speculative bound for step `lane`.
__device__ __forceinline__ float tile_bounds(const ScanArgs& A, const TileDesc& t,
                                             const QueryRefs& Q, const SliceRefs& R, int tj,
                                             int lane) {
  float b = INFINITY;
  if (t.tspec != INFINITY && lane < A.nsteps)
    b = ads_or_bond_bound(t.tspec, Q.ratio[lane], Q.band[lane]);
  if (lane < A.nsteps) R.bnd[tj * kMaxSteps + lane] = b;
  return b;
}

// Park the live slots (al0/al1) of tile tj as sparse items at (step, pos).
__device__ __forceinline__ void park(const SliceRefs& R, TileSum& sum, int tj, int s, int pos,
                                     bool al0, bool al1, float acc0, float acc1, int nsteps,
                                     int& nitems, int lane) {
  const unsigned m0 = __ballot_sync(kFull, al0), m1 = __ballot_sync(kFull, al1);
  if (lane == 0) {
    sum.alive0 = 0;
    sum.alive1 = 0;
    sum.items0 = m0;
    sum.items1 = m1;
    sum.dense_steps = s;
  }
  if (lane >= s && lane < nsteps) sum.cnt[lane] = 0;
  const unsigned lt = (1u << lane) - 1u;
  const int pre = __popc(m0 & lt) + __popc(m1 & lt);
  if (al0) R.items[nitems + pre] = SparseItem{(int16_t)tj, (int16_t)lane, (int16_t)s, (int16_t)pos, acc0};
  if (al1) R.items[nitems + pre + (al0 ? 1 : 0)] = SparseItem{(int16_t)tj, (int16_t)(lane + 32), (int16_t)s, (int16_t)pos, acc1};
  nitems += __popc(m0) + __popc(m1);
}

__device__ __forceinline__ void finish_dense(const ScanArgs& A, const TileDesc& t,
                                             const SliceRefs& R, TileSum& sum, int tj, bool al0,
                                             bool al1, int lane) {
  const unsigned m0 = __ballot_sync(kFull, al0), m1 = __ballot_sync(kFull, al1);
  if (lane == 0) {
    sum.alive0 = m0;
    sum.alive1 = m1;
    sum.items0 = 0;
    sum.items1 = 0;
    sum.dense_steps = A.nsteps;
  }
}

// ----------------------------------------------- dense phase, G = 8, natural order
template <int METRIC>
__device__ __forceinline__ void dense_tile_g8(const ScanArgs& A, const TileDesc& t, int tj,
                                              const QueryRefs& Q, const SliceRefs& R,
                                              int& nitems, int lane) {
  const float* __restrict__ tb = A.tiles + t.tile * A.tile_stride;
  float* __restrict__ part = R.part + (size_t)tj * A.nsteps * kTile;
  TileSum& sum = R.sum[tj];
  const int nsteps = A.nsteps;
  const int s0 = lane, s1 = lane + 32;  // a 256-bit load per slot is contiguous across lanes
  bool al0 = s0 < t.m_tile, al1 = s1 < t.m_tile;
  const bool prune = t.tspec != INFINITY;
  const float mybnd = tile_bounds(A, t, Q, R, tj, lane);
  float acc0 = 0.f, acc1 = 0.f;
  if (t.m_tile <= A.sparse_max) {  // small tile: straight to the sparse phase
    park(R, sum, tj, 0, 0, al0, al1, acc0, acc1, nsteps, nitems, lane);
    return;
  }
  constexpr bool kBsa = METRIC == kMetricL2Bsa;
  float rx0 = 0.f, rx1 = 0.f;  // BSA: residual energies for step s, loaded a step ahead
  if (kBsa) {
    if (al0) rx0 = bsa_resid(A, t.tile, 0, s0);
    if (al1) rx1 = bsa_resid(A, t.tile, 0, s1);
  }
  const int ng = A.d_pad >> 3;
  float n0[8], n1[8];  // prefetched group
#pragma unroll
  for (int e = 0; e < 8; ++e) n0[e] = n1[e] = 0.f;
  {
    const float* p = tb + (size_t)s0 * 8;
    if (al0) ldg8(p, n0);
    if (al1) ldg8(p + 32 * 8, n1);
  }
  int s = 0;
  for (int g = 0; g < ng; ++g) {
    float x0[8], x1[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      x0[e] = n0[e];
      x1[e] = n1[e];
    }
    if (g + 1 < ng) {  // prefetch the next group for the slots alive now
      const float* p = tb + ((size_t)(g + 1) * kTile + s0) * 8;
      if (al0) ldg8(p, n0);
      if (al1) ldg8(p + 32 * 8, n1);
    }
    const float4 qa = *reinterpret_cast<const float4*>(Q.q + g * 8);
    const float4 qb = *reinterpret_cast<const float4*>(Q.q + g * 8 + 4);
    const float qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
    const unsigned bm = Q.bmask[g];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      acc0 = upd<METRIC>(acc0, qv[e], x0[e]);
      acc1 = upd<METRIC>(acc1, qv[e], x1[e]);
      if (bm & (1u << e)) {  // step s ends after dim 8g+e (warp-uniform)
        const float v0 = kBsa ? bsa_est(Q, s, acc0, rx0) : acc0;
        const float v1 = kBsa ? bsa_est(Q, s, acc1, rx1) : acc1;
        part[s * kTile + s0] = al0 ? v0 : INFINITY;
        part[s * kTile + s1] = al1 ? v1 : INFINITY;
        if (prune) {
          const float bs = __shfl_sync(kFull, mybnd, s);
          al0 = al0 && (v0 < bs);
          al1 = al1 && (v1 < bs);
        }
        const int c = __popc(__ballot_sync(kFull, al0)) + __popc(__ballot_sync(kFull, al1));
        if (lane == 0) sum.cnt[s] = c;
        ++s;
        if (s == nsteps) {
          finish_dense(A, t, R, sum, tj, al0, al1, lane);
          return;
        }
        if (c <= A.sparse_max) {
          park(R, sum, tj, s, g * 8 + e + 1, al0, al1, acc0, acc1, nsteps, nitems, lane);
          return;
        }
        if (kBsa) {
          rx0 = al0 ? bsa_resid(A, t.tile, s, s0) : 0.f;
          rx1 = al1 ? bsa_resid(A, t.tile, s, s1) : 0.f;
        }
      }
    }
  }
}

// ----------------------------------- dense phase, generic (G = 1 and/or a visit order)
template <int G, bool ORD, int METRIC>
__device__ __forceinline__ void dense_tile_generic(const ScanArgs& A, int q, const TileDesc& t,
                                                   int tj, const QueryRefs& Q,
                                                   const SliceRefs& R, int& nitems, int lane) {
  const float* __restrict__ tb = A.tiles + t.tile * A.tile_stride;
  const uint16_t* __restrict__ ord = ORD ? warp_order(A, q, t.seg, R, lane) : nullptr;
  float* __restrict__ part = R.part + (size_t)tj * A.nsteps * kTile;
  TileSum& sum = R.sum[tj];
  const int nsteps = A.nsteps;
  const int s0 = lane, s1 = lane + 32;
  bool al0 = s0 < t.m_tile, al1 = s1 < t.m_tile;
  const bool prune = t.tspec != INFINITY;
  const float mybnd = tile_bounds(A, t, Q, R, tj, lane);
  float acc0 = 0.f, acc1 = 0.f;
  if (t.m_tile <= A.sparse_max) {
    park(R, sum, tj, 0, 0, al0, al1, acc0, acc1, nsteps, nitems, lane);
    return;
  }
  constexpr bool kBsa = METRIC == kMetricL2Bsa;
  int a = 0;
  for (int s = 0; s < nsteps; ++s) {
    const int b = Q.ends[s];
    float rx0 = 0.f, rx1 = 0.f;  // BSA: issued before the step's dims are read
    if (kBsa) {
      if (al0) rx0 = bsa_resid(A, t.tile, s, s0);
      if (al1) rx1 = bsa_resid(A, t.tile, s, s1);
    }
    for (int j0 = a; j0 < b; j0 += 8) {
      int dim[8];
      float x0[8], x1[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int j = j0 + e;
        dim[e] = 0;
        x0[e] = x1[e] = 0.f;
        if (j < b) dim[e] = ORD ? (int)ord[j] : j;
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (j0 + e < b) {
          const int dm = dim[e];
          if (G == 1) {  // a 256-byte PDX row: two coalesced 128-byte halves
            if (al0) x0[e] = __ldg(tb + (int64_t)dm * kTile + s0);
            if (al1) x1[e] = __ldg(tb + (int64_t)dm * kTile + s1);
          } else {
            const float* p = tb + ((int64_t)(dm >> 3) * kTile + s0) * 8 + (dm & 7);
            if (al0) x0[e] = __ldg(p);
            if (al1) x1[e] = __ldg(p + 32 * 8);
          }
        }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (j0 + e < b) {
          const float qj = Q.q[dim[e]];
          acc0 = upd<METRIC>(acc0, qj, x0[e]);
          acc1 = upd<METRIC>(acc1, qj, x1[e]);
        }
      }
    }
    const float v0 = kBsa ? bsa_est(Q, s, acc0, rx0) : acc0;
    const float v1 = kBsa ? bsa_est(Q, s, acc1, rx1) : acc1;
    part[s * kTile + s0] = al0 ? v0 : INFINITY;
    part[s * kTile + s1] = al1 ? v1 : INFINITY;
    if (prune) {
      const float bs = __shfl_sync(kFull, mybnd, s);
      al0 = al0 && (v0 < bs);
      al1 = al1 && (v1 < bs);
    }
    const int c = __popc(__ballot_sync(kFull, al0)) + __popc(__ballot_sync(kFull, al1));
    if (lane == 0) sum.cnt[s] = c;
    a = b;
    if (s + 1 < nsteps && c <= A.sparse_max) {
      park(R, sum, tj, s + 1, b, al0, al1, acc0, acc1, nsteps, nitems, lane);
      return;
    }
  }
  finish_dense(A, t, R, sum, tj, al0, al1, lane);
}

// ----------------------------------------------------------- sparse phase
// Lane i finishes item i.  It walks its slot's remaining dims, records the
// partial at each step end, decides against its tile's speculative bound,
// and reports counts / survivors with shared-memory atomics.
template <int G, bool ORD, int METRIC>
__device__ __forceinline__ void sparse_round(const ScanArgs& A, int q, const QueryRefs& Q,
                                             const SliceRefs& R, int base, int nitems, int lane);

template <int G, bool ORD, int METRIC>
__device__ __forceinline__ void sparse_phase(const ScanArgs& A, int q, const QueryRefs& Q,
                                             const SliceRefs& R, int nitems, int lane) {
  if (nitems == 0) return;
  __syncwarp();
  for (int base = 0; base < nitems; base += 32)
    sparse_round<G, ORD, METRIC>(A, q, Q, R, base, nitems, lane);
}

template <int G, bool ORD, int METRIC>
__device__ __forceinline__ void sparse_round(const ScanArgs& A, int q, const QueryRefs& Q,
                                             const SliceRefs& R, int base, int nitems, int lane) {
  const int nsteps = A.nsteps;
  bool act = base + lane < nitems;
  const SparseItem it = act ? R.items[base + lane] : SparseItem{0, 0, 0, 0, 0.f};
  const TileDesc& t = R.desc[it.tj];
  const float* __restrict__ tb = A.tiles + t.tile * A.tile_stride;
  float* __restrict__ part = R.part + (size_t)it.tj * nsteps * kTile;
  TileSum& sum = R.sum[it.tj];
  const float* bnd = R.bnd + it.tj * kMaxSteps;
  const bool prune = t.tspec != INFINITY;
  const int slot = it.slot;
  int s = it.step;
  float acc = it.acc;
  int pos = it.pos;
  constexpr bool kBsa = METRIC == kMetricL2Bsa;
  float rx = (kBsa && act) ? bsa_resid(A, t.tile, s, slot) : 0.f;  // BSA, step s
  if (G == 8 && !ORD) {
    const int ng = A.d_pad >> 3;
    int g = pos >> 3;
    float nx[8];  // prefetched group: one 256-bit load per 8 dims
#pragma unroll
    for (int e = 0; e < 8; ++e) nx[e] = 0.f;
    if (act) ldg8(tb + ((size_t)g * kTile + slot) * 8, nx);
    while (__any_sync(kFull, act)) {
      if (act) {
        float x[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] = nx[e];
        if (g + 1 < ng) ldg8(tb + ((size_t)(g + 1) * kTile + slot) * 8, nx);
        const float4 qa = *reinterpret_cast<const float4*>(Q.q + g * 8);
        const float4 qb = *reinterpret_cast<const float4*>(Q.q + g * 8 + 4);
        const float qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
        const unsigned bm = Q.bmask[g];
        const int e0 = pos - g * 8;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (act && e >= e0) {
            acc = upd<METRIC>(acc, qv[e], x[e]);
            if (bm & (1u << e)) {
              const float v = kBsa ? bsa_est(Q, s, acc, rx) : acc;
              part[s * kTile + slot] = v;
              const bool ok = !prune || v < bnd[s];
              if (ok) atomicAdd(&sum.cnt[s], 1);
              ++s;
              if (!ok) {
                act = false;
              } else if (s == nsteps) {
                atomicOr(slot >= 32 ? &sum.alive1 : &sum.alive0, 1u << (slot & 31));
                act = false;
              } else if (kBsa) {
                rx = bsa_resid(A, t.tile, s, slot);
              }
            }
          }
        }
        ++g;
        pos = g * 8;
      }
    }
  } else {
    // the staged order when the item's segment is the warp's current one
    const uint16_t* __restrict__ ord =
        ORD ? (t.seg == *R.ordseg ? R.ordc : order_of(A, q, t.seg)) : nullptr;
    int end = act ? Q.ends[s] : 0;
    while (__any_sync(kFull, act)) {
      if (act) {
        const int jend = min(end, pos + 8);
        int dim[8];
        float x[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          dim[e] = 0;
          x[e] = 0.f;
          if (pos + e < jend) dim[e] = ORD ? (int)ord[pos + e] : pos + e;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (pos + e < jend) {
            const int dm = dim[e];
            x[e] = G == 1 ? __ldg(tb + (int64_t)dm * kTile + slot)
                          : __ldg(tb + ((int64_t)(dm >> 3) * kTile + slot) * 8 + (dm & 7));
          }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (pos + e < jend) acc = upd<METRIC>(acc, Q.q[dim[e]], x[e]);
        pos = jend;
        if (pos == end) {
          const float v = kBsa ? bsa_est(Q, s, acc, rx) : acc;
          part[s * kTile + slot] = v;
          const bool ok = !prune || v < bnd[s];
          if (ok) atomicAdd(&sum.cnt[s], 1);
          ++s;
          if (!ok) {
            act = false;
          } else if (s == nsteps) {
            atomicOr(slot >= 32 ? &sum.alive1 : &sum.alive0, 1u << (slot & 31));
            act = false;
          } else {
            end = Q.ends[s];
            if (kBsa) rx = bsa_resid(A, t.tile, s, slot);
          }
        }
      }
    }
  }
  __syncwarp();
}

}  // namespace pdx
