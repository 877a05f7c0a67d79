// pdx_scan_kernel: one CTA per query, a ring of tile slots between W COMPUTE
// warps and one COMMIT warp (see pdx_scan.cu for the semantics).
//
//   compute warp: claims `tpw` consecutive tiles of the query's per-tile
//                 visit list (shared-memory atomic), waits for their ring
//                 slots to be free, picks each tile's speculative threshold
//                 from the values the commit warp publishes, scans the
//                 tiles (pdx_scan_spec.cuh) and flags the slots computed.
//   commit warp : commits computed tiles strictly in visit order — exact
//                 threshold chain, top-k pushes, values_touched, survivor
//                 traces — and publishes (tiles committed, T_b of the open
//                 block, current threshold).
// Speculative thresholds are always >= the exact T_b: the published
// threshold only decreases, and a block whose first tile is committed uses
// its recorded T_b.  There is no CTA-wide barrier inside the loop.
#pragma once
#include "pdx_common.cuh"
#include "pdx_scan_spec.cuh"

#ifndef PDX_MBAR_RING
#define PDX_MBAR_RING 1  // compute warps sleep on mbarriers for free ring slots
#endif
#ifndef PDX_MBAR_COMMIT
#define PDX_MBAR_COMMIT 1  // the commit warp sleeps on mbarriers for ready tiles
#endif
#ifndef PDX_MBAR_HINT
#define PDX_MBAR_HINT 1
#endif
#ifndef PDX_SCAN_PROFILE
#define PDX_SCAN_PROFILE 0
#endif
#ifndef PDX_SCAN_MIN_BLOCKS
#define PDX_SCAN_MIN_BLOCKS 3  // 3 query CTAs of 9 warps per SM: <= 75 registers
#endif

namespace pdx {

struct Control {
  int32_t n;          // entries in the top-k (commit warp)
  float tblk;         // T_b of the open block (commit warp)
  int32_t linear;     // open block is linear
  int32_t warm_min;   // smallest survivor count that keeps WARMUP for the open block
  int32_t warm_m;     // the block size warm_min was computed for
  int32_t claim;      // tiles claimed by compute warps
  int32_t com_pub;    // tiles committed (published after tblk_pub / t_pub)
  float tblk_pub;     // T_b of the block whose first tile was committed last
  float t_pub;        // threshold after the last commit
  int32_t ring_waits;  // diagnostics: compute-warp polls for a free ring slot
  int32_t items;       // diagnostics: sparse items
  int64_t touched, total, tlen;
  unsigned long long cyc[4];  // diagnostics: compute-warp cycles in ring wait, dense, sparse, rest
};
static_assert(sizeof(Control) <= 128, "control block");

// Shared-memory carve-up; computed on the host and passed to the kernel so
// the offsets live in the constant bank instead of being rematerialised.
struct ScanSmem {
  int32_t ctl, mbar, ratio, band, bsa, ends, bnd, cnt, wmin, flag, desc, sum, items, wbnd, ids,
      tki, part, tkd, q, bmask, ordc, ordseg, total, rb;
};

inline ScanSmem scan_smem_layout(int W, int tpw, int rb, int k, int nsteps, int d_pad,
                                 bool ord = false) {
  ScanSmem L;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = (o + bytes + 15) & ~(size_t)15;
    return (int32_t)at;
  };
  L.ctl = take(128);
  L.mbar = take(sizeof(uint64_t) * 2 * rb);  // ready[rb], free[rb]
  L.ratio = take(sizeof(double) * kMaxSteps);
  L.band = take(sizeof(double) * kMaxSteps);
  L.bsa = take(sizeof(float) * 3 * kMaxSteps);
  L.ends = take(sizeof(int32_t) * kMaxSteps);
  L.bnd = take(sizeof(float) * kMaxSteps);
  L.cnt = take(sizeof(int32_t) * kMaxSteps);
  L.wmin = take(sizeof(int32_t) * (kTile + 1));
  L.flag = take(sizeof(int32_t) * rb);
  L.desc = take(sizeof(TileDesc) * rb);
  L.sum = take(sizeof(TileSum) * rb);
  L.items = take(sizeof(SparseItem) * kItemsPerWarp * W);
  L.wbnd = take(sizeof(float) * kMaxSteps * W * tpw);
  L.ids = take(0);
  L.tki = take(sizeof(int64_t) * k);
  L.part = take(sizeof(float) * kTile * nsteps * rb);
  L.tkd = take(sizeof(float) * k);
  L.q = take(sizeof(float) * ((d_pad + 7) / 8) * 8);
  L.bmask = take((d_pad + 7) / 8);
  // visit orders: each compute warp keeps its current segment's order on chip
  L.ordc = take(ord ? sizeof(uint16_t) * d_pad * W : 0);
  L.ordseg = take(ord ? sizeof(int32_t) * W : 0);
  L.total = (int32_t)o;
  L.rb = rb;
  return L;
}

// Smallest survivor count p with float64(p / m) >= sf: search.py:148's
// WARMUP test `len(positions) / block.m >= selection_fraction` is then an
// integer compare (the quotient is monotone in p).
__device__ __forceinline__ int warm_min_count(int m, double sf) {
  int p = (int)ceil(sf * (double)m);
  p = p < 0 ? 0 : (p > m ? m : p);
  while (p > 0 && __ddiv_rn((double)(p - 1), (double)m) >= sf) --p;
  while (p < m && __ddiv_rn((double)p, (double)m) < sf) ++p;
  return p;
}

// values_touched of a non-linear block of m vectors given its per-step
// survivor counts (search.py:148-169).
__device__ __forceinline__ int64_t block_touched(int64_t m, int wmin, const int32_t* cnt,
                                                 const int32_t* ends, int nsteps) {
  int64_t touched = 0, prev = m;
  bool warm = true;
  int a = 0;
  for (int s = 0; s < nsteps; ++s) {
    const int w_s = ends[s] - a;
    a = ends[s];
    if (warm && prev >= wmin) {
      touched += m * w_s;
    } else {
      warm = false;
      touched += prev * w_s;
    }
    prev = cnt[s];
  }
  return touched;
}

template <typename T>
__device__ __forceinline__ T vload(const T& x) {
  return *reinterpret_cast<const volatile T*>(&x);
}
template <typename T>
__device__ __forceinline__ void vstore(T& x, T v) {
  *reinterpret_cast<volatile T*>(&x) = v;
}
// acquire / release on a shared-memory word (CTA scope): the data written
// before a release is visible to the warp whose acquire observes the value
__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.b32 %0, [%1];"
               : "=r"(v)
               : "r"((unsigned)__cvta_generic_to_shared(p))
               : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int32_t* p, int v) {
  asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)),
               "r"(v)
               : "memory");
}

// mbarriers (count 1) guarding the ring: ready[slot] completes a phase when
// a compute warp has written the slot's tile, free[slot] when the commit
// warp has consumed it.  A waiting warp sleeps in hardware (try_wait) instead
// of spinning, so the issue slots go to the warps that work.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile(
      "{\n .reg .b64 state;\n mbarrier.arrive.release.cta.shared::cta.b64 state, [%0];\n}" ::"r"(
          smem_u32(b))
      : "memory");
}
// true once the phase with parity `par` has completed; suspends up to `ns`
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t par, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(par), "r"(ns)
      : "memory");
  return ok != 0;
}
// try_wait without a time hint: the hardware suspends the warp for a
// system-defined window and wakes it when the phase completes
__device__ __forceinline__ bool mbar_try_default(uint64_t* b, uint32_t par) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(par)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
#if PDX_MBAR_HINT
  while (!mbar_try(b, par, 1u << 20)) {
  }
#else
  while (!mbar_try_default(b, par)) {
  }
#endif
}

// ------------------------------------------------------------------ top-k
__device__ __forceinline__ float topk_threshold(const Control& c, int k, const float* tkd) {
  return c.n < k ? INFINITY : tkd[k - 1];
}

// Warp-cooperative insertion of one (warp-uniform) candidate into the
// ascending (dist, id) array; TopK.push (search.py:44-51).
__device__ __forceinline__ void topk_insert(Control& c, int k, float* tkd, int64_t* tki, float dv,
                                            int64_t iv, int lane) {
  const int n = c.n;
  if (n == k && !pair_less(dv, iv, tkd[k - 1], tki[k - 1])) return;
  int pos = 0;
  for (int base = 0; base < n; base += 32) {
    const int j = base + lane;
    const bool lt = j < n && pair_less(tkd[j], tki[j], dv, iv);
    pos += __popc(__ballot_sync(kFull, lt));
  }
  const int last = n < k ? n : k - 1;
  for (int hi = last; hi > pos; hi -= 32) {
    const int j = hi - 1 - lane;
    const bool act = j >= pos;
    float dd = 0.f;
    int64_t ii = 0;
    if (act) { dd = tkd[j]; ii = tki[j]; }
    __syncwarp();
    if (act) { tkd[j + 1] = dd; tki[j + 1] = ii; }
    __syncwarp();
  }
  if (lane == 0) {
    tkd[pos] = dv;
    tki[pos] = iv;
    c.n = n < k ? n + 1 : k;
  }
  __syncwarp();
}

__device__ __forceinline__ void topk_push_lanes(Control& c, int k, float* tkd, int64_t* tki,
                                                bool cand, float dv, int64_t iv, int lane) {
  // pre-filter against the current worst (it only improves as we insert)
  if (cand && c.n == k && !pair_less(dv, iv, tkd[k - 1], tki[k - 1])) cand = false;
  unsigned mask = __ballot_sync(kFull, cand);
  while (mask) {
    const int src = __ffs(mask) - 1;
    mask &= mask - 1;
    const float d = __shfl_sync(kFull, dv, src);
    const int64_t i = __shfl_sync(kFull, iv, src);
    topk_insert(c, k, tkd, tki, d, i, lane);
  }
}

// ------------------------------------------------------------------ kernel
template <int G, bool ORD, int METRIC>
__global__ void __launch_bounds__(288, PDX_SCAN_MIN_BLOCKS) pdx_scan_kernel(const ScanArgs A, const ScanSmem L,
                                                       const int tpw) {
  extern __shared__ __align__(16) unsigned char smem[];
  // split mode: CTA b scans range b / nq of query b % nq and writes row b
  const int q = A.nsplit > 1 ? (int)(blockIdx.x % (unsigned)A.nq) : (int)blockIdx.x;
  if (A.only && A.only[q] == 0) return;  // batched path's fallback: flagged queries only
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int RB = L.rb;  // a power of two
  const int RMASK = RB - 1;
  const int nsteps = A.nsteps, k = A.k;

  Control& ctl = *reinterpret_cast<Control*>(smem + L.ctl);
  double* s_ratio = reinterpret_cast<double*>(smem + L.ratio);
  double* s_band = reinterpret_cast<double*>(smem + L.band);
  float* s_bsa = reinterpret_cast<float*>(smem + L.bsa);  // BSA: rq, sqrt(rq), coef per step
  int32_t* s_ends = reinterpret_cast<int32_t*>(smem + L.ends);
  float* s_bnd = reinterpret_cast<float*>(smem + L.bnd);
  int32_t* s_cnt = reinterpret_cast<int32_t*>(smem + L.cnt);
  int32_t* s_wmin = reinterpret_cast<int32_t*>(smem + L.wmin);
  int32_t* s_flag = reinterpret_cast<int32_t*>(smem + L.flag);
  TileDesc* s_desc = reinterpret_cast<TileDesc*>(smem + L.desc);
  TileSum* s_sum = reinterpret_cast<TileSum*>(smem + L.sum);
  int64_t* tki = reinterpret_cast<int64_t*>(smem + L.tki);
  float* s_part = reinterpret_cast<float*>(smem + L.part);
  float* tkd = reinterpret_cast<float*>(smem + L.tkd);
  float* s_q = reinterpret_cast<float*>(smem + L.q);
  uint8_t* s_bmask = reinterpret_cast<uint8_t*>(smem + L.bmask);
  uint64_t* s_ready = reinterpret_cast<uint64_t*>(smem + L.mbar);
  uint64_t* s_free = s_ready + RB;

  // ---- setup
  const float* qg = A.queries + (int64_t)q * A.d;
  const int ngroups = (A.d_pad + 7) / 8;
  for (int j = threadIdx.x; j < ngroups * 8; j += blockDim.x) s_q[j] = j < A.d ? qg[j] : 0.f;
  for (int j = threadIdx.x; j < ngroups; j += blockDim.x) s_bmask[j] = 0;
  if (ORD)  // one staged-order tag per compute warp
    for (int j = threadIdx.x; j < (int)(blockDim.x >> 5) - 1; j += blockDim.x)
      reinterpret_cast<int32_t*>(smem + L.ordseg)[j] = -1;
  for (int j = threadIdx.x; j < RB; j += blockDim.x) {
    s_flag[j] = 0;
    mbar_init(&s_ready[j]);
    mbar_init(&s_free[j]);
  }
  for (int m = threadIdx.x; m <= kTile; m += blockDim.x)
    s_wmin[m] = m > 0 ? warm_min_count(m, A.sf) : 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t start = 0, width = A.initial_step;  // step_schedule (search.py:106-117)
    for (int s = 0; s < nsteps; ++s) {
      const int64_t end = start + width < A.d ? start + width : A.d;
      s_ends[s] = (int32_t)end;
      s_bmask[(end - 1) >> 3] |= (uint8_t)(1u << ((end - 1) & 7));
      start = end;
      width *= 2;
    }
    ctl.n = 0;
    ctl.tblk = INFINITY;
    ctl.linear = 1;
    ctl.warm_min = 0;
    ctl.warm_m = -1;
    ctl.claim = 0;
    ctl.com_pub = 0;
    ctl.tblk_pub = INFINITY;
    ctl.t_pub = INFINITY;
    ctl.touched = ctl.total = ctl.tlen = 0;
    ctl.ring_waits = 0;
    ctl.items = 0;
    ctl.cyc[0] = ctl.cyc[1] = ctl.cyc[2] = ctl.cyc[3] = 0;
  }
  __syncthreads();
  if (threadIdx.x < nsteps) {  // bound factors (bound_factors, pdx_scan.cu: kernel parameters)
    s_ratio[threadIdx.x] = A.factors[threadIdx.x];
    s_band[threadIdx.x] = A.factors[kMaxSteps + threadIdx.x];
    if (METRIC == kMetricL2Bsa) {  // the query's residual energy after this step
      float r = 0.f;
      for (int j = s_ends[threadIdx.x]; j < A.d; ++j) r = __fadd_rn(r, __fmul_rn(s_q[j], s_q[j]));
      s_bsa[threadIdx.x] = r;
      s_bsa[kMaxSteps + threadIdx.x] = __fsqrt_rn(r);
      s_bsa[2 * kMaxSteps + threadIdx.x] = A.bsa_coef[threadIdx.x];
    }
  }
  __syncthreads();
  const TileEntry* vis = A.vis + (int64_t)q * A.vis_qstride;
  int ntiles = A.vis_count[(int64_t)q * A.vis_count_qstride];
  if (A.nsplit > 1) {  // this CTA's range, both ends moved back to a block start
    const int sp = (int)(blockIdx.x / (unsigned)A.nq);
    const int all = ntiles;
    auto start = [&](int x) {
      const int p = (int)((int64_t)x * all / A.nsplit);
      return p >= all ? all : p - vis[p].tib;
    };
    const int t0 = start(sp), t1 = start(sp + 1);
    vis += t0;
    ntiles = t1 - t0;
  }

  if (warp > 0) {
    // ======================================================= compute warp
    const int w = warp - 1;
    QueryRefs Q;
    Q.q = s_q;
    Q.ends = s_ends;
    Q.ratio = s_ratio;
    Q.band = s_band;
    Q.bsa = s_bsa;
    Q.bmask = s_bmask;
    SparseItem* items = reinterpret_cast<SparseItem*>(smem + L.items) + kItemsPerWarp * w;
    float* wbnd = reinterpret_cast<float*>(smem + L.wbnd) + (size_t)w * tpw * kMaxSteps;
    // claims are made one ahead so the next tiles' entries load while the
    // current ones are scanned
    auto claim = [&](TileEntry& e) {
      int n = 0;
      if (lane == 0) n = atomicAdd(&ctl.claim, tpw);
      n = __shfl_sync(kFull, n, 0);
      if (lane < tpw && n + lane < ntiles) e = vis[n + lane];
      return n;
    };
    TileEntry enext = {};
    int nnext = claim(enext);
    // per-phase cycle counters (diagnostics; compiled in with -DPDX_SCAN_PROFILE=1)
    constexpr bool kProf = PDX_SCAN_PROFILE != 0;
    long long c_wait = 0, c_dense = 0, c_sparse = 0, c_all = kProf ? clock64() : 0;
    for (;;) {
      const int n0 = nnext;
      const TileEntry e = enext;
      if (n0 >= ntiles) break;
      const long long c0 = kProf ? clock64() : 0;
      nnext = claim(enext);
      const int nt = min(tpw, ntiles - n0);
      // ring slots n0.. are free once tile n0+nt-1-RB is committed: phase
      // (last/RB - 1) of free[last's slot] (commits are in order)
      const int last = n0 + nt - 1;
#if PDX_MBAR_RING
      if (last >= RB) {
        // A parity wait only tells the current phase from the one before: a
        // warp two ring turns ahead of the commit (possible with lookahead
        // claims) would alias.  First let the commit reach the previous turn.
        while (ld_acquire(&ctl.com_pub) < last + 1 - 2 * RB) __nanosleep(256);
        const uint32_t par = (uint32_t)(last / RB - 1) & 1u;
        if (!mbar_try_default(&s_free[last & RMASK], par)) {
          if (A.debug && lane == 0) atomicAdd(&ctl.ring_waits, 1);
          mbar_wait(&s_free[last & RMASK], par);
        }
      }
#else
      int spins = 0;
      while (ld_acquire(&ctl.com_pub) < last + 1 - RB) {
        __nanosleep(spins < 2 ? 200 : 800);
        ++spins;
      }
      if (A.debug && spins && lane == 0) atomicAdd(&ctl.ring_waits, spins);
#endif
      const long long c1 = kProf ? clock64() : 0;
      c_wait += c1 - c0;
      const int sl = n0 & RMASK;  // RB is a multiple of tpw: the slice is contiguous
      if (lane < nt) {
        TileDesc t;
        t.tile = e.tile;
        t.m_tile = e.m_tile;
        t.seg = e.seg;
        t.block_m = e.block_m;
        t.vis = e.vis;
        t.flags = e.flags;
        if (A.pruner == PDX_PRUNER_NONE || A.dense_spec) {
          t.tspec = INFINITY;
        } else {
          const int first = n0 + lane - e.tib;  // the block's first tile
          const int com = ld_acquire(&ctl.com_pub);
          t.tspec = com > first ? vload(ctl.tblk_pub) : vload(ctl.t_pub);
        }
        s_desc[sl + lane] = t;
      }
      __syncwarp();
      SliceRefs R;
      R.desc = s_desc + sl;
      R.part = s_part + (size_t)sl * nsteps * kTile;
      R.sum = s_sum + sl;
      R.bnd = wbnd;
      R.items = items;
      R.ordc = ORD ? reinterpret_cast<uint16_t*>(smem + L.ordc) + (size_t)w * A.d_pad : nullptr;
      R.ordseg = ORD ? reinterpret_cast<int32_t*>(smem + L.ordseg) + w : nullptr;
      int nitems = 0;
      for (int j = 0; j < nt; ++j) {
        if (G == 8 && !ORD)
          dense_tile_g8<METRIC>(A, R.desc[j], j, Q, R, nitems, lane);
        else
          dense_tile_generic<G, ORD, METRIC>(A, q, R.desc[j], j, Q, R, nitems, lane);
      }
      if (A.debug && lane == 0) atomicAdd(&ctl.items, nitems);
      const long long c2 = kProf ? clock64() : 0;
      c_dense += c2 - c1;
      sparse_phase<G, ORD, METRIC>(A, q, Q, R, nitems, lane);
      if (kProf) c_sparse += clock64() - c2;
      __syncwarp();
      if (lane < nt) {  // values_touched if the commit finds the speculation exact
        const TileDesc& t = R.desc[lane];
        R.sum[lane].touched_spec =
            t.block_m <= kTile ? block_touched(t.block_m, s_wmin[t.block_m], R.sum[lane].cnt,
                                               s_ends, nsteps)
                               : 0;
      }
      __syncwarp();
      if (lane < nt) {
        st_release(&s_flag[sl + lane], 2);
        mbar_arrive(&s_ready[sl + lane]);
      }
    }
    if (kProf && A.debug && lane == 0) {
      c_all = clock64() - c_all;
      atomicAdd(&ctl.cyc[0], (unsigned long long)c_wait);
      atomicAdd(&ctl.cyc[1], (unsigned long long)c_dense);
      atomicAdd(&ctl.cyc[2], (unsigned long long)c_sparse);
      atomicAdd(&ctl.cyc[3], (unsigned long long)(c_all - c_wait - c_dense - c_sparse));
    }
  } else {
    // ======================================================== commit warp
    // The commit warp's state lives in registers (the same value in every
    // lane; the running stats in lane 0): each commit run is on the query's
    // critical path, so it avoids shared-memory round trips it can skip.
    int32_t* tr = A.trace ? A.trace + (int64_t)q * A.trace_cap : nullptr;
    const long long t_start = clock64();
    int64_t dbg_fast = 0, dbg_serial = 0, dbg_replay = 0, dbg_idle = 0;
    float T = INFINITY;      // current threshold, TopK.threshold()
    float tblk = INFINITY;   // T_b of the open block
    bool linear = true;      // the open block is linear
    int warm_min = 0, warm_m = -1;
    int64_t r_touched = 0, r_total = 0, r_tlen = 0;  // lane 0

    // commit one tile (serial path)
    auto commit_one = [&](int sl) {
      const TileDesc t = s_desc[sl];
      const TileSum& sm = s_sum[sl];
      const float* part = s_part + (size_t)sl * nsteps * kTile;
      if (t.flags & 2) {  // first tile of its block: T_b is fixed now
        linear = (t.vis == 0 || A.pruner == PDX_PRUNER_NONE || T == INFINITY);
        tblk = T;
        if (lane < nsteps) {
          s_cnt[lane] = 0;
          if (!linear)
            s_bnd[lane] = ads_or_bond_bound(T, s_ratio[lane], s_band[lane]);
        }
        if (lane == 0) vstore(ctl.tblk_pub, T);
        if (!linear && t.block_m != warm_m) {
          warm_min = t.block_m <= kTile ? s_wmin[t.block_m] : warm_min_count(t.block_m, A.sf);
          warm_m = t.block_m;
        }
        __syncwarp();
      }
      const int s0 = lane, s1 = lane + 32;  // bit `lane` of alive0 / alive1
      bool c0, c1;
      if (linear) {
        c0 = s0 < t.m_tile;
        c1 = s1 < t.m_tile;
      } else if (t.tspec == tblk) {
        // the speculation ran with the exact threshold: its counts and
        // survivors are the reference's
        if (lane < nsteps) s_cnt[lane] += sm.cnt[lane];
        c0 = (sm.alive0 >> lane) & 1;
        c1 = (sm.alive1 >> lane) & 1;
      } else {
        // replay the decisions under T_b from the recorded partials
        ++dbg_replay;
        c0 = s0 < t.m_tile;
        c1 = s1 < t.m_tile;
        int mycnt = 0;
        for (int s = 0; s < nsteps; ++s) {
          if (s == sm.dense_steps) {  // later partials exist only for parked slots
            c0 = c0 && ((sm.items0 >> lane) & 1);
            c1 = c1 && ((sm.items1 >> lane) & 1);
          }
          const float bs = s_bnd[s];
          c0 = c0 && (part[s * kTile + s0] < bs);
          c1 = c1 && (part[s * kTile + s1] < bs);
          const int cnt = __popc(__ballot_sync(kFull, c0)) + __popc(__ballot_sync(kFull, c1));
          if (lane == s) mycnt = cnt;
        }
        if (lane < nsteps) s_cnt[lane] += mycnt;
      }
      if (__any_sync(kFull, c0 || c1)) {
        const float f0 = part[(nsteps - 1) * kTile + s0], f1 = part[(nsteps - 1) * kTile + s1];
        // ids of the (rare) pushed slots come straight from HBM / L2
        const int64_t* gid = A.tile_ids + t.tile * kTile;
        const float key0 = METRIC == PDX_METRIC_IP ? -f0 : f0;
        const float key1 = METRIC == PDX_METRIC_IP ? -f1 : f1;
        const int64_t id0 = c0 ? __ldg(gid + s0) : 0, id1 = c1 ? __ldg(gid + s1) : 0;
        topk_push_lanes(ctl, k, tkd, tki, c0, key0, id0, lane);
        topk_push_lanes(ctl, k, tkd, tki, c1, key1, id1, lane);
        __syncwarp();
        T = topk_threshold(ctl, k, tkd);
      }
      __syncwarp();
      if ((t.flags & 4) && lane == 0) {  // last tile: the block's stats (search.py:132, :169)
        const int64_t m = t.block_m;
        r_total += m * A.d;
        if (linear) {
          r_touched += m * A.d;
          if (tr) {
            if (r_tlen >= 0 && r_tlen + 2 <= A.trace_cap) {
              tr[r_tlen] = 1;
              tr[r_tlen + 1] = (int32_t)m;
              r_tlen += 2;
            } else {
              r_tlen = -1;
            }
          }
        } else {
          r_touched += block_touched(m, warm_min, s_cnt, s_ends, nsteps);
          if (tr) {
            if (r_tlen >= 0 && r_tlen + 1 + nsteps <= A.trace_cap) {
              tr[r_tlen] = nsteps;
              for (int s = 0; s < nsteps; ++s) tr[r_tlen + 1 + s] = s_cnt[s];
              r_tlen += 1 + nsteps;
            } else {
              r_tlen = -1;
            }
          }
        }
      }
      __syncwarp();
    };

    // Commit a run of nr computed tiles starting at ring position com;
    // returns how many were committed.  A leading run of tiles that are
    // whole blocks, non-linear, speculated with the current threshold and
    // without survivors changes nothing but the stats (the threshold stays
    // put), so it is committed in parallel, one tile per lane, with the
    // values_touched the compute warp pre-computed.
    auto commit_run = [&](int com, int nr) -> int {
      bool simple = false;
      int touched = 0, m = 0;
      const TileSum* sm = nullptr;
      if (lane < nr) {
        const int sl = (com + lane) & RMASK;
        const TileDesc& t = s_desc[sl];
        sm = &s_sum[sl];
        m = t.block_m;
        touched = (int)sm->touched_spec;
        simple = t.flags == 6 && t.vis != 0 && A.pruner != PDX_PRUNER_NONE && T != INFINITY &&
                 t.tspec == T && m <= kTile && (sm->alive0 | sm->alive1) == 0;
      }
      const unsigned stop = __ballot_sync(kFull, !simple);
      const int np = min(nr, stop ? __ffs(stop) - 1 : 32);
      if (np == 0) {
        commit_one(com & RMASK);
        ++dbg_serial;
        return 1;
      }
      // per tile: touched <= 64 * d and total = m * d, so 32 of each fit int32
      const int tsum = __reduce_add_sync(kFull, lane < np ? touched : 0);
      const int msum = __reduce_add_sync(kFull, lane < np ? m : 0);
      if (tr) {
        const bool fits = r_tlen >= 0 && r_tlen + (int64_t)np * (1 + nsteps) <= A.trace_cap;
        const int64_t base = __shfl_sync(kFull, r_tlen, 0);
        const int fits0 = __shfl_sync(kFull, (int)fits, 0);  // lane 0 holds the stats
        if (lane < np && fits0) {
          int32_t* rec = tr + base + (int64_t)lane * (1 + nsteps);
          rec[0] = nsteps;
          for (int s = 0; s < nsteps; ++s) rec[1 + s] = sm->cnt[s];
        }
        if (lane == 0) r_tlen = fits ? r_tlen + (int64_t)np * (1 + nsteps) : -1;
      }
      if (lane == 0) {
        r_touched += tsum;
        r_total += (int64_t)msum * A.d;
      }
      dbg_fast += np;
      return np;
    };

    int com = 0, polls = 0;
    long long c_busy = 0;  // profile build: cycles committing (the rest is waiting)
    while (com < ntiles) {
      // never look past one ring turn: lane >= RB would alias an earlier slot
      const bool rdy =
          lane < RB && com + lane < ntiles && ld_acquire(&s_flag[(com + lane) & RMASK]) == 2;
      const unsigned rm = __ballot_sync(kFull, rdy);
      const int nr = (~rm) ? __ffs(~rm) - 1 : 32;
      // batch: a run of tiles costs the commit warp about as much as one
      const int want = min(min(RB, 32) / 2, ntiles - com);
      if (nr == 0 || (nr < want && polls < 3)) {
        // sleep in hardware until the first missing tile is written
        // (bounded while some are ready: a run costs about what one tile does)
        ++dbg_idle;
        ++polls;
#if PDX_MBAR_COMMIT
        const int n = com + nr;
        mbar_try(&s_ready[n & RMASK], (uint32_t)(n / RB) & 1u, nr == 0 ? (1u << 20) : 200u);
#else
        __nanosleep(48);
#endif
        continue;
      }
      polls = 0;
      int done = 0;
      const long long cb = PDX_SCAN_PROFILE ? clock64() : 0;
      while (done < nr) done += commit_run(com + done, nr - done);
      if (PDX_SCAN_PROFILE) c_busy += clock64() - cb;
      if (lane < done) {
        s_flag[(com + lane) & RMASK] = 0;
        mbar_arrive(&s_free[(com + lane) & RMASK]);
      }
      com += done;
      __syncwarp();
      if (lane == 0) {
        vstore(ctl.t_pub, T);
        st_release(&ctl.com_pub, com);
      }
    }
    if (lane == 0) {
      ctl.touched = r_touched;
      ctl.total = r_total;
      ctl.tlen = r_tlen;
    }
    if (A.debug && lane == 0) {
      int64_t* dg = A.debug + (int64_t)q * 16;
      dg[0] = clock64() - t_start;
      dg[1] = ntiles;
      dg[2] = dbg_fast;
      dg[3] = dbg_serial;
      dg[4] = dbg_replay;
      dg[5] = dbg_idle;
      dg[12] = c_busy;
    }
  }
  __syncthreads();
  if (A.debug && threadIdx.x == 0) {
    A.debug[(int64_t)q * 16 + 6] = ctl.ring_waits;
    A.debug[(int64_t)q * 16 + 7] = ctl.items;
    for (int i = 0; i < 4; ++i) A.debug[(int64_t)q * 16 + 8 + i] = (int64_t)ctl.cyc[i];
  }

  // ---- outputs
  const int64_t row = blockIdx.x;  // == q unless split
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const bool v = i < ctl.n;
    A.out_dist[row * k + i] = v ? tkd[i] : INFINITY;
    A.out_ids[row * k + i] = v ? tki[i] : -1;
  }
  if (threadIdx.x == 0) {
    if (A.out_count) A.out_count[row] = ctl.n;
    if (A.nsplit > 1) {  // the split ranges' stats add up (outputs zeroed by the host)
      if (A.out_touched) atomicAdd(reinterpret_cast<unsigned long long*>(&A.out_touched[q]),
                                   (unsigned long long)ctl.touched);
      if (A.out_total) atomicAdd(reinterpret_cast<unsigned long long*>(&A.out_total[q]),
                                 (unsigned long long)ctl.total);
    } else {
      if (A.out_touched) A.out_touched[q] = ctl.touched;
      if (A.out_total) A.out_total[q] = ctl.total;
    }
    if (A.trace_len) A.trace_len[q] = ctl.tlen;
  }
}

}  // namespace pdx
