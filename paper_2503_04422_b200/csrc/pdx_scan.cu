// K5 + K6: the pruned PDX scan with in-CTA top-k (PDXearch on sm_100a).
//
// Reference semantics (search.py:125-205, kernels.py:41-91, pruning.py:83-88):
// blocks are visited in a fixed order; block 0 and every block met while
// the heap is not full are scanned linearly; every other block runs the
// exponential step schedule, after each step pruning against T_b, the k-th
// best distance when the block STARTED (the heap only changes when the
// block's survivors are pushed at its end).
//
// B200 mapping.  One CTA per query: warp 0 is the COMMIT warp, warps 1..W
// are COMPUTE warps.  Rounds are double-buffered: while the compute warps
// scan round r (W x tpw tiles of 64 vectors), the commit warp commits round
// r-1 in visit order and schedules round r+1.
//  * A compute warp scans its tiles SPECULATIVELY (pdx_scan_spec.cuh) with a
//    threshold T' >= T_b (the committed threshold when the tile was
//    scheduled, or T_b itself for a block whose first tile is committed),
//    recording each slot's partial sum after every schedule step plus its
//    own per-step survivor counts and final survivor mask.  Partial sums do
//    not depend on the threshold and both bounds are monotone in T, so the
//    speculative survivors are a superset of the reference's at every step.
//  * The commit warp knows T_b exactly.  If T' == T_b (the usual case: the
//    top-k rarely changes inside the speculation window) the tile's own
//    counts and survivors ARE the reference's; otherwise it replays the
//    decisions from the recorded partials.  It pushes the exact survivors
//    into the top-k and keeps the reference's values_touched / survivors.
// Results, threshold chain, decisions and stats are the reference's.
//
// HBM layout (pdx_b200.h): tiles [d_pad/G][64][G].  G = 8 puts one slot's 8
// consecutive dims in one 32-byte sector: dense early steps read whole 2 KB
// groups (coalesced float4 loads), and a pruned survivor later costs one
// sector per 8 dims instead of one per dim.
#include <cub/block/block_scan.cuh>

#include "pdx_common.cuh"
#include "pdx_scan_spec.cuh"

namespace pdx {

struct Control {
  int32_t n;          // entries in the top-k
  int32_t cur_t;      // next tile within the current visit entry
  int64_t cur_v;      // next visit entry
  int64_t open_vis;   // visit index of a block whose first tile is committed but not its last
  float tblk;         // T_b of the open block
  int32_t linear;     // open block is linear
  int32_t warm_min;   // smallest survivor count that keeps WARMUP for the open block
  int32_t warm_m;     // the block size warm_min was computed for
  int32_t nvalid[3];  // tiles scheduled per round (mod 3)
  int64_t touched, total, tlen;
};
static_assert(sizeof(Control) <= 128, "control block");

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

// Shared-memory carve-up, shared by the kernel and the host launch code.
struct ScanSmem {
  size_t ctl, ratio, band, ends, bnd, cnt, wmin, desc, sum, items, wbnd, ids, tki, part, tkd, q,
      bmask, total;
};

__host__ __device__ inline ScanSmem scan_smem_layout(int W, int tpw, int k, int nsteps, int d_pad) {
  const int nt = 2 * W * tpw;  // tiles in flight (two rounds)
  ScanSmem L;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = (o + bytes + 15) & ~(size_t)15;
    return at;
  };
  L.ctl = take(128);
  L.ratio = take(sizeof(double) * kMaxSteps);
  L.band = take(sizeof(double) * kMaxSteps);
  L.ends = take(sizeof(int32_t) * kMaxSteps);
  L.bnd = take(sizeof(float) * kMaxSteps);
  L.cnt = take(sizeof(int32_t) * kMaxSteps);
  L.wmin = take(sizeof(int32_t) * (kTile + 1));
  L.desc = take(sizeof(TileDesc) * nt);
  L.sum = take(sizeof(TileSum) * nt);
  L.items = take(sizeof(SparseItem) * 32 * W);
  L.wbnd = take(sizeof(float) * kMaxSteps * W * tpw);
  L.ids = take(sizeof(int64_t) * kTile * nt);
  L.tki = take(sizeof(int64_t) * k);
  L.part = take(sizeof(float) * kTile * nsteps * nt);
  L.tkd = take(sizeof(float) * k);
  L.q = take(sizeof(float) * ((d_pad + 7) / 8) * 8);
  L.bmask = take((d_pad + 7) / 8);
  L.total = o;
  return L;
}

// ------------------------------------------------------------------ kernel
template <int G, bool ORD, int METRIC>
__global__ void __launch_bounds__(288) pdx_scan_kernel(const ScanArgs A, const int tpw) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int q = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W = (blockDim.x >> 5) - 1;  // compute warps
  const int RT = W * tpw;               // tiles per round
  const int nsteps = A.nsteps, k = A.k;

  const ScanSmem L = scan_smem_layout(W, tpw, k, nsteps, A.d_pad);
  Control& ctl = *reinterpret_cast<Control*>(smem + L.ctl);
  double* s_ratio = reinterpret_cast<double*>(smem + L.ratio);
  double* s_band = reinterpret_cast<double*>(smem + L.band);
  int32_t* s_ends = reinterpret_cast<int32_t*>(smem + L.ends);
  float* s_bnd = reinterpret_cast<float*>(smem + L.bnd);
  int32_t* s_cnt = reinterpret_cast<int32_t*>(smem + L.cnt);
  TileDesc* s_desc = reinterpret_cast<TileDesc*>(smem + L.desc);
  TileSum* s_sum = reinterpret_cast<TileSum*>(smem + L.sum);
  SparseItem* s_items = reinterpret_cast<SparseItem*>(smem + L.items);
  float* s_wbnd = reinterpret_cast<float*>(smem + L.wbnd);
  int64_t* s_ids = reinterpret_cast<int64_t*>(smem + L.ids);
  int64_t* tki = reinterpret_cast<int64_t*>(smem + L.tki);
  float* s_part = reinterpret_cast<float*>(smem + L.part);
  float* tkd = reinterpret_cast<float*>(smem + L.tkd);
  float* s_q = reinterpret_cast<float*>(smem + L.q);
  uint8_t* s_bmask = reinterpret_cast<uint8_t*>(smem + L.bmask);
  int32_t* s_wmin = reinterpret_cast<int32_t*>(smem + L.wmin);

  // ---- setup
  const float* qg = A.queries + (int64_t)q * A.d;
  const int ngroups = (A.d_pad + 7) / 8;
  for (int j = threadIdx.x; j < ngroups * 8; j += blockDim.x) s_q[j] = j < A.d ? qg[j] : 0.f;
  for (int j = threadIdx.x; j < ngroups; j += blockDim.x) s_bmask[j] = 0;
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
    ctl.cur_t = 0;
    ctl.cur_v = 0;
    ctl.open_vis = -1;
    ctl.tblk = INFINITY;
    ctl.linear = 1;
    ctl.warm_min = 0;
    ctl.warm_m = -1;
    ctl.nvalid[0] = ctl.nvalid[1] = ctl.nvalid[2] = 0;
    ctl.touched = ctl.total = ctl.tlen = 0;
  }
  __syncthreads();
  if (threadIdx.x < nsteps) {
    const double ds = (double)s_ends[threadIdx.x];
    s_ratio[threadIdx.x] = __ddiv_rn(ds, (double)A.ads_d);
    s_band[threadIdx.x] = __dadd_rn(1.0, __ddiv_rn(A.eps0, __dsqrt_rn(ds)));
  }
  const VisitEntry* vis = A.vis + (int64_t)q * A.vis_qstride;
  const int64_t nvis = A.vis_count[(int64_t)q * A.vis_count_qstride];
  int32_t* tr = A.trace ? A.trace + (int64_t)q * A.trace_cap : nullptr;

  // commit warp's register windows of visit entries: lane l holds entry base+l
  int64_t wbase = 0;
  VisitEntry cur = {0, 0, 0}, nxt = {0, 0, 0};

  // schedule RT tiles in visit order into desc buffer `buf` (commit warp)
  auto schedule = [&](int buf, int slot3) {
    const float tlive = topk_threshold(ctl, k, tkd);
    int nvalid = 0;
    int64_t cv = ctl.cur_v;
    int ct = ctl.cur_t;
    for (int w = 0; w < RT; ++w) {
      if (cv >= nvis) break;
      if (cv >= wbase + 32) {  // slide the window; prefetch the one after
        wbase += 32;
        cur = nxt;
        nxt = VisitEntry{0, 0, 0};
        if (wbase + 32 + lane < nvis) nxt = vis[wbase + 32 + lane];
      }
      const int src = (int)(cv - wbase);
      const int64_t tile0 = __shfl_sync(kFull, cur.tile0, src);
      const int m = __shfl_sync(kFull, cur.m, src);
      const int seg = __shfl_sync(kFull, cur.seg, src);
      const int ntl = (m + kTile - 1) / kTile;
      if (lane == 0) {
        TileDesc t;
        t.tile = tile0 + ct;
        t.m_tile = min(kTile, m - kTile * ct);
        t.seg = seg;
        t.block_m = m;
        t.vis = (int32_t)cv;
        t.flags = (ct == 0 ? 2 : 0) | (ct == ntl - 1 ? 4 : 0);
        if (A.pruner == PDX_PRUNER_NONE) t.tspec = INFINITY;
        else t.tspec = (cv == ctl.open_vis) ? ctl.tblk : tlive;
        s_desc[buf * RT + w] = t;
      }
      ++nvalid;
      if (++ct == ntl) {
        ct = 0;
        ++cv;
      }
    }
    if (lane == 0) {
      ctl.cur_v = cv;
      ctl.cur_t = ct;
      ctl.nvalid[slot3] = nvalid;
    }
    __syncwarp();
  };

  // commit the tiles of desc buffer `buf` in visit order (commit warp)
  auto commit = [&](int buf, int nv) {
    int w = 0;
    {
      // Parallel fast path.  A leading run of tiles that are whole blocks,
      // non-linear, speculated with the current threshold and without
      // survivors changes nothing but the stats: the threshold stays put
      // across the run, so every tile's own counts are the reference's.
      const float T = topk_threshold(ctl, k, tkd);
      bool simple = false;
      TileDesc t;
      const TileSum* sm = nullptr;
      if (lane < nv) {
        const int ti = buf * RT + lane;
        t = s_desc[ti];
        sm = &s_sum[ti];
        simple = t.flags == 6 && t.vis != 0 && A.pruner != PDX_PRUNER_NONE && T != INFINITY &&
                 t.tspec == T && t.block_m <= kTile && sm->alive0 == 0 && sm->alive1 == 0;
      }
      const unsigned stop = __ballot_sync(kFull, !simple);
      const int np = min(nv, stop ? __ffs(stop) - 1 : 32);
      if (np > 0) {
        int64_t touched = 0, total = 0;
        if (lane < np) {
          const int64_t m = t.block_m;
          const int wmin = s_wmin[m];
          bool warm = true;
          int64_t prev = m;
          int a = 0;
          for (int s = 0; s < nsteps; ++s) {
            const int w_s = s_ends[s] - a;
            a = s_ends[s];
            if (warm && prev >= wmin) {
              touched += m * w_s;
            } else {
              warm = false;
              touched += prev * w_s;
            }
            prev = sm->cnt[s];
          }
          total = m * A.d;
          if (tr && ctl.tlen >= 0 && ctl.tlen + (int64_t)np * (1 + nsteps) <= A.trace_cap) {
            int32_t* rec = tr + ctl.tlen + (int64_t)lane * (1 + nsteps);
            rec[0] = nsteps;
            for (int s = 0; s < nsteps; ++s) rec[1 + s] = sm->cnt[s];
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          touched += __shfl_xor_sync(kFull, touched, o);
          total += __shfl_xor_sync(kFull, total, o);
        }
        __syncwarp();
        if (lane == 0) {
          ctl.touched += touched;
          ctl.total += total;
          if (tr) {
            if (ctl.tlen >= 0 && ctl.tlen + (int64_t)np * (1 + nsteps) <= A.trace_cap)
              ctl.tlen += (int64_t)np * (1 + nsteps);
            else
              ctl.tlen = -1;
          }
          ctl.open_vis = -1;
        }
        __syncwarp();
        w = np;
      }
    }
    for (; w < nv; ++w) {
      const int ti = buf * RT + w;
      const TileDesc t = s_desc[ti];
      const TileSum& sm = s_sum[ti];
      const float* part = s_part + (size_t)ti * nsteps * kTile;
      if (t.flags & 2) {  // first tile of its block: T_b is fixed now
        const float T = topk_threshold(ctl, k, tkd);
        const int lin = (t.vis == 0 || A.pruner == PDX_PRUNER_NONE || T == INFINITY);
        if (lane < nsteps) {
          s_cnt[lane] = 0;
          if (!lin)
            s_bnd[lane] = ads_or_bond_bound(A.pruner, T, s_ends[lane], A.ads_d, s_ratio[lane],
                                            s_band[lane]);
        }
        if (lane == 0) {
          ctl.tblk = T;
          ctl.linear = lin;
          if (!lin && t.block_m != ctl.warm_m) {
            ctl.warm_min = warm_min_count(t.block_m, A.sf);
            ctl.warm_m = t.block_m;
          }
        }
        __syncwarp();
      }
      const int s0 = 2 * lane, s1 = s0 + 1;
      bool c0, c1;
      if (ctl.linear) {
        c0 = s0 < t.m_tile;
        c1 = s1 < t.m_tile;
      } else if (t.tspec == ctl.tblk) {
        // the speculation ran with the exact threshold: its counts and
        // survivors are the reference's
        if (lane < nsteps) s_cnt[lane] += sm.cnt[lane];
        c0 = (sm.alive0 >> lane) & 1;
        c1 = (sm.alive1 >> lane) & 1;
      } else {
        c0 = s0 < t.m_tile;
        c1 = s1 < t.m_tile;
        int mycnt = 0;
        for (int s = 0; s < nsteps; ++s) {
          if (s == sm.dense_steps) {  // later partials exist only for parked slots
            c0 = c0 && ((sm.items0 >> lane) & 1);
            c1 = c1 && ((sm.items1 >> lane) & 1);
          }
          const float bs = s_bnd[s];
          const float2 pv = *reinterpret_cast<const float2*>(part + s * kTile + s0);
          c0 = c0 && (pv.x < bs);
          c1 = c1 && (pv.y < bs);
          const int cnt = __popc(__ballot_sync(kFull, c0)) + __popc(__ballot_sync(kFull, c1));
          if (lane == s) mycnt = cnt;
        }
        if (lane < nsteps) s_cnt[lane] += mycnt;
      }
      if (__any_sync(kFull, c0 || c1)) {
        const float2 fin = *reinterpret_cast<const float2*>(part + (nsteps - 1) * kTile + s0);
        const int64_t* sid = s_ids + (size_t)ti * kTile;
        const float key0 = METRIC == PDX_METRIC_IP ? -fin.x : fin.x;
        const float key1 = METRIC == PDX_METRIC_IP ? -fin.y : fin.y;
        topk_push_lanes(ctl, k, tkd, tki, c0, key0, c0 ? sid[s0] : 0, lane);
        topk_push_lanes(ctl, k, tkd, tki, c1, key1, c1 ? sid[s1] : 0, lane);
      }
      __syncwarp();
      if (t.flags & 4) {  // last tile: the block's stats (search.py:132, :169)
        if (lane == 0) {
          const int64_t m = t.block_m;
          ctl.total += m * A.d;
          if (ctl.linear) {
            ctl.touched += m * A.d;
            if (tr) {
              if (ctl.tlen >= 0 && ctl.tlen + 2 <= A.trace_cap) {
                tr[ctl.tlen] = 1;
                tr[ctl.tlen + 1] = (int32_t)m;
                ctl.tlen += 2;
              } else {
                ctl.tlen = -1;
              }
            }
          } else {
            bool warm = true;
            int64_t prev = m;
            int a = 0;
            for (int s = 0; s < nsteps; ++s) {
              const int w_s = s_ends[s] - a;
              a = s_ends[s];
              if (warm && prev >= ctl.warm_min) {
                ctl.touched += m * w_s;
              } else {
                warm = false;
                ctl.touched += prev * w_s;
              }
              prev = s_cnt[s];
            }
            if (tr) {
              if (ctl.tlen >= 0 && ctl.tlen + 1 + nsteps <= A.trace_cap) {
                tr[ctl.tlen] = nsteps;
                for (int s = 0; s < nsteps; ++s) tr[ctl.tlen + 1 + s] = s_cnt[s];
                ctl.tlen += 1 + nsteps;
              } else {
                ctl.tlen = -1;
              }
            }
          }
          ctl.open_vis = -1;
        }
      } else if (lane == 0) {
        ctl.open_vis = t.vis;
      }
      __syncwarp();
    }
  };

  if (warp == 0) {
    if (lane < nvis) cur = vis[lane];
    if (32 + lane < nvis) nxt = vis[32 + lane];
    schedule(0, 0);
  }
  __syncthreads();

  for (int r = 0;; ++r) {
    const int nv_cur = ctl.nvalid[r % 3];
    const int nv_prev = r > 0 ? ctl.nvalid[(r + 2) % 3] : 0;
    if (nv_cur == 0 && nv_prev == 0) break;
    if (warp == 0) {
      if (nv_prev) commit((r + 1) & 1, nv_prev);
      schedule((r + 1) & 1, (r + 1) % 3);
    } else {
      const int w = warp - 1, buf = r & 1;
      const int t0 = buf * RT + w * tpw;  // this warp's slice of the round
      const int nt = min(tpw, nv_cur - w * tpw);
      if (nt > 0) {
        SliceRefs R;
        R.desc = s_desc + t0;
        R.part = s_part + (size_t)t0 * nsteps * kTile;
        R.sum = s_sum + t0;
        R.sid = s_ids + (size_t)t0 * kTile;
        R.bnd = s_wbnd + (size_t)w * tpw * kMaxSteps;
        R.items = s_items + 32 * w;
        QueryRefs Q;
        Q.q = s_q;
        Q.ends = s_ends;
        Q.ratio = s_ratio;
        Q.band = s_band;
        Q.bmask = s_bmask;
        int nitems = 0;
        for (int j = 0; j < nt; ++j) {
          if (G == 8 && !ORD)
            dense_tile_g8<METRIC>(A, R.desc[j], j, Q, R, nitems, lane);
          else
            dense_tile_generic<G, ORD, METRIC>(A, q, R.desc[j], j, Q, R, nitems, lane);
        }
        sparse_phase<G, ORD, METRIC>(A, q, Q, R, nitems, lane);
      }
    }
    __syncthreads();
  }

  // ---- outputs
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const bool v = i < ctl.n;
    A.out_dist[(int64_t)q * k + i] = v ? tkd[i] : INFINITY;
    A.out_ids[(int64_t)q * k + i] = v ? tki[i] : -1;
  }
  if (threadIdx.x == 0) {
    if (A.out_count) A.out_count[q] = ctl.n;
    if (A.out_touched) A.out_touched[q] = ctl.touched;
    if (A.out_total) A.out_total[q] = ctl.total;
    if (A.trace_len) A.trace_len[q] = ctl.tlen;
  }
}

// ------------------------------------------------------------ visit lists
// Flattens, per query, the block sequence ivf_search hands to search()
// (index.py:140-149): selected buckets in selection order, each bucket's
// chain in stored order.
__global__ void __launch_bounds__(256) build_visits_kernel(
    const int32_t* __restrict__ seg_bucket, int nseg, const int64_t* __restrict__ bucket_block,
    const int64_t* __restrict__ block_tile, const int32_t* __restrict__ block_m,
    VisitEntry* __restrict__ out, int64_t maxvis, int32_t* __restrict__ counts,
    int32_t* __restrict__ overflow) {
  using Scan = cub::BlockScan<int64_t, 256>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int64_t s_b0[256], s_off[256], s_nb[256];
  __shared__ int64_t running;
  const int q = blockIdx.x;
  if (threadIdx.x == 0) running = 0;
  __syncthreads();
  for (int base = 0; base < nseg; base += 256) {
    const int pseg = base + threadIdx.x;
    int64_t b0 = 0, nb = 0;
    if (pseg < nseg) {
      const int bucket = seg_bucket ? seg_bucket[(int64_t)q * nseg + pseg] : pseg;
      b0 = bucket_block[bucket];
      nb = bucket_block[bucket + 1] - b0;
    }
    int64_t off, tot;
    Scan(tmp).ExclusiveSum(nb, off, tot);
    s_b0[threadIdx.x] = b0;
    s_nb[threadIdx.x] = nb;
    s_off[threadIdx.x] = off;
    __syncthreads();
    const int cnt = min(256, nseg - base);
    for (int i = 0; i < cnt; ++i) {
      for (int64_t j = threadIdx.x; j < s_nb[i]; j += 256) {
        const int64_t v = running + s_off[i] + j;
        if (v < maxvis) {
          const int64_t blk = s_b0[i] + j;
          VisitEntry e;
          e.tile0 = block_tile[blk];
          e.m = block_m[blk];
          e.seg = base + i;
          out[(int64_t)q * maxvis + v] = e;
        } else {
          *overflow = 1;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) running += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) counts[q] = (int32_t)(running < maxvis ? running : maxvis);
}

template <int G, bool ORD, int METRIC>
static cudaError_t launch_scan(const ScanArgs& A, int nq, int W, int tpw, size_t smem,
                               cudaStream_t st) {
  auto fn = pdx_scan_kernel<G, ORD, METRIC>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fn<<<nq, (W + 1) * 32, smem, st>>>(A, tpw);
  return cudaGetLastError();
}

template <int G, bool ORD>
static cudaError_t launch_metric(int metric, const ScanArgs& A, int nq, int W, int tpw,
                                 size_t smem, cudaStream_t st) {
  switch (metric) {
    case PDX_METRIC_L2: return launch_scan<G, ORD, PDX_METRIC_L2>(A, nq, W, tpw, smem, st);
    case PDX_METRIC_L1: return launch_scan<G, ORD, PDX_METRIC_L1>(A, nq, W, tpw, smem, st);
    default: return launch_scan<G, ORD, PDX_METRIC_IP>(A, nq, W, tpw, smem, st);
  }
}

}  // namespace pdx

using namespace pdx;

static int schedule_steps(int d, int initial_step) {
  int n = 0;
  int64_t start = 0, width = initial_step;
  while (start < d) {
    start = start + width < d ? start + width : d;
    width *= 2;
    ++n;
  }
  return n;
}

extern "C" int64_t pdx_search_workspace(const pdx_store* store, int64_t nq, int32_t nseg) {
  if (!store || nq < 0 || nseg < 0) return -1;
  const int64_t maxvis = (int64_t)nseg * store->max_bucket_blocks;
  return 256 + nq * (int64_t)sizeof(int32_t) + 256 + nq * maxvis * (int64_t)sizeof(VisitEntry) + 256;
}

extern "C" int pdx_search(const pdx_store* store, const pdx_search_params* prm,
                          const float* d_queries, int64_t nq, const int32_t* d_seg_bucket,
                          int32_t nseg, const uint16_t* d_orders, int64_t order_qstride,
                          int64_t order_sstride, const pdx_search_out* out, void* d_work,
                          int64_t work_bytes, void* stream) {
  PDX_REQUIRE(store && prm && out, "pdx_search: null argument");
  PDX_REQUIRE(prm->k >= 1, "k must be >= 1");
  PDX_REQUIRE(prm->k <= 4096, "k = %d exceeds this build's limit of 4096", prm->k);
  PDX_REQUIRE(prm->selection_fraction > 0.0 && prm->selection_fraction <= 1.0,
              "selection_fraction must be in (0, 1]");
  PDX_REQUIRE(prm->initial_step >= 1, "initial_step must be >= 1");
  PDX_REQUIRE(prm->metric >= 0 && prm->metric <= 2, "unknown metric %d", prm->metric);
  PDX_REQUIRE(prm->pruner >= 0 && prm->pruner <= 2, "unknown pruner %d", prm->pruner);
  PDX_REQUIRE(!(prm->metric == PDX_METRIC_IP && prm->pruner != PDX_PRUNER_NONE),
              "inner product has no monotone lower bound; use pruner='none' for IP searches");
  PDX_REQUIRE(!(prm->pruner == PDX_PRUNER_ADS && prm->metric != PDX_METRIC_L2),
              "the ads pruner applies to squared L2 only");
  PDX_REQUIRE(prm->pruner != PDX_PRUNER_ADS || prm->ads_epsilon0 > 0.0, "epsilon0 must be positive");
  PDX_REQUIRE(prm->pruner != PDX_PRUNER_ADS || prm->ads_d >= 1, "ads d must be >= 1");
  PDX_REQUIRE(store->d >= 1 && store->d <= 65535, "dimensionality %d unsupported", store->d);
  PDX_REQUIRE(store->group == 1 || store->group == 8, "group must be 1 or 8");
  PDX_REQUIRE(store->d_pad % store->group == 0 && store->d_pad >= store->d, "bad d_pad");
  PDX_REQUIRE(nq >= 0 && nq <= 0x7fffffff, "bad query count");
  PDX_REQUIRE(nseg >= 0, "bad segment count");
  PDX_REQUIRE(d_seg_bucket || nseg <= store->nbuckets, "segments exceed buckets");
  if (nq == 0) return PDX_OK;
  const int nsteps = schedule_steps(store->d, prm->initial_step);
  PDX_REQUIRE(nsteps <= kMaxSteps, "step schedule too long (%d steps)", nsteps);

  int dev = 0, optin = 0;
  PDX_CUDA_CHECK(cudaGetDevice(&dev));
  PDX_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  int W = prm->warps > 0 ? prm->warps : 4;  // compute warps per query CTA
  if (W > 8) W = 8;
  int tpw = prm->tiles_per_warp > 0 ? prm->tiles_per_warp : 2;
  if (tpw > kMaxTpw) tpw = kMaxTpw;
  size_t smem = scan_smem_layout(W, tpw, prm->k, nsteps, store->d_pad).total;
  while ((W > 1 || tpw > 1) && smem > (size_t)optin) {
    if (tpw > 1) tpw /= 2;
    else W /= 2;
    smem = scan_smem_layout(W, tpw, prm->k, nsteps, store->d_pad).total;
  }
  PDX_REQUIRE(smem <= (size_t)optin, "k/d too large for shared memory (%zu bytes)", smem);

  const int64_t maxvis = (int64_t)nseg * store->max_bucket_blocks;
  // visit lists: query-independent when no per-query bucket selection is given
  const int64_t nlists = d_seg_bucket ? nq : 1;
  const int64_t need = pdx_search_workspace(store, nlists, nseg);
  PDX_REQUIRE(d_work && work_bytes >= need, "workspace too small (%lld < %lld)",
              (long long)work_bytes, (long long)need);
  unsigned char* w = reinterpret_cast<unsigned char*>(d_work);
  int32_t* d_overflow = reinterpret_cast<int32_t*>(w);
  int32_t* d_counts = reinterpret_cast<int32_t*>(w + 256);
  VisitEntry* d_vis = reinterpret_cast<VisitEntry*>(
      w + 256 + ((nlists * sizeof(int32_t) + 255) / 256) * 256);
  cudaStream_t st = as_stream(stream);
  PDX_CUDA_CHECK(cudaMemsetAsync(d_overflow, 0, sizeof(int32_t), st));
  if (nseg > 0 && maxvis > 0) {
    build_visits_kernel<<<(unsigned)nlists, 256, 0, st>>>(
        d_seg_bucket, nseg, store->d_bucket_block, store->d_block_tile, store->d_block_m, d_vis,
        maxvis, d_counts, d_overflow);
  } else {
    PDX_CUDA_CHECK(cudaMemsetAsync(d_counts, 0, nlists * sizeof(int32_t), st));
  }
  PDX_LAUNCH_CHECK();

  ScanArgs A;
  memset(&A, 0, sizeof(A));
  A.tiles = store->d_tiles;
  A.tile_ids = store->d_tile_ids;
  A.d = store->d;
  A.d_pad = store->d_pad;
  A.tile_stride = (int64_t)store->d_pad * kTile;
  A.vis = d_vis;
  A.vis_qstride = d_seg_bucket ? maxvis : 0;
  A.vis_count = d_counts;
  A.vis_count_qstride = d_seg_bucket ? 1 : 0;
  A.queries = d_queries;
  A.orders = d_orders;
  A.oqs = order_qstride;
  A.oss = order_sstride;
  A.k = prm->k;
  A.pruner = prm->pruner;
  A.initial_step = prm->initial_step;
  A.nsteps = nsteps;
  A.sf = prm->selection_fraction;
  A.ads_d = prm->ads_d >= 1 ? prm->ads_d : store->d;
  A.eps0 = prm->ads_epsilon0;
  A.out_dist = out->d_dist;
  A.out_ids = out->d_ids;
  A.out_count = out->d_count;
  A.out_touched = out->d_touched;
  A.out_total = out->d_total;
  A.trace = out->d_trace;
  A.trace_cap = out->d_trace ? out->trace_cap : 0;
  A.trace_len = out->d_trace_len;
  PDX_REQUIRE(A.out_dist && A.out_ids, "output buffers required");

  cudaError_t e;
  const bool ord = d_orders != nullptr;
  if (store->group == 8)
    e = ord ? launch_metric<8, true>(prm->metric, A, (int)nq, W, tpw, smem, st)
            : launch_metric<8, false>(prm->metric, A, (int)nq, W, tpw, smem, st);
  else
    e = ord ? launch_metric<1, true>(prm->metric, A, (int)nq, W, tpw, smem, st)
            : launch_metric<1, false>(prm->metric, A, (int)nq, W, tpw, smem, st);
  PDX_CUDA_CHECK(e);
  return PDX_OK;
}
