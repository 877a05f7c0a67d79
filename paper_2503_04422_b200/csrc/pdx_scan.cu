// K5 + K6: the pruned PDX scan with in-CTA top-k (PDXearch on sm_100a).
//
// Reference semantics (search.py:125-205, kernels.py:41-91, pruning.py:83-88):
// blocks are visited in a fixed order; block 0 and every block met while
// the heap is not full are scanned linearly; every other block runs the
// exponential step schedule, after each step pruning against T_b, the k-th
// best distance when the block STARTED (the heap only changes when the
// block's survivors are pushed at its end).
//
// B200 mapping (pdx_scan_kernel.cuh).  One CTA per query: a commit warp and
// W compute warps around a ring of 64-vector tile slots.
//  * Compute warps scan tiles SPECULATIVELY (pdx_scan_spec.cuh) with a
//    threshold T' >= T_b (the committed threshold when the tile was
//    scheduled, or T_b itself for a block whose first tile is committed),
//    recording each slot's partial sum at every step it reaches plus their
//    own per-step survivor counts and final survivor mask.  Partial sums do
//    not depend on the threshold and both bounds are monotone in T, so the
//    speculative survivors are a superset of the reference's at every step.
//  * The commit warp commits tiles in visit order with the exact T_b.  If
//    T' == T_b (the usual case: the top-k rarely changes inside the
//    speculation window) the tile's own counts and survivors ARE the
//    reference's; otherwise it replays the decisions from the recorded
//    partials.  It pushes the exact survivors into the top-k and keeps the
//    reference's values_touched / survivor traces.
// Results, threshold chain, decisions and stats are the reference's.
//
// HBM layout (pdx_b200.h): tiles [d_pad/G][64][G].  G = 8 puts one slot's 8
// consecutive dims in one 32-byte sector: dense early steps read whole 2 KB
// groups (coalesced 256-bit loads), and a pruned survivor later costs one
// sector per 8 dims instead of one per dim.
#include <cub/block/block_scan.cuh>

#include "pdx_common.cuh"
#include "pdx_scan_kernel.cuh"
#include "pdx_batch.cuh"

namespace pdx {

// ------------------------------------------------------------ visit lists
// Flattens, per query, the block sequence ivf_search hands to search()
// (index.py:140-149): selected buckets in selection order, each bucket's
// chain in stored order.
__global__ void __launch_bounds__(256) build_visits_kernel(
    const int32_t* __restrict__ seg_bucket, int nseg, const int64_t* __restrict__ bucket_block,
    const int64_t* __restrict__ block_tile, const int32_t* __restrict__ block_m,
    const int32_t* __restrict__ tile_block, TileEntry* __restrict__ out, int64_t maxtiles,
    int32_t* __restrict__ counts, int32_t* __restrict__ overflow, const int32_t* __restrict__ only) {
  using Scan = cub::BlockScan<int64_t, 256>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int64_t s_b0[256], s_t0[256], s_toff[256], s_boff[256];
  __shared__ int64_t run_t, run_b;
  const int q = blockIdx.x;
  if (only && only[q] == 0) return;
  if (threadIdx.x == 0) run_t = run_b = 0;
  __syncthreads();
  for (int base = 0; base < nseg; base += 256) {
    const int pseg = base + threadIdx.x;
    int64_t b0 = 0, nb = 0, t0 = 0, nt = 0;
    if (pseg < nseg) {
      const int bucket = seg_bucket ? seg_bucket[(int64_t)q * nseg + pseg] : pseg;
      b0 = bucket_block[bucket];
      nb = bucket_block[bucket + 1] - b0;
      t0 = block_tile[b0];
      nt = block_tile[b0 + nb] - t0;  // a bucket's tiles are contiguous
    }
    int64_t toff, ttot, boff, btot;
    Scan(tmp).ExclusiveSum(nt, toff, ttot);
    __syncthreads();
    Scan(tmp).ExclusiveSum(nb, boff, btot);
    s_b0[threadIdx.x] = b0;
    s_t0[threadIdx.x] = t0;
    s_toff[threadIdx.x] = toff;
    s_boff[threadIdx.x] = boff;
    __syncthreads();
    // every tile of this chunk of segments in parallel: tile v of the chunk
    // belongs to the last segment i with toff[i] <= v (binary search)
    const int cnt = min(256, nseg - base);
    for (int64_t vv = threadIdx.x; vv < ttot; vv += 256) {
      int lo = 0, hi = cnt - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_toff[mid] <= vv) lo = mid; else hi = mid - 1;
      }
      const int i = lo;
      const int64_t j = vv - s_toff[i];
      {
        const int64_t v = run_t + vv;
        if (v < maxtiles) {
          const int64_t tile = s_t0[i] + j;
          const int32_t blk = tile_block[tile];
          const int64_t bt = block_tile[blk];
          const int32_t m = block_m[blk];
          const int32_t tib = (int32_t)(tile - bt);
          const int32_t ntl = (int32_t)(block_tile[blk + 1] - bt);
          TileEntry e;
          e.tile = tile;
          e.m_tile = min(kTile, m - kTile * tib);
          e.block_m = m;
          e.seg = base + i;
          e.vis = (int32_t)(run_b + s_boff[i] + (blk - s_b0[i]));
          e.tib = tib;
          e.flags = (tib == 0 ? 2 : 0) | (tib == ntl - 1 ? 4 : 0);
          out[(int64_t)q * maxtiles + v] = e;
        } else {
          *overflow = 1;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      run_t += ttot;
      run_b += btot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) counts[q] = (int32_t)(run_t < maxtiles ? run_t : maxtiles);
}

// Per-step bound factors for ads_or_bond_bound, [0][s] = ratio, [1][s] = band:
// ADS ratio = d'/D and band = 1 + eps0/sqrt(d') in float64 (pruning.py:80-88);
// ratio = band = 1 wherever the comparison is against T itself (BOND, none,
// BSA — whose per-vector estimate is compared with T — and ADS at d' >= D).
// The ADS bound's per-step factors (pruning.py:68-88) in float64, on the
// host: IEEE division, square root and addition, the same values the device
// intrinsics (__ddiv_rn, __dsqrt_rn, __dadd_rn) give.
static void bound_factors(int pruner, int d, int initial_step, int nsteps, int ads_d, double eps0,
                          double* out) {
  int64_t e = 0, width = initial_step;  // step_schedule (search.py:106-117)
  for (int s = 0; s < 2 * kMaxSteps; ++s) out[s] = 1.0;
  for (int s = 0; s < nsteps; ++s, width *= 2) {
    e = e + width < d ? e + width : d;
    double ratio = 1.0, band = 1.0;
    if (pruner == PDX_PRUNER_ADS && e < ads_d) {
      ratio = (double)e / (double)ads_d;
      band = 1.0 + eps0 / sqrt((double)e);
    }
    out[s] = ratio;
    out[kMaxSteps + s] = band;
  }
}

// len(TopK) after a split-mode merge: the valid ids of each row
__global__ void count_valid_kernel(const int64_t* __restrict__ ids, int64_t nq, int k,
                                   int32_t* __restrict__ count) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  int c = 0;
  for (int j = 0; j < k; ++j) c += ids[q * k + j] >= 0;
  count[q] = c;
}

template <int G, bool ORD, int METRIC>
static cudaError_t launch_scan(const ScanArgs& A, const ScanSmem& L, int nq, int W, int tpw,
                               cudaStream_t st) {
  auto fn = pdx_scan_kernel<G, ORD, METRIC>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
  if (e != cudaSuccess) return e;
  // several query CTAs per SM need the full shared-memory carveout
  e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  fn<<<nq, (W + 1) * 32, L.total, st>>>(A, L, tpw);
  return cudaGetLastError();
}

template <int G, bool ORD>
static cudaError_t launch_metric(int metric, const ScanArgs& A, const ScanSmem& L, int nq, int W,
                                 int tpw, cudaStream_t st) {
  switch (metric) {
    case PDX_METRIC_L2: return launch_scan<G, ORD, PDX_METRIC_L2>(A, L, nq, W, tpw, st);
    case PDX_METRIC_L1: return launch_scan<G, ORD, PDX_METRIC_L1>(A, L, nq, W, tpw, st);
    case kMetricL2Bsa:
      if (!ORD) return launch_scan<G, false, kMetricL2Bsa>(A, L, nq, W, tpw, st);
      return cudaErrorInvalidValue;
    default: return launch_scan<G, ORD, PDX_METRIC_IP>(A, L, nq, W, tpw, st);
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
  const int64_t maxvis = (int64_t)nseg * store->max_bucket_tiles;
  return 512 + nq * (int64_t)sizeof(int32_t) + 256 + nq * maxvis * (int64_t)sizeof(TileEntry) + 256;
}

namespace pdx {
int linear_split_scan(const pdx_store* store, int metric, int k, const float* d_queries,
                      int64_t nq, int nsplit, float* tdist, int64_t* tids, int64_t* touched,
                      int64_t* total, cudaStream_t st, bool* applied);
}

static int search_impl(const pdx_store* store, const pdx_search_params* prm,
                       const float* d_queries, int64_t nq, const int32_t* d_seg_bucket,
                       int32_t nseg, const uint16_t* d_orders, int64_t order_qstride,
                       int64_t order_sstride, const pdx_search_out* out, void* d_work,
                       int64_t work_bytes, void* stream, const int32_t* only, bool allow_batched,
                       bool dense_spec = false) {
  PDX_REQUIRE(store && prm && out, "pdx_search: null argument");
  PDX_REQUIRE(prm->k >= 1, "k must be >= 1");
  PDX_REQUIRE(prm->k <= 4096, "k = %d exceeds this build's limit of 4096", prm->k);
  PDX_REQUIRE(prm->selection_fraction > 0.0 && prm->selection_fraction <= 1.0,
              "selection_fraction must be in (0, 1]");
  PDX_REQUIRE(prm->initial_step >= 1, "initial_step must be >= 1");
  PDX_REQUIRE(prm->metric >= 0 && prm->metric <= 2, "unknown metric %d", prm->metric);
  PDX_REQUIRE(prm->pruner >= 0 && prm->pruner <= 3, "unknown pruner %d", prm->pruner);
  PDX_REQUIRE(!(prm->metric == PDX_METRIC_IP && prm->pruner != PDX_PRUNER_NONE),
              "inner product has no monotone lower bound; use pruner='none' for IP searches");
  PDX_REQUIRE(!(prm->pruner == PDX_PRUNER_ADS && prm->metric != PDX_METRIC_L2),
              "the ads pruner applies to squared L2 only");
  PDX_REQUIRE(!(prm->pruner == PDX_PRUNER_BSA && prm->metric != PDX_METRIC_L2),
              "the bsa pruner applies to squared L2 only");
  PDX_REQUIRE(prm->pruner != PDX_PRUNER_BSA || prm->bsa_coef, "bsa needs its coefficients");
  PDX_REQUIRE(prm->pruner != PDX_PRUNER_BSA || !d_orders,
              "bsa visits dimensions in their (principal-axis) order; no visit orders");
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
  PDX_REQUIRE(prm->pruner != PDX_PRUNER_BSA ||
                  (store->d_resid && store->resid_steps == nsteps &&
                   store->resid_initial_step == prm->initial_step),
              "bsa needs the store's residual energies for this step schedule "
              "(pdx_bsa_residuals with initial_step %d)", prm->initial_step);

  if (allow_batched && batched_eligible(store, prm, nq, d_seg_bucket, nseg, d_orders, out))
    return search_batched(store, prm, d_queries, nq, d_seg_bucket, nseg, out, d_work, work_bytes,
                          stream);

  int dev = 0, optin = 0;
  PDX_CUDA_CHECK(cudaGetDevice(&dev));
  PDX_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  int W = prm->warps > 0 ? prm->warps : 8;  // compute warps per query CTA
  if (W > 8) W = 8;
  int tpw = 1;  // tiles per claim: a power of two <= kMaxTpw
  while (tpw * 2 <= (prm->tiles_per_warp > 0 ? prm->tiles_per_warp : 4) && tpw * 2 <= kMaxTpw)
    tpw *= 2;
  int rb = 2 * tpw;  // ring slots: a power of two (masks, not divisions, in the kernel)
  while (rb < (prm->ring_slots > 0 ? prm->ring_slots : W * tpw)) rb *= 2;
  const bool has_ord = d_orders != nullptr;
  ScanSmem L = scan_smem_layout(W, tpw, rb, prm->k, nsteps, store->d_pad, has_ord);
  while (rb > 2 * tpw && L.total > optin) {
    rb /= 2;
    L = scan_smem_layout(W, tpw, rb, prm->k, nsteps, store->d_pad, has_ord);
  }
  PDX_REQUIRE(L.total <= optin, "k/d too large for shared memory (%d bytes)", L.total);

  const int64_t maxvis = (int64_t)nseg * store->max_bucket_tiles;
  // visit lists: query-independent when no per-query bucket selection is given
  const int64_t nlists = d_seg_bucket ? nq : 1;
  const int64_t need = pdx_search_workspace(store, nlists, nseg);
  PDX_REQUIRE(d_work && work_bytes >= need, "workspace too small (%lld < %lld)",
              (long long)work_bytes, (long long)need);
  unsigned char* w = reinterpret_cast<unsigned char*>(d_work);
  int32_t* d_overflow = reinterpret_cast<int32_t*>(w);
  int32_t* d_counts = reinterpret_cast<int32_t*>(w + 512);
  TileEntry* d_vis = reinterpret_cast<TileEntry*>(
      w + 512 + ((nlists * sizeof(int32_t) + 255) / 256) * 256);
  cudaStream_t st = as_stream(stream);
  // (the overflow word is write-only diagnostics: the fallback of a batched
  // search, `only`, skips its reset and saves a graph node)
  if (!only) PDX_CUDA_CHECK(cudaMemsetAsync(d_overflow, 0, sizeof(int32_t), st));
  if (nseg > 0 && maxvis > 0) {
    build_visits_kernel<<<(unsigned)nlists, 256, 0, st>>>(
        d_seg_bucket, nseg, store->d_bucket_block, store->d_block_tile, store->d_block_m,
        store->d_tile_block, d_vis,
        maxvis, d_counts, d_overflow, only);
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
  A.ads_d = (prm->ads_d >= 1 && prm->pruner != PDX_PRUNER_BSA) ? prm->ads_d : store->d;
  bound_factors(prm->pruner, store->d, prm->initial_step, nsteps,
                prm->ads_d >= 1 ? prm->ads_d : store->d, prm->ads_epsilon0, A.factors);
  A.resid = store->d_resid;
  A.bsa_coef = prm->bsa_coef;
  A.eps0 = prm->ads_epsilon0;
  A.out_dist = out->d_dist;
  A.out_ids = out->d_ids;
  A.out_count = out->d_count;
  A.out_touched = out->d_touched;
  A.out_total = out->d_total;
  A.trace = out->d_trace;
  A.trace_cap = out->d_trace ? out->trace_cap : 0;
  A.trace_len = out->d_trace_len;
  A.debug = out->d_debug;
  A.sparse_max = kItemsPerWarp / tpw;
  A.only = only;
  A.dense_spec = dense_spec ? 1 : 0;
  PDX_REQUIRE(A.out_dist && A.out_ids, "output buffers required");

  // split mode: CTA b scans range b / nq of query b % nq into row b of a
  // part-major [nsplit][nq][k] scratch, merged below by K7 (in two levels
  // when nsplit * k exceeds one merge CTA)
  int nsplit = prm->splits > 1 ? prm->splits : 1;
  const int g2 = 8192 / prm->k > 1 ? 8192 / prm->k : 1;  // lists one merge CTA sorts
  int g1 = 1;
  if (nsplit > g2) {
    g1 = (nsplit + g2 - 1) / g2;
    nsplit = g1 * g2;
    PDX_REQUIRE(g1 <= g2, "too many splits (%d) for k = %d", prm->splits, prm->k);
  }
  PDX_REQUIRE(nsplit == 1 || !out->d_trace, "split mode keeps no survivor traces");
  PDX_REQUIRE(nq * nsplit <= 0x7fffffffll, "too many query ranges");
  A.nq = (int32_t)nq;
  A.nsplit = nsplit;
  float* tdist = nullptr;
  int64_t* tids = nullptr;
  if (nsplit > 1) {
    PDX_CUDA_CHECK(cudaMallocAsync(&tdist, sizeof(float) * nq * nsplit * prm->k, st));
    PDX_CUDA_CHECK(cudaMallocAsync(&tids, sizeof(int64_t) * nq * nsplit * prm->k, st));
    A.out_dist = tdist;
    A.out_ids = tids;
    A.out_count = nullptr;
    A.debug = nullptr;
    if (A.out_touched) PDX_CUDA_CHECK(cudaMemsetAsync(A.out_touched, 0, 8 * nq, st));
    if (A.out_total) PDX_CUDA_CHECK(cudaMemsetAsync(A.out_total, 0, 8 * nq, st));
  }

  // keep the stream-ordered pool mapped between calls (split-mode scratch)
  static bool pool_kept = false;
  if (!pool_kept) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool_kept = true;
  }

  cudaError_t e = cudaSuccess;
  const bool ord = d_orders != nullptr;
  const int mt = prm->pruner == PDX_PRUNER_BSA ? kMetricL2Bsa : prm->metric;
  const int grid = (int)(nq * nsplit);
  bool linear = false;  // an unpruned split scan streams (pdx_linear.cu)
  if (nsplit > 1 && prm->pruner == PDX_PRUNER_NONE && !ord && !d_seg_bucket && !only &&
      !out->d_debug && !getenv("PDX_NO_LINEAR"))
    PDX_TRY(linear_split_scan(store, prm->metric, prm->k, d_queries, nq, nsplit, tdist, tids,
                              A.out_touched, A.out_total, st, &linear));
  if (linear) {
  } else if (store->group == 8)
    e = ord ? launch_metric<8, true>(mt, A, L, grid, W, tpw, st)
            : launch_metric<8, false>(mt, A, L, grid, W, tpw, st);
  else
    e = ord ? launch_metric<1, true>(mt, A, L, grid, W, tpw, st)
            : launch_metric<1, false>(mt, A, L, grid, W, tpw, st);
  PDX_CUDA_CHECK(e);
  if (nsplit > 1) {
    int rc = PDX_OK;
    if (g1 == 1) {
      rc = pdx_merge_topk(tdist, tids, nsplit, nq, prm->k, out->d_dist, out->d_ids, stream);
    } else {
      // level 1: rows (a, q) over parts b, where split = b * g1 + a
      float* mdist = nullptr;
      int64_t* mids = nullptr;
      PDX_CUDA_CHECK(cudaMallocAsync(&mdist, sizeof(float) * nq * g1 * prm->k, st));
      PDX_CUDA_CHECK(cudaMallocAsync(&mids, sizeof(int64_t) * nq * g1 * prm->k, st));
      rc = pdx_merge_topk(tdist, tids, g2, nq * g1, prm->k, mdist, mids, stream);
      if (rc == PDX_OK)
        rc = pdx_merge_topk(mdist, mids, g1, nq, prm->k, out->d_dist, out->d_ids, stream);
      cudaFreeAsync(mdist, st);
      cudaFreeAsync(mids, st);
    }
    cudaFreeAsync(tdist, st);
    cudaFreeAsync(tids, st);
    if (rc != PDX_OK) return rc;
    if (out->d_count) {
      count_valid_kernel<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(out->d_ids, nq, prm->k,
                                                                        out->d_count);
      PDX_LAUNCH_CHECK();
    }
  }
  return PDX_OK;
}

int pdx::search_classic(const pdx_store* store, const pdx_search_params* prm,
                        const float* d_queries, int64_t nq, const int32_t* d_seg_bucket,
                        int32_t nseg, const pdx_search_out* out, void* d_work, int64_t work_bytes,
                        void* stream, const int32_t* only, bool dense_spec) {
  return search_impl(store, prm, d_queries, nq, d_seg_bucket, nseg, nullptr, 0, 0, out, d_work,
                     work_bytes, stream, only, false, dense_spec);
}

extern "C" int pdx_search(const pdx_store* store, const pdx_search_params* prm,
                          const float* d_queries, int64_t nq, const int32_t* d_seg_bucket,
                          int32_t nseg, const uint16_t* d_orders, int64_t order_qstride,
                          int64_t order_sstride, const pdx_search_out* out, void* d_work,
                          int64_t work_bytes, void* stream) {
  return search_impl(store, prm, d_queries, nq, d_seg_bucket, nseg, d_orders, order_qstride,
                     order_sstride, out, d_work, work_bytes, stream, nullptr, true);
}
