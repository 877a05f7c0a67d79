/*
 * pdx_b200.h — C-ABI of libpdx_b200.so, the B200 (sm_100a) pruned PDX scan.
 *
 * The reference (`dimscan`, /root/reference/pkg/src/dimscan) is pure
 * Python/numpy and has no FFI or plugin ABI of its own: its boundary is the
 * Python API.  Each entry point below replaces one
 * reference function on the hot path; the reference file:line is cited on
 * each.  The package's Python layer (paper_2503_04422_b200/) binds these
 * with ctypes exactly as INTEGRATION.md shows.
 *
 * Conventions
 *  - Every pointer argument named d_* is DEVICE memory; plain scalars are
 *    host values.  `stream` is a cudaStream_t passed as void* (NULL = the
 *    legacy default stream).  Calls are stream-ordered and asynchronous
 *    unless stated otherwise; the handle-free design means any number of
 *    threads may call concurrently on different streams.
 *  - Return value: PDX_OK (0) or an error code; pdx_last_error() returns
 *    the calling thread's last message.  PDX_EINVAL maps to Python
 *    ValueError (the reference raises ValueError for the same cases,
 *    search.py:70-85, index.py:115-116, kernels.py:35-37).
 *  - Distances are float32 computed with the reference's per-op rounding
 *    (kernels.py:55-61: t = q - x; acc += t*t, no FMA), summed in visit
 *    order, so they are bit-identical to the reference's.
 */
#ifndef PDX_B200_H
#define PDX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDX_ABI_VERSION 3

#define PDX_OK 0
#define PDX_EINVAL 1    /* bad argument (Python: ValueError) */
#define PDX_ECUDA 2     /* CUDA runtime / launch failure */
#define PDX_ENOSUPPORT 3 /* size outside what this build supports */
#define PDX_EFORMAT 4   /* file does not follow the byte layout (Python: FormatError) */
#define PDX_EIO 5       /* open / read / write failure (Python: OSError) */

/* Metric (kernels.py:22-25) */
#define PDX_METRIC_L2 0
#define PDX_METRIC_L1 1
#define PDX_METRIC_IP 2

/* SearchParams.pruner (search.py:65, :78-79).  BSA is not in the reference
 * (SPEC.md:14); it is this build's restatement (DESIGN.md
 * §7), squared L2 on PCA-projected data: after step s (dims [0, e_s) seen)
 *   est = ((partial + rx_s) + rq_s) - (coef_s * sqrt(rx_s)) * sqrt(rq_s)
 * in float32 with per-op rounding, and a vector survives iff est < T.
 * rx_s / rq_s are the residual energies sum_{j=e_s}^{d-1} v_j^2 of vector and
 * query (sequential float32 sums in increasing j); coef_s = 2 * m * c_s with
 * c_s a learned quantile of residual cosines (pdx_bsa_residuals). */
#define PDX_PRUNER_NONE 0
#define PDX_PRUNER_ADS 1
#define PDX_PRUNER_BOND 2
#define PDX_PRUNER_BSA 3

/* OrderCriteria (pruning.py:91-95) */
#define PDX_ORDER_SEQUENTIAL 0
#define PDX_ORDER_DECREASING 1
#define PDX_ORDER_DMEANS 2
#define PDX_ORDER_ZONES 3

/* Number of vectors per HBM tile.  A reference Block (layout.py:53-83) of m
 * vectors occupies ceil(m/64) consecutive tiles. */
#define PDX_TILE 64

/*
 * A device-resident PDX store: the reference's list[Block]
 * (layout.py:93-110) or IvfIndex bucket chains (index.py:75-108) in HBM.
 *
 * tiles  : float32 [ntiles][d_pad/group][64][group].  group = 1 is the
 *          plain PDX block (one 256-byte row per dimension); group = 8 keeps
 *          8 consecutive dimensions of a vector in one 32-byte sector so a
 *          pruned survivor costs one sector per 8 dims.  Padding slots and
 *          padding dims (d..d_pad) are zero.
 * tile_ids : int64 [ntiles][64]  external id per slot, -1 for padding.
 * Logical block b (a reference Block) = tiles block_tile[b] ..
 *          block_tile[b] + ceil(block_m[b]/64) - 1, holding block_m[b] vectors.
 * bucket_block : int64 [nbuckets+1]; bucket c owns logical blocks
 *          [bucket_block[c], bucket_block[c+1]).  A flat store has
 *          nbuckets = 1 covering every block (exact_search, index.py:182-191).
 */
typedef struct pdx_store {
  int32_t d;
  int32_t d_pad;
  int32_t group;
  int32_t nbuckets;
  int64_t ntiles;
  int64_t nblocks;
  const float* d_tiles;
  const int64_t* d_tile_ids;
  const int64_t* d_block_tile;  /* [nblocks+1] first tile of each block (prefix) */
  const int32_t* d_block_m;
  const int64_t* d_bucket_block;
  int32_t max_bucket_blocks; /* max over buckets of (#blocks) */
  int32_t max_bucket_tiles;  /* max over buckets of (#tiles) */
  const int32_t* d_tile_block;  /* [ntiles] logical block of each tile */
  /* BSA only: float32 [ntiles][resid_steps][64] residual energy rx_s of each
   * slot after step s of step_schedule(d, resid_initial_step); NULL otherwise */
  const float* d_resid;
  int32_t resid_steps;
  int32_t resid_initial_step;
} pdx_store;

/* SearchParams (search.py:61-85) + AdsPruner (pruning.py:56-65). */
typedef struct pdx_search_params {
  int32_t k;
  int32_t metric;
  int32_t pruner;
  int32_t initial_step;
  double selection_fraction;
  int32_t ads_d;    /* AdsPruner.d (the reference defaults it to the data d) */
  int32_t warps;    /* compute warps per query CTA (0 = auto) */
  double ads_epsilon0;
  int32_t tiles_per_warp; /* 64-vector tiles a compute warp claims at once (0 = auto) */
  int32_t ring_slots;     /* tiles in flight per query CTA (0 = auto) */
  const float* bsa_coef;  /* BSA: DEVICE float32 [nsteps] coef_s (see PDX_PRUNER_BSA) */
  /* Split mode (> 1): each query's visit list is cut, at block starts, into
   * `splits` ranges scanned by separate CTAs, each with its own threshold
   * chain from +inf; the per-range top-k lists are merged (K7).  Results are
   * the exact top-k for pruner none / BOND (the union of exact local top-ks);
   * values_touched is the split run's own (a throughput mode: the reference
   * has one chain); ADS / BSA become recall-level.  No survivor traces.
   * Lets one query use the whole GPU (batch-1 exact search, C4). */
  int32_t splits;
  /* IVF query batches (per-query bucket selection, 64-vector blocks, G = 8
   * tiles, natural dimension order, pruner ads / bond / bsa, no split):
   *   0 = auto: the bucket-major batched pipeline when the batch has at
   *       least 32 queries, else the per-query scan;
   *   1 = always the per-query scan;  2 = batched whenever eligible.
   * Both give the reference's results, decisions and stats bit for bit
   * (DESIGN.md §3.2); the batched one evaluates each tile once for every
   * query that probes its bucket. */
  int32_t batched;
} pdx_search_params;

/* Outputs of pdx_search.  Per query q (row q of each array):
 *  d_dist/d_ids [nq][k]: TopK.items() (search.py:53-55) ascending by
 *      (distance, id); IP distances are negated (search.py:120-122);
 *      unused rows are +inf / -1 (estimators.py:24-31).
 *  d_count [nq]      : len(TopK)                       (optional)
 *  d_touched/d_total : SearchStats.values_touched / values_total
 *                      (search.py:132, :169, :198)      (optional)
 *  d_trace [nq][trace_cap], d_trace_len [nq]: SearchStats.survivors as
 *      records [len, v1..vlen] per visited block (search.py:133, :170-172);
 *      trace_len = -1 on overflow                     (optional) */
typedef struct pdx_search_out {
  float* d_dist;
  int64_t* d_ids;
  int32_t* d_count;
  int64_t* d_touched;
  int64_t* d_total;
  int32_t* d_trace;
  int64_t trace_cap;
  int64_t* d_trace_len;
  /* optional [nq][16] kernel diagnostics: cycles, tiles, fast-path commits,
   * serial commits, replays, commit-warp idle polls, compute-warp ring
   * waits, sparse items, then compute-warp cycles summed over warps: ring
   * wait, dense phase, sparse phase, the rest */
  int64_t* d_debug;
} pdx_search_out;

int pdx_abi_version(void);
/* Copies the calling thread's last error message; returns its length. */
int pdx_last_error(char* buf, size_t cap);
/* Number of SMs and max opt-in shared memory per block of the current device. */
int pdx_device_info(int32_t* sm_count, int32_t* smem_optin, int32_t* cc_major, int32_t* cc_minor);

/*
 * K1 — PDX transposition / IVF bucket packing.
 * Replaces to_blocks (layout.py:93-110, the transpose at :107-108) and the
 * per-bucket packing of ivf_build (index.py:98-106).
 * d_x: float32 [n][d] row-major; d_slot_src: int64 [ntiles*64] source row of
 * each slot (-1 = padding); d_ids_in: int64 [n] external ids (NULL = row
 * index).  Writes d_tiles (layout above) and d_tile_ids.
 */
int pdx_pack_tiles(const float* d_x, int64_t n, int32_t d, const int64_t* d_slot_src,
                   int64_t ntiles, int32_t group, const int64_t* d_ids_in, float* d_tiles,
                   int64_t* d_tile_ids, void* stream);

/*
 * BSA residual energies of a packed store (PDX_PRUNER_BSA; not in the
 * reference): d_resid[t][s][i] = sum_{j=e_s}^{d-1} x_j^2 for slot i of tile t,
 * e_s the end of step s of step_schedule(d, initial_step) (search.py:106-117),
 * a sequential float32 sum in increasing j.  d_resid: float32
 * [ntiles][nsteps][64] (NULL: only report nsteps); nsteps in *nsteps_out.
 */
int pdx_bsa_residuals(const pdx_store* store, int32_t initial_step, float* d_resid,
                      int32_t* nsteps_out, void* stream);

/*
 * K3 — query / data projection y = x @ M^T (float32).
 * Replaces apply_transform (pruning.py:48-53) as used per query batch at
 * estimators.py:116-117 and at fit time (estimators.py:102-105).  Not
 * bit-identical to numpy's sgemm (neither is any other BLAS); parity tests
 * feed both sides identical rotated floats.
 */
int pdx_project(const float* d_x, int64_t n, int32_t d, const float* d_matrix, float* d_y,
                void* stream);

/*
 * K2 — bucket selection.
 * Replaces ivf_select_buckets (index.py:111-127): float32 centroid
 * distances with the vertical kernel's per-op rounding in natural dim order,
 * then the nprobe smallest (key, bucket) pairs (key = -dist for IP), i.e.
 * numpy's stable argsort.  d_centroids: float32 [nlist][d] row-major.
 * d_scratch: float32 [nq][nlist].  d_sel: int32 [nq][nprobe].
 */
int pdx_select_buckets(const float* d_queries, int64_t nq, int32_t d, const float* d_centroids,
                       int32_t nlist, int32_t metric, int32_t nprobe, float* d_scratch,
                       int32_t* d_sel, void* stream);

/*
 * K4 — query-aware dimension orders.
 * Replaces bond_dimension_order (pruning.py:107-140) with default_zone_width
 * (:98-99): stable float64 sorts, numpy's pairwise float64 sum for zone
 * scores.  d_queries: [nq][d], float32 (queries_f64 = 0, what the scan
 * uses) or float64 (queries_f64 = 1; the reference takes float64 queries,
 * pruning.py:117).  d_means: float64 [nmeans][d].  For output row
 * r = q*nsets + s the means row is d_mean_index[r] (NULL: row 0).
 * d_out: uint16 [nq*nsets][d].  zone_width <= 0 selects the default.
 */
int pdx_dimension_orders(const void* d_queries, int32_t queries_f64, int64_t nq, int32_t d,
                         const double* d_means, const int32_t* d_mean_index, int32_t nsets,
                         int32_t criteria, int32_t zone_width, uint16_t* d_out, void* stream);

/*
 * K5+K6 — the pruned PDX scan with top-k (PDXearch).
 * Replaces search / _linear_block / _search_block (search.py:125-205) with
 * vertical_accumulate(_selected) (kernels.py:41-91), ads_bound
 * (pruning.py:83-88), the BOND test (search.py:165) and TopK (search.py:27-58).
 * The visit order for query q is: for s in 0..nseg-1, every logical block
 * of bucket d_seg_bucket[q*nseg+s] (NULL: bucket s) in stored order — the
 * block list ivf_search builds (index.py:140-149) or exact_search's
 * partition list.  d_orders: NULL (natural order) or uint16 permutations,
 * the one for (q, s) at d_orders + (q*order_qstride + s*order_sstride)*d.
 * Results, the threshold chain, every prune decision and the stats are the
 * reference's (block-synchronous thresholds, search.py:159).
 * d_work/work_bytes: scratch of at least pdx_search_workspace() bytes.
 */
int64_t pdx_search_workspace(const pdx_store* store, int64_t nq, int32_t nseg);
int pdx_search(const pdx_store* store, const pdx_search_params* params, const float* d_queries,
               int64_t nq, const int32_t* d_seg_bucket, int32_t nseg, const uint16_t* d_orders,
               int64_t order_qstride, int64_t order_sstride, const pdx_search_out* out,
               void* d_work, int64_t work_bytes, void* stream);

/*
 * GPU IVF build (next #1): the reference's Lloyd k-means (index.py:27-64)
 * and bucket layout (index.py:98-100) — SIMT float32 kernels and a CUB
 * radix sort, no cuBLAS.
 *   pdx_row_norms: out[i] = sum_j x[i][j]^2 (float32; einsum, index.py:70).
 *   pdx_kmeans_assign: for row i (d_rows[i] when d_rows is not NULL) the
 *     centroid c minimising max(xnorm + cnorm[c] - 2 x.c, 0) (_pairwise_l2,
 *     index.py:67-72), the lowest c among equal minima (np.argmin);
 *     d_min_dist (optional) gets that distance.  d_xnorm is indexed by i.
 *   pdx_bucket_layout: d_order = rows sorted by (bucket, row) (members of
 *     each bucket ascending, np.flatnonzero), d_counts [nlist], d_offsets
 *     [nlist+1] (exclusive sums); call with d_work = NULL for *work_bytes.
 *   pdx_kmeans_update: new[c] = f32(means[c]) if counts[c] > 0 else old[c]
 *     (index.py:45-48, means from pdx_segment_means in float64).
 *   pdx_kmeans_farthest: the member of `bucket` farthest from d_centroid by
 *     the same distance (index.py:52-54); *d_out_key = (gap bits << 32) |
 *     (0xffffffff - row), the largest gap and then the lowest row.
 *   pdx_kmeans_shift: *d_out = max_c ||new_c - old_c|| / (||old_c|| + 1e-30)
 *     in float32 (index.py:57-61).
 *   pdx_gather_rows: d_out[i] = d_x[d_rows[i]] (the sample init, :38-39).
 *   pdx_pack_rows: a chunk of m rows written straight into their slots of
 *     a store (d_dest[i] = tile * 64 + slot, -1 = skip) with their ids: the
 *     chunked build packs without a full copy of the collection.
 */
int pdx_row_norms(const float* d_x, int64_t n, int32_t d, float* d_out, void* stream);
int pdx_kmeans_assign(const float* d_x, const int64_t* d_rows, int64_t n, int32_t d,
                      const float* d_xnorm, const float* d_centroids, const float* d_cnorm,
                      int32_t nlist, int32_t* d_assign, float* d_min_dist, void* stream);
int pdx_bucket_layout(const int32_t* d_assign, int64_t n, int32_t nlist, int64_t* d_order,
                      int64_t* d_counts, int64_t* d_offsets, void* d_work, int64_t* work_bytes,
                      void* stream);
int pdx_kmeans_update(const double* d_means, const int64_t* d_counts, const float* d_old,
                      int32_t nlist, int32_t d, float* d_new, void* stream);
int pdx_kmeans_shift(const float* d_new, const float* d_old, int32_t nlist, int32_t d,
                     float* d_out, void* stream);
int pdx_kmeans_farthest(const float* d_x, int64_t n, int32_t d, const int32_t* d_assign,
                        int32_t bucket, const float* d_centroid, float cnorm, int64_t* d_out_key,
                        void* stream);
int pdx_gather_rows(const float* d_x, int32_t d, const int64_t* d_rows, int64_t m, float* d_out,
                    void* stream);
int pdx_pack_rows(const float* d_x, int64_t m, int32_t d, const int64_t* d_dest,
                  const int64_t* d_ids, const pdx_store* store, void* stream);

/*
 * The vertical kernels as standalone ops: vertical_accumulate
 * (kernels.py:41-62; d_positions NULL: every one of the mp slots) and
 * vertical_accumulate_selected (kernels.py:65-91; the npos listed slots,
 * distinct, others untouched).  d_block f32 [d][mp] (a Block's data),
 * d_query f32 [d], dims [a, b) of the natural order or of d_order (int64
 * permutation of 0..d-1), d_acc f32 [mp] updated in place, each op rounded
 * separately (no FMA), in visit order.  The search kernels fuse the same
 * arithmetic (pdx_search).
 */
int pdx_vertical_accumulate(const float* d_block, int32_t d, int32_t mp, const float* d_query,
                            int32_t a, int32_t b, const int64_t* d_order,
                            const int64_t* d_positions, int32_t npos, int32_t metric,
                            float* d_acc, void* stream);

/*
 * Phase timing of the batched IVF pipeline (pdx_search with per-query bucket
 * selections): with enable = 1 every later batched call records CUDA events
 * on its stream at the phase boundaries (not while the stream is being
 * captured), waits for them at its end and accumulates the device time per
 * phase: [0] plan, [1] phase 1 (bdense + bchain1), [2] T' (incl. the join of
 * the work-list stream), [3] bscan MODE 0, [4] chain, [5] bscan MODE 1,
 * [6] final, [7] fallback.  Copies up to cap accumulated values (ms) to
 * out_ms and the call count to out_calls (either may be NULL); enable >= 0
 * then resets the accumulators and sets the mode, enable < 0 only reads.
 * A call captured into a CUDA graph while enabled records its phase events as
 * external event nodes; after a replay (and a synchronize) enable = 2 adds
 * that replay's phase times to the accumulators (the output arguments are
 * filled first, as always).
 */
int pdx_batch_profile(int32_t enable, double* out_ms, int32_t cap, int64_t* out_calls);

/*
 * K7 — merge of per-shard top-k lists (multi-GPU; no reference counterpart:
 * the reference is single-process).  d_dist/d_ids: [nparts][nq][k] sorted
 * lists (+inf/-1 padded) → the k smallest (dist, id) pairs per query, the
 * TopK tie rule (search.py:45-51).
 */
int pdx_merge_topk(const float* d_dist, const int64_t* d_ids, int32_t nparts, int64_t nq, int32_t k,
                   float* d_out_dist, int64_t* d_out_ids, void* stream);

/*
 * Per-segment float64 means: for segment s, rows d_rows[seg_off[s] ..
 * seg_off[s+1]) of d_x summed in that order in float64, divided by the
 * count.  Replaces compute_means (layout.py:126-138: values.sum(axis=0)/n,
 * numpy's axis-0 reduction adds rows sequentially) for the global / bucket
 * means (index.py:103-104, :178) and the k-means centroid update
 * (index.py:46-48).  Empty segments are left untouched.
 * d_rows NULL = identity (segments of consecutive rows).
 */
int pdx_segment_means(const float* d_x, int32_t d, const int64_t* d_rows, const int64_t* d_seg_off,
                      int32_t nseg, double* d_means, void* stream);

/*
 * Float64 brute-force ground truth (next #3): compute_ground_truth
 * (bench.py:53-67) — horizontal float64 distances (kernels.py:108-119) and
 * the k smallest (key, row) with the lower row on ties.  d_x [n][d] f32,
 * d_queries [nq][d] f32 → d_ids [nq][k] (row indices), d_dist [nq][k] f64.
 */
int pdx_ground_truth(const float* d_x, int64_t n, int32_t d, const float* d_queries, int64_t nq,
                     int32_t k, int32_t metric, int64_t* d_ids, double* d_dist, void* stream);

/*
 * .pdx store interchange, HBM <-> file (storage.py:115-194 of the reference;
 * cli.py:35-76 writes it).  Byte layout, all little-endian:
 *   header "<8sIIQIIII": magic "PDXv1\0\0\0", version 1, flags (1 = rotation,
 *     2 = IVF section), n, d, block_size, block_count, reserved
 *   global means f64 [d]
 *   [flags & 1] transform seed u64, rotation f32 [d][d]
 *   block_count x { m u32, m_padded u32, ids i64 [m], data f32 [d][m_padded] }
 *   [flags & 2] nlist u32, training seed u64, centroids f32 [nlist][d],
 *     bucket offsets u32 [nlist+1] (into the block list), bucket means f64 [nlist][d]
 * Block b becomes ceil(m/64) consecutive tiles of the store (pdx_store); the
 * dims beyond d and slots beyond m are zero.  Saving a loaded store writes
 * the same bytes back.
 */
typedef struct pdx_file_info {
  int64_t n;              /* vectors (header) */
  int32_t d;
  int32_t block_size;
  int64_t nblocks;
  int32_t flags;
  int32_t nlist;          /* 0 without an IVF section */
  uint64_t transform_seed;
  uint64_t training_seed;
  int64_t ntiles;         /* sum over blocks of ceil(m/64) */
  int64_t max_block_bytes; /* largest block record's data, d * m_padded * 4 */
} pdx_file_info;

/* Walks the file's sections (no data read) and validates its framing:
 * bad magic / version, truncation, header n vs the blocks' total. */
int pdx_file_probe(const char* path, pdx_file_info* info);

/* Streams the blocks of `path` into the tile layout of a store with `group`
 * (1 or 8) on `stream`: d_tiles f32 [ntiles][d_pad/group][64][group] (d_pad =
 * d rounded up to group), d_tile_ids i64 [ntiles][64] (-1 padding).  Host
 * outputs: h_block_m / h_block_mpad i32 [nblocks]; h_global_means f64 [d];
 * h_transform f32 [d][d] (flags & 1); h_centroids f32 [nlist][d],
 * h_bucket_offsets i64 [nlist+1], h_bucket_means f64 [nlist][d] (flags & 2).
 * Returns after the device copies complete. */
int pdx_file_load(const char* path, const pdx_file_info* info, int32_t group, float* d_tiles,
                  int64_t* d_tile_ids, int32_t* h_block_m, int32_t* h_block_mpad,
                  double* h_global_means, float* h_transform, float* h_centroids,
                  int64_t* h_bucket_offsets, double* h_bucket_means, void* stream);

/* Writes `store` (its logical blocks in order) as a .pdx file.  h_block_mpad
 * i32 [nblocks] (NULL: m_padded = m); h_transform NULL = no rotation
 * section; nlist 0 = no IVF section (else h_bucket_offsets i64 [nlist+1] are
 * logical-block offsets). */
int pdx_file_save(const char* path, const pdx_store* store, int32_t block_size,
                  const int32_t* h_block_mpad, const double* h_global_means,
                  const float* h_transform, uint64_t transform_seed, int32_t nlist,
                  uint64_t training_seed, const float* h_centroids,
                  const int64_t* h_bucket_offsets, const double* h_bucket_means, void* stream);

/*
 * K8 — batched exact search with tensor-core candidate generation (L2, IP;
 * pruner none), for batches where Q X^T is a real dense GEMM (C4).
 * pdx_k8_candidates runs the whole candidate pass on the tensor cores;
 * pdx_k8_filter is its dense-chunk step (S from the tcgen05 kernel's dense
 * mode, or from any GEMM); pdx_k8_rescore then recomputes the
 * candidates exactly as the scan does.  Results equal pdx_search's (the
 * candidate set provably contains the exact top-k: |S - ref| <= margin *
 * |q| |x|, pdx_k8_margin); a query whose candidates overflow C is reported
 * through d_ccount > C and must be answered by pdx_search.
 *   pdx_k8_norms : squared row norms of float32 [n][d]
 *   pdx_k8_filter: S chunk [nq][R] (row stride ldS) for rows row0..row0+R-1
 *       with their squared norms; d_prev / d_next float32 [nq][k] the k
 *       smallest upper bounds so far (init +inf; swap per chunk); appends
 *       row ids to d_cand [nq][C], counting in d_ccount [nq] (init 0).
 *   pdx_k8_rescore: exact keys of the candidates of a flat store whose
 *       logical blocks all hold part_size vectors (the last may hold fewer),
 *       row r = vector r of block r / part_size; outputs as pdx_search.
 */
int pdx_k8_norms(const float* d_x, int64_t n, int32_t d, float* d_n2, void* stream);
/* pdx_k8_norms over the first d floats of rows ld floats apart. */
int pdx_k8_norms_ld(const float* d_x, int64_t n, int32_t d, int64_t ld, float* d_n2, void* stream);
/*
 * pdx_k8_candidates: the candidate pass on the 5th-generation tensor cores
 * (csrc/pdx_k8tc.cu: tcgen05.mma kind::tf32 with TMEM accumulators, TMA
 * operand staging, the interval filter fused into the TMEM epilogue — the
 * score matrix is never written to HBM except for the first chunk of
 * min(n, 8192) rows, whose k smallest upper bounds seed tau).
 * d_x f32 [n][ld], d_q f32 [nq][ld] (ld a multiple of 4 >= d, 16-B aligned
 * rows, the floats beyond d zero), d_xn2 = pdx_k8_norms_ld of d_x.  Writes
 * d_cand [nq][C] row indices and d_ccount [nq] (> C: overflow, answer that
 * query with pdx_search) — a superset of the exact top-k for
 * pdx_k8_rescore.  d_work NULL: *work_bytes gets the scratch size.
 */
/* pdx_k8_rescore_rows: pdx_k8_rescore from the row-major copy d_x [n][ld]
 * (d_rowids [n]: the id of each row) and ld-strided queries; cmax bounds
 * every query's candidate count (the caller reads d_ccount; larger counts
 * are truncated, so pass the maximum). */
int pdx_k8_rescore_rows(const float* d_x, int64_t ld, int32_t d, const int64_t* d_rowids,
                        const float* d_q, int64_t nq, int32_t metric, int32_t k,
                        const int64_t* d_cand, const int32_t* d_ccount, int32_t C, int32_t cmax,
                        float* d_dist, int64_t* d_ids, void* stream);
int pdx_k8_candidates(const float* d_x, int64_t n, int32_t d, int64_t ld, const float* d_xn2,
                      const float* d_q, int64_t nq, int32_t metric, int32_t k, int64_t* d_cand,
                      int32_t* d_ccount, int32_t C, void* d_work, int64_t* work_bytes,
                      void* stream);
/* The same pass with bf16 MMA operands (tcgen05 kind::f16: twice the
 * tensor-core rate and half the operand bytes of tf32) and the interval
 * widened for their round-to-nearest error, (2 * 2^-8 + 2^-16) |q||x|:
 * d_x16 / d_q16 bf16 [rows][ld16] (pdx_k8_to_bf16 of the float32 rows; ld16
 * a multiple of 8), d_q float32 [nq][ld] (the norms and the L2 expansion
 * are those of the float32 vectors).  More candidates per query than the
 * tf32 pass; the same exactness argument. */
int pdx_k8_candidates_bf16(const void* d_x16, int64_t n, int32_t d, int64_t ld16,
                           const float* d_xn2, const void* d_q16, const float* d_q, int64_t ld,
                           int64_t nq, int32_t metric, int32_t k, int64_t* d_cand,
                           int32_t* d_ccount, int32_t C, void* d_work, int64_t* work_bytes,
                           void* stream);
/* float32 rows (ld apart) -> bf16 rows (ld16 apart, zero padded), round to nearest. */
int pdx_k8_to_bf16(const float* d_x, int64_t n, int32_t d, int64_t ld, int64_t ld16, void* d_y,
                   void* stream);
float pdx_k8_margin(int32_t d, int32_t metric);
int pdx_k8_filter(const float* d_S, int64_t ldS, int64_t nq, int32_t R, int64_t row0,
                  const float* d_xn2, const float* d_qn2, int32_t metric, int32_t d, int32_t k,
                  const float* d_prev, float* d_next, int64_t* d_cand, int32_t* d_ccount,
                  int32_t C, void* stream);
int pdx_k8_rescore(const pdx_store* store, int64_t part_size, const float* d_queries, int64_t nq,
                   int32_t metric, int32_t k, const int64_t* d_cand, const int32_t* d_ccount,
                   int32_t C, float* d_dist, int64_t* d_ids, void* stream);

/*
 * Owning index handle + one-call search: the drop-in boundary a C / C++ /
 * FFI caller binds.  It replaces the estimators' fit /
 * kneighbors pair (estimators.py:54-76, :99-132) and ivf_search /
 * exact_search (index.py:130-191) for a whole query batch, chaining the
 * kernels above inside the library: query projection (K3), bucket
 * selection (K2), dimension orders (K4), the pruned scan with top-k (K5/K6).
 * A handle is not thread-safe; calls are ordered on `stream`.
 */
typedef struct pdx_index pdx_index;

typedef struct pdx_index_desc {
  /* Either borrow a device store (kept alive by the caller) ... */
  const pdx_store* store;
  /* ... or upload host blocks (store == NULL), the reference's Block list:
   * block b holds block_m[b] vectors in a [d][block_mpad[b]] image. */
  int32_t d;
  int32_t group;              /* tile layout: 1 or 8 (0 = 8) */
  int64_t nblocks;
  const float* blocks;        /* images back to back, block order */
  const int32_t* block_m;
  const int32_t* block_mpad;  /* NULL: m_padded = m */
  const int64_t* ids;         /* block_m[b] ids per block, back to back */
  /* metadata (host) */
  const double* global_means; /* [d]: exact_search's order means (NULL: zeros) */
  const float* rotation;      /* [d][d] or NULL: queries are projected q @ R^T first */
  int32_t nlist;              /* 0: flat (exact_search over all blocks) */
  const float* centroids;     /* [nlist][d] */
  const int64_t* bucket_offsets; /* [nlist+1] into the blocks (ignored when borrowing) */
  const double* bucket_means; /* [nlist][d] */
} pdx_index_desc;

int pdx_index_create(const pdx_index_desc* desc, pdx_index** out);
/* Opens a .pdx file (pdx_file_load) into a new handle. */
int pdx_index_open(const char* path, int32_t group, pdx_index** out);
int pdx_index_destroy(pdx_index* index);

typedef struct pdx_query_params {
  int32_t k;
  int32_t metric;            /* PDX_METRIC_* */
  int32_t pruner;            /* PDX_PRUNER_* */
  int32_t criteria;          /* PDX_ORDER_* (BOND only) */
  int32_t zone_width;        /* <= 0: default */
  int32_t nprobe;            /* IVF only */
  double selection_fraction;
  int32_t initial_step;
  int32_t rotate;            /* 1: project queries with the index rotation */
  double epsilon0;
  const float* bsa_coef;     /* host float32 [nsteps] (pruner BSA) */
  int32_t queries_on_device; /* Q is a device pointer */
  int32_t outputs_on_device; /* out_* are device pointers */
  /* Flat index, pruner none, L2 / IP, nq >= 64: answer through K8 (TF32
   * tensor-core candidates + exact rescoring; identical results).  0 = off,
   * 1 = when applicable. */
  int32_t tensor_cores;
} pdx_query_params;

/* Searches nq queries Q [nq][d]; out_dist/out_ids [nq][k] as pdx_search
 * (ascending (distance, id), +inf / -1 padding, IP negated); out_touched /
 * out_total [nq] optional (NULL).  Host outputs are complete on return. */
int pdx_index_search(pdx_index* index, const pdx_query_params* params, const float* Q,
                     int64_t nq, float* out_dist, int64_t* out_ids, int64_t* out_touched,
                     int64_t* out_total, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PDX_B200_H */
