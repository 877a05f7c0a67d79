// Internal entry points shared by pdx_scan.cu and pdx_batch.cu (not ABI).
#pragma once
#include "pdx_common.cuh"

namespace pdx {

// The per-query scan (pdx_scan_kernel) behind pdx_search; `only` (optional,
// [nq]) restricts it to the queries with only[q] != 0, leaving the other
// output rows untouched.  dense_spec: the compute warps scan prune-free
// (T' = +inf) and the commit warp replays every decision — for chains whose
// threshold moves at almost every block (a query's first bucket), where
// pruned speculation would chase long survivor tails one L2 trip at a time.
int search_classic(const pdx_store* store, const pdx_search_params* prm, const float* d_queries,
                   int64_t nq, const int32_t* d_seg_bucket, int32_t nseg,
                   const pdx_search_out* out, void* d_work, int64_t work_bytes, void* stream,
                   const int32_t* only, bool dense_spec = false);

// The bucket-major batched pipeline (pdx_batch.cu) and when pdx_search uses it.
bool batched_eligible(const pdx_store* store, const pdx_search_params* prm, int64_t nq,
                      const int32_t* d_seg_bucket, int32_t nseg, const uint16_t* d_orders,
                      const pdx_search_out* out);
int search_batched(const pdx_store* store, const pdx_search_params* prm, const float* d_queries,
                   int64_t nq, const int32_t* d_seg_bucket, int32_t nseg,
                   const pdx_search_out* out, void* d_work, int64_t work_bytes, void* stream);

}  // namespace pdx
