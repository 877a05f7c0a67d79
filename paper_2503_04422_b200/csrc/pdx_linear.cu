// Pruner-free exact scans split over the whole GPU (pdx_search_params.splits
// with pruner "none": C4 batch 1): a streaming kernel instead of the pruned
// scan's ring of speculative tiles.  With no pruning every value is read
// once and the job is bandwidth work: each warp streams whole tiles (lane l
// owns slots l and l + 32, one 256-bit load per slot and 8-dim group, the
// next group in flight), computes the reference's distances with its
// per-op-rounded sequential arithmetic (kernels.py:41-62, the scan's
// `upd`), and keeps a warp top-k in shared memory behind a threshold
// filter; the CTA merges its warps' lists into row (split * nq + q) of the
// part-major [nsplit][nq][k] scratch that K7 merges (search.py:27-58 order:
// (distance, id), ties to the lower id).  values_touched = values_total =
// every valid slot's d values (an unpruned scan, search.py:132).
#include "pdx_common.cuh"
#include "pdx_sort.cuh"

namespace pdx {
namespace {

constexpr int kLW = 8;    // warps per CTA
constexpr int kLCB = 128;  // per-warp candidate buffer

__device__ __forceinline__ bool kv_less(float a, int64_t ia, float b, int64_t ib) {
  return a < b || (a == b && ia < ib);
}

// warp-wide bitonic sort of n (power of two) (key, id) pairs in shared memory
__device__ void warp_sort(float* key, int64_t* id, int n) {
  const int lane = threadIdx.x & 31;
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < (n >> 1); i += 32) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const float ka = key[lo], kb = key[hi];
        const int64_t va = id[lo], vb = id[hi];
        if (kv_less(kb, vb, ka, va) == asc) {
          key[lo] = kb;
          key[hi] = ka;
          id[lo] = vb;
          id[hi] = va;
        }
      }
      __syncwarp();
    }
  }
}

template <int METRIC>
__global__ void __launch_bounds__(kLW * 32) linear_kernel(
    const float* __restrict__ tiles, const int64_t* __restrict__ tile_ids, int64_t ntiles, int d,
    int d_pad, const float* __restrict__ Q, int64_t nq, int nsplit, int k, int KL,
    float* __restrict__ tdist, int64_t* __restrict__ tids, int64_t* __restrict__ touched,
    int64_t* __restrict__ total) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* qs = reinterpret_cast<float*>(smem);
  float* lkey = qs + d_pad;                              // [kLW][KL]
  int64_t* lid = reinterpret_cast<int64_t*>(lkey + kLW * KL);  // [kLW][KL]
  const int64_t b = blockIdx.x;
  const int64_t q = b % nq;
  const int s = (int)(b / nq);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int j = threadIdx.x; j < d_pad; j += blockDim.x) qs[j] = j < d ? Q[q * d + j] : 0.f;
  for (int i = threadIdx.x; i < kLW * KL; i += blockDim.x) {
    lkey[i] = INFINITY;
    lid[i] = INT64_MAX;
  }
  __syncthreads();
  float* wk = lkey + w * KL;
  int64_t* wi = lid + w * KL;
  // list = wk[0, k) sorted; candidate buffer = wk[k, k + nb)
  int nb = 0;
  float thr = INFINITY;
  int64_t thr_id = INT64_MAX;
  auto merge = [&]() {
    warp_sort(wk, wi, KL);  // the list and the buffer; sentinels sort last
    thr = wk[k - 1];
    thr_id = wi[k - 1];
    for (int i = k + lane; i < KL; i += 32) {
      wk[i] = INFINITY;
      wi[i] = INT64_MAX;
    }
    __syncwarp();
    nb = 0;
  };
  const int64_t t0 = ntiles * s / nsplit, t1 = ntiles * (s + 1) / nsplit;
  const int ng = d_pad >> 3;
  int64_t nvalid = 0;
  for (int64_t t = t0 + w; t < t1; t += kLW) {
    const float* tb = tiles + t * (int64_t)d_pad * kTile;
    const int64_t id0 = __ldg(tile_ids + t * kTile + lane);
    const int64_t id1 = __ldg(tile_ids + t * kTile + 32 + lane);
    float acc0 = 0.f, acc1 = 0.f;
    float x0[8], x1[8], n0[8], n1[8];
    ldg8(tb + lane * 8, n0);
    ldg8(tb + (32 + lane) * 8, n1);
    for (int g = 0; g < ng; ++g) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        x0[e] = n0[e];
        x1[e] = n1[e];
      }
      if (g + 1 < ng) {
        ldg8(tb + ((size_t)(g + 1) * kTile + lane) * 8, n0);
        ldg8(tb + ((size_t)(g + 1) * kTile + 32 + lane) * 8, n1);
      }
      const float4 qa = *reinterpret_cast<const float4*>(qs + g * 8);
      const float4 qb = *reinterpret_cast<const float4*>(qs + g * 8 + 4);
      const float qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
      if (g * 8 + 8 <= d) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          acc0 = upd<METRIC>(acc0, qv[e], x0[e]);
          acc1 = upd<METRIC>(acc1, qv[e], x1[e]);
        }
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (g * 8 + e < d) {
            acc0 = upd<METRIC>(acc0, qv[e], x0[e]);
            acc1 = upd<METRIC>(acc1, qv[e], x1[e]);
          }
      }
    }
    const float k0 = METRIC == PDX_METRIC_IP ? -acc0 : acc0;
    const float k1 = METRIC == PDX_METRIC_IP ? -acc1 : acc1;
    const bool c0 = id0 >= 0 && kv_less(k0, id0, thr, thr_id);
    const bool c1 = id1 >= 0 && kv_less(k1, id1, thr, thr_id);
    nvalid += __popc(__ballot_sync(0xffffffffu, id0 >= 0)) +
              __popc(__ballot_sync(0xffffffffu, id1 >= 0));
    const unsigned m0 = __ballot_sync(0xffffffffu, c0), m1 = __ballot_sync(0xffffffffu, c1);
    const int nc = __popc(m0) + __popc(m1);
    if (nc == 0) continue;
    if (nb + nc > KL - k) merge();
    const unsigned lt = (1u << lane) - 1u;
    const int p0 = k + nb + __popc(m0 & lt);
    if (c0) {
      wk[p0] = k0;
      wi[p0] = id0;
    }
    const int p1 = k + nb + __popc(m0) + __popc(m1 & lt);
    if (c1) {
      wk[p1] = k1;
      wi[p1] = id1;
    }
    nb += nc;
    __syncwarp();
  }
  if (nb) merge();
  if (lane == 0 && nvalid) {
    if (touched) atomicAdd(reinterpret_cast<unsigned long long*>(touched + q),
                           (unsigned long long)(nvalid * d));
    if (total) atomicAdd(reinterpret_cast<unsigned long long*>(total + q),
                         (unsigned long long)(nvalid * d));
  }
  __syncthreads();
  // the CTA's k smallest of its warps' lists (sentinels beyond each list)
  bitonic_sort(lkey, lid, kLW * KL);
  const int64_t row = (int64_t)s * nq + q;
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    tdist[row * k + i] = lkey[i];
    tids[row * k + i] = lid[i] == INT64_MAX ? -1 : lid[i];
  }
}

}  // namespace

// [nsplit][nq][k] part-major top-k lists of an unpruned split scan (see the
// file comment); false when this kernel does not apply (the caller runs the
// pruned scan instead).
int linear_split_scan(const pdx_store* store, int metric, int k, const float* d_queries,
                      int64_t nq, int nsplit, float* tdist, int64_t* tids, int64_t* touched,
                      int64_t* total, cudaStream_t st, bool* applied) {
  *applied = false;
  if (store->group != 8 || k > 512 || metric < 0 || metric > 2) return PDX_OK;
  const int KL = pow2_ceil(k + kLCB);
  const size_t smem = (size_t)store->d_pad * 4 + (size_t)kLW * KL * 12;
  int dev = 0, optin = 0;
  PDX_CUDA_CHECK(cudaGetDevice(&dev));
  PDX_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (smem > (size_t)optin) return PDX_OK;
  const unsigned grid = (unsigned)(nq * nsplit);
#define PDX_LIN(M)                                                                              \
  do {                                                                                          \
    PDX_CUDA_CHECK(cudaFuncSetAttribute(linear_kernel<M>,                                       \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    linear_kernel<M><<<grid, kLW * 32, smem, st>>>(store->d_tiles, store->d_tile_ids,          \
                                                   store->ntiles, store->d, store->d_pad,       \
                                                   d_queries, nq, nsplit, k, KL, tdist, tids,   \
                                                   touched, total);                             \
  } while (0)
  if (metric == PDX_METRIC_L2)
    PDX_LIN(PDX_METRIC_L2);
  else if (metric == PDX_METRIC_L1)
    PDX_LIN(PDX_METRIC_L1);
  else
    PDX_LIN(PDX_METRIC_IP);
#undef PDX_LIN
  PDX_LAUNCH_CHECK();
  *applied = true;
  return PDX_OK;
}

}  // namespace pdx
