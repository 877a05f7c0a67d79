// K4: query-aware dimension orders — bond_dimension_order (pruning.py:107-140).
//
// One CTA per (query, means-row) produces a uint16 permutation:
//   sequential : identity
//   decreasing : stable argsort of -q             (float64)
//   dmeans     : stable argsort of -|q - mu|      (float64)
//   zones      : zones of `zone_width` consecutive dims ranked by the
//                stable argsort of -(sum of gaps), summed with numpy's
//                pairwise float64 association (pruning.py:135 uses
//                ndarray.sum), sequential order inside a zone.
// Stable order == ascending (key, index), which the bitonic sort gives.
#include "pdx_common.cuh"
#include "pdx_sort.cuh"

namespace pdx {

// numpy's pairwise_sum for a contiguous float64 array: 8-way unrolled
// leaves of <= 128 elements, halves split at a multiple of 8.
__device__ double numpy_sum_leaf(const double* x, int m) {
  if (m < 8) {
    double res = 0.0;
    for (int i = 0; i < m; ++i) res = __dadd_rn(res, x[i]);
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = x[j];
  int i;
  for (i = 8; i < m - (m % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], x[i + j]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < m; ++i) res = __dadd_rn(res, x[i]);
  return res;
}

__device__ double numpy_pairwise_sum(const double* a, int n) {
  if (n <= 128) return numpy_sum_leaf(a, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(numpy_pairwise_sum(a, n2), numpy_pairwise_sum(a + n2, n - n2));
}

template <typename QT>
__global__ void __launch_bounds__(512) orders_kernel(const QT* __restrict__ Q, int d,
                                                     const double* __restrict__ means,
                                                     const int32_t* __restrict__ mean_index,
                                                     int nsets, int criteria, int zw,
                                                     uint16_t* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int64_t r = blockIdx.x;  // output row = q*nsets + s
  const int64_t q = r / nsets;
  const int n2 = pow2_ceil(d);
  double* key = reinterpret_cast<double*>(smem);
  int32_t* val = reinterpret_cast<int32_t*>(key + n2);
  double* gaps = reinterpret_cast<double*>(val + ((n2 + 1) & ~1));
  const QT* qv = Q + q * d;
  const double* mu = means + (int64_t)(mean_index ? mean_index[r] : 0) * d;
  uint16_t* o = out + r * d;
  if (criteria == PDX_ORDER_SEQUENTIAL) {
    for (int j = threadIdx.x; j < d; j += blockDim.x) o[j] = (uint16_t)j;
    return;
  }
  if (criteria == PDX_ORDER_DECREASING) {
    for (int j = threadIdx.x; j < n2; j += blockDim.x) {
      key[j] = j < d ? __dadd_rn(-(double)qv[j], 0.0) : INFINITY;
      val[j] = j < d ? j : 0x7fffffff;
    }
    __syncthreads();
    bitonic_sort(key, val, n2);
    for (int j = threadIdx.x; j < d; j += blockDim.x) o[j] = (uint16_t)val[j];
    return;
  }
  for (int j = threadIdx.x; j < d; j += blockDim.x) gaps[j] = fabs(__dsub_rn((double)qv[j], mu[j]));
  __syncthreads();
  if (criteria == PDX_ORDER_DMEANS) {
    for (int j = threadIdx.x; j < n2; j += blockDim.x) {
      key[j] = j < d ? __dadd_rn(-gaps[j], 0.0) : INFINITY;
      val[j] = j < d ? j : 0x7fffffff;
    }
    __syncthreads();
    bitonic_sort(key, val, n2);
    for (int j = threadIdx.x; j < d; j += blockDim.x) o[j] = (uint16_t)val[j];
    return;
  }
  // zones
  const int nz = (d + zw - 1) / zw;
  const int z2 = pow2_ceil(nz);
  for (int z = threadIdx.x; z < z2; z += blockDim.x) {
    if (z < nz) {
      const int s = z * zw;
      const int e = min(s + zw, d);
      key[z] = __dadd_rn(-numpy_pairwise_sum(gaps + s, e - s), 0.0);
      val[z] = z;
    } else {
      key[z] = INFINITY;
      val[z] = 0x7fffffff;
    }
  }
  __syncthreads();
  bitonic_sort(key, val, z2);
  // output: zones in rank order; only the last zone (index nz-1) may be short
  __shared__ int s_lastrank;
  if (threadIdx.x == 0) {
    s_lastrank = nz;
    for (int rk = 0; rk < nz; ++rk)
      if (val[rk] == nz - 1) s_lastrank = rk;
  }
  __syncthreads();
  const int short_len = d - (nz - 1) * zw;
  for (int rk = 0; rk < nz; ++rk) {
    const int z = val[rk];
    const int s = z * zw;
    const int len = (z == nz - 1) ? short_len : zw;
    const int pos = rk * zw - ((s_lastrank < rk) ? (zw - short_len) : 0);
    for (int j = threadIdx.x; j < len; j += blockDim.x) o[pos + j] = (uint16_t)(s + j);
  }
}

}  // namespace pdx

using namespace pdx;

extern "C" int pdx_dimension_orders(const void* d_queries, int32_t queries_f64, int64_t nq,
                                    int32_t d, const double* d_means,
                                    const int32_t* d_mean_index, int32_t nsets, int32_t criteria,
                                    int32_t zone_width, uint16_t* d_out, void* stream) {
  PDX_REQUIRE(d >= 1 && d <= 65535, "dimensionality %d unsupported", d);
  PDX_REQUIRE(nsets >= 1, "nsets must be >= 1");
  PDX_REQUIRE(criteria >= 0 && criteria <= 3, "unknown order criteria %d", criteria);
  if (nq == 0) return PDX_OK;
  cudaStream_t st = as_stream(stream);
  int zw = zone_width;
  if (criteria == PDX_ORDER_ZONES) {
    if (zw <= 0) {
      zw = d / 16 > 8 ? d / 16 : 8;  // default_zone_width (pruning.py:98-99)
      if (zw > d) zw = d;
    }
  }
  const int n2 = pow2_ceil(d);
  const size_t smem = (size_t)n2 * sizeof(double) + (size_t)((n2 + 1) & ~1) * sizeof(int32_t) +
                      (size_t)d * sizeof(double);
  int dev = 0, optin = 0;
  PDX_CUDA_CHECK(cudaGetDevice(&dev));
  PDX_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (smem > (size_t)optin) {
    ::pdx::set_error("dimensionality %d too large for the order kernel", d);
    return PDX_ENOSUPPORT;
  }
  if (queries_f64) {
    PDX_CUDA_CHECK(cudaFuncSetAttribute(orders_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    orders_kernel<double><<<(unsigned)(nq * nsets), 256, smem, st>>>(
        static_cast<const double*>(d_queries), d, d_means, d_mean_index, nsets, criteria, zw, d_out);
  } else {
    PDX_CUDA_CHECK(cudaFuncSetAttribute(orders_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    orders_kernel<float><<<(unsigned)(nq * nsets), 256, smem, st>>>(
        static_cast<const float*>(d_queries), d, d_means, d_mean_index, nsets, criteria, zw, d_out);
  }
  PDX_LAUNCH_CHECK();
  return PDX_OK;
}
