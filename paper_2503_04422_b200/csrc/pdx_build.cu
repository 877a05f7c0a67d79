// GPU IVF build: the reference's Lloyd k-means
// (index.py:27-64) and bucket layout (index.py:98-100) in hand-written
// kernels — no cuBLAS, no ATen.
//
//   pdx_row_norms        ||x_i||^2 in float32 (the einsum of index.py:70)
//   pdx_kmeans_assign    fused distance + argmin: max(xx + cc - 2 x.c, 0)
//                        (index.py:67-72) over every centroid, the lowest
//                        index among equal minima (np.argmin, :44/:63)
//   pdx_bucket_layout    members of every bucket in ascending row order
//                        (np.flatnonzero per bucket, :100): a stable radix
//                        sort of (bucket, row) + counts + offsets
//   pdx_kmeans_update    new centroid = f32(f64 member mean) for non-empty
//                        buckets, else the old one (:45-48)
//   pdx_kmeans_farthest  the repair's farthest member of a bucket (:49-56)
//   pdx_kmeans_shift     max_c ||new_c - old_c|| / (||old_c|| + 1e-30) (:57-61)
//   pdx_gather_rows      x[rows] (the seeded sample init, :38-39)
//   pdx_pack_rows        a chunk of rows scattered straight into their tile
//                        slots (the chunked build: no full host copy)
//
// The distance GEMM runs on the FP32 pipes (FFMA), exact float32 like the
// reference's sgemm (which is itself not bit-pinned: BLAS association).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "pdx_common.cuh"

namespace pdx {
namespace {

// ---------------------------------------------------------------- norms
__global__ void __launch_bounds__(256) row_norms_kernel(const float* __restrict__ x, int64_t n,
                                                        int d, float* __restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  const float* xr = x + r * d;
  float acc = 0.f;
  for (int j = lane; j < d; j += 32) acc = fmaf(xr[j], xr[j], acc);
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[r] = acc;
}

// ------------------------------------------------------- fused assign
// CTA: 128 rows x every centroid, 128 centroids per tile, K chunks of 16.
// 256 threads, an 8x8 register micro-tile each (rows ty*4+{0..3} and
// 64+ty*4+{0..3}, centroids tx*4+{0..3} and 64+tx*4+{0..3}): the classic
// SIMT sgemm shape, operands staged k-major in shared memory so a thread's
// 8 row values and 8 centroid values are two float4 loads each.
constexpr int kAM = 128, kAN = 128, kAK = 16;

__device__ __forceinline__ bool better(float d, int c, float bd, int bc) {
  return d < bd || (d == bd && c < bc);
}

__global__ void __launch_bounds__(256) kmeans_assign_kernel(
    const float* __restrict__ x, const int64_t* __restrict__ rows, int64_t n, int d,
    const float* __restrict__ xx, const float* __restrict__ c, const float* __restrict__ cc,
    int nlist, int32_t* __restrict__ assign, float* __restrict__ mind) {
  __shared__ __align__(16) float Xs[2][kAK][kAM];
  __shared__ __align__(16) float Cs[2][kAK][kAN];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t r0 = (int64_t)blockIdx.x * kAM;
  // loader mapping: 128 rows x 16 k = 2048 floats = 256 threads x 8 (two float4 along k)
  const int lr = tid >> 1, lk = (tid & 1) * 8;
  const int64_t grow = r0 + lr;
  const bool rvalid = grow < n;
  const float* xrow = rvalid ? x + (rows ? rows[grow] : grow) * (int64_t)d : x;
  const bool vec4 = (d & 3) == 0;

  float bestd[8];
  int bestc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    bestd[i] = INFINITY;
    bestc[i] = 0x7fffffff;
  }
  float rxx[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = r0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    rxx[i] = r < n ? xx[r] : 0.f;
  }

  auto load_chunk = [&](float (&xs)[kAK][kAM], float (&cs)[kAK][kAN], int ct, int k0) {
    // rows
    float v[8];
    if (rvalid && vec4 && k0 + lk + 8 <= d) {
      const float4 a = *reinterpret_cast<const float4*>(xrow + k0 + lk);
      const float4 b = *reinterpret_cast<const float4*>(xrow + k0 + lk + 4);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = (rvalid && k0 + lk + q < d) ? xrow[k0 + lk + q] : 0.f;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) xs[lk + q][lr] = v[q];
    // centroids
    const int gc = ct * kAN + lr;
    const bool cvalid = gc < nlist;
    const float* crow = c + (int64_t)(cvalid ? gc : 0) * d;
    if (cvalid && vec4 && k0 + lk + 8 <= d) {
      const float4 a = *reinterpret_cast<const float4*>(crow + k0 + lk);
      const float4 b = *reinterpret_cast<const float4*>(crow + k0 + lk + 4);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = (cvalid && k0 + lk + q < d) ? crow[k0 + lk + q] : 0.f;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) cs[lk + q][lr] = v[q];
  };

  const int ntile = (nlist + kAN - 1) / kAN;
  const int nk = (d + kAK - 1) / kAK;
  for (int ct = 0; ct < ntile; ++ct) {
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    int buf = 0;
    __syncthreads();
    load_chunk(Xs[0], Cs[0], ct, 0);
    __syncthreads();
    for (int kc = 0; kc < nk; ++kc) {
      if (kc + 1 < nk) load_chunk(Xs[buf ^ 1], Cs[buf ^ 1], ct, (kc + 1) * kAK);
#pragma unroll
      for (int k = 0; k < kAK; ++k) {
        const float4 a0 = *reinterpret_cast<const float4*>(&Xs[buf][k][ty * 4]);
        const float4 a1 = *reinterpret_cast<const float4*>(&Xs[buf][k][64 + ty * 4]);
        const float4 b0 = *reinterpret_cast<const float4*>(&Cs[buf][k][tx * 4]);
        const float4 b1 = *reinterpret_cast<const float4*>(&Cs[buf][k][64 + tx * 4]);
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
      buf ^= 1;
    }
    // epilogue: distances of this centroid tile, running (min, lowest index)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int gc = ct * kAN + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (gc >= nlist) continue;
      const float ccv = cc[gc];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float dist =
            fmaxf(__fsub_rn(__fadd_rn(rxx[i], ccv), __fmul_rn(2.0f, acc[i][j])), 0.f);
        if (better(dist, gc, bestd[i], bestc[i])) {
          bestd[i] = dist;
          bestc[i] = gc;
        }
      }
    }
  }
  // reduce over the 16 threads (tx) sharing each row: lanes tx of one half-warp
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float bd = bestd[i];
    int bc = bestc[i];
#pragma unroll
    for (int o = 8; o; o >>= 1) {
      const float od = __shfl_xor_sync(0xffffffffu, bd, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (better(od, oc, bd, bc)) {
        bd = od;
        bc = oc;
      }
    }
    if (tx == 0) {
      const int64_t r = r0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
      if (r < n) {
        assign[r] = bc;
        if (mind) mind[r] = bd;
      }
    }
  }
}

// ---------------------------------------------------------- layout
__global__ void iota_kernel(int64_t* __restrict__ v, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

__global__ void count_kernel(const int32_t* __restrict__ a, int64_t n, int nlist,
                             int64_t* __restrict__ counts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const int b = a[i];
    if (b >= 0 && b < nlist) atomicAdd(reinterpret_cast<unsigned long long*>(counts + b), 1ull);
  }
}

// ---------------------------------------------------------- update
// one warp per centroid: new = f32(mean) if count > 0 else old
__global__ void __launch_bounds__(256) update_kernel(const double* __restrict__ means,
                                                     const int64_t* __restrict__ counts,
                                                     const float* __restrict__ old, int nlist,
                                                     int d, float* __restrict__ out) {
  const int cidx = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (cidx >= nlist) return;
  const bool has = counts[cidx] > 0;
  for (int j = threadIdx.x & 31; j < d; j += 32) {
    const int64_t o = (int64_t)cidx * d + j;
    out[o] = has ? __double2float_rn(means[o]) : old[o];
  }
}

// max over centroids of ||new - old|| / (||old|| + 1e-30), float32 (one warp
// per centroid; the result's bits via atomicMax on the non-negative float)
__global__ void __launch_bounds__(256) shift_kernel(const float* __restrict__ nw,
                                                    const float* __restrict__ old, int nlist,
                                                    int d, float* __restrict__ out) {
  const int cidx = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (cidx >= nlist) return;
  float s = 0.f, o2 = 0.f;
  for (int j = threadIdx.x & 31; j < d; j += 32) {
    const int64_t o = (int64_t)cidx * d + j;
    const float t = __fsub_rn(nw[o], old[o]);
    s = fmaf(t, t, s);
    o2 = fmaf(old[o], old[o], o2);
  }
  for (int m = 16; m; m >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, m);
    o2 += __shfl_xor_sync(0xffffffffu, o2, m);
  }
  if ((threadIdx.x & 31) == 0) {
    const float r = __fdiv_rn(sqrtf(s), __fadd_rn(sqrtf(o2), 1e-30f));
    atomicMax(reinterpret_cast<unsigned int*>(out), __float_as_uint(r));
  }
}

// farthest member of bucket b from centroid cb: max (gap, then lowest row)
__global__ void __launch_bounds__(256) farthest_kernel(const float* __restrict__ x, int64_t n,
                                                       int d, const int32_t* __restrict__ assign,
                                                       int b, const float* __restrict__ cb,
                                                       float ccb,
                                                       unsigned long long* __restrict__ best) {
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= n || assign[r] != b) return;
  const float* xr = x + r * d;
  float dot = 0.f, xx = 0.f;
  for (int j = lane; j < d; j += 32) {
    dot = fmaf(xr[j], cb[j], dot);
    xx = fmaf(xr[j], xr[j], xx);
  }
  for (int m = 16; m; m >>= 1) {
    dot += __shfl_xor_sync(0xffffffffu, dot, m);
    xx += __shfl_xor_sync(0xffffffffu, xx, m);
  }
  if (lane == 0) {
    const float g = fmaxf(__fsub_rn(__fadd_rn(xx, ccb), __fmul_rn(2.0f, dot)), 0.f);
    // larger gap wins; among equal gaps the lower row (np.argmax: first)
    const unsigned long long key =
        ((unsigned long long)__float_as_uint(g) << 32) | (unsigned long long)(0xffffffffu - (uint32_t)r);
    atomicMax(best, key);
  }
}

__global__ void __launch_bounds__(256) gather_rows_kernel(const float* __restrict__ x, int d,
                                                          const int64_t* __restrict__ rows,
                                                          int64_t m, float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= m) return;
  const float* src = x + rows[i] * (int64_t)d;
  for (int j = threadIdx.x & 31; j < d; j += 32) out[i * d + j] = src[j];
}

// one warp per row of the chunk: its tile slot dest[i] (tile * 64 + slot),
// layout [d_pad/G][64][G]; writes the slot's id too
__global__ void __launch_bounds__(256) pack_rows_kernel(const float* __restrict__ x, int64_t m,
                                                        int d, int d_pad, int group,
                                                        const int64_t* __restrict__ dest,
                                                        const int64_t* __restrict__ ids,
                                                        float* __restrict__ tiles,
                                                        int64_t* __restrict__ tile_ids) {
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= m) return;
  const int64_t s = dest[i];
  if (s < 0) return;
  const int64_t t = s >> 6;
  const int slot = (int)(s & 63);
  float* tb = tiles + t * (int64_t)d_pad * 64;
  const float* xr = x + i * (int64_t)d;
  for (int j = threadIdx.x & 31; j < d_pad; j += 32) {
    const float v = j < d ? xr[j] : 0.f;
    if (group == 8)
      tb[((int64_t)(j >> 3) * 64 + slot) * 8 + (j & 7)] = v;
    else
      tb[(int64_t)j * 64 + slot] = v;
  }
  if ((threadIdx.x & 31) == 0) tile_ids[s] = ids[i];
}

}  // namespace
}  // namespace pdx

using namespace pdx;

extern "C" int pdx_row_norms(const float* d_x, int64_t n, int32_t d, float* d_out, void* stream) {
  PDX_REQUIRE(d >= 1 && n >= 0, "bad sizes");
  if (n == 0) return PDX_OK;
  row_norms_kernel<<<(unsigned)((n + 7) / 8), 256, 0, as_stream(stream)>>>(d_x, n, d, d_out);
  PDX_LAUNCH_CHECK();
  return PDX_OK;
}

extern "C" int pdx_kmeans_assign(const float* d_x, const int64_t* d_rows, int64_t n, int32_t d,
                                 const float* d_xnorm, const float* d_centroids,
                                 const float* d_cnorm, int32_t nlist, int32_t* d_assign,
                                 float* d_min_dist, void* stream) {
  PDX_REQUIRE(d >= 1 && n >= 0 && nlist >= 1, "bad sizes");
  PDX_REQUIRE(d_x && d_xnorm && d_centroids && d_cnorm && d_assign, "pdx_kmeans_assign: null");
  if (n == 0) return PDX_OK;
  const int64_t nb = (n + kAM - 1) / kAM;
  PDX_REQUIRE(nb <= 0x7fffffff, "too many rows");
  kmeans_assign_kernel<<<(unsigned)nb, 256, 0, as_stream(stream)>>>(
      d_x, d_rows, n, d, d_xnorm, d_centroids, d_cnorm, nlist, d_assign, d_min_dist);
  PDX_LAUNCH_CHECK();
  return PDX_OK;
}

extern "C" int pdx_bucket_layout(const int32_t* d_assign, int64_t n, int32_t nlist,
                                 int64_t* d_order, int64_t* d_counts, int64_t* d_offsets,
                                 void* d_work, int64_t* work_bytes, void* stream) {
  PDX_REQUIRE(n >= 0 && nlist >= 1 && work_bytes, "bad sizes");
  PDX_REQUIRE(n < ((int64_t)1 << 31), "pdx_bucket_layout: at most 2^31 - 1 rows per call");
  cudaStream_t st = as_stream(stream);
  int bits = 1;
  while ((1ll << bits) < nlist) ++bits;
  // workspace: keys_out i32 [n], iota i64 [n], sort temp, scan temp
  size_t sort_b = 0, scan_b = 0;
  PDX_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, sort_b, (const int32_t*)nullptr,
                                                 (int32_t*)nullptr, (const int64_t*)nullptr,
                                                 (int64_t*)nullptr, (int)n, 0, bits, st));
  PDX_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, scan_b, (const int64_t*)nullptr,
                                               (int64_t*)nullptr, nlist + 1, st));
  auto al = [](int64_t v) { return (v + 255) / 256 * 256; };
  const int64_t need = al(4 * n + 4) + al(8 * n + 8) + al((int64_t)sort_b) + al((int64_t)scan_b) +
                       al(8 * (nlist + 1));
  if (!d_work) {
    *work_bytes = need;
    return PDX_OK;
  }
  PDX_REQUIRE(*work_bytes >= need, "pdx_bucket_layout: workspace too small");
  unsigned char* w = static_cast<unsigned char*>(d_work);
  int32_t* keys_out = reinterpret_cast<int32_t*>(w);
  w += al(4 * n + 4);
  int64_t* iota = reinterpret_cast<int64_t*>(w);
  w += al(8 * n + 8);
  void* sort_tmp = w;
  w += al((int64_t)sort_b);
  void* scan_tmp = w;
  w += al((int64_t)scan_b);
  int64_t* cnt = reinterpret_cast<int64_t*>(w);
  PDX_CUDA_CHECK(cudaMemsetAsync(cnt, 0, 8 * (nlist + 1), st));
  if (n > 0) {
    const unsigned g = (unsigned)((n + 255) / 256);
    iota_kernel<<<g, 256, 0, st>>>(iota, n);
    count_kernel<<<g, 256, 0, st>>>(d_assign, n, nlist, cnt);
    PDX_LAUNCH_CHECK();
    // LSD radix sort is stable: rows stay ascending inside a bucket
    PDX_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(sort_tmp, sort_b, d_assign, keys_out, iota,
                                                   d_order, (int)n, 0, bits, st));
  }
  if (d_counts) PDX_CUDA_CHECK(cudaMemcpyAsync(d_counts, cnt, 8 * nlist, cudaMemcpyDeviceToDevice, st));
  if (d_offsets)
    PDX_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_b, cnt, d_offsets, nlist + 1, st));
  return PDX_OK;
}

extern "C" int pdx_kmeans_update(const double* d_means, const int64_t* d_counts,
                                 const float* d_old, int32_t nlist, int32_t d, float* d_new,
                                 void* stream) {
  PDX_REQUIRE(nlist >= 1 && d >= 1, "bad sizes");
  update_kernel<<<(unsigned)((nlist + 7) / 8), 256, 0, as_stream(stream)>>>(d_means, d_counts,
                                                                            d_old, nlist, d, d_new);
  PDX_LAUNCH_CHECK();
  return PDX_OK;
}

extern "C" int pdx_kmeans_shift(const float* d_new, const float* d_old, int32_t nlist, int32_t d,
                                float* d_out, void* stream) {
  PDX_REQUIRE(nlist >= 1 && d >= 1, "bad sizes");
  cudaStream_t st = as_stream(stream);
  PDX_CUDA_CHECK(cudaMemsetAsync(d_out, 0, sizeof(float), st));
  shift_kernel<<<(unsigned)((nlist + 7) / 8), 256, 0, st>>>(d_new, d_old, nlist, d, d_out);
  PDX_LAUNCH_CHECK();
  return PDX_OK;
}

extern "C" int pdx_kmeans_farthest(const float* d_x, int64_t n, int32_t d, const int32_t* d_assign,
                                   int32_t bucket, const float* d_centroid, float cnorm,
                                   int64_t* d_out_key, void* stream) {
  PDX_REQUIRE(n >= 0 && n < ((int64_t)1 << 32) && d >= 1, "bad sizes");
  cudaStream_t st = as_stream(stream);
  unsigned long long* best = reinterpret_cast<unsigned long long*>(d_out_key);
  PDX_CUDA_CHECK(cudaMemsetAsync(best, 0, 8, st));
  if (n == 0) return PDX_OK;
  farthest_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(d_x, n, d, d_assign, bucket, d_centroid,
                                                           cnorm, best);
  PDX_LAUNCH_CHECK();
  return PDX_OK;
}

extern "C" int pdx_gather_rows(const float* d_x, int32_t d, const int64_t* d_rows, int64_t m,
                               float* d_out, void* stream) {
  PDX_REQUIRE(d >= 1 && m >= 0, "bad sizes");
  if (m == 0) return PDX_OK;
  gather_rows_kernel<<<(unsigned)((m + 7) / 8), 256, 0, as_stream(stream)>>>(d_x, d, d_rows, m,
                                                                             d_out);
  PDX_LAUNCH_CHECK();
  return PDX_OK;
}

extern "C" int pdx_pack_rows(const float* d_x, int64_t m, int32_t d, const int64_t* d_dest,
                             const int64_t* d_ids, const pdx_store* store, void* stream) {
  PDX_REQUIRE(store && d == store->d, "pdx_pack_rows: store dimensionality mismatch");
  PDX_REQUIRE(store->group == 1 || store->group == 8, "group must be 1 or 8");
  if (m == 0) return PDX_OK;
  pack_rows_kernel<<<(unsigned)((m + 7) / 8), 256, 0, as_stream(stream)>>>(
      d_x, m, d, store->d_pad, store->group, d_dest, d_ids, const_cast<float*>(store->d_tiles),
      const_cast<int64_t*>(store->d_tile_ids));
  PDX_LAUNCH_CHECK();
  return PDX_OK;
}
