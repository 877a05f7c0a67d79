// K1 (PDX packing), K3 (projection), K7 (top-k merge), float64 ground truth
// and the ABI's bookkeeping entry points.
#include <mutex>

#include "pdx_common.cuh"
#include "pdx_sort.cuh"

namespace pdx {

static thread_local char g_err[1024] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// ------------------------------------------------------------------- K1
// One CTA per 64-slot tile; a 32-dim chunk at a time is staged in shared
// memory so both the row-major reads (128 B per row) and the tile writes
// (contiguous 256 B rows for group 1, contiguous 2 KB groups for group 8)
// are coalesced.  to_blocks' transpose (layout.py:107-108) with zero
// padding of slots >= m (layout.py:106) and of dims >= d.
constexpr int kPackDims = 32;

__global__ void __launch_bounds__(256) pack_kernel(const float* __restrict__ x, int d, int d_pad,
                                                   int group, const int64_t* __restrict__ src,
                                                   const int64_t* __restrict__ ids_in,
                                                   float* __restrict__ tiles,
                                                   int64_t* __restrict__ tile_ids) {
  __shared__ float buf[kTile][kPackDims + 1];
  __shared__ int64_t rows[kTile];
  const int64_t t = blockIdx.x;
  if (threadIdx.x < kTile) {
    const int64_t r = src[t * kTile + threadIdx.x];
    rows[threadIdx.x] = r;
    tile_ids[t * kTile + threadIdx.x] = r < 0 ? -1 : (ids_in ? ids_in[r] : r);
  }
  __syncthreads();
  float* out = tiles + t * (int64_t)d_pad * kTile;
  for (int c0 = 0; c0 < d_pad; c0 += kPackDims) {
    for (int e = threadIdx.x; e < kTile * kPackDims; e += blockDim.x) {
      const int s = e / kPackDims, j = e % kPackDims;
      const int64_t r = rows[s];
      const int dj = c0 + j;
      buf[s][j] = (r >= 0 && dj < d) ? x[r * d + dj] : 0.f;
    }
    __syncthreads();
    const int nd = min(kPackDims, d_pad - c0);
    if (group == 1) {
      for (int e = threadIdx.x; e < kTile * nd; e += blockDim.x) {
        const int j = e / kTile, s = e % kTile;
        out[(int64_t)(c0 + j) * kTile + s] = buf[s][j];
      }
    } else {  // group 8: [d_pad/8][64][8]; the chunk covers nd/8 whole groups
      float* o = out + (int64_t)(c0 / 8) * kTile * 8;
      for (int e = threadIdx.x; e < kTile * nd; e += blockDim.x) {
        const int g = e / (kTile * 8), rem = e % (kTile * 8);
        const int s = rem / 8, dd = rem % 8;
        o[e] = buf[s][g * 8 + dd];
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------- K3
// y = x @ M^T, float32 (FMA) — apply_transform (pruning.py:48-53).  A CTA
// computes 16 rows x 64 columns (a thread: one row, four columns) over K
// chunks of 32 staged in shared memory: small tiles, so a 1,000-query batch
// still spreads over ~128 CTAs (the projection sits on the search's
// critical path).
// (kPK = 128: a d = 128 projection stages its whole operands with one round of
// loads in flight instead of four load-sync-compute rounds: 16 -> ~7 us)
constexpr int kPR = 16, kPC = 64, kPK = 128;

__global__ void __launch_bounds__(256) project_kernel(const float* __restrict__ x, int64_t n, int d,
                                                      const float* __restrict__ M,
                                                      float* __restrict__ y) {
  __shared__ float xs[kPK][kPR + 1];
  __shared__ float ms[kPK][kPC + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // cols tx*4..+3, row ty
  const int64_t r0 = (int64_t)blockIdx.y * kPR;
  const int c0 = blockIdx.x * kPC;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int j0 = 0; j0 < d; j0 += kPK) {
    for (int e = threadIdx.x; e < kPR * kPK; e += 256) {
      const int r = e / kPK, c = e % kPK;
      const int dj = j0 + c;
      xs[c][r] = (r0 + r < n && dj < d) ? x[(r0 + r) * d + dj] : 0.f;
    }
    for (int e = threadIdx.x; e < kPC * kPK; e += 256) {
      const int r = e / kPK, c = e % kPK;
      const int dj = j0 + c;
      ms[c][r] = (c0 + r < d && dj < d) ? M[(int64_t)(c0 + r) * d + dj] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int jj = 0; jj < kPK; ++jj) {
      const float xv = xs[jj][ty];
      const float4 mv = *reinterpret_cast<const float4*>(&ms[jj][tx * 4]);
      acc[0] = fmaf(xv, mv.x, acc[0]);
      acc[1] = fmaf(xv, mv.y, acc[1]);
      acc[2] = fmaf(xv, mv.z, acc[2]);
      acc[3] = fmaf(xv, mv.w, acc[3]);
    }
    __syncthreads();
  }
  const int64_t r = r0 + ty;
  if (r < n) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + tx * 4 + j;
      if (c < d) y[r * d + c] = acc[j];
    }
  }
}

// ------------------------------------------------------------------- K7
struct DistId {
  float d;
  int64_t i;
};

__global__ void __launch_bounds__(256) merge_kernel(const float* __restrict__ dist,
                                                    const int64_t* __restrict__ ids, int nparts,
                                                    int64_t nq, int k, float* __restrict__ od,
                                                    int64_t* __restrict__ oi) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = nparts * k;
  const int n2 = pow2_ceil(n);
  float* key = reinterpret_cast<float*>(smem);
  int64_t* val = reinterpret_cast<int64_t*>(smem + (((size_t)n2 * 4 + 15) & ~(size_t)15));
  const int64_t q = blockIdx.x;
  for (int e = threadIdx.x; e < n2; e += blockDim.x) {
    if (e < n) {
      const int p = e / k, j = e % k;
      const int64_t off = ((int64_t)p * nq + q) * k + j;
      const int64_t iv = ids[off];
      key[e] = iv < 0 ? INFINITY : dist[off];
      val[e] = iv < 0 ? INT64_MAX : iv;
    } else {
      key[e] = INFINITY;
      val[e] = INT64_MAX;
    }
  }
  __syncthreads();
  bitonic_sort(key, val, n2);
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const bool ok = val[j] != INT64_MAX;
    od[q * k + j] = ok ? key[j] : INFINITY;
    oi[q * k + j] = ok ? val[j] : -1;
  }
}

// ------------------------------------------------------- ground truth (f64)
// compute_ground_truth (bench.py:53-67): horizontal float64 distances
// (kernels.py:108-119) and the k smallest (key, row), lower row on ties.
// Stage 1: each CTA takes 8 queries x a row range; each thread keeps a
// sorted top-k per query in registers-backed local memory; lists go to
// scratch.  Stage 2: per query, a CTA selects over all lists.
constexpr int kGtQ = 8, kGtMaxK = 32, kGtRows = 65536;

template <int METRIC>
__global__ void __launch_bounds__(128) gt_stage1(const float* __restrict__ x, int64_t n, int d,
                                                 const float* __restrict__ Q, int64_t nq, int k,
                                                 double* __restrict__ cd, int64_t* __restrict__ ci) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* qs = reinterpret_cast<double*>(smem);  // [kGtQ][d]
  const int64_t q0 = (int64_t)blockIdx.y * kGtQ;
  for (int e = threadIdx.x; e < kGtQ * d; e += blockDim.x) {
    const int64_t qq = q0 + e / d;
    qs[e] = qq < nq ? (double)Q[qq * d + e % d] : 0.0;
  }
  __syncthreads();
  double bd[kGtQ][kGtMaxK];
  int64_t bi[kGtQ][kGtMaxK];
#pragma unroll
  for (int a = 0; a < kGtQ; ++a)
    for (int j = 0; j < k; ++j) { bd[a][j] = INFINITY; bi[a][j] = INT64_MAX; }
  const int64_t r_begin = (int64_t)blockIdx.x * kGtRows;
  const int64_t r_end = (n < r_begin + kGtRows ? n : r_begin + kGtRows);
  for (int64_t r = r_begin + threadIdx.x; r < r_end; r += blockDim.x) {
    double acc[kGtQ];
#pragma unroll
    for (int a = 0; a < kGtQ; ++a) acc[a] = 0.0;
    const float* xr = x + r * d;
    for (int j = 0; j < d; ++j) {
      const double xv = (double)__ldg(xr + j);
#pragma unroll
      for (int a = 0; a < kGtQ; ++a) {
        const double qv = qs[a * d + j];
        if (METRIC == PDX_METRIC_L2) {
          const double t = xv - qv;
          acc[a] = fma(t, t, acc[a]);
        } else if (METRIC == PDX_METRIC_L1) {
          acc[a] += fabs(xv - qv);
        } else {
          acc[a] = fma(xv, qv, acc[a]);
        }
      }
    }
#pragma unroll
    for (int a = 0; a < kGtQ; ++a) {
      const double key = METRIC == PDX_METRIC_IP ? -acc[a] : acc[a];
      if (key < bd[a][k - 1] || (key == bd[a][k - 1] && r < bi[a][k - 1])) {
        int p = k - 1;
        while (p > 0 && (key < bd[a][p - 1] || (key == bd[a][p - 1] && r < bi[a][p - 1]))) {
          bd[a][p] = bd[a][p - 1];
          bi[a][p] = bi[a][p - 1];
          --p;
        }
        bd[a][p] = key;
        bi[a][p] = r;
      }
    }
  }
  // lists: [nq][nblocks_x * blockDim][k]
  const int64_t lists = (int64_t)gridDim.x * blockDim.x;
  const int64_t lid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int a = 0; a < kGtQ; ++a) {
    const int64_t qq = q0 + a;
    if (qq >= nq) continue;
    for (int j = 0; j < k; ++j) {
      cd[(qq * lists + lid) * k + j] = bd[a][j];
      ci[(qq * lists + lid) * k + j] = bi[a][j];
    }
  }
}

__global__ void __launch_bounds__(512) gt_stage2(const double* __restrict__ cd,
                                                 const int64_t* __restrict__ ci, int64_t ncand,
                                                 int k, int metric, int64_t* __restrict__ oi,
                                                 double* __restrict__ od) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int chunk = 2048;
  const int n2 = pow2_ceil(k + chunk);
  double* bk = reinterpret_cast<double*>(smem);
  int64_t* bv = reinterpret_cast<int64_t*>(bk + n2);
  const int64_t q = blockIdx.x;
  const double* dq = cd + q * ncand;
  const int64_t* iq = ci + q * ncand;
  block_top_p<double, int64_t>((int)ncand, k, chunk, bk, bv, INFINITY, INT64_MAX,
                               [&](int i, double& kk, int64_t& vv) {
                                 kk = dq[i];
                                 vv = iq[i];
                               });
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    oi[q * k + j] = bv[j];
    od[q * k + j] = metric == PDX_METRIC_IP ? -bk[j] : bk[j];
  }
}

// ------------------------------------------------------- segment means
// One CTA per segment, a thread per dimension (column); rows are added in
// segment order, float64, as numpy's axis-0 sum does.
__global__ void __launch_bounds__(128) segment_means_kernel(const float* __restrict__ x, int d,
                                                            const int64_t* __restrict__ rows,
                                                            const int64_t* __restrict__ off,
                                                            double* __restrict__ means) {
  const int s = blockIdx.x;
  const int64_t b = off[s], e = off[s + 1];
  if (e <= b) return;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double acc = 0.0;
    int64_t i = b;
    for (; i + 4 <= e; i += 4) {
      const int64_t r0 = rows ? rows[i] : i, r1 = rows ? rows[i + 1] : i + 1;
      const int64_t r2 = rows ? rows[i + 2] : i + 2, r3 = rows ? rows[i + 3] : i + 3;
      const float v0 = __ldg(x + r0 * d + j), v1 = __ldg(x + r1 * d + j);
      const float v2 = __ldg(x + r2 * d + j), v3 = __ldg(x + r3 * d + j);
      acc = __dadd_rn(acc, (double)v0);
      acc = __dadd_rn(acc, (double)v1);
      acc = __dadd_rn(acc, (double)v2);
      acc = __dadd_rn(acc, (double)v3);
    }
    for (; i < e; ++i) acc = __dadd_rn(acc, (double)__ldg(x + (rows ? rows[i] : i) * d + j));
    means[(int64_t)s * d + j] = __ddiv_rn(acc, (double)(e - b));
  }
}

}  // namespace pdx

using namespace pdx;

extern "C" int pdx_segment_means(const float* d_x, int32_t d, const int64_t* d_rows,
                                 const int64_t* d_seg_off, int32_t nseg, double* d_means,
                                 void* stream) {
  PDX_REQUIRE(d >= 1 && nseg >= 0, "bad sizes");
  if (nseg == 0) return PDX_OK;
  segment_means_kernel<<<(unsigned)nseg, 128, 0, as_stream(stream)>>>(d_x, d, d_rows, d_seg_off,
                                                                      d_means);
  PDX_LAUNCH_CHECK();
  return PDX_OK;
}

namespace pdx {
// BSA residual energies (pdx_bsa_residuals): one thread per slot; each step's
// suffix sum is its own sequential float32 chain in increasing dim order, the
// definition the C oracle restates.
__global__ void __launch_bounds__(256) bsa_resid_kernel(const float* __restrict__ tiles, int64_t ntiles,
                                                        int d, int d_pad, int group,
                                                        int initial_step, int nsteps,
                                                        float* __restrict__ out) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= ntiles * 64) return;
  const int64_t t = gid >> 6;
  const int i = (int)(gid & 63);
  const float* tb = tiles + t * (int64_t)d_pad * 64;
  int64_t e = 0, width = initial_step;
  for (int s = 0; s < nsteps; ++s, width *= 2) {
    e = e + width < d ? e + width : d;
    float r = 0.f;
    for (int j = (int)e; j < d; ++j) {
      const float x = group == 8 ? tb[((int64_t)(j >> 3) * 64 + i) * 8 + (j & 7)]
                                 : tb[(int64_t)j * 64 + i];
      r = __fadd_rn(r, __fmul_rn(x, x));
    }
    out[(t * nsteps + s) * 64 + i] = r;
  }
}
}  // namespace pdx

extern "C" int pdx_bsa_residuals(const pdx_store* store, int32_t initial_step, float* d_resid,
                                 int32_t* nsteps_out, void* stream) {
  PDX_REQUIRE(store && nsteps_out, "pdx_bsa_residuals: null argument");
  PDX_REQUIRE(initial_step >= 1, "initial_step must be >= 1");
  PDX_REQUIRE(store->group == 1 || store->group == 8, "group must be 1 or 8");
  int n = 0;
  for (int64_t e = 0, w = initial_step; e < store->d; w *= 2, ++n) e = e + w < store->d ? e + w : store->d;
  *nsteps_out = n;
  if (store->ntiles == 0 || !d_resid) return PDX_OK;  // NULL output: size query
  const int64_t threads = store->ntiles * 64;
  pdx::bsa_resid_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, pdx::as_stream(stream)>>>(
      store->d_tiles, store->ntiles, store->d, store->d_pad, store->group, initial_step, n,
      d_resid);
  PDX_LAUNCH_CHECK();
  return PDX_OK;
}

extern "C" int pdx_abi_version(void) { return PDX_ABI_VERSION; }

extern "C" int pdx_last_error(char* buf, size_t cap) {
  const size_t n = strlen(pdx::g_err);
  if (buf && cap) {
    const size_t c = n < cap - 1 ? n : cap - 1;
    memcpy(buf, pdx::g_err, c);
    buf[c] = 0;
  }
  return (int)n;
}

extern "C" int pdx_device_info(int32_t* sm_count, int32_t* smem_optin, int32_t* cc_major,
                               int32_t* cc_minor) {
  int dev = 0;
  PDX_CUDA_CHECK(cudaGetDevice(&dev));
  int v = 0;
  if (sm_count) { PDX_CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev)); *sm_count = v; }
  if (smem_optin) { PDX_CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)); *smem_optin = v; }
  if (cc_major) { PDX_CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, dev)); *cc_major = v; }
  if (cc_minor) { PDX_CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, dev)); *cc_minor = v; }
  return PDX_OK;
}

extern "C" int pdx_pack_tiles(const float* d_x, int64_t n, int32_t d, const int64_t* d_slot_src,
                              int64_t ntiles, int32_t group, const int64_t* d_ids_in,
                              float* d_tiles, int64_t* d_tile_ids, void* stream) {
  PDX_REQUIRE(d >= 1, "dimensionality must be >= 1");
  PDX_REQUIRE(group == 1 || group == 8, "group must be 1 or 8");
  PDX_REQUIRE(n >= 0 && ntiles >= 0, "bad sizes");
  if (ntiles == 0) return PDX_OK;
  const int d_pad = group == 8 ? (d + 7) / 8 * 8 : d;
  pack_kernel<<<(unsigned)ntiles, 256, 0, as_stream(stream)>>>(d_x, d, d_pad, group, d_slot_src,
                                                               d_ids_in, d_tiles, d_tile_ids);
  PDX_LAUNCH_CHECK();
  return PDX_OK;
}

extern "C" int pdx_project(const float* d_x, int64_t n, int32_t d, const float* d_matrix,
                           float* d_y, void* stream) {
  PDX_REQUIRE(d >= 1 && n >= 0, "bad sizes");
  PDX_REQUIRE(d_x != d_y, "pdx_project: output must not alias input");
  if (n == 0) return PDX_OK;
  const int64_t per = (int64_t)65535 * kPR;  // rows per launch (grid.y limit)
  for (int64_t r = 0; r < n; r += per) {
    const int64_t m = n - r < per ? n - r : per;
    dim3 grid((d + kPC - 1) / kPC, (unsigned)((m + kPR - 1) / kPR));
    project_kernel<<<grid, 256, 0, as_stream(stream)>>>(d_x + r * d, m, d, d_matrix, d_y + r * d);
    PDX_LAUNCH_CHECK();
  }
  return PDX_OK;
}

// The reference's vertical kernels as a standalone op (kernels.py:41-91):
// one thread per slot (or per listed position), dims [a, b) of the natural
// order or of d_order, each float32 op rounded on its own.
template <int METRIC>
__global__ void __launch_bounds__(128) vacc_kernel(const float* __restrict__ block, int mp,
                                                   const float* __restrict__ q, int a, int b,
                                                   const int64_t* __restrict__ order,
                                                   const int64_t* __restrict__ pos, int npos,
                                                   float* __restrict__ acc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= npos) return;
  const int64_t slot = pos ? pos[t] : t;
  float v = acc[slot];
  for (int i = a; i < b; ++i) {
    const int64_t j = order ? order[i] : i;
    v = upd<METRIC>(v, q[j], block[j * mp + slot]);
  }
  acc[slot] = v;
}

extern "C" int pdx_vertical_accumulate(const float* d_block, int32_t d, int32_t mp,
                                       const float* d_query, int32_t a, int32_t b,
                                       const int64_t* d_order, const int64_t* d_positions,
                                       int32_t npos, int32_t metric, float* d_acc, void* stream) {
  PDX_REQUIRE(d >= 1 && mp >= 0, "bad block shape");
  PDX_REQUIRE(0 <= a && a <= b && b <= d, "dimension range [%d, %d) out of bounds for d=%d", a, b,
              d);
  PDX_REQUIRE(metric >= 0 && metric <= 2, "unknown metric %d", metric);
  const int n = d_positions ? npos : mp;
  if (n <= 0 || a == b) return PDX_OK;
  cudaStream_t st = as_stream(stream);
  const unsigned g = (unsigned)((n + 127) / 128);
  if (metric == PDX_METRIC_L2)
    vacc_kernel<PDX_METRIC_L2><<<g, 128, 0, st>>>(d_block, mp, d_query, a, b, d_order, d_positions,
                                                  n, d_acc);
  else if (metric == PDX_METRIC_L1)
    vacc_kernel<PDX_METRIC_L1><<<g, 128, 0, st>>>(d_block, mp, d_query, a, b, d_order, d_positions,
                                                  n, d_acc);
  else
    vacc_kernel<PDX_METRIC_IP><<<g, 128, 0, st>>>(d_block, mp, d_query, a, b, d_order, d_positions,
                                                  n, d_acc);
  PDX_LAUNCH_CHECK();
  return PDX_OK;
}

extern "C" int pdx_merge_topk(const float* d_dist, const int64_t* d_ids, int32_t nparts, int64_t nq,
                              int32_t k, float* d_out_dist, int64_t* d_out_ids, void* stream) {
  PDX_REQUIRE(nparts >= 1 && k >= 1, "bad merge sizes");
  if (nq == 0) return PDX_OK;
  const int n2 = pow2_ceil(nparts * k);
  const size_t smem = (((size_t)n2 * 4 + 15) & ~(size_t)15) + (size_t)n2 * 8;
  int dev = 0, optin = 0;
  PDX_CUDA_CHECK(cudaGetDevice(&dev));
  PDX_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (smem > (size_t)optin) {
    pdx::set_error("merge of %d x %d candidates exceeds shared memory", nparts, k);
    return PDX_ENOSUPPORT;
  }
  PDX_CUDA_CHECK(cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  merge_kernel<<<(unsigned)nq, 256, smem, as_stream(stream)>>>(d_dist, d_ids, nparts, nq, k,
                                                               d_out_dist, d_out_ids);
  PDX_LAUNCH_CHECK();
  return PDX_OK;
}

extern "C" int pdx_ground_truth(const float* d_x, int64_t n, int32_t d, const float* d_queries,
                                int64_t nq, int32_t k, int32_t metric, int64_t* d_ids,
                                double* d_dist, void* stream) {
  PDX_REQUIRE(k >= 1 && k <= kGtMaxK, "ground truth supports 1 <= k <= %d", kGtMaxK);
  PDX_REQUIRE(n >= k, "k larger than the collection");
  PDX_REQUIRE(d >= 1 && metric >= 0 && metric <= 2, "bad arguments");
  if (nq == 0) return PDX_OK;
  cudaStream_t st = as_stream(stream);
  const int64_t nbx = (n + kGtRows - 1) / kGtRows;
  const int64_t ncand = nbx * 128 * k;
  PDX_REQUIRE(ncand < (1ll << 31), "collection too large for the ground-truth kernel");
  double* cd = nullptr;
  int64_t* ci = nullptr;
  PDX_CUDA_CHECK(cudaMallocAsync(&cd, (size_t)nq * ncand * sizeof(double), st));
  PDX_CUDA_CHECK(cudaMallocAsync(&ci, (size_t)nq * ncand * sizeof(int64_t), st));
  const size_t sm1 = (size_t)kGtQ * d * sizeof(double);
  dim3 g1((unsigned)nbx, (unsigned)((nq + kGtQ - 1) / kGtQ));
  if (metric == PDX_METRIC_L2) {
    PDX_CUDA_CHECK(cudaFuncSetAttribute(gt_stage1<PDX_METRIC_L2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
    gt_stage1<PDX_METRIC_L2><<<g1, 128, sm1, st>>>(d_x, n, d, d_queries, nq, k, cd, ci);
  } else if (metric == PDX_METRIC_L1) {
    PDX_CUDA_CHECK(cudaFuncSetAttribute(gt_stage1<PDX_METRIC_L1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
    gt_stage1<PDX_METRIC_L1><<<g1, 128, sm1, st>>>(d_x, n, d, d_queries, nq, k, cd, ci);
  } else {
    PDX_CUDA_CHECK(cudaFuncSetAttribute(gt_stage1<PDX_METRIC_IP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
    gt_stage1<PDX_METRIC_IP><<<g1, 128, sm1, st>>>(d_x, n, d, d_queries, nq, k, cd, ci);
  }
  PDX_LAUNCH_CHECK();
  const int n2 = pow2_ceil(k + 2048);
  const size_t sm2 = (size_t)n2 * 16;
  PDX_CUDA_CHECK(cudaFuncSetAttribute(gt_stage2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
  gt_stage2<<<(unsigned)nq, 512, sm2, st>>>(cd, ci, ncand, k, metric, d_ids, d_dist);
  PDX_LAUNCH_CHECK();
  PDX_CUDA_CHECK(cudaFreeAsync(cd, st));
  PDX_CUDA_CHECK(cudaFreeAsync(ci, st));
  return PDX_OK;
}
