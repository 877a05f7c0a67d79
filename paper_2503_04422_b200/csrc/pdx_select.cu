// K2: IVF bucket selection — ivf_select_buckets (index.py:111-127).
//
// Stage 1: every (query, centroid) float32 distance with the vertical
// kernel's per-op rounding, summed over dims 0..d-1 in order (exactly what
// vertical_accumulate over the centroid chain computes, index.py:120-124).
// It is a dense nq x nlist x d product, tiled 64x64 through shared memory;
// the sequential, unfused accumulation is what keeps the distances (and so
// the bucket order and every later decision) bit-identical to the
// reference, which is why this is not a tensor-core GEMM.
// Stage 2: per query the nprobe smallest (key, bucket) pairs, key = dist
// (or -dist for IP) — numpy's stable argsort followed by [:nprobe].
#include <cub/block/block_radix_sort.cuh>

#include <algorithm>

#include "pdx_common.cuh"
#include "pdx_sort.cuh"

namespace pdx {

constexpr int kQT = 32, kCT = 64, kDC = 16;  // 2 x 4 outputs per thread (4 = two f32x2 pairs)

// (q - c0)^2, (q - c1)^2 as one FADD2 (q broadcast) + FMUL2, each lane rounded
// on its own; the accumulation stays scalar (an f32x2 add after an f32x2
// multiply is contracted into FFMA2 by ptxas).
__device__ __forceinline__ float2 sqdiff_pair(float q, float c0, float c1) {
  unsigned long long cc, qq, t, p;
  asm("mov.b64 %0, {%1, %2};" : "=l"(cc) : "f"(c0), "f"(c1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(qq) : "f"(q));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(qq), "l"(cc));
  asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(p) : "l"(t));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(p));
  return r;
}

// acc + (q - c)^2 for a centroid pair, all three steps f32x2: FADD2 (q
// broadcast), the square as FFMA2 with a +0 addend — the exact square rounded
// once, bit-identical to mul.rn (a square is never -0) — and FADD2; ptxas does
// not contract FFMA2 + FADD2, so each op stays separately rounded (the
// vertical kernel's arithmetic) at 3 instructions per dim and pair.
__device__ __forceinline__ unsigned long long sqacc_pair(unsigned long long acc, float q,
                                                         unsigned long long cc) {
  unsigned long long qq, z, t, p, r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(qq) : "f"(q));
  asm("mov.b64 %0, {%1, %1};" : "=l"(z) : "f"(0.0f));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(qq), "l"(cc));
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(p) : "l"(t), "l"(z));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(acc), "l"(p));
  return r;
}

template <int METRIC>
__global__ void __launch_bounds__(256) centroid_dist_kernel(const float* __restrict__ Q, int64_t nq,
                                                            const float* __restrict__ Cm, int nlist,
                                                            int d, float* __restrict__ out) {
  __shared__ __align__(16) float qs[kDC][kQT + 4];
  __shared__ __align__(16) float cs[kDC][kCT + 4];
  constexpr int RI = kQT / 16;  // query rows per thread
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t q0 = (int64_t)blockIdx.y * kQT;
  const int c0 = blockIdx.x * kCT;
  float acc[RI][4];
  unsigned long long acc2[RI][2];  // L2: the accumulators as centroid pairs
#pragma unroll
  for (int i = 0; i < RI; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    acc2[i][0] = acc2[i][1] = 0ull;  // (+0, +0)
  }
  // the next chunk's operands are loaded into registers while this chunk is
  // evaluated (every CTA is resident at once: the kernel's time is one CTA's
  // chain of load - store - evaluate rounds)
  constexpr int NQL = (kQT * kDC) / 256, NCL = (kCT * kDC) / 256;
  float rq[NQL], rc[NCL];
  auto load_chunk = [&](const int j0) {
#pragma unroll
    for (int it = 0; it < NQL; ++it) {
      const int e = threadIdx.x + 256 * it;
      const int r = e / kDC, c = e % kDC;
      const int64_t qr = q0 + r;
      const int dj = j0 + c;
      rq[it] = (qr < nq && dj < d) ? Q[qr * d + dj] : 0.f;
    }
#pragma unroll
    for (int it = 0; it < NCL; ++it) {
      const int e = threadIdx.x + 256 * it;
      const int r = e / kDC, c = e % kDC;
      const int dj = j0 + c;
      const int cr = c0 + r;
      rc[it] = (cr < nlist && dj < d) ? Cm[(int64_t)cr * d + dj] : 0.f;
    }
  };
  load_chunk(0);
  for (int j0 = 0; j0 < d; j0 += kDC) {
#pragma unroll
    for (int it = 0; it < NQL; ++it) {
      const int e = threadIdx.x + 256 * it;
      qs[e % kDC][e / kDC] = rq[it];
    }
#pragma unroll
    for (int it = 0; it < NCL; ++it) {
      const int e = threadIdx.x + 256 * it;
      cs[e % kDC][e / kDC] = rc[it];
    }
    __syncthreads();
    if (j0 + kDC < d) load_chunk(j0 + kDC);
    const int jn = min(kDC, d - j0);
    auto dim_step = [&](const int jj) {
      float qv[RI], cv[4];
      static_assert(RI == 2, "the query pair is one 64-bit shared-memory load");
      const float2 q2 = *reinterpret_cast<const float2*>(&qs[jj][ty * RI]);
      qv[0] = q2.x;
      qv[1] = q2.y;
      const float4 c4 = *reinterpret_cast<const float4*>(&cs[jj][tx * 4]);
      cv[0] = c4.x; cv[1] = c4.y; cv[2] = c4.z; cv[3] = c4.w;
      if (METRIC == PDX_METRIC_L2) {
        unsigned long long c01, c23;
        asm("mov.b64 %0, {%1, %2};" : "=l"(c01) : "f"(cv[0]), "f"(cv[1]));
        asm("mov.b64 %0, {%1, %2};" : "=l"(c23) : "f"(cv[2]), "f"(cv[3]));
#pragma unroll
        for (int i = 0; i < RI; ++i) {
          acc2[i][0] = sqacc_pair(acc2[i][0], qv[i], c01);
          acc2[i][1] = sqacc_pair(acc2[i][1], qv[i], c23);
        }
      } else {
#pragma unroll
        for (int i = 0; i < RI; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = upd<METRIC>(acc[i][j], qv[i], cv[j]);
      }
    };
    if (jn == kDC) {  // a full chunk: straight-line code (the loop was ~30% of the instructions)
#pragma unroll
      for (int jj = 0; jj < kDC; ++jj) dim_step(jj);
    } else {
      for (int jj = 0; jj < jn; ++jj) dim_step(jj);
    }
    __syncthreads();
  }
  if (METRIC == PDX_METRIC_L2) {
#pragma unroll
    for (int i = 0; i < RI; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[i][2 * h]), "=f"(acc[i][2 * h + 1]) : "l"(acc2[i][h]));
  }
#pragma unroll
  for (int i = 0; i < RI; ++i) {
    const int64_t qr = q0 + ty * RI + i;
    if (qr >= nq) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cr = c0 + tx * 4 + j;
      if (cr < nlist) out[qr * nlist + cr] = acc[i][j];
    }
  }
}

constexpr int kSelChunk = 2048;

// nprobe <= 32, nlist <= 1024: one warp per query.  Keys are (order-preserving
// key << 32 | bucket), so ties go to the lower bucket (numpy's stable
// argsort).  The nprobe-th smallest of the 32 lane minima bounds the answer
// from above (those minima are nprobe real keys); the keys at or below it
// (~3 nprobe for typical data) are sorted by a warp bitonic sort in shared
// memory.  A query with more than kWarpSelCap candidates takes nprobe rounds
// of a warp-wide minimum instead.
constexpr int kWarpSelCap = 256;

__global__ void __launch_bounds__(256) select_warp_kernel(const float* __restrict__ dists,
                                                          int64_t nq, int nlist, int nprobe,
                                                          int negate,
                                                          int32_t* __restrict__ sel) {
  __shared__ uint64_t s_c[8][kWarpSelCap];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t q = (int64_t)blockIdx.x * 8 + w;
  if (q >= nq) return;
  uint64_t* c = s_c[w];
  const float* row = dists + q * nlist;
  constexpr int PER = 1024 / 32;
  uint64_t key[PER];
  uint64_t mn = ~0ull;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int i = j * 32 + lane;
    key[j] = ~0ull;
    if (i < nlist) {
      const float f = row[i];
      key[j] = ((uint64_t)float_key(negate ? -f : f) << 32) | (uint32_t)i;
    }
    mn = key[j] < mn ? key[j] : mn;
  }
  // bitonic sort of the 32 lane minima (ascending across lanes)
  uint64_t v = mn;
  for (int size = 2; size <= 32; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const uint64_t o = __shfl_xor_sync(0xffffffffu, v, stride);
      const bool lower = (lane & stride) == 0, asc = (lane & size) == 0;
      v = (lower == asc) ? (o < v ? o : v) : (o > v ? o : v);
    }
  const uint64_t U = __shfl_sync(0xffffffffu, v, nprobe - 1);
  int cnt = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) cnt += key[j] <= U;
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (total > kWarpSelCap) {
    // rare (skewed rows): nprobe rounds of a warp-wide minimum, each taken
    // out of its lane's registers (the keys are distinct: bucket in the low bits)
    for (int r = 0; r < nprobe; ++r) {
      uint64_t lm = ~0ull;
#pragma unroll
      for (int j = 0; j < PER; ++j) lm = key[j] < lm ? key[j] : lm;
      uint64_t gm = lm;
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t t = __shfl_xor_sync(0xffffffffu, gm, o);
        gm = t < gm ? t : gm;
      }
#pragma unroll
      for (int j = 0; j < PER; ++j)
        if (key[j] == gm) key[j] = ~0ull;
      if (lane == 0) sel[q * nprobe + r] = (int32_t)(uint32_t)gm;
    }
    return;
  }
  int at = incl - cnt;
#pragma unroll
  for (int j = 0; j < PER; ++j)
    if (key[j] <= U) c[at++] = key[j];
  int n2 = 32;
  while (n2 < total) n2 <<= 1;
  for (int i = total + lane; i < n2; i += 32) c[i] = ~0ull;
  __syncwarp();
  for (int size = 2; size <= n2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = lane; t < n2 / 2; t += 32) {
        const int i = 2 * t - (t & (stride - 1)), jn = i + stride;  // stride: a power of two
        const bool asc = (i & size) == 0;
        const uint64_t a = c[i], b = c[jn];
        if ((a > b) == asc) {
          c[i] = b;
          c[jn] = a;
        }
      }
      __syncwarp();
    }
  if (lane < nprobe) sel[q * nprobe + lane] = (int32_t)(uint32_t)c[lane];
}

__global__ void __launch_bounds__(512) select_kernel(const float* __restrict__ dists, int nlist,
                                                     int nprobe, int negate,
                                                     int32_t* __restrict__ sel) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n2 = pow2_ceil(nprobe + min(kSelChunk, nlist));
  uint64_t* bk = reinterpret_cast<uint64_t*>(smem);
  int32_t* bv = reinterpret_cast<int32_t*>(bk + n2);
  const float* row = dists + (int64_t)blockIdx.x * nlist;
  block_top_p<uint64_t, int32_t>(nlist, nprobe, min(kSelChunk, nlist), bk, bv, ~0ull, 0x7fffffff,
                                 [&](int i, uint64_t& k, int32_t& v) {
                                   const float f = row[i];
                                   k = ((uint64_t)float_key(negate ? -f : f) << 32) | (uint32_t)i;
                                   v = i;
                                 });
  for (int i = threadIdx.x; i < nprobe; i += blockDim.x)
    sel[(int64_t)blockIdx.x * nprobe + i] = bv[i];
}

// Stage 2 for nlist <= 256 * IPT: a stable block radix sort of the 32-bit
// order-preserving keys with the bucket index as value (loaded in index
// order, so equal keys keep ascending buckets: numpy's stable argsort).
template <int IPT>
__global__ void __launch_bounds__(256) select_radix_kernel(const float* __restrict__ dists,
                                                           int nlist, int nprobe, int negate,
                                                           int32_t* __restrict__ sel,
                                                           const int32_t* __restrict__ only,
                                                           int64_t nq) {
  using Sort = cub::BlockRadixSort<uint32_t, 256, IPT, int32_t>;
  __shared__ typename Sort::TempStorage tmp;
  // one query per CTA, or (with `only`) a grid-stride loop over the flagged ones
  for (int64_t qb = blockIdx.x; qb < nq; qb += gridDim.x) {
  if (only && !only[qb]) continue;
  __syncthreads();  // tmp is reused across iterations
  const float* row = dists + qb * nlist;
  uint32_t key[IPT];
  int32_t val[IPT];
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const int i = threadIdx.x * IPT + j;  // blocked arrangement = index order
    const float f = i < nlist ? row[i] : 0.f;
    key[j] = i < nlist ? float_key(negate ? -f : f) : 0xffffffffu;
    val[j] = i;
  }
  Sort(tmp).Sort(key, val);
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const int r = threadIdx.x * IPT + j;
    if (r < nprobe) sel[qb * nprobe + r] = val[j];
  }
  }
}

}  // namespace pdx

using namespace pdx;

extern "C" int pdx_select_buckets(const float* d_queries, int64_t nq, int32_t d,
                                  const float* d_centroids, int32_t nlist, int32_t metric,
                                  int32_t nprobe, float* d_scratch, int32_t* d_sel, void* stream) {
  PDX_REQUIRE(nlist >= 1, "nlist must be >= 1");
  PDX_REQUIRE(nprobe >= 1 && nprobe <= nlist, "nprobe must be in [1, %d], got %d", nlist, nprobe);
  PDX_REQUIRE(nprobe <= 4096, "nprobe %d exceeds this build's limit of 4096", nprobe);
  PDX_REQUIRE(d >= 1, "dimensionality must be >= 1");
  PDX_REQUIRE(metric >= 0 && metric <= 2, "unknown metric");
  PDX_REQUIRE(nq >= 0 && nq < (1ll << 31) * kQT, "bad query count");
  if (nq == 0) return PDX_OK;
  cudaStream_t st = as_stream(stream);
  dim3 grid((nlist + kCT - 1) / kCT, (unsigned)((nq + kQT - 1) / kQT));
  switch (metric) {
    case PDX_METRIC_L2:
      centroid_dist_kernel<PDX_METRIC_L2><<<grid, 256, 0, st>>>(d_queries, nq, d_centroids, nlist, d, d_scratch);
      break;
    case PDX_METRIC_L1:
      centroid_dist_kernel<PDX_METRIC_L1><<<grid, 256, 0, st>>>(d_queries, nq, d_centroids, nlist, d, d_scratch);
      break;
    default:
      centroid_dist_kernel<PDX_METRIC_IP><<<grid, 256, 0, st>>>(d_queries, nq, d_centroids, nlist, d, d_scratch);
  }
  PDX_LAUNCH_CHECK();
  const int neg = metric == PDX_METRIC_IP;
  if (nlist <= 1024 && nprobe <= 32) {
    select_warp_kernel<<<(unsigned)((nq + 7) / 8), 256, 0, st>>>(d_scratch, nq, nlist, nprobe,
                                                                 neg, d_sel);
    PDX_LAUNCH_CHECK();
    return PDX_OK;
  }
  if (nlist <= 256 * 4) {
    select_radix_kernel<4><<<(unsigned)nq, 256, 0, st>>>(d_scratch, nlist, nprobe, neg, d_sel,
                                                         nullptr, nq);
    PDX_LAUNCH_CHECK();
    return PDX_OK;
  }
  if (nlist <= 256 * 8) {
    select_radix_kernel<8><<<(unsigned)nq, 256, 0, st>>>(d_scratch, nlist, nprobe, neg, d_sel,
                                                         nullptr, nq);
    PDX_LAUNCH_CHECK();
    return PDX_OK;
  }
  const int n2 = pow2_ceil(nprobe + (nlist < kSelChunk ? nlist : kSelChunk));
  const size_t smem = (size_t)n2 * (sizeof(uint64_t) + sizeof(int32_t));
  PDX_CUDA_CHECK(cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  select_kernel<<<(unsigned)nq, 512, smem, st>>>(d_scratch, nlist, nprobe, metric == PDX_METRIC_IP, d_sel);
  PDX_LAUNCH_CHECK();
  return PDX_OK;
}
