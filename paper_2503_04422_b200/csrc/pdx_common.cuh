// Shared helpers for the sm_100a PDX kernels (internal; not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "../../include/pdx_b200.h"

namespace pdx {

constexpr int kTile = PDX_TILE;
constexpr int kMaxSteps = 20;  // step_schedule length cap: d <= 65535, initial_step >= 1

// ------------------------------------------------------------ errors (host)
void set_error(const char* fmt, ...);

#define PDX_REQUIRE(cond, ...)        \
  do {                                \
    if (!(cond)) {                    \
      ::pdx::set_error(__VA_ARGS__);  \
      return PDX_EINVAL;              \
    }                                 \
  } while (0)

#define PDX_CUDA_CHECK(expr)                                                        \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      ::pdx::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return PDX_ECUDA;                                                             \
    }                                                                               \
  } while (0)

#define PDX_LAUNCH_CHECK() PDX_CUDA_CHECK(cudaGetLastError())
#define PDX_TRY(expr)              \
  do {                             \
    const int _rc = (expr);        \
    if (_rc != PDX_OK) return _rc; \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------- device helpers
// The reference's vertical kernels (kernels.py:55-61): every float32 op is
// rounded on its own (numpy ufuncs never fuse), so use the _rn intrinsics,
// which nvcc never contracts into FMA.
// Scan-kernel-internal metric tag: squared L2 with the BSA residual bound.
constexpr int kMetricL2Bsa = 3;

template <int METRIC>
__device__ __forceinline__ float upd(float acc, float q, float x) {
  if (METRIC == PDX_METRIC_L2 || METRIC == kMetricL2Bsa) {
    const float t = __fsub_rn(q, x);
    return __fadd_rn(acc, __fmul_rn(t, t));
  } else if (METRIC == PDX_METRIC_L1) {
    return __fadd_rn(acc, fabsf(__fsub_rn(q, x)));
  } else {
    return __fadd_rn(acc, __fmul_rn(q, x));
  }
}

// Order-preserving uint32 image of a float (ascending); -0.0 is folded into
// +0.0 first so that equal floats (numpy's comparison) give equal keys.
__device__ __forceinline__ uint32_t float_key(float f) {
  f = __fadd_rn(f, 0.0f);
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ uint64_t double_key(double f) {
  f = __dadd_rn(f, 0.0);
  uint64_t u = (uint64_t)__double_as_longlong(f);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// (dist, id) lexicographic order of TopK (search.py:45-51).
__device__ __forceinline__ bool pair_less(float d0, int64_t i0, float d1, int64_t i1) {
  return d0 < d1 || (d0 == d1 && i0 < i1);
}

__device__ __forceinline__ float4 ldg4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ float2 ldg2(const float* p) {
  return __ldg(reinterpret_cast<const float2*>(p));
}
// One 256-bit load (LDG.E.ENL2.256): the 8 dims of one slot in a G = 8 tile
// group, a full 32-byte sector.  p must be 32-byte aligned.
__device__ __forceinline__ void ldg8(const float* p, float (&x)[8]) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]),
                 "=f"(x[6]), "=f"(x[7])
               : "l"(p));
}
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

}  // namespace pdx
