// Shared definitions for the sm_100a eigen-update kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace eigb {

// Error carried from the device layer to the C-ABI (include/eigmod_b200.h):
// code 1 = invalid argument, 2 = numerical (stage set), 3 = CUDA failure.
struct Error : std::runtime_error {
  int code;
  std::string stage;
  Error(int c, std::string st, const std::string& msg)
      : std::runtime_error(st.empty() ? msg : "[" + st + "] " + msg), code(c), stage(std::move(st)) {}
};

#define EIGB_CUDA(x)                                                                         \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess)                                                                   \
      throw ::eigb::Error(3, "cuda", std::string(#x) + ": " + cudaGetErrorString(e_));       \
  } while (0)

void note_launch();
#define EIGB_LAUNCH_CHECK()          \
  do {                               \
    EIGB_CUDA(cudaGetLastError());   \
    ::eigb::note_launch();           \
  } while (0)

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Padded rank used by the templated kernels: the smallest of {1,2,4,8,16,32}
// >= k. Padding columns of U are zero with sign +1, which adds a decoupled +1
// to S(x) and changes neither the inertia count nor the null vector.
inline int padded_rank(int64_t k) {
  int p = 1;
  while (p < k) p <<= 1;
  return p;
}
constexpr int kMaxRank = 32;

// Relative thresholds of the reference (proj/include/eigmod/secular.hpp:66-67,
// proj/src/secular.cpp:306-330, proj/src/rootfind.cpp:328).
constexpr double kPoleMergeRelGap = 1e-12;
constexpr double kWeightDeflationRel = 1e-14;
constexpr double kRowMassRel = 1e-12;
constexpr double kColumnDropRel = 1e-15;
// exact mode (the solve): rows coupling below this fraction of the problem
// scale decouple unchanged
constexpr double kExactCouplingRel = 1e-13;
// Exact-mode run threshold (near-equal poles are merged and
// Householder-compressed when closer than this, relative to max(1,|lambda|)).
constexpr double kExactRunRelGap = 1e-10;

}  // namespace eigb

// ------------------------------------------------------------------ device side
#ifdef __CUDACC__
namespace eigb {

// FP64 reciprocal: MUFU.RCP64H seed + two Newton steps (relative error
// ~1 ulp, not correctly rounded). x must be finite and nonzero.
__device__ __forceinline__ double rcp64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// One Newton step only (relative error ~1e-13): for the scalar presolve,
// whose root is a start refined by the S solver (stops at 1e-6 |delta|).
__device__ __forceinline__ double rcp64_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__host__ __device__ __forceinline__ int64_t cdiv_dev(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Number of entries < x / <= x in an ascending array (binary search).
__device__ __forceinline__ int64_t dev_n_less(const double* d, int64_t n, double x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t m = (lo + hi) >> 1;
    if (d[m] < x) lo = m + 1; else hi = m;
  }
  return lo;
}
__device__ __forceinline__ int64_t dev_n_leq(const double* d, int64_t n, double x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t m = (lo + hi) >> 1;
    if (d[m] <= x) lo = m + 1; else hi = m;
  }
  return lo;
}

// The same within a known window: the count lies in [a, b] (every d[i < a]
// is below x, every d[i >= b] above it), so only log2(b - a) probes.
__device__ __forceinline__ int64_t dev_n_less_in(const double* d, int64_t a, int64_t b, double x) {
  while (a < b) {
    const int64_t m = (a + b) >> 1;
    if (d[m] < x) a = m + 1; else b = m;
  }
  return a;
}
__device__ __forceinline__ int64_t dev_n_leq_in(const double* d, int64_t a, int64_t b, double x) {
  while (a < b) {
    const int64_t m = (a + b) >> 1;
    if (d[m] <= x) a = m + 1; else b = m;
  }
  return a;
}

}  // namespace eigb
#endif
