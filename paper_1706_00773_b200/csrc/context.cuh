// The device context behind the C ABI (include/eigmod_b200.h) and the host
// helpers shared by the entry points in capi.cu, eigpair.cu and multi.cu.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/eigmod_b200.h"
#include "pipeline.cuh"

using eigb::Error;

struct eigmod_b200_ctx {
  int device = 0;
  cudaStream_t own = nullptr, stream = nullptr;
  int sms = 148;
  eigb::DeviceScratch ws;
  eigb::Plan plan;
  bool have_plan = false;
  eigb::RootRecords recs{};
  double run_rel = eigb::kExactRunRelGap;
  eigb::SolveOptions sopt;
  const double* lam = nullptr;  // the plan's own copy of lambda (workspace "plan_lam")
  cudaStream_t copy = nullptr;   // D2H stream of the blocked host path
  std::vector<cudaEvent_t> blk_ev;
  std::string err, stage;
  // per-stage CUDA-event timing (option "timing"): 0 K1 project, 1 K2 plan,
  // 2 K3 solve, 3 K4 columns, 4 K5 GEMM, 5 sign rule
  // assemble_eigenvectors reuses the plan and root records of the last
  // update_eigenvalues call when the caller hands back that call's plan
  // (same lambda, U, signs and roots): plan_key hashes those inputs.
  uint64_t plan_key = 0;
  bool plan_key_valid = false;
  std::vector<double> plan_roots;  // the secular roots (ascending) of the cached plan
  // stage launches (K1 projections, K2 plans, K3 solves, K4/K5 column builds)
  int64_t stage_calls[4] = {0, 0, 0, 0};
  bool timing = false;
  // option "compact_gemm": back-transform over the reduced rows when the plan
  // has decoupled columns (capi.cu finish_compact)
  bool compact_gemm = true;
  cudaEvent_t ev[8] = {};
  double stage_ms[8] = {};
  int64_t timed_calls = 0;
  void mark(int i) {
    if (!timing) return;
    if (!ev[i]) EIGB_CUDA(cudaEventCreate(&ev[i]));
    EIGB_CUDA(cudaEventRecord(ev[i], stream));
  }
  // staged entry points: add stages [i0, i1) once their end mark completed
  void accumulate(int i0, int i1) {
    if (!timing || !ev[i1]) return;
    EIGB_CUDA(cudaEventSynchronize(ev[i1]));
    for (int i = i0; i < i1; ++i) {
      float ms = 0.f;
      if (ev[i] && cudaEventElapsedTime(&ms, ev[i], ev[i + 1]) == cudaSuccess) stage_ms[i] += ms;
    }
  }
};

namespace eigb_capi {

inline void check_basic(int64_t n, int64_t k, const int* signs) {
  // proj/src/core.cpp:89-97 (validate_update)
  if (n < 1) throw Error(1, "", "LowRankUpdate: dimension mismatch");
  if (k < 1 || k > n) throw Error(1, "", "LowRankUpdate: rank out of range");
  if (k > eigb::kMaxRank) throw Error(1, "", "LowRankUpdate: rank above 32 is not supported");
  if (signs)
    for (int64_t r = 0; r < k; ++r)
      if (signs[r] != 1 && signs[r] != -1)
        throw Error(1, "", "LowRankUpdate: signs must be +1/-1");
}

inline void check_finite(const double* p, int64_t cnt, const char* what) {
  for (int64_t i = 0; i < cnt; ++i)
    if (!std::isfinite(p[i])) throw Error(1, "", std::string("LowRankUpdate: non-finite ") + what);
}

inline void check_ascending(const double* lam, int64_t n) {
  // proj/src/secular.cpp:281-283, surfaced as NumericalError("deflate")
  for (int64_t i = 0; i + 1 < n; ++i)
    if (!(lam[i] <= lam[i + 1]))
      throw Error(2, "deflate", "deflate_problem: eigenvalues not ascending");
}

inline void check_ascending_invalid(const double* lam, int64_t n) {
  // proj/src/secular.cpp:281-283 called directly (the CLI locate path)
  for (int64_t i = 0; i + 1 < n; ++i)
    if (!(lam[i] <= lam[i + 1]))
      throw Error(1, "", "deflate_problem: eigenvalues not ascending");
}

// FNV-1a over the bytes of the eigenvalue stage's inputs (the plan key)
struct Fnv {
  uint64_t h = 1469598103934665603ull;
  void add(const void* p, size_t bytes) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < bytes; ++i) h = (h ^ b[i]) * 1099511628211ull;
  }
  template <class T>
  void add_value(T v) { add(&v, sizeof(v)); }
};

inline uint64_t plan_key_of(const double* lambda, const double* u, const int* signs, int64_t n,
                     int64_t k) {
  Fnv f;
  f.add_value(n);
  f.add_value(k);
  f.add(lambda, 8 * (size_t)n);
  if (k > 0) {
    f.add(u, 8 * (size_t)n * (size_t)k);
    f.add(signs, 4 * (size_t)k);
  }
  return f.h;
}

template <class F>
int guarded(eigmod_b200_ctx* ctx, F&& f) {
  if (!ctx) return EIGMOD_B200_INVALID_ARGUMENT;
  try {
    EIGB_CUDA(cudaSetDevice(ctx->device));
    f();
    ctx->err.clear();
    ctx->stage.clear();
    return EIGMOD_B200_OK;
  } catch (const Error& e) {
    ctx->err = e.what();
    ctx->stage = e.stage;
    if (e.code == EIGMOD_B200_CUDA) (void)cudaGetLastError();  // clear a non-sticky error
    return e.code;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    ctx->stage = "cuda";
    (void)cudaGetLastError();  // a non-sticky error must not poison the next call
    return EIGMOD_B200_CUDA;
  }
}

// pipeline stages on one context (capi.cu)
void project(eigmod_b200_ctx* c, const double* q, const double* kmat, int64_t n, int64_t k,
             int64_t lo, int64_t hi, double* u_out);
void plan_groups(eigmod_b200_ctx* c, const double* lam, const double* u, const int* signs,
                 int64_t n, int64_t k, double run_rel, bool spec = false);
void plan_from_u(eigmod_b200_ctx* c, const double* lam, const double* u, const int* signs,
                 int64_t n, int64_t k, double run_rel, bool fuse = false);
void solve(eigmod_b200_ctx* c, int64_t j0, int64_t j1);
// root records of [j0, j0 + cnt) packed as eigmod_b200_record_width(kp)
// doubles each (the all-gather payload), and all records back from it
void pack_records_dev(eigmod_b200_ctx* c, int64_t j0, int64_t cnt, double* out);
void unpack_records_dev(eigmod_b200_ctx* c, const double* in, int64_t cnt);
void finish(eigmod_b200_ctx* c, const double* q, const double* lam_in, int64_t c0, int64_t c1,
            double* lam_out, double* q_out, int64_t ldq, double* host_q_out = nullptr,
            int64_t host_ld = 0);

}  // namespace eigb_capi
