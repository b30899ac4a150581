// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (eigmod, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets
// the Python tests, the golden-vector generator and bench.py's CPU-baseline
// leg call the reference's own entry points through ctypes:
//   transform_update          proj/include/eigmod/secular.hpp:28
//   secular_weights           proj/include/eigmod/secular.hpp:34
//   deflate_problem           proj/include/eigmod/secular.hpp:69
//   update_eigenvalues_full   proj/include/eigmod/rootfind.hpp:51-53
//   assemble_eigenvectors     proj/include/eigmod/eigvec.hpp:29-31
//   update_decomposition      proj/include/eigmod/eigvec.hpp:35-36
//   random_instance           proj/include/eigmod/core.hpp:17-20
//   jacobi_evd                proj/include/eigmod/baseline.hpp:15
//   locate (CLI path)         proj/tools/eigmod.cpp:143-161 over locate.hpp:31,50
//   reconstruct/apply_update  proj/include/eigmod/core.hpp:11-14
//   ortho_error               proj/include/eigmod/kernels.hpp:36
//   read/write CSV, Matrix Market   proj/include/eigmod/io.hpp:17-33
// Return codes follow the product C-ABI (include/eigmod_b200.h):
// 0 ok, 1 std::invalid_argument, 2 NumericalError (stage in the message
// buffer as "[stage] msg"), 4 any other exception.
#include <omp.h>

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <optional>
#include <string>
#include <vector>

#include "eigmod/baseline.hpp"
#include "eigmod/core.hpp"
#include "eigmod/eigvec.hpp"
#include "eigmod/io.hpp"
#include "eigmod/kernels.hpp"
#include "eigmod/locate.hpp"
#include "eigmod/rootfind.hpp"
#include "eigmod/secular.hpp"
#include "eigmod/types.hpp"

using namespace eigmod;

namespace {

void put_msg(char* buf, std::size_t len, const std::string& s) {
  if (!buf || len == 0) return;
  std::size_t m = s.size() < len - 1 ? s.size() : len - 1;
  std::memcpy(buf, s.data(), m);
  buf[m] = 0;
}

template <class F>
int guarded(char* msg, std::size_t len, F&& f) {
  try {
    f();
    put_msg(msg, len, "");
    return 0;
  } catch (const NumericalError& e) {
    put_msg(msg, len, e.what());
    return 2;
  } catch (const std::invalid_argument& e) {
    put_msg(msg, len, e.what());
    return 1;
  } catch (const std::exception& e) {
    put_msg(msg, len, e.what());
    return 4;
  }
}

Matrix to_matrix(const double* p, std::int64_t r, std::int64_t c) {
  Matrix m(static_cast<std::size_t>(r), static_cast<std::size_t>(c));
  if (r * c) std::memcpy(m.data(), p, sizeof(double) * r * c);
  return m;
}

SpectralDecomposition to_decomp(const double* q, const double* lambda, std::int64_t n) {
  SpectralDecomposition d;
  d.q = to_matrix(q, n, n);
  d.lambda.assign(lambda, lambda + n);
  return d;
}

LowRankUpdate to_update(const double* kmat, const int* signs, std::int64_t n, std::int64_t k) {
  LowRankUpdate u;
  u.kmat = to_matrix(kmat, n, k);
  u.signs.assign(signs, signs + k);
  return u;
}

TransformedUpdate to_tu(const double* u, const int* signs, std::int64_t n, std::int64_t k) {
  TransformedUpdate tu;
  tu.u = to_matrix(u, n, k);
  tu.signs.assign(signs, signs + k);
  return tu;
}

void copy_vec(const Vec& v, double* out) {
  if (!v.empty()) std::memcpy(out, v.data(), sizeof(double) * v.size());
}

void copy_idx(const std::vector<std::size_t>& v, std::int64_t* out) {
  for (std::size_t i = 0; i < v.size(); ++i) out[i] = static_cast<std::int64_t>(v[i]);
}

// io.hpp: FormatError maps to return code 3.
template <class F>
int io_guarded(char* msg, std::size_t len, F&& f) {
  try {
    f();
    put_msg(msg, len, "");
    return 0;
  } catch (const FormatError& e) {
    put_msg(msg, len, e.what());
    return 3;
  } catch (const std::exception& e) {
    put_msg(msg, len, e.what());
    return 4;
  }
}

}  // namespace

extern "C" {

void ref_set_parallel(int on) { kernels::set_parallel(on != 0); }
int ref_worker_count() { return kernels::worker_count(); }
// OpenMP team size of the reference's parallel paths (torchrun exports
// OMP_NUM_THREADS=1 to every rank; the reference arm wants all host cores)
void ref_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }

int ref_random_instance(std::int64_t n, std::int64_t k, double norm, std::uint64_t seed, double* q,
                        double* lambda, double* kmat, char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    auto [d, u] = random_instance(n, k, norm, seed);
    std::memcpy(q, d.q.data(), sizeof(double) * n * n);
    copy_vec(d.lambda, lambda);
    std::memcpy(kmat, u.kmat.data(), sizeof(double) * n * k);
  });
}

int ref_transform_update(const double* q, const double* lambda, const double* kmat,
                         const int* signs, std::int64_t n, std::int64_t k, double* u_out,
                         char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    const TransformedUpdate tu =
        transform_update(to_decomp(q, lambda, n), to_update(kmat, signs, n, k));
    std::memcpy(u_out, tu.u.data(), sizeof(double) * n * k);
  });
}

int ref_secular_weights(const double* lambda, const double* u, const int* signs, std::int64_t n,
                        std::int64_t k, double* alpha_out, char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    const Vec lam(lambda, lambda + n);
    copy_vec(secular_weights(lam, to_tu(u, signs, n, k)), alpha_out);
  });
}

// Deflation record. Output arrays must hold n entries each; counts are
// written to counts[0..2] = (npoles, nunchanged, ncollided).
int ref_deflate_problem(const double* lambda, const double* u, const int* signs, std::int64_t n,
                        std::int64_t k, double* poles, double* weights, std::int64_t* pole_origin,
                        std::int64_t* unchanged, std::int64_t* collided, std::int64_t* counts,
                        char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    const Vec lam(lambda, lambda + n);
    const DeflatedProblem dp = deflate_problem(lam, to_tu(u, signs, n, k));
    copy_vec(dp.coeffs.poles, poles);
    copy_vec(dp.coeffs.weights, weights);
    copy_idx(dp.pole_origin, pole_origin);
    copy_idx(dp.unchanged, unchanged);
    copy_idx(dp.collided, collided);
    counts[0] = static_cast<std::int64_t>(dp.coeffs.size());
    counts[1] = static_cast<std::int64_t>(dp.unchanged.size());
    counts[2] = static_cast<std::int64_t>(dp.collided.size());
  });
}

// Location vector of the CLI locate path: transform_update is the caller's
// (u given), then deflate_problem and locate_rank2 / locate_rank_k exactly as
// cmd_locate does. counts_out holds n + 1 entries.
int ref_locate_from_u(const double* lambda, const double* u, const int* signs, std::int64_t n,
                      std::int64_t k, std::int64_t* counts_out, std::int64_t* ncounts_out,
                      char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    const Vec lam(lambda, lambda + n);
    const TransformedUpdate tu = to_tu(u, signs, n, k);
    const DeflatedProblem dp = deflate_problem(lam, tu);
    LocationVector loc;
    if (dp.coeffs.size() == 0) {
      loc.counts.assign(1, 0);
    } else if (tu.rank() == 2) {
      loc = locate_rank2(dp.coeffs, classify_shift(tu.signs));
    } else {
      loc = locate_rank_k(dp.coeffs, tu.signs).loc;
    }
    for (std::size_t i = 0; i < loc.counts.size(); ++i) counts_out[i] = loc.counts[i];
    *ncounts_out = static_cast<std::int64_t>(loc.counts.size());
  });
}

// locate_rank2 / locate_rank_k (locate.hpp:31,50) on given coefficients
// (rank2 when signs has two entries, with classify_shift).
int ref_locate_coeffs(const double* poles, const double* weights, std::int64_t m,
                      const int* signs, std::int64_t k, std::int64_t* counts_out, char* msg,
                      std::size_t len) {
  return guarded(msg, len, [&] {
    const SecularCoefficients c = make_secular(Vec(poles, poles + m), Vec(weights, weights + m));
    const std::vector<int> sg(signs, signs + k);
    const LocationVector loc = k == 2 ? locate_rank2(c, classify_shift(sg)) : locate_rank_k(c, sg).loc;
    for (std::size_t i = 0; i < loc.counts.size(); ++i) counts_out[i] = loc.counts[i];
  });
}

// crossing_count (secular.hpp:48), solve_rank1 (rootfind.hpp:33),
// null_problem / null_direction / update_eigenvector (eigvec.hpp:15-26).
int ref_crossing_count(const double* poles, const double* weights, std::int64_t m, double lo,
                       double hi, int samples, std::int64_t* out, char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    const SecularCoefficients c = make_secular(Vec(poles, poles + m), Vec(weights, weights + m));
    *out = crossing_count(c, lo, hi, samples);
  });
}

int ref_solve_rank1(const double* poles, const double* zeta, std::int64_t n, double sigma,
                    double tol, double* roots_out, char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    copy_vec(solve_rank1(Vec(poles, poles + n), Vec(zeta, zeta + n), sigma, tol), roots_out);
  });
}

int ref_null_problem(const double* u, const int* signs, const double* lambda, std::int64_t n,
                     std::int64_t k, double lambda_new, double* m_out, char* msg,
                     std::size_t len) {
  return guarded(msg, len, [&] {
    const Matrix m = null_problem(to_tu(u, signs, n, k), Vec(lambda, lambda + n), lambda_new);
    std::memcpy(m_out, m.data(), sizeof(double) * k * k);
  });
}

int ref_null_direction(const double* m, std::int64_t k, double* dir_out, double* resid_out,
                       char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    const NullDirection nd = null_direction(to_matrix(m, k, k));
    copy_vec(nd.direction, dir_out);
    *resid_out = nd.residual;
  });
}

int ref_update_eigenvector(const double* q, const double* lambda, const double* kmat,
                           const int* signs, std::int64_t n, std::int64_t k, double lambda_new,
                           double* v_out, char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    copy_vec(update_eigenvector(to_decomp(q, lambda, n), to_update(kmat, signs, n, k), lambda_new),
             v_out);
  });
}

// core.hpp:11 reconstruct (Q diag(lambda) Q^T, symmetrized) and core.hpp:14
// apply_update (a + sum_r s_r k_r k_r^T, symmetrized); kernels.hpp:36
// ortho_error (max |A^T A - I|).
int ref_reconstruct(const double* q, const double* lambda, std::int64_t n, double* out,
                    char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    const SymmetricDense a = reconstruct(to_decomp(q, lambda, n));
    std::memcpy(out, a.entries.data(), sizeof(double) * n * n);
  });
}

int ref_apply_update(const double* a, const double* kmat, const int* signs, std::int64_t n,
                     std::int64_t k, double* out, char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    SymmetricDense s;
    s.n = static_cast<std::size_t>(n);
    s.entries = to_matrix(a, n, n);
    const SymmetricDense r = apply_update(s, to_update(kmat, signs, n, k));
    std::memcpy(out, r.entries.data(), sizeof(double) * n * n);
  });
}

double ref_ortho_error(const double* a, std::int64_t rows, std::int64_t cols) {
  return kernels::ortho_error(to_matrix(a, rows, cols));
}

int ref_write_csv(const char* path, const double* m, std::int64_t rows, std::int64_t cols,
                  const int* signs, std::int64_t nsigns, char* msg, std::size_t len) {
  return io_guarded(msg, len, [&] {
    std::optional<std::vector<int>> s;
    if (signs) s = std::vector<int>(signs, signs + nsigns);
    write_csv_matrix(path, to_matrix(m, rows, cols), s);
  });
}

// shape_out = (rows, cols, nsigns); values_out / signs_out sized by the caller
// (call once with null buffers to get the shape).
int ref_read_csv(const char* path, std::int64_t* shape_out, double* values_out, int* signs_out,
                 char* msg, std::size_t len) {
  return io_guarded(msg, len, [&] {
    const CsvMatrix c = read_csv_matrix(path);
    shape_out[0] = static_cast<std::int64_t>(c.values.rows());
    shape_out[1] = static_cast<std::int64_t>(c.values.cols());
    shape_out[2] = c.signs ? static_cast<std::int64_t>(c.signs->size()) : -1;
    if (values_out && c.values.rows() * c.values.cols())
      std::memcpy(values_out, c.values.data(), sizeof(double) * c.values.rows() * c.values.cols());
    if (signs_out && c.signs)
      for (std::size_t i = 0; i < c.signs->size(); ++i) signs_out[i] = (*c.signs)[i];
  });
}

int ref_write_mm(const char* path, const double* a, std::int64_t n, char* msg, std::size_t len) {
  return io_guarded(msg, len, [&] {
    write_matrix_market(path, SymmetricDense::from(to_matrix(a, n, n)));
  });
}

int ref_read_mm(const char* path, std::int64_t* n_out, double* a_out, char* msg, std::size_t len) {
  return io_guarded(msg, len, [&] {
    const SymmetricDense s = read_matrix_market(path);
    *n_out = static_cast<std::int64_t>(s.n);
    if (a_out) std::memcpy(a_out, s.entries.data(), sizeof(double) * s.n * s.n);
  });
}

double ref_default_tolerance(const double* lambda, const double* kmat, const int* signs,
                             std::int64_t n, std::int64_t k) {
  const Vec lam(lambda, lambda + n);
  return default_tolerance(lam, to_update(kmat, signs, n, k));
}

// Eigenvalue stage. values_out (n), roots_out (n), nroots_out (1).
// stage_seconds receives the wall time of the call.
int ref_update_eigenvalues_full(const double* q, const double* lambda, const double* kmat,
                                const int* signs, std::int64_t n, std::int64_t k, double tol,
                                int strategy, double* values_out, double* roots_out,
                                std::int64_t* nroots_out, double* stage_seconds, char* msg,
                                std::size_t len) {
  return guarded(msg, len, [&] {
    const auto d = to_decomp(q, lambda, n);
    const auto u = to_update(kmat, signs, n, k);
    const auto t0 = std::chrono::steady_clock::now();
    const EigenvalueUpdate plan = update_eigenvalues_full(
        d, u, tol, strategy ? LocateStrategy::sturm : LocateStrategy::automatic);
    const auto t1 = std::chrono::steady_clock::now();
    if (stage_seconds) *stage_seconds = std::chrono::duration<double>(t1 - t0).count();
    copy_vec(plan.values, values_out);
    copy_vec(plan.roots, roots_out);
    *nroots_out = static_cast<std::int64_t>(plan.roots.size());
  });
}

// Both stages, timed separately (the bench.cpp:188-222 split):
// stage_seconds[0] = update_eigenvalues_full, [1] = assemble_eigenvectors.
int ref_update_pairs(const double* q, const double* lambda, const double* kmat, const int* signs,
                     std::int64_t n, std::int64_t k, double tol, int reorthogonalize,
                     double* lambda_out, double* q_out, double* stage_seconds, char* msg,
                     std::size_t len) {
  return guarded(msg, len, [&] {
    const auto d = to_decomp(q, lambda, n);
    const auto u = to_update(kmat, signs, n, k);
    const auto t0 = std::chrono::steady_clock::now();
    const EigenvalueUpdate plan = update_eigenvalues_full(d, u, tol);
    const auto t1 = std::chrono::steady_clock::now();
    const SpectralDecomposition out = assemble_eigenvectors(d, plan, reorthogonalize != 0);
    const auto t2 = std::chrono::steady_clock::now();
    if (stage_seconds) {
      stage_seconds[0] = std::chrono::duration<double>(t1 - t0).count();
      stage_seconds[1] = std::chrono::duration<double>(t2 - t1).count();
    }
    copy_vec(out.lambda, lambda_out);
    std::memcpy(q_out, out.q.data(), sizeof(double) * n * n);
  });
}

// BASELINE.md §3 timing of the two stages with the failure record: out3[0]
// seconds of update_eigenvalues_full, out3[1] of assemble_eigenvectors,
// out3[2] the stage that threw (0 none, 1 eigenvalues, 2 eigenvectors); the
// time of a failing stage is its time to failure. q_out may be null (the
// eigenvalue stage only).
int ref_timed_pairs(const double* q, const double* lambda, const double* kmat, const int* signs,
                    std::int64_t n, std::int64_t k, double tol, double* lambda_out, double* q_out,
                    double* out3, char* msg, std::size_t len) {
  out3[0] = out3[1] = out3[2] = 0.0;
  return guarded(msg, len, [&] {
    const auto d = to_decomp(q, lambda, n);
    const auto u = to_update(kmat, signs, n, k);
    auto t0 = std::chrono::steady_clock::now();
    auto since = [&] {
      return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    std::optional<EigenvalueUpdate> plan;
    try {
      plan.emplace(update_eigenvalues_full(d, u, tol));
    } catch (...) {
      out3[0] = since();
      out3[2] = 1.0;
      throw;
    }
    out3[0] = since();
    copy_vec(plan->values, lambda_out);
    if (!q_out) return;
    t0 = std::chrono::steady_clock::now();
    try {
      const SpectralDecomposition out = assemble_eigenvectors(d, *plan, false);
      out3[1] = since();
      copy_vec(out.lambda, lambda_out);
      std::memcpy(q_out, out.q.data(), sizeof(double) * n * n);
    } catch (...) {
      out3[1] = since();
      out3[2] = 2.0;
      throw;
    }
  });
}

// Full update with the reference's own metrics (residual_fro, ortho_err,
// wall_time) in metrics[0..2].
int ref_update_decomposition(const double* q, const double* lambda, const double* kmat,
                             const int* signs, std::int64_t n, std::int64_t k, double tol,
                             int reorthogonalize, double* lambda_out, double* q_out,
                             double* metrics, char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    const UpdateResult r = update_decomposition(to_decomp(q, lambda, n),
                                                to_update(kmat, signs, n, k), tol,
                                                reorthogonalize != 0);
    copy_vec(r.decomposition.lambda, lambda_out);
    std::memcpy(q_out, r.decomposition.q.data(), sizeof(double) * n * n);
    metrics[0] = r.residual_fro;
    metrics[1] = r.ortho_err;
    metrics[2] = r.wall_time;
  });
}

// Eigenvalues of the symmetric matrix a (n x n) by the reference's Jacobi
// oracle (ascending).
int ref_jacobi_eigenvalues(const double* a, std::int64_t n, double* out, char* msg,
                           std::size_t len) {
  return guarded(msg, len, [&] {
    const SymmetricDense s = SymmetricDense::from(to_matrix(a, n, n));
    copy_vec(jacobi_evd(s).lambda, out);
  });
}

// Secular function of the deflated problem (secular.hpp:44-47).
int ref_eval_secular(const double* poles, const double* weights, std::int64_t m, double leading,
                     double x, double* f_out, char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    const SecularCoefficients c =
        make_secular(Vec(poles, poles + m), Vec(weights, weights + m), leading);
    *f_out = eval_secular(c, x);
  });
}

}  // extern "C"

// ---- handles for sampling the reference's per-eigenpair work at full size
// (bench.py --impl reference): the reference's own kernels on persistent
// operands, so each timed step only pays for the sampled work.
extern "C" {

void* ref_matrix_new(const double* data, std::int64_t rows, std::int64_t cols) {
  return new Matrix(to_matrix(data, rows, cols));
}
void ref_matrix_free(void* h) { delete static_cast<Matrix*>(h); }
// rows x cols filled with v (a timing operand: the i-l-j kernel's cost does
// not depend on the values)
void* ref_matrix_const(std::int64_t rows, std::int64_t cols, double v) {
  return new Matrix(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols), v);
}

// C = A * B with the reference's back-transform kernel (kernels.cpp:32-48,
// called at eigvec.cpp:339). b: A.cols() x bcols, c_out: A.rows() x bcols.
int ref_gemm_nn(void* a, const double* b, std::int64_t bcols, double* c_out, char* msg,
                std::size_t len) {
  return guarded(msg, len, [&] {
    const Matrix& A = *static_cast<Matrix*>(a);
    const Matrix B = to_matrix(b, static_cast<std::int64_t>(A.cols()), bcols);
    const Matrix Cm = kernels::gemm_nn(A, B);
    std::memcpy(c_out, Cm.data(), sizeof(double) * Cm.rows() * Cm.cols());
  });
}

// Same kernel with both operands persistent (no per-call copy of B): the
// sampled rows of Q' = Q X against the full n x n X (bench.py).
int ref_gemm_nn_hh(void* a, void* b, double* c_out, char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    const Matrix Cm = kernels::gemm_nn(*static_cast<Matrix*>(a), *static_cast<Matrix*>(b));
    std::memcpy(c_out, Cm.data(), sizeof(double) * Cm.rows() * Cm.cols());
  });
}

void* ref_tu_new(const double* u, const int* signs, std::int64_t n, std::int64_t k) {
  return new TransformedUpdate(to_tu(u, signs, n, k));
}
void ref_tu_free(void* h) { delete static_cast<TransformedUpdate*>(h); }

// One eigenvector of the reference's assembly (eigvec.cpp:133-153): the
// null problem M(root) (eigvec.cpp:187-202), its null direction
// (eigvec.cpp:157-185) and the resolvent w_s = (U beta)_s / (lambda_s - root).
int ref_basis_vector(void* tu_h, const double* lambda, std::int64_t n, double root, double* w_out,
                     double* resid_out, char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    const TransformedUpdate& tu = *static_cast<TransformedUpdate*>(tu_h);
    const Vec lam(lambda, lambda + n);
    const Matrix m = null_problem(tu, lam, root);
    const NullDirection nd = null_direction(m);
    const std::size_t k = tu.rank();
    double norm2 = 0.0;
    for (std::int64_t s = 0; s < n; ++s) {
      double ub = 0.0;
      for (std::size_t r = 0; r < k; ++r) ub += tu.u(s, r) * nd.direction[r];
      w_out[s] = ub / (lambda[s] - root);
      norm2 += w_out[s] * w_out[s];
    }
    const double inv = 1.0 / std::sqrt(norm2);
    for (std::int64_t s = 0; s < n; ++s) w_out[s] *= inv;
    *resid_out = nd.residual;
  });
}

// The reference's bracket solver (rootfind.hpp:35-36 / rootfind.cpp:89-229)
// on its secular function with the given poles and weights.
int ref_dnc_solve(const double* poles, const double* weights, std::int64_t m, double lo, double hi,
                  std::int64_t expected, double tol, double* roots_out, std::int64_t* nroots,
                  char* msg, std::size_t len) {
  return guarded(msg, len, [&] {
    const SecularCoefficients c = make_secular(Vec(poles, poles + m), Vec(weights, weights + m), 1.0);
    const Vec r = dnc_solve(c, RootBracket{lo, hi, static_cast<long>(expected)}, tol);
    copy_vec(r, roots_out);
    *nroots = static_cast<std::int64_t>(r.size());
  });
}

}  // extern "C"
