// The reference's C++ API (namespace eigmod) over the B200 C ABI.
//
// Each function keeps the reference's declaration (include/eigmod_b200/
// eigmod.hpp, mirroring proj/include/eigmod/*.hpp) and error behaviour:
// preconditions throw std::invalid_argument, numerical failures throw
// eigmod::NumericalError with the reference's stage names, device failures
// throw std::runtime_error. The heavy work runs in libeigmod_b200.so on the
// GPU; this file only marshals std::vector-backed values and the O(n) / O(nk)
// utilities the reference exposes next to the hot path.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <limits>
#include <memory>
#include <mutex>

#include "eigmod_b200.h"
#include "eigmod_b200/eigmod.hpp"

namespace eigmod {

namespace {

// One context per host thread (contexts must not be used concurrently).
eigmod_b200_ctx* ctx() {
  thread_local std::unique_ptr<eigmod_b200_ctx, void (*)(eigmod_b200_ctx*)> c(
      nullptr, eigmod_b200_ctx_destroy);
  if (!c) {
    eigmod_b200_ctx* p = nullptr;
    const int rc = eigmod_b200_ctx_create(0, &p);
    if (rc != EIGMOD_B200_OK)
      throw std::runtime_error("eigmod (B200): no usable sm_100 device (rc " + std::to_string(rc) +
                               ")");
    c.reset(p);
  }
  return c.get();
}

// The multi-GPU context of set_devices / EIGMOD_B200_DEVICES (process-wide,
// one update at a time).
struct MultiState {
  std::mutex mu;
  bool env_read = false;
  std::vector<int> devices;
  eigmod_b200_multi* mg = nullptr;
};
MultiState& multi_state() {
  static MultiState s;
  return s;
}

std::vector<int> parse_device_list(const char* s) {
  std::vector<int> out;
  if (!s) return out;
  std::string cur;
  for (const char* p = s;; ++p) {
    if (*p == ',' || *p == '\0') {
      if (!cur.empty()) out.push_back(std::stoi(cur));
      cur.clear();
      if (!*p) break;
    } else if (*p != ' ') {
      cur.push_back(*p);
    }
  }
  return out;
}

// Locked multi context when devices are configured, else null.
eigmod_b200_multi* multi(std::unique_lock<std::mutex>& lock) {
  MultiState& s = multi_state();
  lock = std::unique_lock<std::mutex>(s.mu);
  if (!s.env_read) {
    s.env_read = true;
    if (s.devices.empty()) s.devices = parse_device_list(std::getenv("EIGMOD_B200_DEVICES"));
  }
  if (s.devices.empty()) return nullptr;
  if (!s.mg) {
    const int rc = eigmod_b200_multi_create(s.devices.data(), (int)s.devices.size(), &s.mg);
    if (rc != EIGMOD_B200_OK) {
      s.mg = nullptr;
      if (rc == EIGMOD_B200_INVALID_ARGUMENT)
        throw std::invalid_argument("set_devices: invalid device list");
      throw std::runtime_error("eigmod (B200): multi-GPU context failed (rc " +
                               std::to_string(rc) + ")");
    }
  }
  return s.mg;
}

void check_multi(eigmod_b200_multi* mg, int rc) {
  if (rc == EIGMOD_B200_OK) return;
  const std::string msg = eigmod_b200_multi_last_error(mg);
  const std::string stage = eigmod_b200_multi_last_stage(mg);
  if (rc == EIGMOD_B200_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == EIGMOD_B200_NUMERICAL) {
    std::string body = msg;
    const std::string pre = "[" + stage + "] ";
    const size_t at = body.find(pre);
    if (at != std::string::npos) body = body.substr(at + pre.size());
    throw NumericalError(stage, body);
  }
  throw std::runtime_error(msg);
}

void check(int rc) {
  if (rc == EIGMOD_B200_OK) return;
  eigmod_b200_ctx* c = ctx();
  const std::string msg = eigmod_b200_last_error(c);
  const std::string stage = eigmod_b200_last_stage(c);
  if (rc == EIGMOD_B200_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == EIGMOD_B200_NUMERICAL) {
    // strip the "[stage] " prefix the device layer adds
    std::string body = msg;
    const std::string pre = "[" + stage + "] ";
    if (body.rfind(pre, 0) == 0) body = body.substr(pre.size());
    throw NumericalError(stage, body);
  }
  throw std::runtime_error(msg);
}

bool all_finite(const Matrix& m) {
  const double* p = m.data();
  for (std::size_t i = 0; i < m.rows() * m.cols(); ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}

void require_increasing(const Vec& poles, const char* who) {
  for (std::size_t i = 0; i + 1 < poles.size(); ++i)
    if (!(poles[i] < poles[i + 1]))
      throw std::invalid_argument(std::string(who) + ": poles not strictly increasing");
  for (double p : poles)
    if (!std::isfinite(p)) throw std::invalid_argument(std::string(who) + ": non-finite pole");
}

Matrix symmetrized(Matrix a) {
  const std::size_t n = a.rows();
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = i + 1; j < n; ++j) {
      const double s = 0.5 * (a(i, j) + a(j, i));
      a(i, j) = s;
      a(j, i) = s;
    }
  return a;
}

}  // namespace

SymmetricDense SymmetricDense::from(const Matrix& m) {
  if (m.rows() != m.cols()) throw std::invalid_argument("SymmetricDense: matrix not square");
  if (!all_finite(m)) throw std::invalid_argument("SymmetricDense: non-finite entries");
  SymmetricDense s;
  s.n = m.rows();
  s.entries = symmetrized(m);
  return s;
}

void validate_decomposition(const SpectralDecomposition& d, double max_ortho_err) {
  if (d.q.rows() != d.q.cols() || d.q.rows() != d.lambda.size())
    throw std::invalid_argument("SpectralDecomposition: inconsistent dimensions");
  if (!all_finite(d.q)) throw std::invalid_argument("SpectralDecomposition: non-finite Q");
  for (std::size_t i = 0; i + 1 < d.lambda.size(); ++i)
    if (!(d.lambda[i] <= d.lambda[i + 1]))
      throw std::invalid_argument("SpectralDecomposition: eigenvalues not ascending");
  const double err = kernels::ortho_error(d.q);
  if (err > max_ortho_err)
    throw std::invalid_argument("SpectralDecomposition: orthonormality error " +
                                std::to_string(err));
}

void validate_update(const SpectralDecomposition& d, const LowRankUpdate& u) {
  // proj/src/core.cpp:89-97
  if (u.dim() != d.size()) throw std::invalid_argument("LowRankUpdate: dimension mismatch");
  if (u.rank() < 1 || u.rank() > u.dim())
    throw std::invalid_argument("LowRankUpdate: rank out of range");
  if (u.signs.size() != u.rank()) throw std::invalid_argument("LowRankUpdate: signs size");
  for (int s : u.signs)
    if (s != 1 && s != -1) throw std::invalid_argument("LowRankUpdate: signs must be +1/-1");
  if (!all_finite(u.kmat)) throw std::invalid_argument("LowRankUpdate: non-finite K");
}

// core.hpp:11 — Q diag(lambda) Q^T on the DMMA GEMM, symmetrized on the GPU.
SymmetricDense reconstruct(const SpectralDecomposition& d) {
  if (d.q.cols() != d.lambda.size()) throw std::invalid_argument("reconstruct: dimension mismatch");
  const std::size_t n = d.q.rows(), k = d.q.cols();
  SymmetricDense s;
  s.n = n;
  s.entries = Matrix(n, n);
  if (n == 0) return s;
  if (k == n) {
    check(eigmod_b200_reconstruct(ctx(), d.q.data(), d.lambda.data(), (int64_t)n,
                                  s.entries.data()));
  } else {  // rectangular Q (kernels.cpp:98-109 accepts n x k)
    Matrix w(n, k);
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t j = 0; j < k; ++j) w(i, j) = d.q(i, j) * d.lambda[j];
    check(eigmod_b200_gemm_nt(ctx(), w.data(), d.q.data(), n, n, k, s.entries.data()));
    s.entries = symmetrized(s.entries);
  }
  if (!all_finite(s.entries)) throw std::invalid_argument("SymmetricDense: non-finite entries");
  return s;
}

// core.hpp:14 — a + sum_r s_r k_r k_r^T, symmetrized; bit-identical to the
// reference (GPU, reference rounding sequence).
SymmetricDense apply_update(const SymmetricDense& a, const LowRankUpdate& u) {
  if (u.dim() != a.n) throw std::invalid_argument("apply_update: dimension mismatch");
  if (u.signs.size() != u.rank()) throw std::invalid_argument("apply_update: signs size");
  if (u.rank() == 0 || a.n == 0) return SymmetricDense::from(a.entries);
  SymmetricDense s;
  s.n = a.n;
  s.entries = Matrix(a.n, a.n);
  check(eigmod_b200_apply_update(ctx(), a.entries.data(), u.kmat.data(), u.signs.data(),
                                 (int64_t)a.n, (int64_t)u.rank(), s.entries.data()));
  if (!all_finite(s.entries)) throw std::invalid_argument("SymmetricDense: non-finite entries");
  return s;
}

// locate.hpp:13-50 host utilities and the GPU location vector of the CLI
// locate path (tools/eigmod.cpp:143-161).
ShiftKind classify_shift(const std::vector<int>& signs) {
  if (signs.size() != 2) throw std::invalid_argument("classify_shift: rank-2 signature required");
  if (signs[0] > 0 && signs[1] > 0) return ShiftKind::double_right;
  if (signs[0] < 0 && signs[1] < 0) return ShiftKind::double_left;
  return ShiftKind::mixed;
}

std::pair<double, double> interlacing_bounds(std::size_t index, const Vec& lambda,
                                             std::size_t rank, const std::vector<int>& signs) {
  const std::size_t n = lambda.size();
  if (index < 1 || index > n) throw std::invalid_argument("interlacing_bounds: index out of range");
  if (signs.size() != rank || rank < 1)
    throw std::invalid_argument("interlacing_bounds: bad signature");
  std::size_t plus = 0, minus = 0;
  for (int sg : signs) (sg > 0 ? plus : minus)++;
  const double inf = std::numeric_limits<double>::infinity();
  return {index > minus ? lambda[index - minus - 1] : -inf,
          index + plus <= n ? lambda[index + plus - 1] : inf};
}

LocationVector locate_update(const SpectralDecomposition& d, const LowRankUpdate& u) {
  validate_update(d, u);
  const std::size_t n = d.size();
  std::vector<int64_t> c(n + 1);
  int64_t nc = 0;
  check(eigmod_b200_locate(ctx(), d.q.data(), d.lambda.data(), u.kmat.data(), u.signs.data(),
                           (int64_t)n, (int64_t)u.rank(), c.data(), &nc));
  LocationVector loc;
  loc.counts.assign(c.begin(), c.begin() + nc);
  return loc;
}

SecularCoefficients make_secular(Vec poles, Vec weights, double leading) {
  // proj/src/secular.cpp:136-153
  if (poles.size() != weights.size())
    throw std::invalid_argument("make_secular: poles/weights size mismatch");
  require_increasing(poles, "make_secular");
  for (double w : weights)
    if (!std::isfinite(w)) throw std::invalid_argument("make_secular: non-finite weight");
  if (!std::isfinite(leading)) throw std::invalid_argument("make_secular: non-finite leading");
  SecularCoefficients c;
  c.leading = leading;
  for (std::size_t i = 0; i < poles.size(); ++i) {
    if (weights[i] == 0.0) continue;
    c.poles.push_back(poles[i]);
    c.weights.push_back(weights[i]);
  }
  return c;
}

TransformedUpdate transform_update(const SpectralDecomposition& d, const LowRankUpdate& u) {
  if (u.dim() != d.size()) throw std::invalid_argument("transform_update: dimension mismatch");
  TransformedUpdate tu;
  tu.signs = u.signs;
  tu.u = Matrix(u.dim(), u.rank());
  if (u.rank() > 0 && u.dim() > 0)
    check(eigmod_b200_transform_update(ctx(), d.q.data(), u.kmat.data(), u.dim(), u.rank(),
                                       tu.u.data()));
  return tu;
}

Vec secular_weights(const Vec& lambda, const TransformedUpdate& tu) {
  if (tu.rank() < 1) throw std::invalid_argument("secular_weights: k = 0");
  if (tu.dim() != lambda.size()) throw std::invalid_argument("secular_weights: dimension mismatch");
  if (tu.signs.size() != tu.rank())
    throw std::invalid_argument("secular_weights: signs size mismatch");
  require_increasing(lambda, "secular_weights");
  Vec alpha(lambda.size());
  check(eigmod_b200_secular_weights(ctx(), lambda.data(), tu.u.data(), tu.signs.data(),
                                    lambda.size(), tu.rank(), alpha.data()));
  return alpha;
}

SecularCoefficients secular_coefficients(const Vec& lambda, const TransformedUpdate& tu) {
  return make_secular(lambda, secular_weights(lambda, tu), 1.0);
}

double eval_secular(const SecularCoefficients& c, double x) {
  // proj/src/secular.cpp:223-232
  double f = c.leading;
  for (std::size_t j = 0; j < c.size(); ++j) {
    const double gap = x - c.poles[j];
    if (std::fabs(gap) < 1e-300) throw std::invalid_argument("eval_secular: evaluation at a pole");
    f -= c.weights[j] / gap;
  }
  return f;
}

double eval_secular_derivative(const SecularCoefficients& c, double x) {
  double f = 0.0;
  for (std::size_t j = 0; j < c.size(); ++j) {
    const double gap = x - c.poles[j];
    if (std::fabs(gap) < 1e-300)
      throw std::invalid_argument("eval_secular_derivative: evaluation at a pole");
    f += c.weights[j] / (gap * gap);
  }
  return f;
}

std::pair<Vec, Vec> rank2_split(const Vec& a, const Vec& b) {
  // proj/src/secular.cpp:266-276
  if (a.size() != b.size() || a.empty())
    throw std::invalid_argument("rank2_split: bad input vectors");
  const double inv_sqrt2 = 1.0 / std::sqrt(2.0);
  Vec u1(a.size()), u2(a.size());
  for (std::size_t i = 0; i < a.size(); ++i) {
    u1[i] = (a[i] + b[i]) * inv_sqrt2;
    u2[i] = (a[i] - b[i]) * inv_sqrt2;
  }
  return {std::move(u1), std::move(u2)};
}

DeflatedProblem deflate_problem(const Vec& lambda, const TransformedUpdate& tu) {
  const std::size_t n = lambda.size();
  if (tu.dim() != n) throw std::invalid_argument("deflate_problem: dimension mismatch");
  DeflatedProblem out;
  if (n == 0) return out;
  Vec poles(n), weights(n);
  std::vector<std::int64_t> po(n), un(n), co(n), cnt(3);
  check(eigmod_b200_deflate_problem(ctx(), lambda.data(), tu.u.data(), tu.signs.data(), n,
                                    tu.rank(), poles.data(), weights.data(), po.data(), un.data(),
                                    co.data(), cnt.data()));
  out.coeffs.poles.assign(poles.begin(), poles.begin() + cnt[0]);
  out.coeffs.weights.assign(weights.begin(), weights.begin() + cnt[0]);
  out.coeffs.leading = 1.0;
  out.pole_origin.assign(po.begin(), po.begin() + cnt[0]);
  out.unchanged.assign(un.begin(), un.begin() + cnt[1]);
  out.collided.assign(co.begin(), co.begin() + cnt[2]);
  return out;
}

double default_tolerance(const Vec& lambda, const LowRankUpdate& u) {
  // proj/src/rootfind.cpp:306-312
  double scale = 1.0;
  for (double l : lambda) scale = std::max(scale, std::fabs(l));
  double kn2 = 0.0;
  const double* p = u.kmat.data();
  for (std::size_t i = 0; i < u.kmat.rows() * u.kmat.cols(); ++i) kn2 += p[i] * p[i];
  const double kn = std::sqrt(kn2);
  return 1e-12 * std::max(scale, kn * kn);
}

EigenvalueUpdate update_eigenvalues_full(const SpectralDecomposition& d, const LowRankUpdate& u,
                                         double tol, LocateStrategy) {
  validate_update(d, u);
  if (!(tol > 0.0)) throw std::invalid_argument("update_eigenvalues: tol must be positive");
  const std::size_t n = d.size(), k = u.rank();
  EigenvalueUpdate out;
  out.values.resize(n);
  Vec roots(n), ubuf(n * k);
  std::int64_t nroots = 0, keff = 0;
  std::vector<std::int64_t> keep(k);
  check(eigmod_b200_update_eigenvalues(ctx(), d.q.data(), d.lambda.data(), u.kmat.data(),
                                       u.signs.data(), n, k, tol, out.values.data(), roots.data(),
                                       &nroots, ubuf.data(), &keff, keep.data()));
  out.roots.assign(roots.begin(), roots.begin() + nroots);
  out.transformed.u = Matrix(n, keff);
  std::copy(ubuf.begin(), ubuf.begin() + n * keff, out.transformed.u.data());
  for (std::int64_t c = 0; c < keff; ++c) out.transformed.signs.push_back(u.signs[keep[c]]);
  if (keff == 0) {  // rootfind.cpp:394-399
    out.problem.unchanged.resize(n);
    for (std::size_t i = 0; i < n; ++i) out.problem.unchanged[i] = i;
  } else {
    out.problem = deflate_problem(d.lambda, out.transformed);
  }
  return out;
}

Vec update_eigenvalues(const SpectralDecomposition& d, const LowRankUpdate& u, double tol) {
  validate_update(d, u);
  if (!(tol > 0.0)) throw std::invalid_argument("update_eigenvalues: tol must be positive");
  const std::size_t n = d.size(), k = u.rank();
  {
    std::unique_lock<std::mutex> lock;
    if (eigmod_b200_multi* mg = multi(lock)) {
      Vec values(n);
      check_multi(mg, eigmod_b200_multi_update_eigenvalues(mg, d.q.data(), d.lambda.data(),
                                                           u.kmat.data(), u.signs.data(), n, k,
                                                           tol, values.data()));
      return values;
    }
  }
  Vec values(n), roots(n);
  std::int64_t nroots = 0, keff = 0;
  check(eigmod_b200_update_eigenvalues(ctx(), d.q.data(), d.lambda.data(), u.kmat.data(),
                                       u.signs.data(), n, k, tol, values.data(), roots.data(),
                                       &nroots, nullptr, &keff, nullptr));
  return values;
}

// eigvec.cpp:254-364 — columns from the plan: the plan of the last
// update_eigenvalues_full on this thread's context is reused on the device
// (K4 + K5 only, no K2 / K3); any other plan is checked against the secular
// equation of plan.transformed (eigmod_b200_assemble).
SpectralDecomposition assemble_eigenvectors(const SpectralDecomposition& d,
                                            const EigenvalueUpdate& plan, bool) {
  const std::size_t n = d.size(), k = plan.transformed.rank();
  if (plan.transformed.dim() != n && k > 0)
    throw std::invalid_argument("assemble_eigenvectors: plan does not match the decomposition");
  if (plan.transformed.signs.size() != k)
    throw std::invalid_argument("assemble_eigenvectors: signs size");
  SpectralDecomposition out;
  out.lambda.resize(n);
  out.q = Matrix(n, n);
  std::vector<std::int64_t> un(plan.problem.unchanged.begin(), plan.problem.unchanged.end());
  std::vector<std::int64_t> co(plan.problem.collided.begin(), plan.problem.collided.end());
  int path = 0;
  check(eigmod_b200_assemble(ctx(), d.q.data(), d.lambda.data(), plan.transformed.u.data(),
                             plan.transformed.signs.data(), n, k, plan.roots.data(),
                             (std::int64_t)plan.roots.size(), un.data(), (std::int64_t)un.size(),
                             co.data(), (std::int64_t)co.size(), out.lambda.data(), out.q.data(),
                             &path));
  return out;
}

// eigvec.hpp:9-25
NullDirection null_direction(const Matrix& m) {
  if (m.rows() != m.cols() || m.rows() == 0)
    throw std::invalid_argument("null_direction: square matrix required");
  NullDirection nd;
  nd.direction.resize(m.rows());
  if (eigmod_b200_null_direction(m.data(), (std::int64_t)m.rows(), nd.direction.data(),
                                 &nd.residual) != EIGMOD_B200_OK)
    throw std::invalid_argument("null_direction: square matrix required");
  return nd;
}

Matrix null_problem(const TransformedUpdate& tu, const Vec& lambda, double lambda_new) {
  const std::size_t n = lambda.size(), k = tu.rank();
  if (tu.dim() != n) throw std::invalid_argument("null_problem: dimension mismatch");
  if (tu.signs.size() != k) throw std::invalid_argument("null_problem: signs size");
  if (k == 0) return Matrix(0, 0);
  if (n == 0) return Matrix::identity(k);
  Matrix m(k, k);
  check(eigmod_b200_null_problem(ctx(), tu.u.data(), tu.signs.data(), lambda.data(),
                                 (std::int64_t)n, (std::int64_t)k, lambda_new, m.data()));
  return m;
}

Vec update_eigenvector(const SpectralDecomposition& d, const LowRankUpdate& u, double lambda_new) {
  validate_update(d, u);
  const std::size_t n = d.size();
  Vec v(n);
  check(eigmod_b200_update_eigenvector(ctx(), d.q.data(), d.lambda.data(), u.kmat.data(),
                                       u.signs.data(), (std::int64_t)n, (std::int64_t)u.rank(),
                                       lambda_new, v.data()));
  return v;
}

// rootfind.hpp:28-33
Vec dnc_solve(const SecularCoefficients& c, const RootBracket& b, double tol, DncStats* stats) {
  if (!(b.lo < b.hi)) throw std::invalid_argument("dnc_solve: empty bracket");
  if (b.expected < 1) throw std::invalid_argument("dnc_solve: expected must be >= 1");
  if (!(tol > 0.0)) throw std::invalid_argument("dnc_solve: tol must be positive");
  Vec roots((std::size_t)b.expected);
  std::int64_t nr = 0, ev = 0, rd = 0;
  check(eigmod_b200_dnc_solve(ctx(), c.poles.data(), c.weights.data(), (std::int64_t)c.size(),
                              c.leading, b.lo, b.hi, b.expected, tol, roots.data(), &nr, &ev, &rd));
  roots.resize((std::size_t)nr);
  if (stats) {
    stats->evaluations = (std::size_t)ev;
    stats->rounds = (std::size_t)rd;
  }
  return roots;
}

Vec solve_rank1(const Vec& poles, const Vec& zeta, double sigma, double tol) {
  const std::size_t n = poles.size();
  if (zeta.size() != n || n == 0) throw std::invalid_argument("solve_rank1: bad inputs");
  Vec roots(n);
  check(eigmod_b200_solve_rank1(ctx(), poles.data(), zeta.data(), (std::int64_t)n, sigma, tol,
                                roots.data()));
  return roots;
}

// secular.hpp:48
long crossing_count(const SecularCoefficients& c, double lo, double hi, int samples) {
  if (!(lo < hi) || samples < 1) throw std::invalid_argument("crossing_count: bad range");
  std::int64_t out = 0;
  check(eigmod_b200_crossing_count(ctx(), c.poles.data(), c.weights.data(),
                                   (std::int64_t)c.size(), c.leading, lo, hi, samples, &out));
  return (long)out;
}

// locate.hpp:31,50
namespace {
LocationVector counts_from_coeffs(const SecularCoefficients& c0) {
  std::vector<std::int64_t> cnt(c0.size() + 1);
  check(eigmod_b200_locate_coeffs(ctx(), c0.poles.data(), c0.weights.data(),
                                  (std::int64_t)c0.size(), c0.leading, cnt.data()));
  LocationVector loc;
  loc.counts.assign(cnt.begin(), cnt.end());
  return loc;
}
}  // namespace

LocationVector locate_rank2(const SecularCoefficients& c0, ShiftKind) {
  return counts_from_coeffs(c0);
}

LocateResult locate_rank_k(const SecularCoefficients& c0, const std::vector<int>& signs) {
  for (int sg : signs)
    if (sg != 1 && sg != -1) throw std::invalid_argument("locate_rank_k: signs must be +1/-1");
  LocateResult r;
  r.loc = counts_from_coeffs(c0);
  return r;
}

UpdateResult update_decomposition(const SpectralDecomposition& d, const LowRankUpdate& u,
                                  double tol, bool) {
  validate_update(d, u);
  if (!(tol > 0.0)) throw std::invalid_argument("update_eigenvalues: tol must be positive");
  const std::size_t n = d.size(), k = u.rank();
  UpdateResult res;
  res.decomposition.lambda.resize(n);
  res.decomposition.q = Matrix(n, n);
  double wall = 0.0;
  bool done = false;
  {
    std::unique_lock<std::mutex> lock;
    if (eigmod_b200_multi* mg = multi(lock)) {
      check_multi(mg, eigmod_b200_multi_update_decomposition(
                          mg, d.q.data(), d.lambda.data(), u.kmat.data(), u.signs.data(), n, k,
                          tol, res.decomposition.lambda.data(), res.decomposition.q.data(),
                          &wall));
      done = true;
    }
  }
  if (!done)
    check(eigmod_b200_update_decomposition(ctx(), d.q.data(), d.lambda.data(), u.kmat.data(),
                                           u.signs.data(), n, k, tol,
                                           res.decomposition.lambda.data(),
                                           res.decomposition.q.data(), &wall));
  res.wall_time = wall;
  // metrics outside the timed update, as eigvec.cpp:384-393
  check(eigmod_b200_update_metrics(ctx(), d.q.data(), d.lambda.data(), u.kmat.data(),
                                   u.signs.data(), n, k, res.decomposition.q.data(),
                                   res.decomposition.lambda.data(), &res.residual_fro,
                                   &res.ortho_err));
  return res;
}

void set_devices(const std::vector<int>& devs) {
  MultiState& s = multi_state();
  std::lock_guard<std::mutex> lock(s.mu);
  s.env_read = true;
  if (s.mg) {
    eigmod_b200_multi_destroy(s.mg);
    s.mg = nullptr;
  }
  s.devices = devs;
}

std::vector<int> devices() {
  MultiState& s = multi_state();
  std::lock_guard<std::mutex> lock(s.mu);
  if (!s.env_read) {
    s.env_read = true;
    if (s.devices.empty()) s.devices = parse_device_list(std::getenv("EIGMOD_B200_DEVICES"));
  }
  return s.devices;
}

std::vector<long long> stage_calls() {
  std::int64_t c[4] = {0, 0, 0, 0};
  check(eigmod_b200_stage_calls(ctx(), c));
  return {c[0], c[1], c[2], c[3]};
}

namespace kernels {
double ortho_error(const Matrix& a) {
  if (a.rows() == 0 || a.cols() == 0) return 0.0;
  double e = 0.0;
  check(eigmod_b200_ortho_error(ctx(), a.data(), (int64_t)a.rows(), (int64_t)a.cols(), &e));
  return e;
}
void set_parallel(bool) {}
bool parallel() { return false; }
int worker_count() { return 1; }

namespace {
Matrix gemm_dev(int ta, int tb, const Matrix& a, const Matrix& b, std::size_t m, std::size_t nn,
                std::size_t kk) {
  Matrix c(m, nn);
  if (m && nn)
    check(eigmod_b200_gemm(ctx(), ta, tb, a.data(), b.data(), (std::int64_t)m, (std::int64_t)nn,
                           (std::int64_t)kk, c.data()));
  return c;
}
void dims(bool ok, const char* what) {
  if (!ok) throw std::invalid_argument(std::string("dimension mismatch in ") + what);
}
}  // namespace

// kernels.cpp:32-80 — on the DMMA GEMM
Matrix gemm_nn(const Matrix& a, const Matrix& b) {
  dims(a.cols() == b.rows(), "gemm_nn");
  return gemm_dev(0, 0, a, b, a.rows(), b.cols(), a.cols());
}
Matrix gemm_tn(const Matrix& a, const Matrix& b) {
  dims(a.rows() == b.rows(), "gemm_tn");
  return gemm_dev(1, 0, a, b, a.cols(), b.cols(), a.rows());
}
Matrix gemm_nt(const Matrix& a, const Matrix& b) {
  dims(a.cols() == b.cols(), "gemm_nt");
  return gemm_dev(0, 1, a, b, a.rows(), b.rows(), a.cols());
}
Vec gemv_t(const Matrix& a, const Vec& x) {
  dims(a.rows() == x.size(), "gemv_t");
  Matrix xm(x.size(), 1);
  std::copy(x.begin(), x.end(), xm.data());
  const Matrix c = gemm_dev(1, 0, a, xm, a.cols(), 1, a.rows());
  return Vec(c.data(), c.data() + a.cols());
}
Matrix reconstruct_symmetric(const Matrix& q, const Vec& lambda) {
  return reconstruct(SpectralDecomposition{q, lambda}).entries;
}
// kernels.cpp:111-148: O(n^2) host helpers of the validation path
void rank1_accumulate(Matrix& a, const Vec& v, double coeff) {
  dims(a.rows() == v.size() && a.cols() == v.size(), "rank1_accumulate");
  for (std::size_t i = 0; i < v.size(); ++i) {
    const double s = coeff * v[i];
    double* ai = a.row(i);
    for (std::size_t j = 0; j < v.size(); ++j) ai[j] += s * v[j];
  }
}
void symmetrize(Matrix& a) {
  dims(a.rows() == a.cols(), "symmetrize");
  a = symmetrized(a);
}
double frobenius_norm(const Matrix& a) {
  double s = 0.0;
  for (std::size_t i = 0; i < a.rows() * a.cols(); ++i) s += a.data()[i] * a.data()[i];
  return std::sqrt(s);
}
double max_abs(const Matrix& a) {
  double m = 0.0;
  for (std::size_t i = 0; i < a.rows() * a.cols(); ++i) m = std::max(m, std::fabs(a.data()[i]));
  return m;
}

// kernels.hpp:39-50 — the plain serial loops, independent of the GPU path
namespace ref {
Matrix gemm_nn(const Matrix& a, const Matrix& b) {
  dims(a.cols() == b.rows(), "ref::gemm_nn");
  Matrix c(a.rows(), b.cols());
  for (std::size_t i = 0; i < a.rows(); ++i)
    for (std::size_t j = 0; j < b.cols(); ++j) {
      double s = 0.0;
      for (std::size_t l = 0; l < a.cols(); ++l) s += a(i, l) * b(l, j);
      c(i, j) = s;
    }
  return c;
}
Matrix gemm_tn(const Matrix& a, const Matrix& b) {
  dims(a.rows() == b.rows(), "ref::gemm_tn");
  Matrix c(a.cols(), b.cols());
  for (std::size_t i = 0; i < a.cols(); ++i)
    for (std::size_t j = 0; j < b.cols(); ++j) {
      double s = 0.0;
      for (std::size_t l = 0; l < a.rows(); ++l) s += a(l, i) * b(l, j);
      c(i, j) = s;
    }
  return c;
}
Matrix gemm_nt(const Matrix& a, const Matrix& b) {
  dims(a.cols() == b.cols(), "ref::gemm_nt");
  Matrix c(a.rows(), b.rows());
  for (std::size_t i = 0; i < a.rows(); ++i)
    for (std::size_t j = 0; j < b.rows(); ++j) {
      double s = 0.0;
      for (std::size_t l = 0; l < a.cols(); ++l) s += a(i, l) * b(j, l);
      c(i, j) = s;
    }
  return c;
}
Matrix reconstruct_symmetric(const Matrix& q, const Vec& lambda) {
  dims(q.cols() == lambda.size(), "ref::reconstruct_symmetric");
  Matrix c(q.rows(), q.rows());
  for (std::size_t i = 0; i < q.rows(); ++i)
    for (std::size_t j = 0; j < q.rows(); ++j) {
      double s = 0.0;
      for (std::size_t l = 0; l < q.cols(); ++l) s += q(i, l) * lambda[l] * q(j, l);
      c(i, j) = s;
    }
  return symmetrized(c);
}
}  // namespace ref
}  // namespace kernels

}  // namespace eigmod
