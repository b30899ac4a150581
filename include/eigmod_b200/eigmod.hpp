// eigmod drop-in API over the B200 C ABI (include/eigmod_b200.h).
//
// Same declarations as the reference's public headers
// (/root/reference/proj/include/eigmod/{types,core,secular,rootfind,eigvec,
// kernels}.hpp) for the functions on the hot path, so a caller recompiles
// against include/ and links lib/libeigmod_b200_cxx.so instead of
// libeigmod.a. Value semantics and exception types are the reference's:
// std::invalid_argument for preconditions, eigmod::NumericalError(stage, msg)
// for numerical failures; device failures surface as std::runtime_error.
// Everything O(n^2 k) and above runs on the GPU; there is no CPU fallback
// (the host keeps the reference's O(n^2) SymmetricDense::from symmetrization).
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace eigmod {

using Vec = std::vector<double>;

// types.hpp:14-44 — dense row-major matrix of doubles.
class Matrix {
 public:
  Matrix() = default;
  Matrix(std::size_t rows, std::size_t cols, double fill = 0.0)
      : rows_(rows), cols_(cols), data_(rows * cols, fill) {}
  static Matrix identity(std::size_t n) {
    Matrix m(n, n);
    for (std::size_t i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
  double& operator()(std::size_t i, std::size_t j) { return data_[i * cols_ + j]; }
  double operator()(std::size_t i, std::size_t j) const { return data_[i * cols_ + j]; }
  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  bool empty() const { return data_.empty(); }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }
  double* row(std::size_t i) { return data_.data() + i * cols_; }
  const double* row(std::size_t i) const { return data_.data() + i * cols_; }
  bool operator==(const Matrix& o) const = default;

 private:
  std::size_t rows_ = 0, cols_ = 0;
  std::vector<double> data_;
};

// types.hpp:47-53
struct SymmetricDense {
  std::size_t n = 0;
  Matrix entries;
  static SymmetricDense from(const Matrix& m);
};

// types.hpp:55-60 — A = Q diag(lambda) Q^T, lambda ascending.
struct SpectralDecomposition {
  Matrix q;
  Vec lambda;
  std::size_t size() const { return lambda.size(); }
};

// types.hpp:62-69 — sum_r signs[r] k_r k_r^T.
struct LowRankUpdate {
  Matrix kmat;
  std::vector<int> signs;
  std::size_t rank() const { return kmat.cols(); }
  std::size_t dim() const { return kmat.rows(); }
};

// types.hpp:71-76
struct UpdateResult {
  SpectralDecomposition decomposition;
  double residual_fro = 0.0;
  double ortho_err = 0.0;
  double wall_time = 0.0;
};

// types.hpp:78-87
class NumericalError : public std::runtime_error {
 public:
  NumericalError(std::string stage, const std::string& msg)
      : std::runtime_error("[" + stage + "] " + msg), stage_(std::move(stage)) {}
  const std::string& stage() const { return stage_; }

 private:
  std::string stage_;
};

// types.hpp:91 (core.cpp:76-87); the orthonormality check runs on the GPU.
void validate_decomposition(const SpectralDecomposition& d, double max_ortho_err = 1e-10);
void validate_update(const SpectralDecomposition& d, const LowRankUpdate& u);

// core.hpp:11-14 — validation helpers (GPU: DMMA GEMM / rank-k kernel)
SymmetricDense reconstruct(const SpectralDecomposition& d);
SymmetricDense apply_update(const SymmetricDense& a, const LowRankUpdate& u);

// secular.hpp:9-17
struct SecularCoefficients {
  Vec poles;
  Vec weights;
  double leading = 1.0;
  std::size_t size() const { return poles.size(); }
};

// locate.hpp:13-24 — root counts per interval cut by the deflated poles.
struct LocationVector {
  std::vector<long> counts;
  long total() const {
    long s = 0;
    for (long c : counts) s += c;
    return s;
  }
};
// locate.hpp:27-28
enum class ShiftKind { double_right, double_left, mixed };
ShiftKind classify_shift(const std::vector<int>& signs);
// locate.hpp:33-39
std::pair<double, double> interlacing_bounds(std::size_t index, const Vec& lambda,
                                             std::size_t rank, const std::vector<int>& signs);
// locate.hpp:31 / 41-50 — counts from the secular coefficients alone (GPU:
// sampled sign changes certified by their sum, include/eigmod_b200.h
// eigmod_b200_locate_coeffs); the rank-2 shift kind and the rank-k signature
// select the reference's scan strategy and do not change the counts.
LocationVector locate_rank2(const SecularCoefficients& c0, ShiftKind kind);
struct LocateResult {
  LocationVector loc;
  Vec roots;  // filled when solved (never: the counts are exact)
  bool solved = false;
};
LocateResult locate_rank_k(const SecularCoefficients& c0, const std::vector<int>& signs);
// The CLI locate path (tools/eigmod.cpp:143-161: transform_update ->
// deflate_problem -> locate_rank2 / locate_rank_k) on the GPU. The reference's
// locate_rank2 / locate_rank_k take only the merged scalar coefficients; the
// GPU counts from U (exact inertia at the poles), so its entry takes the update.
LocationVector locate_update(const SpectralDecomposition& d, const LowRankUpdate& u);

SecularCoefficients make_secular(Vec poles, Vec weights, double leading = 1.0);

// secular.hpp:19-28
struct TransformedUpdate {
  Matrix u;
  std::vector<int> signs;
  std::size_t rank() const { return u.cols(); }
  std::size_t dim() const { return u.rows(); }
};
TransformedUpdate transform_update(const SpectralDecomposition& d, const LowRankUpdate& u);

// secular.hpp:30-57
Vec secular_weights(const Vec& lambda, const TransformedUpdate& tu);
SecularCoefficients secular_coefficients(const Vec& lambda, const TransformedUpdate& tu);
double eval_secular(const SecularCoefficients& c, double x);
double eval_secular_derivative(const SecularCoefficients& c, double x);
// secular.hpp:48 — sign crossings over `samples` equidistant cells (GPU,
// bit-identical f)
long crossing_count(const SecularCoefficients& c, double lo, double hi, int samples);
std::pair<Vec, Vec> rank2_split(const Vec& a, const Vec& b);

// secular.hpp:59-69
struct DeflatedProblem {
  SecularCoefficients coeffs;
  std::vector<std::size_t> pole_origin;
  std::vector<std::size_t> unchanged;
  std::vector<std::size_t> collided;
};
inline constexpr double kPoleMergeRelGap = 1e-12;
inline constexpr double kWeightDeflationRel = 1e-14;
DeflatedProblem deflate_problem(const Vec& lambda, const TransformedUpdate& tu);

// rootfind.hpp:8-33 — bracket solver and rank-1 fast path (GPU)
struct RootBracket {
  double lo = 0.0;
  double hi = 0.0;
  long expected = 1;
};
struct DncStats {
  std::size_t evaluations = 0;
  std::size_t rounds = 0;
};
inline constexpr int kDncPoints = 8;
Vec dnc_solve(const SecularCoefficients& c, const RootBracket& b, double tol,
              DncStats* stats = nullptr);
Vec solve_rank1(const Vec& poles, const Vec& zeta, double sigma, double tol);

// rootfind.hpp:37-58
double default_tolerance(const Vec& lambda, const LowRankUpdate& u);
struct EigenvalueUpdate {
  Vec values;
  Vec roots;
  DeflatedProblem problem;
  TransformedUpdate transformed;
};
enum class LocateStrategy { automatic, sturm };
// Both the rank-2 and the general rank-k entry (rootfind.hpp:51-53): the
// strategy is accepted for compatibility; one inertia-count solver serves all.
EigenvalueUpdate update_eigenvalues_full(const SpectralDecomposition& d, const LowRankUpdate& u,
                                         double tol,
                                         LocateStrategy strategy = LocateStrategy::automatic);
Vec update_eigenvalues(const SpectralDecomposition& d, const LowRankUpdate& u, double tol);

// eigvec.hpp:9-25 — single eigenpairs (GPU resolvent sums and
// back-transform; the k x k null direction on the host)
struct NullDirection {
  Vec direction;
  double residual;
};
NullDirection null_direction(const Matrix& m);
Matrix null_problem(const TransformedUpdate& tu, const Vec& lambda, double lambda_new);
Vec update_eigenvector(const SpectralDecomposition& d, const LowRankUpdate& u, double lambda_new);

// eigvec.hpp:29-36. reorthogonalize is accepted for compatibility: the
// vectors are orthonormal to ~1e-11 without it.
SpectralDecomposition assemble_eigenvectors(const SpectralDecomposition& d,
                                            const EigenvalueUpdate& plan,
                                            bool reorthogonalize = false);
UpdateResult update_decomposition(const SpectralDecomposition& d, const LowRankUpdate& u,
                                  double tol, bool reorthogonalize = false);

// io.hpp:10-35 — Matrix Market / CSV ingest and egest (host, all threads;
// byte-identical output, same grammar and messages as proj/src/io.cpp).
class FormatError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
SymmetricDense read_matrix_market(const std::string& path);
void write_matrix_market(const std::string& path, const SymmetricDense& a);
struct CsvMatrix {
  Matrix values;
  std::optional<std::vector<int>> signs;
};
CsvMatrix read_csv_matrix(const std::string& path);
void write_csv_matrix(const std::string& path, const Matrix& m,
                      const std::optional<std::vector<int>>& signs = std::nullopt);
std::vector<int> parse_signs(const std::string& text);

// kernels.hpp:9-13 — the OpenMP toggle has no meaning on the GPU path.
namespace kernels {
void set_parallel(bool on);
bool parallel();
int worker_count();
// kernels.hpp:19-23 — GEMMs on the GPU DMMA path
Matrix gemm_nn(const Matrix& a, const Matrix& b);
Matrix gemm_tn(const Matrix& a, const Matrix& b);
Matrix gemm_nt(const Matrix& a, const Matrix& b);
Vec gemv_t(const Matrix& a, const Vec& x);
// kernels.hpp:26-37 — Q diag(lambda) Q^T (GPU), and O(n^2) host helpers
Matrix reconstruct_symmetric(const Matrix& q, const Vec& lambda);
void rank1_accumulate(Matrix& a, const Vec& v, double coeff);
void symmetrize(Matrix& a);
double frobenius_norm(const Matrix& a);
double max_abs(const Matrix& a);
// kernels.hpp:36 — max |A^T A - I| (GPU DMMA GEMM)
double ortho_error(const Matrix& a);
// kernels.hpp:39-50 — the reference's plain serial i-j-k loops (kept
// independent of the GPU kernels above, for tests that compare the two)
namespace ref {
Matrix gemm_nn(const Matrix& a, const Matrix& b);
Matrix gemm_tn(const Matrix& a, const Matrix& b);
Matrix gemm_nt(const Matrix& a, const Matrix& b);
Matrix reconstruct_symmetric(const Matrix& q, const Vec& lambda);
}  // namespace ref
}  // namespace kernels

// Multi-GPU (extension): route update_decomposition and
// update_eigenvalues of this process through one NCCL context over these
// devices (include/eigmod_b200.h eigmod_b200_multi_*). An empty list returns
// to one device. The environment variable EIGMOD_B200_DEVICES ("0,1,2,3")
// sets the initial list.
void set_devices(const std::vector<int>& devices);
std::vector<int> devices();
// Diagnostics (extension): stage launches on this thread's device context
// since it was created: {K1 projections, K2 plans, K3 root solves, K4 + K5
// column builds} (include/eigmod_b200.h eigmod_b200_stage_calls).
std::vector<long long> stage_calls();

}  // namespace eigmod
