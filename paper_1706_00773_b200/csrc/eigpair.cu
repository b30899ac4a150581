// Single-eigenpair and secular-function entry points of the reference API on
// the GPU (the public functions next to the batched path).
//
//   null_problem         eigvec.hpp:19  / eigvec.cpp:187-202
//   update_eigenvector   eigvec.hpp:25  / eigvec.cpp:204-252 (bordered system of
//                        eigvec.cpp:75-119 for a root on an old eigenvalue)
//   crossing_count       secular.hpp:48 / secular.cpp:245-264
//   dnc_solve            rootfind.hpp:28 / rootfind.cpp:89-229
//   solve_rank1          rootfind.hpp:33 / rootfind.cpp:231-304
//   locate_rank2 / _k    locate.hpp:31,50 (counts from the coefficients)
//   kernels::gemm_nn/tn/nt, gemv_t   kernels.hpp:19-23
//
// The O(n k^2) resolvent sums, the O(n k) resolvent vectors, the O(n^2)
// back-transform of one vector and every secular-function evaluation run on
// the device; the host keeps only k x k algebra (the null direction of a
// k x k matrix) and the orchestration of the bracket subdivision.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "context.cuh"

using namespace eigb_capi;
using eigb::cdiv;

namespace {

// ---------------------------------------------------------------- kernels
// f(x) = leading - sum_j w_j / (x - p_j) summed in ascending pole order with
// the reference's rounding (secular.cpp:223-243: one rounded division and one
// rounded subtraction per pole, no contraction), and f'(x) = sum_j w_j /
// (x - p_j)^2. One thread per point; hit = 1 where |x - p_j| < 1e-300 (the
// reference throws there).
__global__ void secular_eval_kernel(const double* __restrict__ poles,
                                    const double* __restrict__ w, int64_t m, double leading,
                                    const double* __restrict__ xs, int64_t npts,
                                    double* __restrict__ f_out, double* __restrict__ fp_out,
                                    int* __restrict__ hit_out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= npts) return;
  const double x = xs[t];
  double f = leading, fp = 0.0;
  int hit = 0;
  for (int64_t j = 0; j < m; ++j) {
    const double gap = __dsub_rn(x, poles[j]);
    if (fabs(gap) < 1e-300) {
      hit = 1;
      break;
    }
    f = __dsub_rn(f, __ddiv_rn(w[j], gap));
    if (fp_out) fp = __dadd_rn(fp, __ddiv_rn(w[j], __dmul_rn(gap, gap)));
  }
  f_out[t] = f;
  if (fp_out) fp_out[t] = fp;
  if (hit_out) hit_out[t] = hit;
}

// Lipschitz bound of f on [a, b] (rootfind.cpp:102-118): sum |w_j| / dist^2,
// +inf when a pole lies in [a, b]. One thread per segment.
__global__ void slope_bound_kernel(const double* __restrict__ poles, const double* __restrict__ w,
                                   int64_t m, const double* __restrict__ a,
                                   const double* __restrict__ b, int64_t nseg,
                                   double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nseg) return;
  const double lo = a[t], hi = b[t];
  double l = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    const double p = poles[j];
    double dist;
    if (p <= lo) dist = lo - p;
    else if (p >= hi) dist = p - hi;
    else { l = INFINITY; break; }
    if (dist <= 0.0) { l = INFINITY; break; }
    l += fabs(w[j]) / (dist * dist);
  }
  out[t] = l;
}

// Partial resolvent sums G = sum_s u_s u_s^T / (lambda_s - x) over this CTA's
// rows, rows with |lambda_s - x| < excl skipped (excl = 0: none; a row with
// |gap| < 1e-300 then sets *hit). Thread t owns entries t, t + 256, ... of
// the k x k matrix; rows staged in shared memory.
constexpr int kGramRows = 128;
__global__ void __launch_bounds__(256) gram_partial_kernel(const double* __restrict__ u, int kp,
                                                           int k, const double* __restrict__ lam,
                                                           int64_t n, double x, double excl,
                                                           double* __restrict__ part,
                                                           int* __restrict__ hit) {
  __shared__ double su[kGramRows][33];
  __shared__ double sr[kGramRows];
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int kk = k * k;
  for (int64_t r0 = (int64_t)blockIdx.x * kGramRows; r0 < n; r0 += (int64_t)gridDim.x * kGramRows) {
    const int rows = (int)(n - r0 < kGramRows ? n - r0 : kGramRows);
    for (int e = threadIdx.x; e < rows * k; e += blockDim.x) {
      const int r = e / k, c = e - r * k;
      su[r][c] = u[(r0 + r) * kp + c];
    }
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
      const double gap = lam[r0 + r] - x;
      double inv = 1.0 / gap;
      if (fabs(gap) < excl) inv = 0.0;
      else if (fabs(gap) < 1e-300) { inv = 0.0; *hit = 1; }
      sr[r] = inv;
    }
    __syncthreads();
    for (int q = 0; q < 4; ++q) {
      const int e = threadIdx.x + 256 * q;
      if (e >= kk) break;
      const int rr = e / k, cc = e - rr * k;
      double s = acc[q];
      for (int r = 0; r < rows; ++r) s += su[r][rr] * sr[r] * su[r][cc];
      acc[q] = s;
    }
    __syncthreads();
  }
  for (int q = 0; q < 4; ++q) {
    const int e = threadIdx.x + 256 * q;
    if (e < kk) part[(size_t)blockIdx.x * kk + e] = acc[q];
  }
}

// Fixed-order sum of the per-CTA partials (deterministic).
__global__ void sum_partials_kernel(const double* __restrict__ part, int nblocks, int cnt,
                                    double* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= cnt) return;
  double s = 0.0;
  for (int b = 0; b < nblocks; ++b) s += part[(size_t)b * cnt + e];
  out[e] = s;
}

// w_s = coef * (u_s . beta) / (lambda_s - x) (rows with |gap| < excl: 0, and
// row `idx` >= 0 takes beta[k]); per-CTA partial sums of w_s^2.
__global__ void __launch_bounds__(256) resolvent_vector_kernel(
    const double* __restrict__ u, int kp, int k, const double* __restrict__ lam, int64_t n,
    double x, double excl, double coef, const double* __restrict__ beta, int64_t idx,
    double* __restrict__ w, double* __restrict__ part) {
  __shared__ double sb[33];
  __shared__ double red[8];
  if (threadIdx.x <= k) sb[threadIdx.x] = beta[threadIdx.x];
  __syncthreads();
  double ss = 0.0;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    double v;
    if (s == idx) {
      v = sb[k];
    } else {
      const double gap = lam[s] - x;
      if (fabs(gap) < excl) {
        v = 0.0;
      } else {
        double ub = 0.0;
        for (int r = 0; r < k; ++r) ub += u[s * kp + r] * sb[r];
        v = coef * ub / gap;
      }
    }
    w[s] = v;
    ss += v * v;
  }
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < 8; ++q) t += red[q];
    part[blockIdx.x] = t;
  }
}

// v_i = scale * sum_j Q[i, j] w_j (one warp per row, coalesced rows of Q).
__global__ void __launch_bounds__(256) gemv_rows_kernel(const double* __restrict__ q, int64_t n,
                                                        const double* __restrict__ w,
                                                        const double* __restrict__ norm2,
                                                        double* __restrict__ v) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double* qr = q + row * n;
  double s = 0.0;
  for (int64_t j = lane; j < n; j += 32) s += __ldcs(qr + j) * w[j];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) v[row] = s * rsqrt(*norm2);
}

// out (cols x rows) = in (rows x cols)^T, 32 x 32 shared-memory tiles; out
// rows padded to ldo.
__global__ void transpose_kernel(const double* __restrict__ in, int64_t rows, int64_t cols,
                                 double* __restrict__ out, int64_t ldo) {
  __shared__ double tile[32][33];
  const int64_t bx = (int64_t)blockIdx.x * 32, by = (int64_t)blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = by + i, c = bx + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = bx + i, r = by + threadIdx.x;
    if (c < cols && r < rows) out[c * ldo + r] = tile[threadIdx.x][i];
  }
}

// ------------------------------------------------------------ host helpers
// Smallest singular direction of a k x k matrix m: the eigenvector of m^T m
// for its smallest eigenvalue (cyclic Jacobi rotations on the k x k Gram
// matrix, as eigvec.cpp:157-185 specifies), unit length; residual ||m d||_2.
void null_direction_host(const double* m, int k, double* dir, double* resid) {
  std::vector<double> b((size_t)k * k), v((size_t)k * k, 0.0);
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) {
      double s = 0.0;
      for (int r = 0; r < k; ++r) s += m[r * k + i] * m[r * k + j];
      b[i * k + j] = s;
    }
  for (int i = 0; i < k; ++i) v[i * k + i] = 1.0;
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0, mx = 0.0;
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) {
        mx = std::max(mx, std::fabs(b[i * k + j]));
        if (j > i) off += b[i * k + j] * b[i * k + j];
      }
    if (off < 1e-30 * (1.0 + mx)) break;
    for (int p = 0; p < k; ++p)
      for (int q = p + 1; q < k; ++q) {
        const double bpq = b[p * k + q];
        if (bpq == 0.0) continue;
        const double theta = (b[q * k + q] - b[p * k + p]) / (2.0 * bpq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(1.0 + theta * theta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = t * c;
        for (int i = 0; i < k; ++i) {  // B <- B R (columns p, q)
          const double x = b[i * k + p], y = b[i * k + q];
          b[i * k + p] = c * x - s * y;
          b[i * k + q] = s * x + c * y;
        }
        for (int j = 0; j < k; ++j) {  // B <- R^T B (rows p, q)
          const double x = b[p * k + j], y = b[q * k + j];
          b[p * k + j] = c * x - s * y;
          b[q * k + j] = s * x + c * y;
        }
        b[p * k + q] = b[q * k + p] = 0.0;
        for (int i = 0; i < k; ++i) {  // V <- V R
          const double x = v[i * k + p], y = v[i * k + q];
          v[i * k + p] = c * x - s * y;
          v[i * k + q] = s * x + c * y;
        }
      }
  }
  int imin = 0;
  for (int i = 1; i < k; ++i)
    if (b[i * k + i] < b[imin * k + imin]) imin = i;
  double nn = 0.0;
  for (int i = 0; i < k; ++i) dir[i] = v[i * k + imin], nn += dir[i] * dir[i];
  const double inv = 1.0 / std::sqrt(nn);
  for (int i = 0; i < k; ++i) dir[i] *= inv;
  double r2 = 0.0;
  for (int i = 0; i < k; ++i) {
    double mi = 0.0;
    for (int j = 0; j < k; ++j) mi += m[i * k + j] * dir[j];
    r2 += mi * mi;
  }
  *resid = std::sqrt(r2);
}

double fro(const std::vector<double>& a) {
  double s = 0.0;
  for (double x : a) s += x * x;
  return std::sqrt(s);
}

unsigned grid_for(int64_t n, int per) { return (unsigned)std::max<int64_t>(1, cdiv(n, per)); }

// G (k x k, host) = sum over rows of u_s u_s^T / (lambda_s - x) on the device.
std::vector<double> gram_dev(eigmod_b200_ctx* c, const double* du, int kp, int k, const double* dl,
                             int64_t n, double x, double excl, bool* hit) {
  const int blocks = (int)std::min<int64_t>(2 * c->sms, std::max<int64_t>(1, cdiv(n, kGramRows)));
  double* part = c->ws.get_f64("ep_gram_part", (size_t)blocks * k * k);
  double* g = c->ws.get_f64("ep_gram", (size_t)k * k);
  int* dh = c->ws.get_i32("ep_hit", 1);
  EIGB_CUDA(cudaMemsetAsync(dh, 0, 4, c->stream));
  gram_partial_kernel<<<blocks, 256, 0, c->stream>>>(du, kp, k, dl, n, x, excl, part, dh);
  EIGB_LAUNCH_CHECK();
  sum_partials_kernel<<<grid_for(k * k, 128), 128, 0, c->stream>>>(part, blocks, k * k, g);
  EIGB_LAUNCH_CHECK();
  std::vector<double> h((size_t)k * k);
  int hh = 0;
  EIGB_CUDA(cudaMemcpyAsync(h.data(), g, 8 * h.size(), cudaMemcpyDeviceToHost, c->stream));
  EIGB_CUDA(cudaMemcpyAsync(&hh, dh, 4, cudaMemcpyDeviceToHost, c->stream));
  EIGB_CUDA(cudaStreamSynchronize(c->stream));
  if (hit) *hit = hh != 0;
  return h;
}

// v = Q w / ||w|| for w_s = coef (u_s . beta) / (lambda_s - x) (see
// resolvent_vector_kernel); result on the host with the reference's sign rule
// (largest-magnitude entry positive, eigvec.cpp:54-60).
void backtransform_vector(eigmod_b200_ctx* c, const double* dq, const double* du, int kp, int k,
                          const double* dl, int64_t n, double x, double excl, double coef,
                          const std::vector<double>& beta, int64_t idx, double* v_out) {
  auto st = c->stream;
  double* db = c->ws.get_f64("ep_beta", 33);
  double* dw = c->ws.get_f64("ep_w", n);
  const int blocks = (int)std::min<int64_t>(2 * c->sms, std::max<int64_t>(1, cdiv(n, 256)));
  double* part = c->ws.get_f64("ep_wpart", blocks);
  double* nrm = c->ws.get_f64("ep_wnorm", 1);
  double* dv = c->ws.get_f64("ep_v", n);
  EIGB_CUDA(cudaMemcpyAsync(db, beta.data(), 8 * beta.size(), cudaMemcpyHostToDevice, st));
  resolvent_vector_kernel<<<blocks, 256, 0, st>>>(du, kp, k, dl, n, x, excl, coef, db, idx, dw,
                                                  part);
  EIGB_LAUNCH_CHECK();
  sum_partials_kernel<<<1, 32, 0, st>>>(part, blocks, 1, nrm);
  EIGB_LAUNCH_CHECK();
  double hn = 0.0;
  EIGB_CUDA(cudaMemcpyAsync(&hn, nrm, 8, cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaStreamSynchronize(st));
  if (!(hn > 0.0) || !std::isfinite(hn))
    throw Error(2, "eigvec", "degenerate eigenvector (zero or non-finite norm)");
  gemv_rows_kernel<<<grid_for(n * 32, 256), 256, 0, st>>>(dq, n, dw, nrm, dv);
  EIGB_LAUNCH_CHECK();
  EIGB_CUDA(cudaMemcpyAsync(v_out, dv, 8 * n, cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaStreamSynchronize(st));
  int64_t imax = 0;
  for (int64_t i = 1; i < n; ++i)
    if (std::fabs(v_out[i]) > std::fabs(v_out[imax])) imax = i;
  if (v_out[imax] < 0.0)
    for (int64_t i = 0; i < n; ++i) v_out[i] = -v_out[i];
}

// Secular coefficients resident on the device for repeated evaluation.
struct DevSecular {
  eigmod_b200_ctx* c;
  const double* p;   // device copies
  const double* w;
  int64_t m;
  double leading;
  const double* hp;  // the caller's host arrays (O(m) host scans)
  const double* hw;
  int64_t evals = 0;
  // f (and f') at xs; hit[i] = 1 where x_i is within 1e-300 of a pole
  void eval(const std::vector<double>& xs, std::vector<double>& f, std::vector<int>* hit = nullptr,
            std::vector<double>* fp = nullptr) {
    const int64_t np = (int64_t)xs.size();
    f.assign(np, 0.0);
    if (np == 0) return;
    evals += np;
    double* dx = c->ws.get_f64("sec_x", np);
    double* df = c->ws.get_f64("sec_f", np);
    double* dfp = fp ? c->ws.get_f64("sec_fp", np) : nullptr;
    int* dh = c->ws.get_i32("sec_hit", np);
    EIGB_CUDA(cudaMemcpyAsync(dx, xs.data(), 8 * np, cudaMemcpyHostToDevice, c->stream));
    secular_eval_kernel<<<grid_for(np, 128), 128, 0, c->stream>>>(p, w, m, leading, dx, np, df,
                                                                  dfp, dh);
    EIGB_LAUNCH_CHECK();
    EIGB_CUDA(cudaMemcpyAsync(f.data(), df, 8 * np, cudaMemcpyDeviceToHost, c->stream));
    if (fp) {
      fp->assign(np, 0.0);
      EIGB_CUDA(cudaMemcpyAsync(fp->data(), dfp, 8 * np, cudaMemcpyDeviceToHost, c->stream));
    }
    std::vector<int> hh(np);
    EIGB_CUDA(cudaMemcpyAsync(hh.data(), dh, 4 * np, cudaMemcpyDeviceToHost, c->stream));
    EIGB_CUDA(cudaStreamSynchronize(c->stream));
    if (hit) *hit = std::move(hh);
  }
  std::vector<double> slope_bounds(const std::vector<double>& a, const std::vector<double>& b) {
    const int64_t ns = (int64_t)a.size();
    std::vector<double> out(ns);
    if (ns == 0) return out;
    double* da = c->ws.get_f64("sec_sa", ns);
    double* db = c->ws.get_f64("sec_sb", ns);
    double* dout = c->ws.get_f64("sec_so", ns);
    EIGB_CUDA(cudaMemcpyAsync(da, a.data(), 8 * ns, cudaMemcpyHostToDevice, c->stream));
    EIGB_CUDA(cudaMemcpyAsync(db, b.data(), 8 * ns, cudaMemcpyHostToDevice, c->stream));
    slope_bound_kernel<<<grid_for(ns, 128), 128, 0, c->stream>>>(p, w, m, da, db, ns, dout);
    EIGB_LAUNCH_CHECK();
    EIGB_CUDA(cudaMemcpyAsync(out.data(), dout, 8 * ns, cudaMemcpyDeviceToHost, c->stream));
    EIGB_CUDA(cudaStreamSynchronize(c->stream));
    return out;
  }
};

DevSecular upload_secular(eigmod_b200_ctx* c, const double* poles, const double* weights,
                          int64_t m, double leading) {
  double* dp = c->ws.get_f64("sec_p", std::max<int64_t>(m, 1));
  double* dw = c->ws.get_f64("sec_w", std::max<int64_t>(m, 1));
  if (m > 0) {
    EIGB_CUDA(cudaMemcpyAsync(dp, poles, 8 * m, cudaMemcpyHostToDevice, c->stream));
    EIGB_CUDA(cudaMemcpyAsync(dw, weights, 8 * m, cudaMemcpyHostToDevice, c->stream));
  }
  return DevSecular{c, dp, dw, m, leading, poles, weights};
}

void check_secular(const double* poles, const double* weights, int64_t m, double leading,
                   const char* who) {
  // make_secular's preconditions (secular.cpp:136-153)
  for (int64_t j = 0; j < m; ++j) {
    if (!std::isfinite(poles[j])) throw Error(1, "", std::string(who) + ": non-finite pole");
    if (!std::isfinite(weights[j])) throw Error(1, "", std::string(who) + ": non-finite weight");
    if (j + 1 < m && !(poles[j] < poles[j + 1]))
      throw Error(1, "", std::string(who) + ": poles not strictly increasing");
  }
  if (!std::isfinite(leading)) throw Error(1, "", std::string(who) + ": non-finite leading");
}

double residual_scale_host(const double* poles, const double* w, int64_t m, double x) {
  double mass = 0.0, dist = INFINITY;
  for (int64_t j = 0; j < m; ++j) mass += std::fabs(w[j]), dist = std::min(dist, std::fabs(x - poles[j]));
  return 1.0 + mass / std::max(dist, 1e-300);
}

// newton_polish (rootfind.cpp:36-51) of several iterates at once: up to 3
// guarded Newton steps each, keeping the best |f| inside (lo, hi).
void newton_polish_batch(DevSecular& sec, std::vector<double>& x, const std::vector<double>& lo,
                         const std::vector<double>& hi) {
  const size_t nb = x.size();
  std::vector<double> f, fp, fb(nb);
  std::vector<int> hit;
  sec.eval(x, f, &hit, &fp);
  for (size_t i = 0; i < nb; ++i) fb[i] = std::fabs(f[i]);
  std::vector<char> live(nb, 1);
  for (int it = 0; it < 3; ++it) {
    std::vector<double> nx;
    std::vector<size_t> who;
    for (size_t i = 0; i < nb; ++i) {
      if (!live[i] || hit[i]) { live[i] = 0; continue; }
      if (!std::isfinite(fp[i]) || std::fabs(fp[i]) < 1e-300) { live[i] = 0; continue; }
      const double next = x[i] - f[i] / fp[i];
      if (!(next > lo[i] && next < hi[i])) { live[i] = 0; continue; }
      nx.push_back(next);
      who.push_back(i);
    }
    if (nx.empty()) break;
    std::vector<double> f2, fp2;
    std::vector<int> h2;
    sec.eval(nx, f2, &h2, &fp2);
    for (size_t t = 0; t < who.size(); ++t) {
      const size_t i = who[t];
      if (h2[t] || std::fabs(f2[t]) >= fb[i]) { live[i] = 0; continue; }
      x[i] = nx[t];
      f[i] = f2[t];
      fp[i] = fp2[t];
      fb[i] = std::fabs(f2[t]);
      hit[i] = 0;
    }
  }
}

struct Seg {
  double lo, hi, flo, fhi;
  bool sc() const { return (flo < 0.0) != (fhi < 0.0); }
};

constexpr int kDncPoints = 8;                 // rootfind.hpp:21
constexpr int64_t kMaxEvals = int64_t(1) << 22;  // rootfind.cpp:18

// rootfind.cpp:89-229 with every round's evaluations batched on the device:
// all live segments are subdivided at their kDncPoints equidistant interior
// points together (the reference's grid), root-free segments are dropped by
// the Lipschitz bound, and once the sign-change segments account for the
// missing roots they are refined together by 32-section to tol and polished.
std::vector<double> dnc_solve_dev(DevSecular& sec, double lo, double hi, int64_t expected,
                                  double tol, int64_t* rounds_out) {
  std::vector<double> roots;
  std::vector<double> f1;
  auto f_at = [&](double x, int* hit) {
    std::vector<int> h;
    sec.eval({x}, f1, &h);
    if (hit) *hit = h[0];
    return f1[0];
  };
  double flo = f_at(lo, nullptr), fhi = f_at(hi, nullptr);
  for (int t = 0; t < 4 && flo == 0.0; ++t) lo += tol / 8.0, flo = f_at(lo, nullptr);
  for (int t = 0; t < 4 && fhi == 0.0; ++t) hi -= tol / 8.0, fhi = f_at(hi, nullptr);
  std::vector<Seg> segs;
  auto push_all = [&](std::vector<Seg>& cand) {
    std::vector<double> a, b;
    std::vector<size_t> idx;
    for (size_t i = 0; i < cand.size(); ++i)
      if (!cand[i].sc()) a.push_back(cand[i].lo), b.push_back(cand[i].hi), idx.push_back(i);
    std::vector<char> keep(cand.size(), 1);
    if (!idx.empty()) {
      const std::vector<double> l = sec.slope_bounds(a, b);
      for (size_t t = 0; t < idx.size(); ++t) {
        const Seg& s = cand[idx[t]];
        if (std::min(std::fabs(s.flo), std::fabs(s.fhi)) > l[t] * (s.hi - s.lo)) keep[idx[t]] = 0;
      }
    }
    for (size_t i = 0; i < cand.size(); ++i)
      if (keep[i]) segs.push_back(cand[i]);
  };
  {
    std::vector<Seg> c0{{lo, hi, flo, fhi}};
    push_all(c0);
  }
  int64_t depth = 0;
  while (!segs.empty()) {
    const int64_t needed = expected - (int64_t)roots.size();
    if (needed <= 0) break;
    if (sec.evals > kMaxEvals) throw Error(2, "rootfind", "evaluation budget exhausted in bracket");
    std::vector<Seg> sc, other;
    for (const Seg& s : segs) (s.sc() ? sc : other).push_back(s);
    if ((int64_t)sc.size() >= needed) {
      // every sign-change segment holds one root: 32-section to tol
      std::sort(sc.begin(), sc.end(), [](const Seg& a, const Seg& b) { return a.lo < b.lo; });
      sc.resize(needed);
      for (int round = 0; round < 64; ++round) {
        std::vector<size_t> wide;
        for (size_t i = 0; i < sc.size(); ++i)
          if (sc[i].hi - sc[i].lo > tol) wide.push_back(i);
        if (wide.empty()) break;
        constexpr int kSec = 31;
        std::vector<double> xs;
        for (size_t i : wide)
          for (int t = 1; t <= kSec; ++t)
            xs.push_back(sc[i].lo + (sc[i].hi - sc[i].lo) * t / (kSec + 1));
        std::vector<double> fx;
        std::vector<int> hx;
        sec.eval(xs, fx, &hx);
        for (size_t q = 0; q < wide.size(); ++q) {
          Seg& s = sc[wide[q]];
          double plo = s.lo, pflo = s.flo;
          bool done = false;
          for (int t = 0; t < kSec && !done; ++t) {
            const double x = xs[q * kSec + t], fv = fx[q * kSec + t];
            if (hx[q * kSec + t]) continue;
            if (fv == 0.0) { s.lo = s.hi = x; s.flo = s.fhi = 0.0; done = true; break; }
            if ((fv < 0.0) != (pflo < 0.0)) { s.lo = plo; s.flo = pflo; s.hi = x; s.fhi = fv; done = true; }
            plo = x, pflo = fv;
          }
          if (!done) s.lo = plo, s.flo = pflo;  // the change is in the last cell
        }
        if (sec.evals > kMaxEvals) throw Error(2, "rootfind", "evaluation budget exhausted in bracket");
      }
      std::vector<double> x, l, h;
      for (const Seg& s : sc) x.push_back(0.5 * (s.lo + s.hi)), l.push_back(s.lo), h.push_back(s.hi);
      newton_polish_batch(sec, x, l, h);
      roots.insert(roots.end(), x.begin(), x.end());
      break;
    }
    // subdivide every live segment (narrow ones resolve as roots / tangencies)
    ++depth;
    std::vector<Seg> next;
    std::vector<double> xs;
    std::vector<size_t> wide;
    std::vector<double> tang_x, tang_lo, tang_hi;
    for (size_t i = 0; i < segs.size(); ++i) {
      const Seg& s = segs[i];
      if (s.hi - s.lo < tol) {
        const double mid = 0.5 * (s.lo + s.hi);
        if (s.sc()) {
          tang_x.push_back(mid), tang_lo.push_back(s.lo), tang_hi.push_back(s.hi);
        } else {
          int hit = 0;
          const double fm = f_at(mid, &hit);
          if (hit) continue;
          double xstar = mid, fstar = std::fabs(fm);
          if (std::fabs(s.flo) < fstar) xstar = s.lo, fstar = std::fabs(s.flo);
          if (std::fabs(s.fhi) < fstar) xstar = s.hi, fstar = std::fabs(s.fhi);
          // tangency: an even pair collapsed below tol (rootfind.cpp:188-193)
          if (fstar <= std::sqrt(tol) * residual_scale_host(sec.hp, sec.hw, sec.m, xstar)) {
            const int64_t need = expected - (int64_t)roots.size();
            for (int64_t t = 0; t < std::min<int64_t>(2, need); ++t) roots.push_back(xstar);
          }
        }
        continue;
      }
      wide.push_back(i);
      const double hstep = (s.hi - s.lo) / (kDncPoints + 1);
      for (int t = 1; t <= kDncPoints; ++t) xs.push_back(s.lo + hstep * t);
    }
    if (!tang_x.empty()) {
      newton_polish_batch(sec, tang_x, tang_lo, tang_hi);
      for (double x : tang_x)
        if ((int64_t)roots.size() < expected) roots.push_back(x);
    }
    std::vector<double> fx;
    std::vector<int> hx;
    sec.eval(xs, fx, &hx);
    for (size_t q = 0; q < wide.size(); ++q) {
      const Seg& s = segs[wide[q]];
      const double hstep = (s.hi - s.lo) / (kDncPoints + 1);
      double px = s.lo, pf = s.flo;
      for (int t = 1; t <= kDncPoints + 1; ++t) {
        double x, fv;
        if (t <= kDncPoints) {
          x = xs[q * kDncPoints + t - 1];
          fv = fx[q * kDncPoints + t - 1];
          if (fv == 0.0 || hx[q * kDncPoints + t - 1]) {  // nudge off an exact zero
            x += hstep * 1e-9;
            fv = f_at(x, nullptr);
          }
        } else {
          x = s.hi, fv = s.fhi;
        }
        next.push_back({px, x, pf, fv});
        px = x, pf = fv;
      }
    }
    segs.clear();
    push_all(next);
  }
  if (rounds_out) *rounds_out = depth;
  std::sort(roots.begin(), roots.end());
  return roots;
}

}  // namespace

extern "C" {

int eigmod_b200_null_direction(const double* m, int64_t k, double* dir_out, double* resid_out) {
  if (!m || !dir_out || !resid_out || k < 1) return EIGMOD_B200_INVALID_ARGUMENT;
  null_direction_host(m, (int)k, dir_out, resid_out);
  return EIGMOD_B200_OK;
}

int eigmod_b200_null_problem(eigmod_b200_ctx* ctx, const double* u, const int* signs,
                             const double* lambda, int64_t n, int64_t k, double lambda_new,
                             double* m_out) {
  return guarded(ctx, [&] {
    if (k < 1 || k > eigb::kMaxRank) throw Error(1, "", "null_problem: rank out of range");
    if (n < 1) throw Error(1, "", "null_problem: dimension mismatch");
    const int kp = eigb::padded_rank(k);
    std::vector<double> up((size_t)n * kp, 0.0);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t c = 0; c < k; ++c) up[i * kp + c] = u[i * k + c];
    double* du = ctx->ws.get_f64("ep_u", up.size());
    double* dl = ctx->ws.get_f64("ep_l", n);
    EIGB_CUDA(cudaMemcpyAsync(du, up.data(), 8 * up.size(), cudaMemcpyHostToDevice, ctx->stream));
    EIGB_CUDA(cudaMemcpyAsync(dl, lambda, 8 * n, cudaMemcpyHostToDevice, ctx->stream));
    bool hit = false;
    const std::vector<double> g = gram_dev(ctx, du, kp, (int)k, dl, n, lambda_new, 0.0, &hit);
    if (hit) throw Error(1, "", "null_problem: lambda_new equals an old eigenvalue");
    // M = I + J U^T (Lambda - lambda' I)^{-1} U (eigvec.cpp:187-202)
    for (int64_t r = 0; r < k; ++r)
      for (int64_t c = 0; c < k; ++c)
        m_out[r * k + c] = (r == c ? 1.0 : 0.0) + signs[r] * g[r * k + c];
  });
}

int eigmod_b200_update_eigenvector(eigmod_b200_ctx* ctx, const double* q, const double* lambda,
                                   const double* kmat, const int* signs, int64_t n, int64_t k,
                                   double lambda_new, double* v_out) {
  return guarded(ctx, [&] {
    check_basic(n, k, signs);
    check_finite(kmat, n * k, "K");
    if (!std::isfinite(lambda_new)) throw Error(1, "", "update_eigenvector: non-finite eigenvalue");
    auto st = ctx->stream;
    double scale = 1.0;  // lambda_scale (eigvec.cpp:62-66)
    int64_t nearest = 0;
    double gap = INFINITY;
    for (int64_t i = 0; i < n; ++i) {
      scale = std::max(scale, std::fabs(lambda[i]));
      const double g = std::fabs(lambda[i] - lambda_new);
      if (g < gap) gap = g, nearest = i;
    }
    const int kp = eigb::padded_rank(k);
    double* dq = ctx->ws.get_f64("h_q", (size_t)n * n);
    double* dk = ctx->ws.get_f64("h_k", (size_t)n * k);
    double* du = ctx->ws.get_f64("h_u", (size_t)n * kp);
    double* dl = ctx->ws.get_f64("h_l", n);
    EIGB_CUDA(cudaMemcpyAsync(dq, q, 8 * n * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dk, kmat, 8 * n * k, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dl, lambda, 8 * n, cudaMemcpyHostToDevice, st));
    project(ctx, dq, dk, n, k, 0, n, du);  // U = Q^T K (K1)
    if (gap < 1e-12 * scale) {
      // on an old eigenvalue: the old vector unless its row still couples
      // (row_is_negligible, eigvec.cpp:122-127), then the bordered system
      std::vector<double> row(kp), un2(k);
      double* dn = ctx->ws.get_f64("ep_cn", k);
      eigb::column_norms2_dev(du, n, kp, (int)k, dn, st);
      EIGB_CUDA(cudaMemcpyAsync(row.data(), du + nearest * kp, 8 * kp, cudaMemcpyDeviceToHost, st));
      EIGB_CUDA(cudaMemcpyAsync(un2.data(), dn, 8 * k, cudaMemcpyDeviceToHost, st));
      EIGB_CUDA(cudaStreamSynchronize(st));
      double rm = 0.0, fn2 = 0.0;
      for (int64_t r = 0; r < k; ++r) rm += row[r] * row[r], fn2 += un2[r];
      if (!(rm <= 1e-12 * (1.0 + fn2))) {
        const double pole = lambda[nearest];
        const double merge_gap = eigb::kPoleMergeRelGap * scale;
        const std::vector<double> g = gram_dev(ctx, du, kp, (int)k, dl, n, pole, merge_gap, nullptr);
        const int kb = (int)k + 1;
        std::vector<double> bm((size_t)kb * kb, 0.0);
        for (int r = 0; r < k; ++r) {
          for (int c = 0; c < k; ++c) bm[r * kb + c] = (r == c ? 1.0 : 0.0) + signs[r] * g[r * k + c];
          bm[r * kb + k] = -(double)signs[r] * row[r];
          bm[k * kb + r] = row[r];
        }
        std::vector<double> beta(kb);
        double resid = 0.0;
        null_direction_host(bm.data(), kb, beta.data(), &resid);
        if (!(resid > 1e-6 * std::max(1.0, fro(bm)))) {
          backtransform_vector(ctx, dq, du, kp, (int)k, dl, n, pole, merge_gap, -1.0, beta,
                               nearest, v_out);
          return;
        }
      }
      for (int64_t i = 0; i < n; ++i) v_out[i] = q[i * n + nearest];
      return;
    }
    const std::vector<double> g = gram_dev(ctx, du, kp, (int)k, dl, n, lambda_new, 0.0, nullptr);
    std::vector<double> m((size_t)k * k);
    for (int64_t r = 0; r < k; ++r)
      for (int64_t c = 0; c < k; ++c) m[r * k + c] = (r == c ? 1.0 : 0.0) + signs[r] * g[r * k + c];
    std::vector<double> beta(k);
    double resid = 0.0;
    null_direction_host(m.data(), (int)k, beta.data(), &resid);
    if (resid > 1e-6 * std::max(1.0, fro(m)))  // basis_vector_for_root, eigvec.cpp:133-138
      throw Error(2, "eigvec", "null problem is full rank: " + std::to_string(lambda_new) +
                                   " is not an updated eigenvalue");
    backtransform_vector(ctx, dq, du, kp, (int)k, dl, n, lambda_new, 0.0, 1.0, beta, -1, v_out);
  });
}

int eigmod_b200_secular_eval(eigmod_b200_ctx* ctx, const double* poles, const double* weights,
                             int64_t m, double leading, const double* xs, int64_t npts,
                             double* f_out, double* fp_out, int* hit_out) {
  return guarded(ctx, [&] {
    if (m < 0 || npts < 0) throw Error(1, "", "secular_eval: negative size");
    check_secular(poles, weights, m, leading, "make_secular");
    DevSecular sec = upload_secular(ctx, poles, weights, m, leading);
    std::vector<double> x(xs, xs + npts), f, fp;
    std::vector<int> hit;
    sec.eval(x, f, &hit, fp_out ? &fp : nullptr);
    std::copy(f.begin(), f.end(), f_out);
    if (fp_out) std::copy(fp.begin(), fp.end(), fp_out);
    if (hit_out) std::copy(hit.begin(), hit.end(), hit_out);
  });
}

int eigmod_b200_crossing_count(eigmod_b200_ctx* ctx, const double* poles, const double* weights,
                               int64_t m, double leading, double lo, double hi, int samples,
                               int64_t* count_out) {
  return guarded(ctx, [&] {
    if (!(lo < hi) || samples < 1) throw Error(1, "", "crossing_count: bad range");
    check_secular(poles, weights, m, leading, "make_secular");
    DevSecular sec = upload_secular(ctx, poles, weights, m, leading);
    std::vector<double> x(samples + 1), f;
    for (int s = 0; s <= samples; ++s)  // secular.cpp:251
      x[s] = lo + (hi - lo) * static_cast<double>(s) / static_cast<double>(samples);
    std::vector<int> hit;
    sec.eval(x, f, &hit);
    int64_t crossings = 0;
    double prev = 0.0;
    bool have = false;
    for (int s = 0; s <= samples; ++s) {
      if (hit[s] || f[s] == 0.0) continue;
      if (have && (prev < 0.0) != (f[s] < 0.0)) ++crossings;
      prev = f[s];
      have = true;
    }
    *count_out = crossings;
  });
}

int eigmod_b200_dnc_solve(eigmod_b200_ctx* ctx, const double* poles, const double* weights,
                          int64_t m, double leading, double lo, double hi, int64_t expected,
                          double tol, double* roots_out, int64_t* nroots_out, int64_t* evals_out,
                          int64_t* rounds_out) {
  return guarded(ctx, [&] {
    if (!(lo < hi)) throw Error(1, "", "dnc_solve: empty bracket");
    if (expected < 1) throw Error(1, "", "dnc_solve: expected must be >= 1");
    if (!(tol > 0.0)) throw Error(1, "", "dnc_solve: tol must be positive");
    check_secular(poles, weights, m, leading, "make_secular");
    DevSecular sec = upload_secular(ctx, poles, weights, m, leading);
    int64_t rounds = 0;
    std::vector<double> r = dnc_solve_dev(sec, lo, hi, expected, tol, &rounds);
    if (evals_out) *evals_out = sec.evals;
    if (rounds_out) *rounds_out = rounds;
    if ((int64_t)r.size() < expected)
      throw Error(2, "rootfind",
                  "bracket [" + std::to_string(lo) + ", " + std::to_string(hi) + "] resolved " +
                      std::to_string(r.size()) + " of " + std::to_string(expected) + " roots");
    std::copy(r.begin(), r.end(), roots_out);
    *nroots_out = (int64_t)r.size();
  });
}

// Rank-1 fast path (rootfind.cpp:231-304) on the batched solver: the
// eigenvalues of diag(poles) + sigma zeta zeta^T, i.e. the update U = zeta
// sqrt|sigma| with signature sign(sigma).
int eigmod_b200_solve_rank1(eigmod_b200_ctx* ctx, const double* poles, const double* zeta,
                            int64_t n, double sigma, double tol, double* roots_out) {
  return guarded(ctx, [&] {
    if (n < 1) throw Error(1, "", "solve_rank1: bad inputs");
    for (int64_t i = 0; i + 1 < n; ++i)
      if (!(poles[i] < poles[i + 1]))
        throw Error(1, "", "solve_rank1: poles not strictly increasing");
    if (sigma == 0.0) {
      std::copy(poles, poles + n, roots_out);
      return;
    }
    for (int64_t i = 0; i < n; ++i)
      if (zeta[i] == 0.0) throw Error(1, "", "solve_rank1: zero zeta (deflate first)");
    if (!(tol > 0.0)) throw Error(1, "", "solve_rank1: tol must be positive");
    const double s = std::sqrt(std::fabs(sigma));
    const int sg = sigma > 0.0 ? 1 : -1;
    auto st = ctx->stream;
    double* dl = ctx->ws.get_f64("h_l", n);
    double* du = ctx->ws.get_f64("h_u", n);
    double* dlo = ctx->ws.get_f64("h_lo", n);
    std::vector<double> u(n);
    for (int64_t i = 0; i < n; ++i) u[i] = zeta[i] * s;
    EIGB_CUDA(cudaMemcpyAsync(dl, poles, 8 * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(du, u.data(), 8 * n, cudaMemcpyHostToDevice, st));
    plan_from_u(ctx, dl, du, &sg, n, 1, ctx->run_rel);
    solve(ctx, 0, ctx->plan.nred);
    finish(ctx, nullptr, nullptr, 0, 0, dlo, nullptr, n);
    EIGB_CUDA(cudaMemcpyAsync(roots_out, dlo, 8 * n, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaStreamSynchronize(st));
  });
}

// Root counts per interval of the poles of a secular function (locate.hpp:
// 13-50 from the coefficients alone): f is sampled on the device in every
// interval (geometrically towards both poles; the outer intervals end at the
// root bound |x - p| <= sum |w| / |leading|), and the sign changes per
// interval are lower bounds on its root count. f * prod (x - p_j) is a
// polynomial of degree m, so once the lower bounds sum to m every count is
// exact; the sampling doubles until they do (NumericalError "locate"
// otherwise: complex roots, or roots closer than the sampling resolves).
int eigmod_b200_locate_coeffs(eigmod_b200_ctx* ctx, const double* poles, const double* weights,
                              int64_t m, double leading, int64_t* counts_out) {
  return guarded(ctx, [&] {
    check_secular(poles, weights, m, leading, "make_secular");
    if (m == 0) {
      counts_out[0] = 0;
      return;
    }
    if (leading == 0.0) throw Error(1, "", "locate: leading coefficient must be nonzero");
    double wsum = 0.0;
    for (int64_t j = 0; j < m; ++j) wsum += std::fabs(weights[j]);
    const double bound = wsum / std::fabs(leading) * (1.0 + 1e-12) + 1e-300;
    DevSecular sec = upload_secular(ctx, poles, weights, m, leading);
    for (int samples = 16; samples <= 4096; samples *= 4) {
      std::vector<double> xs;
      xs.reserve((size_t)(m + 1) * samples);
      const int half = samples / 2;
      for (int64_t i = 0; i <= m; ++i) {
        const double a = i == 0 ? poles[0] - bound : poles[i - 1];
        const double b = i == m ? poles[m - 1] + bound : poles[i];
        const double wdt = b - a;
        // geometric from both ends: offsets wdt * 2^-t, t = 1 .. 52 spread
        // over half the samples each (the midpoint included once)
        for (int t = 0; t < samples; ++t) {
          double x;
          if (t < half) {
            const double e = -52.0 * (half - 1 - t) / std::max(1, half - 1) - 1.0;
            x = a + wdt * std::exp2(e);
          } else {
            const double e = -52.0 * (t - half) / std::max(1, half - 1) - 1.0;
            x = b - wdt * std::exp2(e);
          }
          xs.push_back(x);
        }
        std::sort(xs.end() - samples, xs.end());
      }
      std::vector<double> f;
      std::vector<int> hit;
      sec.eval(xs, f, &hit);
      int64_t total = 0;
      for (int64_t i = 0; i <= m; ++i) {
        int64_t c = 0;
        double prev = 0.0;
        bool have = false;
        for (int t = 0; t < samples; ++t) {
          const size_t q = (size_t)i * samples + t;
          if (hit[q] || f[q] == 0.0) continue;
          if (have && (prev < 0.0) != (f[q] < 0.0)) ++c;
          prev = f[q];
          have = true;
        }
        counts_out[i] = c;
        total += c;
      }
      if (total == m) return;
    }
    throw Error(2, "locate", "root accounting incomplete");
  });
}

// C (m x nn) = op(A) op(B), row-major host buffers (kernels.hpp:19-21:
// gemm_nn, gemm_tn, gemm_nt), on the DMMA GEMM: the operands are brought to
// the K-contiguous layout it takes by device transposes.
int eigmod_b200_gemm(eigmod_b200_ctx* ctx, int trans_a, int trans_b, const double* a,
                     const double* b, int64_t m, int64_t nn, int64_t kk, double* c) {
  return guarded(ctx, [&] {
    if (m < 0 || nn < 0 || kk < 0) throw Error(1, "", "gemm: negative size");
    if (m == 0 || nn == 0) return;
    auto st = ctx->stream;
    if (kk == 0) {
      std::fill(c, c + m * nn, 0.0);
      return;
    }
    const int64_t kp = kk + (kk & 1);  // the DMMA kernel wants an even inner dimension
    double* da = ctx->ws.get_f64("g_a", (size_t)m * kp);
    double* db = ctx->ws.get_f64("g_b", (size_t)nn * kp);
    double* dt = ctx->ws.get_f64("g_t", (size_t)std::max(m, nn) * kk);
    double* dc = ctx->ws.get_f64("g_c", (size_t)m * nn);
    double* ones = ctx->ws.get_f64("g_ones", nn);
    std::vector<double> h(nn, 1.0);
    EIGB_CUDA(cudaMemcpyAsync(ones, h.data(), 8 * nn, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemset2DAsync(da, 8 * kp, 0, 8 * kp, m, st));
    EIGB_CUDA(cudaMemset2DAsync(db, 8 * kp, 0, 8 * kp, nn, st));
    const dim3 tb(32, 8);
    // A' = op(A), m x kk row-major
    if (!trans_a) {
      EIGB_CUDA(cudaMemcpy2DAsync(da, 8 * kp, a, 8 * kk, 8 * kk, m, cudaMemcpyHostToDevice, st));
    } else {  // A is kk x m
      EIGB_CUDA(cudaMemcpyAsync(dt, a, 8 * kk * m, cudaMemcpyHostToDevice, st));
      transpose_kernel<<<dim3((unsigned)cdiv(m, 32), (unsigned)cdiv(kk, 32)), tb, 0, st>>>(
          dt, kk, m, da, kp);
      EIGB_LAUNCH_CHECK();
    }
    // B' = op(B)^T, nn x kk row-major
    if (trans_b) {  // B is nn x kk
      EIGB_CUDA(cudaMemcpy2DAsync(db, 8 * kp, b, 8 * kk, 8 * kk, nn, cudaMemcpyHostToDevice, st));
    } else {  // B is kk x nn
      EIGB_CUDA(cudaMemcpyAsync(dt, b, 8 * kk * nn, cudaMemcpyHostToDevice, st));
      transpose_kernel<<<dim3((unsigned)cdiv(nn, 32), (unsigned)cdiv(kk, 32)), tb, 0, st>>>(
          dt, kk, nn, db, kp);
      EIGB_LAUNCH_CHECK();
    }
    eigb::gemm_nt_dev(da, db, m, nn, kp, dc, nn, ones, nullptr, st);
    EIGB_CUDA(cudaMemcpyAsync(c, dc, 8 * m * nn, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
