/* CPU oracle for the rank-k eigen-update hot path. TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference computation (paths relative to
 * /root/reference/proj). Only tests/, __graft_entry__.smoke() and bench.py's
 * CPU-baseline leg load this file's library — as the checker, never as the
 * product. Built with -ffp-contract=off so the parts restated in the
 * reference's own loop order (transform, deflation weights) are bit-identical
 * to the reference compiled -O3 for x86-64 (no FMA contraction).
 *
 * Root location: the reference locates roots with parity scans and secular
 * Sturm chains (locate.cpp, sturm.cpp) and solves with dnc_solve
 * (rootfind.cpp:89-229); that machinery throws or returns wrong roots at the
 * BASELINE scales. The oracle instead computes the same
 * roots — the n eigenvalues of diag(d) + U J U^T, i.e. the zeros of the
 * reference's det M(x) (eigvec.cpp:187-202) — by bisection on the exact
 * inertia count #eig < x = #{d_i < x} + m - nu(S(x)), S(x) = J + U^T (D-x)^-1 U
 * (SURVEY.md App. B), to one ulp of a shifted origin. Parity with the real
 * reference where it succeeds is pinned by tests/test_oracle.py.
 */
#include "eigmod_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define EO_MAXK 64

/* ---------------------------------------------------------------- U = Q^T K */
/* kernels.cpp:50-65 (gemm_tn): c[i][j] += a[l][i] * b[l][j], l ascending. */
void eo_transform(const double* q, const double* kmat, int64_t n, int64_t k, double* u) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double* ci = u + i * k;
    for (int64_t j = 0; j < k; ++j) ci[j] = 0.0;
    for (int64_t l = 0; l < n; ++l) {
      const double ali = q[l * n + i];
      const double* bl = kmat + l * k;
      for (int64_t j = 0; j < k; ++j) ci[j] += ali * bl[j];
    }
  }
}

/* rootfind.cpp:318-340 */
int64_t eo_drop_zero_columns(const double* u, int64_t n, int64_t k, int64_t* keep) {
  double colnorm[EO_MAXK];
  double maxnorm = 0.0;
  for (int64_t j = 0; j < k; ++j) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += u[i * k + j] * u[i * k + j];
    colnorm[j] = sqrt(s);
    if (colnorm[j] > maxnorm) maxnorm = colnorm[j];
  }
  const double drop = 1e-15 * (maxnorm > 1.0 ? maxnorm : 1.0);
  int64_t m = 0;
  for (int64_t j = 0; j < k; ++j)
    if (colnorm[j] > drop) keep[m++] = j;
  return m;
}

/* ------------------------------------------------------- small dense algebra */
/* secular.cpp:14-38: LU with partial pivoting, det accumulated on the fly. */
static int lu_factor(double* m, int k, int* piv, double* det) {
  for (int i = 0; i < k; ++i) piv[i] = i;
  *det = 1.0;
  for (int col = 0; col < k; ++col) {
    int best = col;
    for (int i = col + 1; i < k; ++i)
      if (fabs(m[i * k + col]) > fabs(m[best * k + col])) best = i;
    if (best != col) {
      for (int j = 0; j < k; ++j) {
        double t = m[col * k + j];
        m[col * k + j] = m[best * k + j];
        m[best * k + j] = t;
      }
      int t = piv[col];
      piv[col] = piv[best];
      piv[best] = t;
      *det = -*det;
    }
    const double pivot = m[col * k + col];
    *det *= pivot;
    if (pivot == 0.0) return 0;
    for (int i = col + 1; i < k; ++i) {
      const double f = m[i * k + col] / pivot;
      m[i * k + col] = f;
      for (int j = col + 1; j < k; ++j) m[i * k + j] -= f * m[col * k + j];
    }
  }
  return 1;
}

static double det_by_lu(const double* a, int k) {
  double m[EO_MAXK * EO_MAXK];
  int piv[EO_MAXK];
  double det;
  memcpy(m, a, sizeof(double) * k * k);
  lu_factor(m, k, piv, &det);
  return det;
}

/* secular.cpp:49-124: explicit cofactors for k <= 3, LU det*inverse when the
 * pivots are healthy (min > 1e-8 max), cofactor expansion otherwise. */
static void adjugate(const double* m, int k, double* adj) {
  memset(adj, 0, sizeof(double) * k * k);
  if (k == 1) {
    adj[0] = 1.0;
    return;
  }
#define M(i, j) m[(i) * k + (j)]
  if (k == 2) {
    adj[0] = M(1, 1);
    adj[1] = -M(0, 1);
    adj[2] = -M(1, 0);
    adj[3] = M(0, 0);
    return;
  }
  if (k == 3) {
    adj[0] = M(1, 1) * M(2, 2) - M(1, 2) * M(2, 1);
    adj[1] = M(0, 2) * M(2, 1) - M(0, 1) * M(2, 2);
    adj[2] = M(0, 1) * M(1, 2) - M(0, 2) * M(1, 1);
    adj[3] = M(1, 2) * M(2, 0) - M(1, 0) * M(2, 2);
    adj[4] = M(0, 0) * M(2, 2) - M(0, 2) * M(2, 0);
    adj[5] = M(0, 2) * M(1, 0) - M(0, 0) * M(1, 2);
    adj[6] = M(1, 0) * M(2, 1) - M(1, 1) * M(2, 0);
    adj[7] = M(0, 1) * M(2, 0) - M(0, 0) * M(2, 1);
    adj[8] = M(0, 0) * M(1, 1) - M(0, 1) * M(1, 0);
    return;
  }
  double lu[EO_MAXK * EO_MAXK];
  int piv[EO_MAXK];
  double det, maxpiv = 0.0, minpiv = 0.0;
  memcpy(lu, m, sizeof(double) * k * k);
  if (lu_factor(lu, k, piv, &det)) {
    maxpiv = fabs(lu[0]);
    minpiv = maxpiv;
    for (int i = 1; i < k; ++i) {
      const double p = fabs(lu[i * k + i]);
      if (p > maxpiv) maxpiv = p;
      if (p < minpiv) minpiv = p;
    }
  }
  if (minpiv > 1e-8 * maxpiv) {
    double x[EO_MAXK];
    for (int j = 0; j < k; ++j) {
      for (int i = 0; i < k; ++i) x[i] = (piv[i] == j) ? det : 0.0;
      for (int i = 1; i < k; ++i)
        for (int l = 0; l < i; ++l) x[i] -= lu[i * k + l] * x[l];
      for (int ii = k; ii-- > 0;) {
        for (int l = ii + 1; l < k; ++l) x[ii] -= lu[ii * k + l] * x[l];
        x[ii] /= lu[ii * k + ii];
      }
      for (int i = 0; i < k; ++i) adj[i * k + j] = x[i];
    }
    return;
  }
  double minor[EO_MAXK * EO_MAXK];
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) {
      int mr = 0;
      for (int r = 0; r < k; ++r) {
        if (r == i) continue;
        int mc = 0;
        for (int c = 0; c < k; ++c) {
          if (c == j) continue;
          minor[mr * (k - 1) + mc] = M(r, c);
          ++mc;
        }
        ++mr;
      }
      const double cof = (((i + j) % 2) ? -1.0 : 1.0) * det_by_lu(minor, k - 1);
      adj[j * k + i] = cof;
    }
#undef M
}

/* secular.cpp:168-202 (group_weights). Groups are contiguous runs
 * [gstart[g], gstart[g]+glen[g]) as the reference's run detection makes them. */
static void group_weights(const double* rep, const int64_t* gstart, const int64_t* glen,
                          int64_t ng, const double* u, const int* signs, int64_t k,
                          double* alpha) {
#pragma omp parallel for schedule(static)
  for (int64_t g = 0; g < ng; ++g) {
    double m[EO_MAXK * EO_MAXK], adj[EO_MAXK * EO_MAXK];
    memset(m, 0, sizeof(double) * k * k);
    for (int64_t r = 0; r < k; ++r) m[r * k + r] = 1.0;
    for (int64_t h = 0; h < ng; ++h) {
      if (h == g) continue;
      const double inv_gap = 1.0 / (rep[h] - rep[g]);
      for (int64_t s = gstart[h]; s < gstart[h] + glen[h]; ++s) {
        const double* ws = u + s * k;
        for (int64_t r = 0; r < k; ++r) {
          const double f = (double)signs[r] * ws[r] * inv_gap;
          for (int64_t c = 0; c < k; ++c) m[r * k + c] += f * ws[c];
        }
      }
    }
    adjugate(m, (int)k, adj);
    double a = 0.0;
    for (int64_t s = gstart[g]; s < gstart[g] + glen[g]; ++s) {
      const double* ws = u + s * k;
      for (int64_t r = 0; r < k; ++r) {
        double t = 0.0;
        for (int64_t c = 0; c < k; ++c) t += adj[r * k + c] * (double)signs[c] * ws[c];
        a += ws[r] * t;
      }
    }
    alpha[g] = a;
  }
}

int eo_secular_weights(const double* lambda, const double* u, const int* signs, int64_t n,
                       int64_t k, double* alpha) {
  if (k < 1 || k > EO_MAXK) return 1;
  for (int64_t i = 0; i + 1 < n; ++i)
    if (!(lambda[i] < lambda[i + 1])) return 1;
  int64_t* gs = (int64_t*)malloc(sizeof(int64_t) * n);
  int64_t* gl = (int64_t*)malloc(sizeof(int64_t) * n);
  for (int64_t i = 0; i < n; ++i) gs[i] = i, gl[i] = 1;
  group_weights(lambda, gs, gl, n, u, signs, k, alpha);
  free(gs);
  free(gl);
  return 0;
}

/* Runs of near-equal poles (secular.cpp:285-302): a value joins the current run
 * when lambda[i] - lambda[last member] < rel * scale; rep = run mean. */
/* scale_override > 0: the exact mode's scale max(max|lambda|, ||U||_F^2)
 * (scale invariance); otherwise the reference's max(1, max|lambda|). */
static int64_t make_runs_s(const double* lambda, int64_t n, double rel, double scale_override,
                           int64_t* gstart, int64_t* glen, double* rep) {
  double scale = 1.0;
  for (int64_t i = 0; i < n; ++i)
    if (fabs(lambda[i]) > scale) scale = fabs(lambda[i]);
  if (scale_override > 0.0) scale = scale_override;
  const double gap = rel * scale;
  int64_t ng = 0;
  /* exact mode: a run never spans more than the gap (merging moves every
   * member by less than the gap); the reference chains consecutive gaps */
  const int width_limited = scale_override > 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double ref = (width_limited && ng > 0) ? lambda[gstart[ng - 1]] : (i > 0 ? lambda[i - 1] : 0.0);
    if (ng > 0 && lambda[i] - ref < gap) {
      glen[ng - 1]++;
    } else {
      gstart[ng] = i;
      glen[ng] = 1;
      ++ng;
    }
  }
  for (int64_t g = 0; g < ng; ++g) {
    double s = 0.0;
    for (int64_t i = gstart[g]; i < gstart[g] + glen[g]; ++i) s += lambda[i];
    rep[g] = s / (double)glen[g];
  }
  return ng;
}

static int64_t make_runs(const double* lambda, int64_t n, double rel, int64_t* gstart,
                         int64_t* glen, double* rep) {
  return make_runs_s(lambda, n, rel, 0.0, gstart, glen, rep);
}

static double frob2(const double* u, int64_t cnt) {
  double s = 0.0;
  for (int64_t i = 0; i < cnt; ++i) s += u[i] * u[i];
  const double fn = sqrt(s);
  return fn * fn;
}

/* Classification of secular.cpp:306-337. kind[g]: 0 survives, 1 unchanged,
 * 2 collided. */
static void classify(const double* alpha, const int64_t* gstart, const int64_t* glen, int64_t ng,
                     const double* u, int64_t n, int64_t k, int* kind) {
  double alpha_mass = 0.0;
  for (int64_t g = 0; g < ng; ++g) alpha_mass += fabs(alpha[g]);
  const double drop = 1e-14 * (1.0 + alpha_mass);
  const double u_mass = frob2(u, n * k);
  for (int64_t g = 0; g < ng; ++g) {
    kind[g] = 0;
    if (fabs(alpha[g]) <= drop) {
      double row_mass = 0.0;
      for (int64_t i = gstart[g]; i < gstart[g] + glen[g]; ++i)
        for (int64_t r = 0; r < k; ++r) row_mass += u[i * k + r] * u[i * k + r];
      kind[g] = (row_mass <= 1e-12 * (1.0 + u_mass)) ? 1 : 2;
    }
  }
}

/* Exact mode (the solve): a group decouples unchanged when its rows couple
 * to the rest by less than 1e-13 of the scale s; no collided class. */
static void classify_exact(const int64_t* gstart, const int64_t* glen, int64_t ng,
                           const double* u, int64_t n, int64_t k, double scale, int* kind) {
  const double fn = sqrt(frob2(u, n * k));
  for (int64_t g = 0; g < ng; ++g) {
    double row_mass = 0.0;
    for (int64_t i = gstart[g]; i < gstart[g] + glen[g]; ++i)
      for (int64_t r = 0; r < k; ++r) row_mass += u[i * k + r] * u[i * k + r];
    kind[g] = (sqrt(row_mass) * fn <= 1e-13 * scale) ? 1 : 0;
  }
}

int eo_deflate(const double* lambda, const double* u, const int* signs, int64_t n, int64_t k,
               double merge_rel, double* poles, double* weights, int64_t* pole_origin,
               int64_t* unchanged, int64_t* collided, int64_t* counts) {
  if (k < 1 || k > EO_MAXK) return 1;
  for (int64_t i = 0; i + 1 < n; ++i)
    if (!(lambda[i] <= lambda[i + 1])) return 1;
  int64_t* gs = (int64_t*)malloc(sizeof(int64_t) * n);
  int64_t* gl = (int64_t*)malloc(sizeof(int64_t) * n);
  double* rep = (double*)malloc(sizeof(double) * n);
  double* alpha = (double*)malloc(sizeof(double) * n);
  int* kind = (int*)malloc(sizeof(int) * n);
  const int64_t ng = make_runs(lambda, n, merge_rel, gs, gl, rep);
  group_weights(rep, gs, gl, ng, u, signs, k, alpha);
  classify(alpha, gs, gl, ng, u, n, k, kind);
  int64_t np = 0, nu = 0, nc = 0;
  for (int64_t g = 0; g < ng; ++g) {
    if (kind[g] == 1) {
      for (int64_t i = gs[g]; i < gs[g] + gl[g]; ++i) unchanged[nu++] = i;
      continue;
    }
    if (kind[g] == 2) {
      collided[nc++] = gs[g];
    } else {
      poles[np] = rep[g];
      weights[np] = alpha[g];
      pole_origin[np] = gs[g];
      ++np;
    }
    for (int64_t i = gs[g] + 1; i < gs[g] + gl[g]; ++i) unchanged[nu++] = i;
  }
  counts[0] = np;
  counts[1] = nu;
  counts[2] = nc;
  free(gs), free(gl), free(rep), free(alpha), free(kind);
  return 0;
}

/* ------------------------------------------------ symmetric k x k eigensolver */
/* Cyclic Jacobi (same scheme as eigvec.cpp:17-54) on a symmetric matrix;
 * eigenvalues in w, eigenvectors in the columns of v. */
static void sym_evd(const double* a_in, int k, double* w, double* v) {
  double a[EO_MAXK * EO_MAXK];
  memcpy(a, a_in, sizeof(double) * k * k);
  for (int i = 0; i < k * k; ++i) v[i] = 0.0;
  for (int i = 0; i < k; ++i) v[i * k + i] = 1.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    double off = 0.0, amax = 0.0;
    for (int p = 0; p < k; ++p)
      for (int q = 0; q < k; ++q) {
        if (p != q) off += a[p * k + q] * a[p * k + q];
        if (fabs(a[p * k + q]) > amax) amax = fabs(a[p * k + q]);
      }
    if (off <= 1e-36 * amax * amax || off == 0.0) break;
    for (int p = 0; p < k; ++p)
      for (int q = p + 1; q < k; ++q) {
        const double apq = a[p * k + q];
        if (apq == 0.0) continue;
        const double tau = (a[q * k + q] - a[p * k + p]) / (2.0 * apq);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
        for (int i = 0; i < k; ++i) {
          const double aip = a[i * k + p], aiq = a[i * k + q];
          a[i * k + p] = c * aip - s * aiq;
          a[i * k + q] = s * aip + c * aiq;
        }
        for (int j = 0; j < k; ++j) {
          const double apj = a[p * k + j], aqj = a[q * k + j];
          a[p * k + j] = c * apj - s * aqj;
          a[q * k + j] = s * apj + c * aqj;
        }
        a[p * k + q] = a[q * k + p] = 0.0;
        for (int i = 0; i < k; ++i) {
          const double vip = v[i * k + p], viq = v[i * k + q];
          v[i * k + p] = c * vip - s * viq;
          v[i * k + q] = s * vip + c * viq;
        }
      }
  }
  for (int i = 0; i < k; ++i) w[i] = a[i * k + i];
}

/* ------------------------------------------------------ secular matrix S(x) */
/* S = J + sum_i u_i u_i^T / diff_i, diff_i = (d_i - d_o) - delta. Returns the
 * number of poles below x, or -1 when x hits a pole exactly. */
static int64_t eval_S(const double* d, const double* ut, const int* signs, int64_t n, int64_t k,
                      int64_t o, double delta, double* S) {
  const double dob = (o >= 0) ? d[o] : 0.0;
  memset(S, 0, sizeof(double) * k * k);
  int64_t below = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double diff = (d[i] - dob) - delta;
    if (diff == 0.0) return -1;
    if (diff < 0.0) ++below;
    const double inv = 1.0 / diff;
    const double* ui = ut + i * k;
    for (int64_t r = 0; r < k; ++r) {
      const double f = ui[r] * inv;
      for (int64_t c = r; c < k; ++c) S[r * k + c] += f * ui[c];
    }
  }
  for (int64_t r = 0; r < k; ++r) {
    S[r * k + r] += (double)signs[r];
    for (int64_t c = 0; c < r; ++c) S[r * k + c] = S[c * k + r];
  }
  return below;
}

static int64_t count_at(const double* d, const double* ut, const int* signs, int64_t n,
                        int64_t k, int64_t o, double delta, int64_t m_neg, int* hit) {
  double S[EO_MAXK * EO_MAXK], w[EO_MAXK], v[EO_MAXK * EO_MAXK];
  const int64_t below = eval_S(d, ut, signs, n, k, o, delta, S);
  if (below < 0) {
    *hit = 1;
    return 0;
  }
  *hit = 0;
  sym_evd(S, (int)k, w, v);
  int64_t nu = 0;
  for (int64_t r = 0; r < k; ++r)
    if (w[r] < 0.0) ++nu;
  return below + m_neg - nu;
}

int64_t eo_count_below(const double* d, const double* ut, const int* signs, int64_t n, int64_t k,
                       double x) {
  int64_t m_neg = 0;
  for (int64_t r = 0; r < k; ++r) m_neg += signs[r] < 0;
  int hit;
  const int64_t c = count_at(d, ut, signs, n, k, -1, x, m_neg, &hit);
  return hit ? -1 : c;
}

/* Eigenvalue count at a pole value v itself (the limit from either side):
 * T = J + sum over the rows off v of u u^T/(d - v), restricted to the
 * orthogonal complement of the rows R at v (their span gets |R| huge
 * eigenvalues of either sign), nu = its negative inertia; then
 * #eig < v = #eig <= v = #{d < v} + m - nu when the restriction is
 * nonsingular. Returns -1 if v has no rows. */
static int64_t n_less(const double* d, int64_t n, double x);
static int64_t n_leq(const double* d, int64_t n, double x);
static int64_t count_at_pole(const double* d, const double* ut, const int* signs, int64_t n,
                             int64_t k, double v, int64_t m_neg, int64_t* zeros) {
  const int64_t p0 = n_less(d, n, v), p1 = n_leq(d, n, v);
  if (p1 <= p0) return -1;
  double T[EO_MAXK * EO_MAXK];
  memset(T, 0, sizeof(double) * k * k);
  for (int64_t s = 0; s < n; ++s) {
    if (s >= p0 && s < p1) continue;
    const double inv = 1.0 / (d[s] - v);
    const double* ws = ut + s * k;
    for (int64_t r = 0; r < k; ++r)
      for (int64_t c = 0; c < k; ++c) T[r * k + c] += ws[r] * inv * ws[c];
  }
  for (int64_t r = 0; r < k; ++r) T[r * k + r] += (double)signs[r];
  /* orthonormal basis of span(R) by modified Gram-Schmidt, then its
   * complement: basis Z of k - q vectors from the identity columns */
  double Bs[EO_MAXK * EO_MAXK];
  int q = 0;
  for (int64_t t = p0; t < p1 && q < k; ++t) {
    double v2[EO_MAXK], nn = 0.0, n0 = 0.0;
    for (int64_t c = 0; c < k; ++c) v2[c] = ut[t * k + c], n0 += v2[c] * v2[c];
    for (int rep = 0; rep < 2; ++rep)
      for (int b = 0; b < q; ++b) {
        double dp = 0.0;
        for (int64_t c = 0; c < k; ++c) dp += Bs[b * EO_MAXK + c] * v2[c];
        for (int64_t c = 0; c < k; ++c) v2[c] -= dp * Bs[b * EO_MAXK + c];
      }
    for (int64_t c = 0; c < k; ++c) nn += v2[c] * v2[c];
    if (!(nn > 1e-28 * n0)) continue;
    nn = 1.0 / sqrt(nn);
    for (int64_t c = 0; c < k; ++c) Bs[q * EO_MAXK + c] = v2[c] * nn;
    ++q;
  }
  int nz = q;
  for (int64_t e = 0; e < k && nz < k; ++e) {
    double v2[EO_MAXK], nn = 0.0;
    for (int64_t c = 0; c < k; ++c) v2[c] = (c == e) ? 1.0 : 0.0;
    for (int rep = 0; rep < 2; ++rep)
      for (int b = 0; b < nz; ++b) {
        double dp = 0.0;
        for (int64_t c = 0; c < k; ++c) dp += Bs[b * EO_MAXK + c] * v2[c];
        for (int64_t c = 0; c < k; ++c) v2[c] -= dp * Bs[b * EO_MAXK + c];
      }
    for (int64_t c = 0; c < k; ++c) nn += v2[c] * v2[c];
    if (!(nn > 1e-6)) continue;
    nn = 1.0 / sqrt(nn);
    for (int64_t c = 0; c < k; ++c) Bs[nz * EO_MAXK + c] = v2[c] * nn;
    ++nz;
  }
  const int kc = nz - q;
  int64_t nu = 0;
  *zeros = 0;
  if (kc > 0) {
    double M[EO_MAXK * EO_MAXK], w[EO_MAXK], V[EO_MAXK * EO_MAXK];
    for (int a = 0; a < kc; ++a)
      for (int b = 0; b < kc; ++b) {
        double acc = 0.0;
        for (int64_t r = 0; r < k; ++r) {
          double tr = 0.0;
          for (int64_t c = 0; c < k; ++c) tr += T[r * k + c] * Bs[(q + b) * EO_MAXK + c];
          acc += Bs[(q + a) * EO_MAXK + r] * tr;
        }
        M[a * kc + b] = acc;
      }
    sym_evd(M, kc, w, V);
    double wmax = 0.0;
    for (int a = 0; a < kc; ++a) wmax = fmax(wmax, fabs(w[a]));
    for (int a = 0; a < kc; ++a) {
      if (fabs(w[a]) <= 1e-14 * wmax) ++*zeros; /* eigenvalue of A' exactly at v */
      else if (w[a] < 0.0) ++nu;
    }
  }
  return p0 + m_neg - nu; /* #eig <= v; #eig < v is this minus *zeros */
}

/* #{d_i < x} and #{d_i <= x} by binary search. */
static int64_t n_less(const double* d, int64_t n, double x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (d[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}
static int64_t n_leq(const double* d, int64_t n, double x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (d[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

/* Root j of diag(d) + U J U^T (ascending). Bisection in x until the bracket
 * holds exactly this root and no pole, then bisection in delta relative to
 * the nearer bracketing pole, down to one ulp of delta. *collided is set when
 * the bracket collapses onto a pole (no pole-free isolation possible). */
static void solve_one(const double* d, const double* ut, const int* signs, int64_t n, int64_t k,
                      int64_t m_neg, int64_t p_pos, double lo_clip, double hi_clip, int64_t j,
                      double* root, int64_t* origin, double* delta, int* collided,
                      int64_t* evals) {
  double lo = (j - m_neg >= 0) ? d[j - m_neg] : lo_clip;
  double hi = (j + p_pos <= n - 1) ? d[j + p_pos] : hi_clip;
  int lo_ok = 0, hi_ok = 0;  /* endpoint evaluated with count == j / == j+1 */
  int64_t ne = 0;
  double last_pole = NAN;    /* pole value whose limit count was taken */
  *collided = 0;
  for (int it = 0; it < 4000; ++it) {
    if (lo_ok && hi_ok && n_less(d, n, hi) == n_leq(d, n, lo)) break; /* isolated */
    /* exactly one pole value v in [lo, hi] that is inside or an uncertified
     * endpoint: split the bracket at the pole itself (its limit count says on
     * which side root j lies; both sides empty means the root is v) */
    {
      const int64_t a = n_less(d, n, lo), b = n_leq(d, n, hi); /* poles in [lo, hi] */
      if (b > a && d[a] == d[b - 1]) {
        const double v = d[a];
        const int inside = v > lo && v < hi;
        const int open_end = (v == hi && !hi_ok) || (v == lo && !lo_ok);
        if ((inside || open_end) && v != last_pole) {
          last_pole = v;
          int64_t zeros = 0;
          const int64_t cplus = count_at_pole(d, ut, signs, n, k, v, m_neg, &zeros);
          const int64_t cminus = cplus - zeros;
          ++ne;
          if (cminus >= j + 1) {
            hi = v;
            hi_ok = (cminus == j + 1);
          } else if (cplus <= j) {
            lo = v;
            lo_ok = (cplus == j);
          } else { /* the root sits on v (a collision) */
            lo = hi = v;
            break;
          }
          if (lo == hi) break;
          continue;
        }
      }
    }
    double mid = 0.5 * (lo + hi);
    if (!(mid > lo && mid < hi)) break;
    int hit;
    int64_t c = count_at(d, ut, signs, n, k, -1, mid, m_neg, &hit);
    ++ne;
    if (hit) {
      double alt = nextafter(mid, hi);
      if (!(alt < hi)) alt = nextafter(mid, lo);
      if (!(alt > lo && alt < hi)) break;
      mid = alt;
      c = count_at(d, ut, signs, n, k, -1, mid, m_neg, &hit);
      ++ne;
      if (hit) break;
    }
    if (c >= j + 1) {
      hi = mid;
      hi_ok = (c == j + 1);
    } else {
      lo = mid;
      lo_ok = (c == j);
    }
  }
  const int isolated = lo_ok && hi_ok && n_less(d, n, hi) == n_leq(d, n, lo);
  if (!isolated) {
    /* Bracket at ulp width. A pole inside [lo, hi] means the root sits on
     * the pole (a collision, eigvec.cpp:303-323). */
    int64_t o = -1;
    const int64_t a = n_less(d, n, lo); /* first pole >= lo */
    if (a < n && d[a] <= hi) {
      o = a;
      const double mid = 0.5 * (lo + hi);
      for (int64_t b = a + 1; b < n && d[b] <= hi; ++b)
        if (fabs(d[b] - mid) < fabs(d[o] - mid)) o = b;
    }
    if (o >= 0) {
      *root = d[o];
      *origin = o;
      *delta = 0.0;
      *collided = 1;
    } else {
      *root = 0.5 * (lo + hi);
      int64_t near = n_less(d, n, *root);
      if (near >= n) near = n - 1;
      if (near > 0 && fabs(d[near - 1] - *root) < fabs(d[near] - *root)) near -= 1;
      *origin = near;
      *delta = *root - d[near];
    }
    *evals += ne;
    return;
  }
  /* Shifted origin: nearer of the two bracketing poles. */
  const int64_t a = n_leq(d, n, lo) - 1; /* largest pole <= lo */
  const int64_t b = a + 1;               /* smallest pole >= hi */
  const double mid = 0.5 * (lo + hi);
  int64_t o;
  if (a < 0) o = b;
  else if (b >= n) o = a;
  else o = (mid - d[a] <= d[b] - mid) ? a : b;
  double dlo = lo - d[o], dhi = hi - d[o];
  for (int it = 0; it < 4000; ++it) {
    const double dm = 0.5 * (dlo + dhi);
    if (!(dm > dlo && dm < dhi)) break;
    int hit;
    const int64_t c = count_at(d, ut, signs, n, k, o, dm, m_neg, &hit);
    ++ne;
    if (hit) break;
    if (c >= j + 1) dhi = dm; else dlo = dm;
  }
  *origin = o;
  *delta = 0.5 * (dlo + dhi);
  *root = d[o] + *delta;
  *evals += ne;
}

static void clips(const double* d, const double* ut, const int* signs, int64_t n, int64_t k,
                  double* lo_clip, double* hi_clip) {
  double pos = 0.0, neg = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t r = 0; r < k; ++r) {
      const double v = ut[i * k + r] * ut[i * k + r];
      if (signs[r] > 0) pos += v; else neg += v;
    }
  double scale = pos + neg;
  for (int64_t i = 0; i < n; ++i)
    if (fabs(d[i]) > scale) scale = fabs(d[i]);
  const double pad = 1e-9 * (scale > 0.0 ? scale : 1.0);
  *lo_clip = d[0] - neg * (1.0 + 1e-12) - pad;
  *hi_clip = d[n - 1] + pos * (1.0 + 1e-12) + pad;
}

int eo_solve_roots(const double* d, const double* ut, const int* signs, int64_t n, int64_t k,
                   int64_t j0, int64_t j1, double* roots, int64_t* roots_origin,
                   double* roots_delta, int64_t* evals) {
  if (k < 1 || k > EO_MAXK || n < 1) return 1;
  int64_t m_neg = 0;
  for (int64_t r = 0; r < k; ++r) m_neg += signs[r] < 0;
  const int64_t p_pos = k - m_neg;
  double lo_clip, hi_clip;
  clips(d, ut, signs, n, k, &lo_clip, &hi_clip);
  int64_t total = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : total)
  for (int64_t j = j0; j < j1; ++j) {
    int col;
    int64_t e = 0;
    solve_one(d, ut, signs, n, k, m_neg, p_pos, lo_clip, hi_clip, j, &roots[j - j0],
              &roots_origin[j - j0], &roots_delta[j - j0], &col, &e);
    total += e;
  }
  if (evals) *evals = total;
  return 0;
}

/* ------------------------------------------------------------------ vectors */
/* Null vector of S at the root: eigenvector of the eigenvalue of smallest
 * magnitude (replaces the M^T M route of eigvec.cpp:157-185 by the symmetric
 * S = J M; same null space). */
static void null_vector_S(const double* d, const double* ut, const int* signs, int64_t n,
                          int64_t k, int64_t o, double delta, double* y) {
  double S[EO_MAXK * EO_MAXK], w[EO_MAXK], v[EO_MAXK * EO_MAXK];
  eval_S(d, ut, signs, n, k, o, delta, S);
  sym_evd(S, (int)k, w, v);
  int imin = 0;
  for (int r = 1; r < k; ++r)
    if (fabs(w[r]) < fabs(w[imin])) imin = r;
  for (int r = 0; r < k; ++r) y[r] = v[r * k + imin];
}

/* eigvec.cpp:75-119 (basis_vector_for_collision) on the reduced problem:
 * bordered system [[M_i, -J w_i],[w_i^T, 0]], smallest singular direction via
 * M^T M + Jacobi, vector from the resolvent at the pole. Returns 0 on
 * rejection (caller falls back to e_idx, eigvec.cpp:298). */
/* Vector of a root lambda = v + delta at or next to the pole value v = d[idx]
 * (eigvec.cpp:75-119, the bordered system), generalised to a multiple pole
 * and to delta != 0: R = the rows at v (within merge_gap of it; a compressed
 * run keeps up to k of them). With z = J U^T x and xi = x_R,
 *   (I + J T(lambda)) z - J U_R^T xi = 0,   U_R z - delta xi = 0,
 * T(lambda) the pole sum over the rows outside R; x_s = -(u_s . z) /
 * ((d_s - v) - delta) outside R and xi on R. Unlike the formula
 * x_s = (u_s . y) / (d_s - lambda) this keeps x_R accurate when delta is far
 * below the pole's coupling (0/0 in the formula). With delta = 0 the null
 * space holds one direction per root on v; the which-th root takes the
 * eigenvector of B^T B with the which-th smallest eigenvalue. */
static int collision_vector(const double* d, const double* ut, const int* signs, int64_t n,
                            int64_t k, int64_t idx, double delta, double merge_gap, int which,
                            double* w_out) {
  const double pole = d[idx];
  int64_t r0 = idx, r1 = idx + 1;
  while (r0 > 0 && fabs(d[r0 - 1] - pole) < merge_gap) --r0;
  while (r1 < n && fabs(d[r1] - pole) < merge_gap) ++r1;
  const int64_t nr = r1 - r0;
  if (nr > EO_MAXK) return 0;
  const int64_t K1 = k + nr;
  enum { MK = 2 * EO_MAXK };
  static _Thread_local double B[MK * MK], BtB[MK * MK], V[MK * MK];
  double w[MK];
  memset(B, 0, sizeof(double) * K1 * K1);
  for (int64_t r = 0; r < k; ++r) B[r * K1 + r] = 1.0;
  for (int64_t s = 0; s < n; ++s) {
    if (s >= r0 && s < r1) continue;
    const double gap = (d[s] - pole) - delta;
    const double* ws = ut + s * k;
    for (int64_t r = 0; r < k; ++r) {
      const double f = (double)signs[r] * ws[r] / gap;
      for (int64_t c = 0; c < k; ++c) B[r * K1 + c] += f * ws[c];
    }
  }
  for (int64_t t = 0; t < nr; ++t) {
    const double* wi = ut + (r0 + t) * k;
    for (int64_t r = 0; r < k; ++r) {
      B[r * K1 + k + t] = -(double)signs[r] * wi[r];
      B[(k + t) * K1 + r] = wi[r];
    }
    B[(k + t) * K1 + k + t] = -delta;
  }
  for (int64_t i = 0; i < K1; ++i)
    for (int64_t j = 0; j < K1; ++j) {
      double s2 = 0.0;
      for (int64_t l = 0; l < K1; ++l) s2 += B[l * K1 + i] * B[l * K1 + j];
      BtB[i * K1 + j] = s2;
    }
  sym_evd(BtB, (int)K1, w, V);
  /* the which-th smallest eigenvalue (ties broken by index) */
  int pick = -1;
  for (int rank = 0; rank <= which; ++rank) {
    int best = -1;
    for (int r = 0; r < K1; ++r) {
      int taken = 0;
      /* r already used by a smaller rank? */
      for (int q = 0; q < K1; ++q)
        if (q != r && (w[q] < w[r] || (w[q] == w[r] && q < r))) ++taken;
      if (taken == rank) best = r;
    }
    pick = best;
  }
  if (pick < 0) return 0;
  double dir[MK], nrm = 0.0, fro = 0.0, res = 0.0;
  for (int r = 0; r < K1; ++r) dir[r] = V[r * K1 + pick], nrm += dir[r] * dir[r];
  nrm = sqrt(nrm);
  for (int r = 0; r < K1; ++r) dir[r] /= nrm;
  for (int64_t i = 0; i < K1 * K1; ++i) fro += B[i] * B[i];
  if (which == 0) {
    /* B^T B squares the conditioning: two inverse-iteration steps on B itself
     * (LU with partial pivoting; exact zero pivots replaced by eps ||B||) */
    static _Thread_local double L[MK * MK];
    int piv[MK];
    memcpy(L, B, sizeof(double) * K1 * K1);
    const double tiny = DBL_EPSILON * sqrt(fro);
    for (int c = 0; c < K1; ++c) {
      int pr = c;
      for (int r = c + 1; r < K1; ++r)
        if (fabs(L[r * K1 + c]) > fabs(L[pr * K1 + c])) pr = r;
      piv[c] = pr;
      if (pr != c)
        for (int t = 0; t < K1; ++t) {
          const double x = L[c * K1 + t];
          L[c * K1 + t] = L[pr * K1 + t];
          L[pr * K1 + t] = x;
        }
      if (fabs(L[c * K1 + c]) < tiny) L[c * K1 + c] = (L[c * K1 + c] < 0.0 ? -tiny : tiny);
      for (int r = c + 1; r < K1; ++r) {
        const double f = L[r * K1 + c] / L[c * K1 + c];
        L[r * K1 + c] = f;
        for (int t = c + 1; t < K1; ++t) L[r * K1 + t] -= f * L[c * K1 + t];
      }
    }
    for (int it = 0; it < 2; ++it) {
      double x[MK];
      memcpy(x, dir, sizeof(double) * K1);
      for (int c = 0; c < K1; ++c) {
        const double t2 = x[c];
        x[c] = x[piv[c]];
        x[piv[c]] = t2;
      }
      for (int r = 1; r < K1; ++r)
        for (int c = 0; c < r; ++c) x[r] -= L[r * K1 + c] * x[c];
      for (int r = K1 - 1; r >= 0; --r) {
        for (int c = r + 1; c < K1; ++c) x[r] -= L[r * K1 + c] * x[c];
        x[r] /= L[r * K1 + r];
      }
      double xn = 0.0;
      for (int r = 0; r < K1; ++r) xn += x[r] * x[r];
      if (!(xn > 0.0) || !isfinite(xn)) break;
      xn = 1.0 / sqrt(xn);
      for (int r = 0; r < K1; ++r) dir[r] = x[r] * xn;
    }
  }
  for (int64_t i = 0; i < K1; ++i) {
    double mi = 0.0;
    for (int64_t j = 0; j < K1; ++j) mi += B[i * K1 + j] * dir[j];
    res += mi * mi;
  }
  if (sqrt(res) > 1e-6 * fmax(1.0, sqrt(fro))) return 0;
  double norm2 = 0.0;
  for (int64_t s = 0; s < n; ++s) {
    w_out[s] = 0.0;
    if (s >= r0 && s < r1) {
      w_out[s] = dir[k + (s - r0)];
    } else {
      double ub = 0.0;
      for (int64_t r = 0; r < k; ++r) ub += ut[s * k + r] * dir[r];
      w_out[s] = -ub / ((d[s] - pole) - delta);
    }
    norm2 += w_out[s] * w_out[s];
  }
  if (!(norm2 > 0.0) || !isfinite(norm2)) return 0;
  const double inv = 1.0 / sqrt(norm2);
  for (int64_t s = 0; s < n; ++s) w_out[s] *= inv;
  return 1;
}

/* ---------------------------------------------------------------- back-GEMM */
void eo_gemm_nt(const double* a, const double* b, int64_t m, int64_t nn, int64_t l, double* c) {
  const int64_t BI = 64, BJ = 64;
#pragma omp parallel for schedule(dynamic) collapse(2)
  for (int64_t i0 = 0; i0 < m; i0 += BI)
    for (int64_t j0 = 0; j0 < nn; j0 += BJ) {
      const int64_t i1 = i0 + BI < m ? i0 + BI : m, j1 = j0 + BJ < nn ? j0 + BJ : nn;
      for (int64_t i = i0; i < i1; ++i)
        for (int64_t j = j0; j < j1; ++j) {
          const double* ai = a + i * l;
          const double* bj = b + j * l;
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
          int64_t t = 0;
          for (; t + 3 < l; t += 4) {
            s0 += ai[t] * bj[t];
            s1 += ai[t + 1] * bj[t + 1];
            s2 += ai[t + 2] * bj[t + 2];
            s3 += ai[t + 3] * bj[t + 3];
          }
          for (; t < l; ++t) s0 += ai[t] * bj[t];
          c[i * nn + j] = (s0 + s1) + (s2 + s3);
        }
    }
}

/* -------------------------------------------------------------- full update */
typedef struct {
  double value;
  int kind;        /* 0 root, 1 decoupled (unit vector), 2 decoupled (group rotation) */
  int64_t payload; /* root index / original index / group */
  int64_t sub;     /* rotation row for kind 2 */
  int64_t order;   /* insertion order for the stable merge */
} entry_t;

static int cmp_entry(const void* a, const void* b) {
  const entry_t* x = (const entry_t*)a;
  const entry_t* y = (const entry_t*)b;
  if (x->value < y->value) return -1;
  if (x->value > y->value) return 1;
  return (x->order > y->order) - (x->order < y->order);
}

int eo_update(const double* q, const double* lambda, const double* kmat, const int* signs,
              int64_t n, int64_t k, double run_rel, double* lambda_out, double* q_out,
              int64_t* info) {
  /* core.cpp:89-97 validate_update */
  if (n < 1 || k < 1 || k > n || k > EO_MAXK) return 1;
  for (int64_t r = 0; r < k; ++r)
    if (signs[r] != 1 && signs[r] != -1) return 1;
  for (int64_t i = 0; i < n * k; ++i)
    if (!isfinite(kmat[i])) return 1;
  for (int64_t i = 0; i + 1 < n; ++i)
    if (!(lambda[i] <= lambda[i + 1])) return 1;
  for (int i = 0; i < 4; ++i) info[i] = 0;

  double* u_full = (double*)malloc(sizeof(double) * n * k);
  eo_transform(q, kmat, n, k, u_full);
  int64_t keep[EO_MAXK];
  const int exact = run_rel != 1e-12;
  int64_t ke;
  if (exact) { /* columns relative to the largest one only */
    double colnorm[EO_MAXK], maxnorm = 0.0;
    for (int64_t j = 0; j < k; ++j) {
      double s2 = 0.0;
      for (int64_t i = 0; i < n; ++i) s2 += u_full[i * k + j] * u_full[i * k + j];
      colnorm[j] = sqrt(s2);
      if (colnorm[j] > maxnorm) maxnorm = colnorm[j];
    }
    ke = 0;
    for (int64_t j = 0; j < k; ++j)
      if (colnorm[j] > 1e-15 * maxnorm && colnorm[j] > 0.0) keep[ke++] = j;
  } else {
    ke = eo_drop_zero_columns(u_full, n, k, keep);
  }
  if (ke == 0) { /* rootfind.cpp:394-399: nothing couples */
    memcpy(lambda_out, lambda, sizeof(double) * n);
    if (q_out) memcpy(q_out, q, sizeof(double) * n * n);
    info[1] = n;
    free(u_full);
    return 0;
  }
  double* u = (double*)malloc(sizeof(double) * n * ke);
  int sg[EO_MAXK];
  for (int64_t jj = 0; jj < ke; ++jj) sg[jj] = signs[keep[jj]];
  for (int64_t i = 0; i < n; ++i)
    for (int64_t jj = 0; jj < ke; ++jj) u[i * ke + jj] = u_full[i * k + keep[jj]];
  free(u_full);

  /* Deflation (secular.cpp:278-340 rules) with the requested run threshold. */
  int64_t* gs = (int64_t*)malloc(sizeof(int64_t) * n);
  int64_t* gl = (int64_t*)malloc(sizeof(int64_t) * n);
  double* rep = (double*)malloc(sizeof(double) * n);
  double* alpha = (double*)malloc(sizeof(double) * n);
  int* kind = (int*)malloc(sizeof(int) * n);
  double escale = 0.0;
  if (exact) { /* max(max|lambda|, max_r ||u_r||^2): the size of A' */
    for (int64_t r = 0; r < ke; ++r) {
      double c2 = 0.0;
      for (int64_t i = 0; i < n; ++i) c2 += u[i * ke + r] * u[i * ke + r];
      if (c2 > escale) escale = c2;
    }
    for (int64_t i = 0; i < n; ++i)
      if (fabs(lambda[i]) > escale) escale = fabs(lambda[i]);
    if (!(escale > 0.0)) escale = 1.0;
  }
  const int64_t ng = make_runs_s(lambda, n, run_rel, escale, gs, gl, rep);
  group_weights(rep, gs, gl, ng, u, sg, ke, alpha);
  if (exact)
    classify_exact(gs, gl, ng, u, n, ke, escale, kind);
  else
    classify(alpha, gs, gl, ng, u, n, ke, kind);
  const double u_norm = sqrt(frob2(u, n * ke));
  /* numerical rank of a compressed run; exact mode: directions coupling below
   * 1e-13 of the scale decouple (the unchanged rule of classify_exact) */
  double rank_thr = DBL_EPSILON * u_norm;
  if (exact && u_norm > 0.0 && 1e-13 * escale / u_norm > rank_thr) rank_thr = 1e-13 * escale / u_norm;

  /* Reduced problem: singleton groups keep their row; multi-member groups are
   * compressed by a Householder QR of their rows (rows >= rank decouple at
   * rep); unchanged groups decouple at their own values. */
  double* d = (double*)malloc(sizeof(double) * n);
  double* ut = (double*)malloc(sizeof(double) * n * ke);
  int64_t* red_group = (int64_t*)malloc(sizeof(int64_t) * n); /* group of reduced row */
  int64_t* red_t = (int64_t*)malloc(sizeof(int64_t) * n);     /* rotated row index */
  double** rot = (double**)calloc(ng, sizeof(double*));       /* H per multi group */
  entry_t* ent = (entry_t*)malloc(sizeof(entry_t) * n);
  int64_t nent = 0, N = 0;
  for (int64_t g = 0; g < ng; ++g) {
    const int64_t m = gl[g], s0 = gs[g];
    if (kind[g] == 1) {
      for (int64_t i = s0; i < s0 + m; ++i)
        ent[nent] = (entry_t){lambda[i], 1, i, 0, 0}, ++nent;
      continue;
    }
    if (m == 1) {
      d[N] = lambda[s0];
      memcpy(ut + N * ke, u + s0 * ke, sizeof(double) * ke);
      red_group[N] = g;
      red_t[N] = -1;
      ++N;
      continue;
    }
    /* Householder QR of the m x ke block B; H accumulated explicitly. */
    double* B = (double*)malloc(sizeof(double) * m * ke);
    double* H = (double*)malloc(sizeof(double) * m * m);
    double* v = (double*)malloc(sizeof(double) * m);
    memcpy(B, u + s0 * ke, sizeof(double) * m * ke);
    for (int64_t i = 0; i < m * m; ++i) H[i] = 0.0;
    for (int64_t i = 0; i < m; ++i) H[i * m + i] = 1.0;
    const int64_t steps = m < ke ? m : ke;
    /* column pivoting (largest remaining column): rank-revealing, so a
     * numerically dependent run row ends up with a tiny residual row */
    int64_t used = 0; /* bit mask of pivot columns (ke <= 64) */
    for (int64_t c = 0; c < steps; ++c) {
      int64_t pc = -1;
      double best = 0.0;
      for (int64_t jj = 0; jj < ke; ++jj) {
        if ((used >> jj) & 1) continue;
        double s2 = 0.0;
        for (int64_t i = c; i < m; ++i) s2 += B[i * ke + jj] * B[i * ke + jj];
        if (s2 > best) best = s2, pc = jj;
      }
      if (pc < 0) break;
      used |= (int64_t)1 << pc;
      const double nrm = sqrt(best);
      const double al = B[c * ke + pc] >= 0.0 ? -nrm : nrm;
      double vn = 0.0;
      for (int64_t i = c; i < m; ++i) {
        v[i] = B[i * ke + pc] - (i == c ? al : 0.0);
        vn += v[i] * v[i];
      }
      if (vn == 0.0) continue;
      const double beta = 2.0 / vn;
      for (int64_t j = 0; j < ke; ++j) {
        double s = 0.0;
        for (int64_t i = c; i < m; ++i) s += v[i] * B[i * ke + j];
        s *= beta;
        for (int64_t i = c; i < m; ++i) B[i * ke + j] -= s * v[i];
      }
      for (int64_t j = 0; j < m; ++j) {
        double s = 0.0;
        for (int64_t i = c; i < m; ++i) s += v[i] * H[i * m + j];
        s *= beta;
        for (int64_t i = c; i < m; ++i) H[i * m + j] -= s * v[i];
      }
    }
    rot[g] = H;
    for (int64_t t = 0; t < m; ++t) {
      double rn = 0.0;
      for (int64_t j = 0; j < ke; ++j) rn += B[t * ke + j] * B[t * ke + j];
      if (t < steps && sqrt(rn) > rank_thr) {
        d[N] = rep[g];
        memcpy(ut + N * ke, B + t * ke, sizeof(double) * ke);
        red_group[N] = g;
        red_t[N] = t;
        ++N;
      } else {
        ent[nent] = (entry_t){rep[g], 2, g, t, 0};
        ++nent;
      }
    }
    free(B);
    free(v);
  }

  /* Roots of the reduced problem. */
  double* root = (double*)malloc(sizeof(double) * (N > 0 ? N : 1));
  int64_t* rorig = (int64_t*)malloc(sizeof(int64_t) * (N > 0 ? N : 1));
  double* rdel = (double*)malloc(sizeof(double) * (N > 0 ? N : 1));
  int* rcol = (int*)malloc(sizeof(int) * (N > 0 ? N : 1));
  int64_t evals = 0;
  if (N > 0) {
    int64_t m_neg = 0;
    for (int64_t r = 0; r < ke; ++r) m_neg += sg[r] < 0;
    double lo_clip, hi_clip;
    clips(d, ut, sg, N, ke, &lo_clip, &hi_clip);
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : evals)
    for (int64_t j = 0; j < N; ++j) {
      int64_t e = 0;
      solve_one(d, ut, sg, N, ke, m_neg, ke - m_neg, lo_clip, hi_clip, j, &root[j], &rorig[j],
                &rdel[j], &rcol[j], &e);
      evals += e;
    }
  }

  /* Merge: roots first, then decoupled entries in insertion order (stable). */
  entry_t* all = (entry_t*)malloc(sizeof(entry_t) * n);
  int64_t na = 0;
  for (int64_t j = 0; j < N; ++j) all[na] = (entry_t){root[j], 0, j, 0, na}, ++na;
  for (int64_t e = 0; e < nent; ++e) {
    all[na] = ent[e];
    all[na].order = na;
    ++na;
  }
  if (na != n) {
    /* accounting failure (rootfind.cpp:468-470 "merge") */
    free(all); free(root); free(rorig); free(rdel); free(rcol);
    free(d); free(ut); free(red_group); free(red_t); free(ent);
    for (int64_t g = 0; g < ng; ++g) free(rot[g]);
    free(rot); free(gs); free(gl); free(rep); free(alpha); free(kind); free(u);
    return 2;
  }
  qsort(all, n, sizeof(entry_t), cmp_entry);
  for (int64_t c = 0; c < n; ++c) lambda_out[c] = all[c].value;
  info[0] = N;
  info[1] = n - N;
  info[3] = evals;
  int64_t ncol = 0;
  for (int64_t j = 0; j < N; ++j) ncol += rcol[j];
  info[2] = ncol;

  if (q_out) {
    double scale = 1.0;
    for (int64_t i = 0; i < n; ++i)
      if (fabs(lambda[i]) > scale) scale = fabs(lambda[i]);
    if (exact) scale = escale;
    const double merge_gap = 1e-12 * scale;
    double* xt = (double*)calloc((size_t)n * n, sizeof(double));
    unsigned char* computed = (unsigned char*)calloc(n, 1);
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t c = 0; c < n; ++c) {
      double* row = xt + c * n;
      const entry_t* e = &all[c];
      if (e->kind == 1) {
        row[e->payload] = 1.0;
        continue;
      }
      computed[c] = 1;
      if (e->kind == 2) {
        const int64_t g = e->payload, t = e->sub;
        for (int64_t s = 0; s < gl[g]; ++s) row[gs[g] + s] = rot[g][t * gl[g] + s];
        continue;
      }
      const int64_t j = e->payload;
      double* xr = (double*)malloc(sizeof(double) * N);
      int ok = 0;
      int which = 0; /* earlier roots on the same pole value (adjacent in j) */
      if (rcol[j])
        for (int64_t j2 = j - 1; j2 >= 0 && rcol[j2] &&
                                 fabs(d[rorig[j2]] - d[rorig[j]]) < merge_gap; --j2)
          ++which;
      /* origin on a multiple pole: the shifted bordered system */
      const int64_t oj = rorig[j];
      int multi = (oj > 0 && d[oj - 1] == d[oj]) || (oj + 1 < N && d[oj + 1] == d[oj]);
      if (multi && !rcol[j]) {
        /* only next to the pole: |delta| below 1e-6 of the coupling of its
         * rows; far roots take the formula (the bordered system loses ~1e-9
         * at large delta) */
        double ur2 = 0.0;
        for (int64_t r = oj; r >= 0 && d[r] == d[oj]; --r)
          for (int64_t c2 = 0; c2 < ke; ++c2) ur2 += ut[r * ke + c2] * ut[r * ke + c2];
        for (int64_t r = oj + 1; r < N && d[r] == d[oj]; ++r)
          for (int64_t c2 = 0; c2 < ke; ++c2) ur2 += ut[r * ke + c2] * ut[r * ke + c2];
        multi = fabs(rdel[j]) < 1e-6 * ur2;
      }
      if (rcol[j]) ok = collision_vector(d, ut, sg, N, ke, oj, 0.0, merge_gap, which, xr);
      else if (multi) ok = collision_vector(d, ut, sg, N, ke, oj, rdel[j], 0.0, 0, xr);
      if (rcol[j] && !ok) {
        for (int64_t i = 0; i < N; ++i) xr[i] = 0.0;
        xr[rorig[j]] = 1.0;
        ok = 1;
      }
      if (!ok) {
        double y[EO_MAXK];
        null_vector_S(d, ut, sg, N, ke, rorig[j], rdel[j], y);
        double nrm2 = 0.0;
        for (int64_t i = 0; i < N; ++i) {
          double t = 0.0;
          for (int64_t r = 0; r < ke; ++r) t += ut[i * ke + r] * y[r];
          xr[i] = t / ((d[i] - d[rorig[j]]) - rdel[j]);
          nrm2 += xr[i] * xr[i];
        }
        const double inv = 1.0 / sqrt(nrm2);
        for (int64_t i = 0; i < N; ++i) xr[i] *= inv;
      }
      /* back to original coordinates */
      for (int64_t i = 0; i < N; ++i) {
        const int64_t g = red_group[i];
        if (red_t[i] < 0) {
          row[gs[g]] = xr[i];
        } else {
          const double* H = rot[g];
          const int64_t m = gl[g], t = red_t[i];
          for (int64_t s = 0; s < m; ++s) row[gs[g] + s] += H[t * m + s] * xr[i];
        }
      }
      free(xr);
    }
    eo_gemm_nt(q, xt, n, n, n, q_out);
    /* eigvec.cpp:340-347 sign rule on computed columns */
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n; ++c) {
      if (!computed[c]) continue;
      int64_t imax = 0;
      for (int64_t i = 1; i < n; ++i)
        if (fabs(q_out[i * n + c]) > fabs(q_out[imax * n + c])) imax = i;
      if (q_out[imax * n + c] < 0.0)
        for (int64_t i = 0; i < n; ++i) q_out[i * n + c] = -q_out[i * n + c];
    }
    free(xt);
    free(computed);
  }
  free(all); free(root); free(rorig); free(rdel); free(rcol);
  free(d); free(ut); free(red_group); free(red_t); free(ent);
  for (int64_t g = 0; g < ng; ++g) free(rot[g]);
  free(rot); free(gs); free(gl); free(rep); free(alpha); free(kind); free(u);
  return 0;
}

/* ------------------------------------------------------------ location vector */
/* Location vector of the CLI locate path (tools/eigmod.cpp:143-161): the
 * poles v_g of the reference deflation record (secular.cpp:278-340, run
 * threshold 1e-12) and, per open interval between consecutive poles, the
 * number of updated eigenvalues (the meaning of locate.hpp:13-18). The
 * reference reaches it by weight-sign parity scans plus Sturm counts
 * (locate.cpp:70-252); this restatement uses the eigenvalue count instead:
 * #eig < v_g = #{poles below v_g} + m - nu_g, with nu_g the negative inertia
 * of T_g = J + sum over the other coupled rows u u^T/(lambda - v_g) on the
 * orthogonal complement of u_g (the limit of S(x) as x -> v_g from below).
 * Collided poles (kind 2) stay in T but are neither boundaries nor counted,
 * as they leave the reference's secular coefficients. Returns 0; 1 invalid
 * input; 3 a merged multi-row run with k >= 2 (the reference's merged pole
 * is inexact there, locate.hpp has no exact meaning to restate). */
int eo_locate(const double* lambda, const double* u, const int* signs, int64_t n, int64_t k,
              int64_t* counts, int64_t* ncounts) {
  if (k < 1 || k > EO_MAXK || n < 0) return 1;
  for (int64_t i = 0; i + 1 < n; ++i)
    if (!(lambda[i] <= lambda[i + 1])) return 1;
  int64_t keep[EO_MAXK];
  const int64_t k2 = eo_drop_zero_columns(u, n, k, keep);
  if (n == 0 || k2 == 0) {
    counts[0] = 0;
    *ncounts = 1;
    return 0;
  }
  double* u2 = (double*)malloc(sizeof(double) * n * k2);
  int s2[EO_MAXK];
  int64_t m_neg = 0;
  for (int64_t c = 0; c < k2; ++c) s2[c] = signs[keep[c]], m_neg += s2[c] < 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t c = 0; c < k2; ++c) u2[i * k2 + c] = u[i * k + keep[c]];
  int64_t* gs = (int64_t*)malloc(sizeof(int64_t) * n);
  int64_t* gl = (int64_t*)malloc(sizeof(int64_t) * n);
  double* rep = (double*)malloc(sizeof(double) * n);
  double* alpha = (double*)malloc(sizeof(double) * n);
  int* kind = (int*)malloc(sizeof(int) * n);
  const int64_t ng = make_runs(lambda, n, 1e-12, gs, gl, rep);
  group_weights(rep, gs, gl, ng, u2, s2, k2, alpha);
  classify(alpha, gs, gl, ng, u2, n, k2, kind);
  int rc = 0;
  for (int64_t g = 0; g < ng; ++g)
    if (kind[g] == 0 && gl[g] > 1 && k2 >= 2) rc = 3;
  int64_t nb = 0, below = 0, prev = 0;
  for (int64_t g = 0; g < ng && rc == 0; ++g) {
    if (kind[g] != 0) continue;
    const double v = rep[g];
    double T[EO_MAXK * EO_MAXK];
    memset(T, 0, sizeof(double) * k2 * k2);
    for (int64_t h = 0; h < ng; ++h) {
      if (h == g || kind[h] == 1) continue;
      for (int64_t s = gs[h]; s < gs[h] + gl[h]; ++s) {
        const double inv = 1.0 / (lambda[s] - v);
        const double* ws = u2 + s * k2;
        for (int64_t r = 0; r < k2; ++r)
          for (int64_t c = 0; c < k2; ++c) T[r * k2 + c] += ws[r] * inv * ws[c];
      }
    }
    for (int64_t r = 0; r < k2; ++r) T[r * k2 + r] += (double)s2[r];
    /* complement of u_g: eigenvectors of the projector-deflated T. With the
     * unit vector e = u_g/|u_g|, B = (I - e e^T) T (I - e e^T) has e as an
     * exact null direction; its other eigenpairs are those of T restricted
     * to the complement. */
    int64_t nu = 0;
    if (k2 > 1) {
      const double* ug = u2 + gs[g] * k2;
      double e[EO_MAXK], nrm = 0.0;
      for (int64_t c = 0; c < k2; ++c) nrm += ug[c] * ug[c];
      nrm = sqrt(nrm);
      for (int64_t c = 0; c < k2; ++c) e[c] = ug[c] / nrm;
      double Te[EO_MAXK], eTe = 0.0;
      for (int64_t r = 0; r < k2; ++r) {
        Te[r] = 0.0;
        for (int64_t c = 0; c < k2; ++c) Te[r] += T[r * k2 + c] * e[c];
        eTe += e[r] * Te[r];
      }
      double B[EO_MAXK * EO_MAXK], w[EO_MAXK], V[EO_MAXK * EO_MAXK];
      for (int64_t r = 0; r < k2; ++r)
        for (int64_t c = 0; c < k2; ++c)
          B[r * k2 + c] = T[r * k2 + c] - e[r] * Te[c] - Te[r] * e[c] + e[r] * e[c] * eTe;
      sym_evd(B, (int)k2, w, V);
      /* drop the eigenpair along e */
      int64_t skip = 0;
      double best = -1.0;
      for (int64_t j = 0; j < k2; ++j) {
        double d = 0.0;
        for (int64_t r = 0; r < k2; ++r) d += V[r * k2 + j] * e[r];
        if (fabs(d) > best) best = fabs(d), skip = j;
      }
      for (int64_t j = 0; j < k2; ++j)
        if (j != skip && w[j] < 0.0) ++nu;
    }
    const int64_t cb = below + m_neg - nu;
    counts[nb++] = cb - prev;
    prev = cb;
    below += 1;
  }
  if (rc == 0) {
    if (nb == 0) {
      counts[0] = 0;
      *ncounts = 1;
    } else {
      counts[nb] = below - prev;
      *ncounts = nb + 1;
    }
  }
  free(u2), free(gs), free(gl), free(rep), free(alpha), free(kind);
  return rc;
}
