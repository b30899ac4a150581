// K4: eigenvector columns X (stored transposed, Xt[c, :] = column c of the
// in-basis eigenvector matrix) and the final column order (sm_100a).
//
// Column order (proj/src/eigvec.cpp:260-278): roots, then decoupled pairs,
// stable-merged by value. Root columns follow the reference formula
// w_s = (U y)_s / (lambda_s - lambda') (eigvec.cpp:133-153) with y the null
// vector of S(lambda') from the solver and the difference formed in the
// solver's shifted origin, (d_s - d_o) - delta; the norm is left to the
// GEMM epilogue (column scale). Roots that sit on a pole use the reference's
// bordered system (eigvec.cpp:75-119). Decoupled pairs are unit vectors
// (unchanged, eigvec.cpp:288-291) or rows of a run's Householder rotation.
// Xt is written row by row with coalesced stores: HBM-bound (8 n^2 bytes).
#include "pipeline.cuh"

#include <cfloat>
#include <cstdlib>
#include <string>

#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/sequence.h>
#include <thrust/sort.h>

namespace eigb {

namespace {

__global__ void root_order_check_kernel(const double* v, int64_t n, int* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i + 1 < n && v[i + 1] < v[i]) atomicOr(bad, 1);
}

__global__ void merge_kernel(const double* __restrict__ rv, const int64_t* __restrict__ rperm,
                             int64_t nr, const double* __restrict__ dv,
                             const int64_t* __restrict__ dsrc, int64_t nd,
                             int* __restrict__ kind, int64_t* __restrict__ payload,
                             double* __restrict__ value) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nr) {
    const double x = rv[t];
    const int64_t c = t + dev_n_less(dv, nd, x);  // roots precede equal decoupled values
    kind[c] = 0;
    payload[c] = rperm ? rperm[t] : t;
    value[c] = x;
  } else if (t < nr + nd) {
    const int64_t e = t - nr;
    const double x = dv[e];
    const int64_t c = e + dev_n_leq(rv, nr, x);
    kind[c] = dsrc[e] >= 0 ? 1 : 2;
    payload[c] = e;
    value[c] = x;
  }
}

// Small symmetric Jacobi (eigvec.cpp:17-54 scheme) for the bordered system.
__device__ void sym_evd_dev(double* a, int k, double* v) {
  for (int i = 0; i < k * k; ++i) v[i] = 0.0;
  for (int i = 0; i < k; ++i) v[i * k + i] = 1.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    double off = 0.0, amax = 0.0;
    for (int p = 0; p < k; ++p)
      for (int q = 0; q < k; ++q) {
        if (p != q) off += a[p * k + q] * a[p * k + q];
        amax = fmax(amax, fabs(a[p * k + q]));
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
}

// Bordered systems, 32 roots per CTA (proj/src/eigvec.cpp:75-119 generalised):
// a root lambda = v + delta at or next to the pole value v = d[o], R = the rows
// within gap of v (a compressed run keeps up to k of them). With z = J U^T x and
// xi = x_R: (I + J T(lambda)) z - J U_R^T xi = 0, U_R z - delta xi = 0, T the
// pole pass at lambda over the rows outside R. Used for collided roots (delta
// = 0; the which-th root on v takes the which-th smallest direction of B^T B)
// and for roots whose origin is a multiple pole, where the formula
// x_s = (u_s . y)/(d_s - lambda) is 0/0 on R. The direction of B^T B is refined
// by two inverse-iteration steps on B (LU, partial pivoting). Output per root
// (stride kCollStride(KP)): z (KP), xi (KP), r0, |R|, delta, v.
template <int KP>
constexpr int kCollStride = 2 * KP + 4;

// Slots of a batch of 32 bordered roots: pole value, delta, and the row of R
// when R is the origin row alone (-1: the rows within gap of v).
__device__ __forceinline__ void collision_slots(const ReducedView& rp, const int64_t* list,
                                                int64_t cnt, const int64_t* origin,
                                                const double* rdelta, const int* mark, int64_t b0,
                                                double* dob, double* delta, int* active, int* hit,
                                                int64_t* xrow) {
  const int t = threadIdx.x;
  if (t < 32) {
    const int64_t q = b0 + t;
    active[t] = q < cnt;
    double v = 0.0, dl = 0.0;
    int64_t xr = -1;
    if (q < cnt) {
      const int64_t j = list[q];
      v = rp.d[origin[j]];
      const bool coll = (mark[j] & 1) != 0;
      dl = coll ? 0.0 : rdelta[j];
      // a root next to (not on) a multiple pole: R = its origin row alone; the
      // other rows at v stay in T at the finite difference -delta
      if (!coll) xr = origin[j];
    }
    dob[t] = v;
    delta[t] = dl;
    xrow[t] = xr;
    hit[t] = 0;
  }
}

// The pole pass of collision_kernel split over gridDim.y pole slices (one
// bordered root would otherwise run the whole pass on one CTA): slice s
// writes its partial sums to partial[(blockIdx.x * S + s)][32][OUT].
template <int KP>
__global__ void __launch_bounds__(kPassThreads, KP <= 16 ? 2 : 1) collision_pass_kernel(
    ReducedView rp, const int64_t* __restrict__ list, int64_t cnt, const int64_t* __restrict__ origin,
    const double* __restrict__ rdelta, const int* __restrict__ mark, double gap,
    double* __restrict__ partial) {
  using C = PassCfg<KP>;
  extern __shared__ __align__(16) double smem[];
  __shared__ double dob[32], delta[32];
  __shared__ int active[32], hit[32];
  __shared__ int64_t xrow[32];
  const int64_t b0 = (int64_t)blockIdx.x * 32;
  collision_slots(rp, list, cnt, origin, rdelta, mark, b0, dob, delta, active, hit, xrow);
  const int S = gridDim.y, s = blockIdx.y;
  const int64_t chunk = cdiv_dev(rp.n, (int64_t)S);
  const int64_t plo = (s * chunk < rp.n) ? s * chunk : rp.n;
  const int64_t pcnt = ((plo + chunk < rp.n) ? plo + chunk : rp.n) - plo;
  __syncthreads();
  if (threadIdx.x < 32 && xrow[threadIdx.x] >= 0) {  // slice-local row index (none: never matches)
    const int64_t xl = xrow[threadIdx.x] - plo;
    xrow[threadIdx.x] = (xl >= 0 && xl < pcnt) ? xl : INT64_MAX;
  }
  __syncthreads();
  PassSlots sl{dob, delta, nullptr, active, hit, xrow};
  PassOpts o;
  o.exclude_zero = true;
  o.excl_gap = gap;
  secular_pass<KP>(rp.d + plo, rp.u + plo * KP, pcnt, sl, o, smem);
  const double* red = pass_result<KP>(smem);
  double* out = partial + ((size_t)blockIdx.x * S + s) * C::RED_DOUBLES;
  for (int e = threadIdx.x; e < C::RED_DOUBLES; e += kPassThreads) out[e] = red[e];
}

template <int KP>
__global__ void __launch_bounds__(kPassThreads, 1) collision_kernel(
    ReducedView rp, const int64_t* __restrict__ list, int64_t cnt, const int64_t* __restrict__ origin,
    const double* __restrict__ rdelta, const int* __restrict__ mark, const int* __restrict__ which,
    double gap, double* __restrict__ colldir, int* __restrict__ collok, double* __restrict__ scratch,
    const double* __restrict__ yall, const double* __restrict__ partial, int splits) {
  using C = PassCfg<KP>;
  constexpr int MK = 2 * KP;
  extern __shared__ __align__(16) double smem[];
  __shared__ double dob[32], delta[32];
  __shared__ int active[32], hit[32];
  __shared__ int64_t xrow[32];
  const int t = threadIdx.x;
  const int64_t b0 = (int64_t)blockIdx.x * 32;
  collision_slots(rp, list, cnt, origin, rdelta, mark, b0, dob, delta, active, hit, xrow);
  __syncthreads();
  double* red = const_cast<double*>(pass_result<KP>(smem));
  if (splits > 1) {  // the slices' partial sums, in slice order
    const double* pb = partial + (size_t)blockIdx.x * splits * C::RED_DOUBLES;
    for (int e = t; e < C::RED_DOUBLES; e += kPassThreads) {
      double v = 0.0;
      for (int s = 0; s < splits; ++s) v += pb[(size_t)s * C::RED_DOUBLES + e];
      red[e] = v;
    }
    __syncthreads();
  } else {
    PassSlots sl{dob, delta, nullptr, active, hit, xrow};
    PassOpts o;
    o.exclude_zero = true;
    o.excl_gap = gap;  // rows within gap of v: the bordered block
    secular_pass<KP>(rp.d, rp.u, rp.n, sl, o, smem);
  }
  if (t < 32 && active[t]) {
    const int64_t j = list[b0 + t];
    const int64_t N = rp.n;
    const double v = dob[t], dl = delta[t];
    int64_t r0 = dev_n_leq(rp.d, N, v - gap), r1 = dev_n_less(rp.d, N, v + gap);
    if (xrow[t] >= 0) r0 = xrow[t], r1 = r0 + 1;
    const int nr = (int)(r1 - r0);
    double* out = colldir + j * kCollStride<KP>;
    if (nr < 1 || nr > KP) {
      collok[j] = 2;
      return;
    }
    const int k = rp.k, K1 = k + nr;
    double* B = scratch + ((size_t)blockIdx.x * 32 + t) * 4 * MK * MK;
    double* BtB = B + MK * MK;
    double* V = BtB + MK * MK;
    double* L = V + MK * MK;
    const double* rb = red + t * C::OUT;
    for (int r = 0; r < K1 * K1; ++r) B[r] = 0.0;
    for (int r = 0; r < k; ++r)
      for (int c = 0; c < k; ++c) {
        const double tv = (r <= c) ? rb[C::pidx(r, c)] : rb[C::pidx(c, r)];
        B[r * K1 + c] = (r == c ? 1.0 : 0.0) + (double)rp.sgn[r] * tv;
      }
    for (int tt = 0; tt < nr; ++tt) {
      const double* wi = rp.u + (r0 + tt) * KP;
      for (int r = 0; r < k; ++r) {
        B[r * K1 + k + tt] = -(double)rp.sgn[r] * wi[r];
        B[(k + tt) * K1 + r] = wi[r];
      }
      B[(k + tt) * K1 + k + tt] = -dl;
    }
    double fro = 0.0;
    for (int i = 0; i < K1 * K1; ++i) fro += B[i] * B[i];
    const int w = (mark[j] & 1) ? which[j] : 0;
    double dir[MK];
    const double* yj = yall + j * KP;
    double uy = 0.0;
    for (int r = 0; r < k; ++r) uy += rp.u[r0 * KP + r] * yj[r];
    if (!(mark[j] & 1) && nr == 1 && dl != 0.0 && isfinite(uy / dl)) {
      // a root next to its pole (R = its origin row, delta != 0): the solver's
      // null vector y of S(lambda) already solves the bordered system
      // (z = y, xi = u_o.y / delta); the inverse iterations on B below refine it
      double nrm = 0.0;
      for (int r = 0; r < k; ++r) dir[r] = yj[r], nrm += dir[r] * dir[r];
      dir[k] = uy / dl;
      nrm += dir[k] * dir[k];
      nrm = rsqrt(nrm);
      for (int r = 0; r < K1; ++r) dir[r] *= nrm;
    } else {
      for (int i = 0; i < K1; ++i)
        for (int jj = 0; jj < K1; ++jj) {
          double s = 0.0;
          for (int l = 0; l < K1; ++l) s += B[l * K1 + i] * B[l * K1 + jj];
          BtB[i * K1 + jj] = s;
        }
      sym_evd_dev(BtB, K1, V);
      // the which-th smallest eigenvalue of B^T B (ties by index)
      int pick = -1;
      for (int r = 0; r < K1; ++r) {
        int below = 0;
        for (int q = 0; q < K1; ++q)
          if (q != r && (BtB[q * K1 + q] < BtB[r * K1 + r] ||
                         (BtB[q * K1 + q] == BtB[r * K1 + r] && q < r)))
            ++below;
        if (below == w) pick = r;
      }
      if (pick < 0) {
        collok[j] = 2;
        return;
      }
      double nrm = 0.0;
      for (int r = 0; r < K1; ++r) dir[r] = V[r * K1 + pick], nrm += dir[r] * dir[r];
      nrm = rsqrt(nrm);
      for (int r = 0; r < K1; ++r) dir[r] *= nrm;
    }
    if (w == 0) {  // B^T B squares the conditioning: refine on B itself
      int piv[MK];
      for (int r = 0; r < K1 * K1; ++r) L[r] = B[r];
      const double tiny = DBL_EPSILON * sqrt(fro);
      for (int c = 0; c < K1; ++c) {
        int pr = c;
        for (int r = c + 1; r < K1; ++r)
          if (fabs(L[r * K1 + c]) > fabs(L[pr * K1 + c])) pr = r;
        piv[c] = pr;
        if (pr != c)
          for (int q = 0; q < K1; ++q) {
            const double x = L[c * K1 + q];
            L[c * K1 + q] = L[pr * K1 + q];
            L[pr * K1 + q] = x;
          }
        if (fabs(L[c * K1 + c]) < tiny) L[c * K1 + c] = (L[c * K1 + c] < 0.0 ? -tiny : tiny);
        for (int r = c + 1; r < K1; ++r) {
          const double f = L[r * K1 + c] / L[c * K1 + c];
          L[r * K1 + c] = f;
          for (int q = c + 1; q < K1; ++q) L[r * K1 + q] -= f * L[c * K1 + q];
        }
      }
      for (int it = 0; it < 2; ++it) {
        double x[MK];
        for (int r = 0; r < K1; ++r) x[r] = dir[r];
        for (int c = 0; c < K1; ++c) {
          const double x2 = x[c];
          x[c] = x[piv[c]];
          x[piv[c]] = x2;
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
        xn = rsqrt(xn);
        for (int r = 0; r < K1; ++r) dir[r] = x[r] * xn;
      }
    }
    double res = 0.0;
    for (int i = 0; i < K1; ++i) {
      double mi = 0.0;
      for (int l = 0; l < K1; ++l) mi += B[i * K1 + l] * dir[l];
      res += mi * mi;
    }
    const int ok = sqrt(res) <= 1e-6 * fmax(1.0, sqrt(fro));
    for (int r = 0; r < KP; ++r) out[r] = (r < k) ? dir[r] : 0.0;
    for (int r = 0; r < KP; ++r) out[KP + r] = (r < nr) ? dir[k + r] : 0.0;
    out[2 * KP] = (double)r0;
    out[2 * KP + 1] = (double)nr;
    out[2 * KP + 2] = dl;
    out[2 * KP + 3] = v;
    collok[j] = ok ? 1 : 2;
  }
}

// mark[j]: bit 0 collided (flag), bit 1 origin on a multiple pole and the root
// within 1e-6 of its rows' coupling, bit 2 the
// root is so close to its pole that the formula's y loses the small
// components (|delta| < 1e-6 |u_o|^2: S(lambda) has a term |u_o|^2/|delta|
// above 1e6 times its O(1) part); which[j]: earlier collided roots on the
// same pole value (adjacent in j).
__global__ void bordered_mark_kernel(const double* __restrict__ d, const double* __restrict__ u,
                                     int kp, int64_t N, const int64_t* __restrict__ origin,
                                     const double* __restrict__ rdelta,
                                     const int* __restrict__ flags, int64_t nr,
                                     int* __restrict__ mark, int* __restrict__ which,
                                     int* __restrict__ collok, int allow_multi) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nr) return;
  const int64_t o = origin[j];
  const double v = d[o];
  const bool coll = (flags[j] & 1) != 0;
  bool multi = allow_multi && ((o > 0 && d[o - 1] == v) || (o + 1 < N && d[o + 1] == v));
  double uo2 = 0.0;
  for (int c = 0; c < kp; ++c) uo2 += u[o * kp + c] * u[o * kp + c];
  const bool near = allow_multi && !coll && fabs(rdelta[j]) < 1e-6 * uo2;
  if (multi && !coll) {
    // the same rule for a multiple pole, with the coupling of all its rows: a
    // root far from it (|delta| >= 1e-6 sum |u_r|^2, e.g. the outer roots of
    // an update much larger than A) takes the formula, whose y is accurate
    // there; the bordered system loses ~1e-9 at such delta
    // (tests/test_stress.py::test_far_roots_of_a_clustered_spectrum)
    double ur2 = uo2;
    for (int64_t r = o - 1; r >= 0 && d[r] == v; --r)
      for (int c = 0; c < kp; ++c) ur2 += u[r * kp + c] * u[r * kp + c];
    for (int64_t r = o + 1; r < N && d[r] == v; ++r)
      for (int c = 0; c < kp; ++c) ur2 += u[r * kp + c] * u[r * kp + c];
    multi = fabs(rdelta[j]) < 1e-6 * ur2;
  }
  mark[j] = (coll ? 1 : 0) | (multi ? 2 : 0) | (near ? 4 : 0);
  collok[j] = 0;
  int w = 0;
  if (coll)
    for (int64_t j2 = j - 1; j2 >= 0 && (flags[j2] & 1) && d[origin[j2]] == v; --j2) ++w;
  which[j] = w;
}

// Per-column parameters of a tile (shared memory).
template <int KP>
struct XtCol {
  int kind;      // 0 root, 1 unit, 2 rotation, -1 outside [c0, c1)
  int mode;      // roots: 0 formula, 1 bordered (collided), 2 collided fallback e_o
  int64_t o;     // roots: origin pole; unit: source index; rotation: group
  int64_t t;     // rotation row
  double dob, del;
  double y[KP + 1];
  const double* cd;  // mode 1: the root's bordered-system record (collision_kernel)
};

// Value of reduced coordinate r for column parameters cp (eigvec.cpp:133-153
// formula in the solver's shifted origin, or the bordered-system vector of
// eigvec.cpp:75-119 for a root sitting on pole o).
template <int KP>
__device__ __forceinline__ double red_value(const ReducedView& rp, int64_t r, const double* ur,
                                            const XtCol<KP>& cp, double gap) {
  double t = 0.0;
#pragma unroll
  for (int c = 0; c < KP; ++c) t = fma(ur[c], cp.y[c], t);
  const double dr = rp.d[r];
  if (cp.mode == 0) return t * rcp64((dr - cp.dob) - cp.del);
  if (cp.mode == 2) return (r == cp.o) ? 1.0 : 0.0;
  // bordered system: xi on the rows of the pole, -(u_r . z)/((d_r - v) - delta)
  const double* cd = cp.cd;
  const int64_t r0 = (int64_t)cd[2 * KP], nr = (int64_t)cd[2 * KP + 1];
  if (r >= r0 && r < r0 + nr) return cd[KP + (r - r0)];
  double tz = 0.0;
#pragma unroll
  for (int c = 0; c < KP; ++c) tz = fma(ur[c], cd[c], tz);
  (void)gap;
  return -tz / ((dr - cd[2 * KP + 3]) - cd[2 * KP + 2]);
}

constexpr int kXtThreads = 256;
constexpr int kXtCols = 16;

// One CTA = 256 original indices x 16 columns. Each thread loads its row of U
// once and produces 16 entries of Xt (coalesced stores along the row index);
// squared norms are reduced per CTA and finished by xt_norm_kernel in a
// fixed order (deterministic).
template <int KP>
__global__ void __launch_bounds__(kXtThreads) xt_tile_kernel(
    ReducedView rp, int64_t n, const int* __restrict__ ckind, const int64_t* __restrict__ cpay,
    const int64_t* __restrict__ origin, const double* __restrict__ delta,
    const int* __restrict__ flags, const double* __restrict__ yall,
    const double* __restrict__ colldir, const int* __restrict__ collok,
    const int64_t* __restrict__ orig_map, const int64_t* __restrict__ dec_src,
    const int64_t* __restrict__ gstart, const int64_t* __restrict__ glen,
    const int64_t* __restrict__ hoff, const double* __restrict__ hbuf,
    const int64_t* __restrict__ rank, const int64_t* __restrict__ off_red, double gap,
    int64_t c0, int64_t c1, double* __restrict__ xt, double* __restrict__ part) {
  __shared__ XtCol<KP> cols[kXtCols];
  __shared__ double red[kXtThreads / 32][kXtCols];
  const int64_t cb = c0 + (int64_t)blockIdx.y * kXtCols;
  if (threadIdx.x < kXtCols) {
    XtCol<KP>& cp = cols[threadIdx.x];
    const int64_t c = cb + threadIdx.x;
    if (c >= c1) {
      cp.kind = -1;
    } else {
      cp.kind = ckind[c];
      const int64_t pay = cpay[c];
      if (cp.kind == 0) {
        const int64_t j = pay;
        cp.o = origin[j];
        cp.dob = rp.d[cp.o];
        cp.del = delta[j];
        const bool coll = (flags[j] & 1) != 0;
        cp.mode = (collok[j] == 1) ? 1 : ((collok[j] == 2 && coll) ? 2 : 0);
        cp.cd = colldir + j * kCollStride<KP>;
        for (int q = 0; q <= KP; ++q) cp.y[q] = (q < KP) ? yall[j * KP + q] : 0.0;
      } else {
        const int64_t src = dec_src[pay];
        if (cp.kind == 1) {
          cp.o = src;
        } else {
          const int64_t code = -(src + 2);
          cp.o = code / 65536;
          cp.t = code % 65536;
        }
      }
    }
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * kXtThreads + threadIdx.x;
  const bool valid = i < n;
  const int64_t r = valid ? orig_map[i] : -1;
  double ur[KP];
  if (r >= 0) {
    if constexpr (KP >= 2) {
#pragma unroll
      for (int c = 0; c < KP; c += 2) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(rp.u + r * KP + c));
        ur[c] = v.x;
        ur[c + 1] = v.y;
      }
    } else {
      ur[0] = rp.u[r];
    }
  }
  double ss[kXtCols];
#pragma unroll
  for (int q = 0; q < kXtCols; ++q) {
    const XtCol<KP>& cp = cols[q];
    double x = 0.0;
    if (cp.kind == 0) {
      if (r >= 0) {
        x = red_value<KP>(rp, r, ur, cp, gap);
      } else if (r <= -2) {  // member of a compressed run: rotate back
        const int64_t g = -2 - r;
        const int64_t s0 = gstart[g], m = glen[g];
        const double* H = hbuf + hoff[g];
        for (int64_t tt = 0; tt < rank[g]; ++tt) {
          const int64_t rr = off_red[g] + tt;
          double uu[KP];
#pragma unroll
          for (int c = 0; c < KP; ++c) uu[c] = rp.u[rr * KP + c];
          x += H[tt * m + (i - s0)] * red_value<KP>(rp, rr, uu, cp, gap);
        }
      }
    } else if (cp.kind == 1) {
      x = (i == cp.o) ? 1.0 : 0.0;
    } else if (cp.kind == 2) {
      const int64_t s0 = gstart[cp.o], m = glen[cp.o];
      x = (i >= s0 && i < s0 + m) ? hbuf[hoff[cp.o] + cp.t * m + (i - s0)] : 0.0;
    }
    if (valid && cp.kind >= 0) __stcs(xt + (cb + q - c0) * n + i, x);
    ss[q] = x * x;
  }
  // per-CTA column sums (fixed order: warp shuffles, then warps 0..7)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < kXtCols; ++q) {
    const double v = warp_sum(ss[q]);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < kXtCols) {
    double tsum = 0.0;
    for (int w = 0; w < kXtThreads / 32; ++w) tsum += red[w][threadIdx.x];
    const int64_t c = cb + threadIdx.x;
    if (c < c1) part[(c - c0) * gridDim.x + blockIdx.x] = tsum;
  }
}

__global__ void xt_norm_kernel(const double* __restrict__ part, int64_t nchunks, int64_t c0,
                               int64_t c1, const int* __restrict__ ckind,
                               double* __restrict__ colscale, int* __restrict__ cmode) {
  const int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c1) return;
  const int kind = ckind[c];
  double s = 0.0;
  for (int64_t b = 0; b < nchunks; ++b) s += part[(c - c0) * nchunks + b];
  colscale[c - c0] = (kind == 0 && s > 0.0) ? 1.0 / sqrt(s) : 1.0;
  cmode[c - c0] = (kind != 1);  // sign rule on computed columns (eigvec.cpp:340-347)
}

// K4 v2: one CTA = 64 original indices x 64 columns. The dot products
// (U y)_r of the whole tile are a 64 x 64 x KP register-blocked product from
// shared memory (4 x 4 entries per thread, LDS.128 operands); the epilogue
// divides by (d_r - d_o) - delta (one MUFU reciprocal + Newton per entry),
// stages the tile transposed in shared memory for coalesced streaming stores
// of Xt rows, and leaves per-tile column sums of squares (fixed order). Tiles
// that touch collided roots, unit / rotation columns or rows of compressed
// runs take the per-entry path of xt_tile_kernel.
constexpr int kXt2 = 64;

template <int KP>
struct Xt2Smem {
  static constexpr int YS = KP + 2;  // padded row stride: conflict-free LDS.128
  double ut[kXt2 * YS];
  double yt[kXt2 * YS];
  double out[kXt2 * (kXt2 + 1)];
  double ss[16 * kXt2];
  double dr[kXt2], cdob[kXt2], cdel[kXt2];
  int64_t row[kXt2], co[kXt2], ct[kXt2], cj[kXt2];
  int ckind[kXt2], cmode[kXt2];
  int special;
};

template <int KP>
__global__ void __launch_bounds__(256, 2) xt_tile64_kernel(
    ReducedView rp, int64_t n, const int* __restrict__ ckind, const int64_t* __restrict__ cpay,
    const int64_t* __restrict__ origin, const double* __restrict__ delta,
    const int* __restrict__ flags, const double* __restrict__ yall,
    const double* __restrict__ colldir, const int* __restrict__ collok,
    const int64_t* __restrict__ orig_map, const int64_t* __restrict__ dec_src,
    const int64_t* __restrict__ gstart, const int64_t* __restrict__ glen,
    const int64_t* __restrict__ hoff, const double* __restrict__ hbuf,
    const int64_t* __restrict__ rank, const int64_t* __restrict__ off_red, double gap,
    int64_t c0, int64_t c1, int64_t tiles_per_split, double* __restrict__ xt,
    double* __restrict__ part) {
  using S = Xt2Smem<KP>;
  constexpr int YS = S::YS;
  extern __shared__ __align__(16) unsigned char smraw[];
  S& sm = *reinterpret_cast<S*>(smraw);
  const int t = threadIdx.x;
  const int64_t cb = c0 + (int64_t)blockIdx.y * kXt2;
  const int64_t ntiles = cdiv_dev(n, kXt2);
  const int64_t tile0 = (int64_t)blockIdx.x * tiles_per_split;
  const int64_t tile1 = (tile0 + tiles_per_split < ntiles) ? tile0 + tiles_per_split : ntiles;
  if (t == 0) sm.special = 0;
  __syncthreads();
  // ---- this CTA's 64 column parameters, once
  if (t < kXt2) {
    const int64_t c = cb + t;
    int kind = -1, mode = 0;
    int64_t o = 0, tt = 0, cjj = -1;
    double dob = 0.0, del = 0.0;
    double* y = sm.yt + t * YS;
    for (int q = 0; q < YS; ++q) y[q] = 0.0;
    if (c < c1) {
      kind = ckind[c];
      const int64_t pay = cpay[c];
      if (kind == 0) {
        const int64_t j = pay;
        o = origin[j];
        dob = rp.d[o];
        del = delta[j];
        const bool coll = (flags[j] & 1) != 0;
        mode = (collok[j] == 1) ? 1 : ((collok[j] == 2 && coll) ? 2 : 0);
        cjj = j;
        for (int q = 0; q <= KP; ++q) y[q] = (q < KP) ? yall[j * KP + q] : 0.0;
      } else {
        const int64_t src = dec_src[pay];
        if (kind == 1) {
          o = src;
        } else {
          const int64_t code = -(src + 2);
          o = code / 65536;
          tt = code % 65536;
        }
      }
      if (kind != 0 || mode != 0) atomicOr(&sm.special, 1);
    }
    sm.ckind[t] = kind;
    sm.cmode[t] = mode;
    sm.cj[t] = cjj;
    sm.co[t] = o;
    sm.ct[t] = tt;
    sm.cdob[t] = dob;
    sm.cdel[t] = del;
  }
  __syncthreads();
  const int cols_special = sm.special;
  const int tr = t >> 4, tc = t & 15;
  double ssum[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t tile = tile0; tile < tile1; ++tile) {
    const int64_t i0 = tile * kXt2;
    // ---- row tile: reduced index, pole and U row of 64 original indices
    if (t < kXt2) {
      const int64_t i = i0 + t;
      const int64_t r = (i < n) ? orig_map[i] : -1;
      sm.row[t] = r;
      sm.dr[t] = (r >= 0) ? rp.d[r] : 0.0;
    }
    if (t == 0) sm.special = cols_special;
    __syncthreads();
    for (int e = t; e < kXt2 * YS; e += 256) {
      const int rr = e / YS, q = e - rr * YS;
      const int64_t r = sm.row[rr];
      sm.ut[e] = (r >= 0 && q < KP) ? rp.u[r * KP + q] : 0.0;
    }
    if (t < kXt2 && sm.row[t] <= -2) atomicOr(&sm.special, 1);
    __syncthreads();
    if (!sm.special) {
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
      if constexpr (KP >= 2) {
#pragma unroll
        for (int c = 0; c < KP; c += 2) {
          double2 ua[4], yb[4];
#pragma unroll
          for (int a = 0; a < 4; ++a)
            ua[a] = *reinterpret_cast<const double2*>(sm.ut + (tr + 16 * a) * YS + c);
#pragma unroll
          for (int b = 0; b < 4; ++b)
            yb[b] = *reinterpret_cast<const double2*>(sm.yt + (tc + 16 * b) * YS + c);
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              acc[a][b] = fma(ua[a].x, yb[b].x, acc[a][b]);
              acc[a][b] = fma(ua[a].y, yb[b].y, acc[a][b]);
            }
        }
      } else {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b)
            acc[a][b] = sm.ut[(tr + 16 * a) * YS] * sm.yt[(tc + 16 * b) * YS];
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int rr = tr + 16 * a;
        const bool live = sm.row[rr] >= 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int q = tc + 16 * b;
          double x = 0.0;
          if (live && sm.ckind[q] == 0)
            x = acc[a][b] * rcp64((sm.dr[rr] - sm.cdob[q]) - sm.cdel[q]);
          sm.out[q * (kXt2 + 1) + rr] = x;
          ssum[b] = fma(x, x, ssum[b]);
        }
      }
    } else {
      // per-entry path (xt_tile_kernel semantics)
      for (int a = 0; a < 4; ++a) {
        const int rr = tr + 16 * a;
        const int64_t i = i0 + rr;
        const int64_t r = sm.row[rr];
        for (int b = 0; b < 4; ++b) {
          const int q = tc + 16 * b;
          XtCol<KP> cp;
          cp.kind = sm.ckind[q];
          cp.mode = sm.cmode[q];
          cp.o = sm.co[q];
          cp.t = sm.ct[q];
          cp.dob = sm.cdob[q];
          cp.del = sm.cdel[q];
          cp.cd = colldir + (sm.cj[q] >= 0 ? sm.cj[q] : 0) * kCollStride<KP>;
          for (int c = 0; c <= KP; ++c) cp.y[c] = sm.yt[q * YS + c];
          double x = 0.0;
          if (i < n) {
            if (cp.kind == 0) {
              if (r >= 0) {
                double ur[KP];
                for (int c = 0; c < KP; ++c) ur[c] = sm.ut[rr * YS + c];
                x = red_value<KP>(rp, r, ur, cp, gap);
              } else if (r <= -2) {  // member of a compressed run: rotate back
                const int64_t g = -2 - r;
                const int64_t s0 = gstart[g], m = glen[g];
                const double* H = hbuf + hoff[g];
                for (int64_t k2 = 0; k2 < rank[g]; ++k2) {
                  const int64_t r2 = off_red[g] + k2;
                  double uu[KP];
                  for (int c = 0; c < KP; ++c) uu[c] = rp.u[r2 * KP + c];
                  x += H[k2 * m + (i - s0)] * red_value<KP>(rp, r2, uu, cp, gap);
                }
              }
            } else if (cp.kind == 1) {
              x = (i == cp.o) ? 1.0 : 0.0;
            } else if (cp.kind == 2) {
              const int64_t s0 = gstart[cp.o], m = glen[cp.o];
              x = (i >= s0 && i < s0 + m) ? hbuf[hoff[cp.o] + cp.t * m + (i - s0)] : 0.0;
            }
          }
          sm.out[q * (kXt2 + 1) + rr] = x;
          ssum[b] = fma(x, x, ssum[b]);
        }
      }
    }
    __syncthreads();
    // coalesced streaming stores: a warp writes 32 consecutive rows of a column
    for (int e = t; e < kXt2 * kXt2; e += 256) {
      const int q = e >> 6, rr = e & 63;
      const int64_t c = cb + q, i = i0 + rr;
      if (c < c1 && i < n) __stcs(xt + (c - c0) * n + i, sm.out[q * (kXt2 + 1) + rr]);
    }
  }
  // column sums of squares: thread (tr, tc) holds rows tr, tr+16, .. of
  // columns tc + 16 b over this CTA's tiles; combine over tr in order
  __syncthreads();
#pragma unroll
  for (int b = 0; b < 4; ++b) sm.ss[tr * kXt2 + tc + 16 * b] = ssum[b];
  __syncthreads();
  if (t < kXt2) {
    double s2 = 0.0;
    for (int w = 0; w < 16; ++w) s2 += sm.ss[w * kXt2 + t];
    const int64_t c = cb + t;
    if (c < c1) part[(c - c0) * gridDim.x + blockIdx.x] = s2;
  }
}

// K4 v3 (plans without compressed runs: every column is a root -- by the
// formula, the bordered-system vector of a collided / near-pole root, or its
// e_o fallback -- or a unit vector): lane = original index, R rows per
// thread (rows lane + 32 a of the warp's block), 64 columns per CTA with
// their y in shared memory (LDS.128 broadcasts, each reused for R rows), Xt
// written straight from registers (warp-coalesced rows), column sums of
// squares staged per batch of 8 columns and reduced in a fixed order. Other
// plans use xt_tile64_kernel, whose tiles fall back to the general rules.
template <int KP>
struct XtRowsCfg {
  static constexpr int R = KP >= 32 ? 1 : (KP >= 16 ? 2 : 4);  // rows per thread (registers)
  static constexpr int ROWS = 8 * 32 * R;           // rows per CTA
  static constexpr int YS = KP + 2;
};

template <int KP>
__global__ void __launch_bounds__(256, KP >= 32 ? 1 : 2) xt_rows_kernel(
    ReducedView rp, int64_t n, const int* __restrict__ ckind, const int64_t* __restrict__ cpay,
    const int64_t* __restrict__ origin, const double* __restrict__ delta,
    const int* __restrict__ flags, const double* __restrict__ yall,
    const double* __restrict__ colldir, const int* __restrict__ collok,
    const int64_t* __restrict__ orig_map, const int64_t* __restrict__ dec_src,
    const int64_t* __restrict__ gstart, const int64_t* __restrict__ glen,
    const int64_t* __restrict__ hoff, const double* __restrict__ hbuf,
    const int64_t* __restrict__ rank, const int64_t* __restrict__ off_red, double gap,
    int64_t c0, int64_t c1, double* __restrict__ xt, double* __restrict__ part) {
  using RC = XtRowsCfg<KP>;
  constexpr int R = RC::R, YS = RC::YS;
  __shared__ __align__(16) double yt[kXt2 * YS];
  __shared__ double cdob[kXt2], cdel[kXt2];
  __shared__ int64_t co[kXt2], ct[kXt2], cj[kXt2];
  __shared__ int ck[kXt2], cm[kXt2];
  __shared__ double red[kXt2];
  __shared__ double sb[8][256];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t cb = c0 + (int64_t)blockIdx.y * kXt2;
  if (t < kXt2) {
    const int64_t c = cb + t;
    int kind = -1, mode = 0;
    int64_t o = 0, tt = 0, jr = 0;
    double dob = 0.0, del = 0.0;
    double* y = yt + t * YS;
    for (int q = 0; q < YS; ++q) y[q] = 0.0;
    if (c < c1) {
      kind = ckind ? ckind[c] : 0;
      const int64_t pay = ckind ? cpay[c] : c;
      if (kind == 0) {
        const int64_t j = pay;
        jr = j;
        o = origin[j];
        dob = rp.d[o];
        del = delta[j];
        const bool coll = (flags[j] & 1) != 0;
        mode = (collok[j] == 1) ? 1 : ((collok[j] == 2 && coll) ? 2 : 0);
        if (mode == 1)  // the bordered-system vector z (as y)
          for (int q = 0; q <= KP; ++q) y[q] = (q < KP) ? colldir[j * kCollStride<KP> + q] : 0.0;
        else
          for (int q = 0; q <= KP; ++q) y[q] = (q < KP) ? yall[j * KP + q] : 0.0;
      } else {
        const int64_t src = dec_src[pay];
        if (kind == 1) {
          o = src;
        } else {
          const int64_t code = -(src + 2);
          o = code / 65536;
          tt = code % 65536;
        }
      }
    }
    ck[t] = kind;
    cm[t] = mode;
    co[t] = o;
    ct[t] = tt;
    cj[t] = jr;
    cdob[t] = dob;
    cdel[t] = del;
  }
  // this thread's rows
  const int64_t ib = (int64_t)blockIdx.x * RC::ROWS + warp * 32 * R + lane;
  int64_t rr[R];
  double ur[R][KP], drow[R];
#pragma unroll
  for (int a = 0; a < R; ++a) {
    const int64_t i = ib + 32 * a;
    rr[a] = (i < n) ? orig_map[i] : -1;
    drow[a] = (rr[a] >= 0) ? rp.d[rr[a]] : 0.0;
    if constexpr (KP >= 2) {
#pragma unroll
      for (int c = 0; c < KP; c += 2) {
        const double2 v = (rr[a] >= 0) ? __ldg(reinterpret_cast<const double2*>(rp.u + rr[a] * KP + c))
                                      : make_double2(0.0, 0.0);
        ur[a][c] = v.x;
        ur[a][c + 1] = v.y;
      }
    } else {
      ur[a][0] = (rr[a] >= 0) ? rp.u[rr[a]] : 0.0;
    }
  }
  __syncthreads();
  // columns in batches of 8: per-thread sums of squares staged in shared
  // memory and reduced once per batch (warp w takes column q0 + w; fixed order).
  // Entries of special columns or rows take the general rules.
  for (int q0 = 0; q0 < kXt2; q0 += 8) {
    double s2[8];
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) s2[qq] = 0.0;
#pragma unroll
    for (int qq = 0; qq < 8; qq += 2) {
      const int q = q0 + qq;
      // two columns, even/odd partial dot products: 4 R independent chains
      double e0[R], o0[R], e1[R], o1[R];
#pragma unroll
      for (int a = 0; a < R; ++a) e0[a] = o0[a] = e1[a] = o1[a] = 0.0;
      if constexpr (KP >= 2) {
#pragma unroll
        for (int cc = 0; cc < KP; cc += 2) {
          const double2 y0 = *reinterpret_cast<const double2*>(yt + q * YS + cc);
          const double2 y1 = *reinterpret_cast<const double2*>(yt + (q + 1) * YS + cc);
#pragma unroll
          for (int a = 0; a < R; ++a) {
            e0[a] = fma(ur[a][cc], y0.x, e0[a]);
            o0[a] = fma(ur[a][cc + 1], y0.y, o0[a]);
            e1[a] = fma(ur[a][cc], y1.x, e1[a]);
            o1[a] = fma(ur[a][cc + 1], y1.y, o1[a]);
          }
        }
      } else {
#pragma unroll
        for (int a = 0; a < R; ++a) {
          e0[a] = ur[a][0] * yt[q * YS];
          e1[a] = ur[a][0] * yt[(q + 1) * YS];
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int qh = q + h;
        const int64_t c = cb + qh;
        const int kind = ck[qh];
        const bool colfast = kind == 0;
        const double dob = cdob[qh], del = cdel[qh];
#pragma unroll
        for (int a = 0; a < R; ++a) {
          const double dot = h ? (e1[a] + o1[a]) : (e0[a] + o0[a]);
          const int64_t i = ib + 32 * a;
          double x;
          if (colfast && cm[qh] == 0) {
            x = (rr[a] >= 0) ? dot * rcp64((drow[a] - dob) - del) : 0.0;
          } else if (colfast && cm[qh] == 2) {  // collided fallback e_o
            x = (rr[a] >= 0 && rr[a] == co[qh]) ? 1.0 : 0.0;
          } else if (colfast) {  // bordered system (red_value mode 1); dot = u_r . z
            const double* cd = colldir + cj[qh] * kCollStride<KP>;
            const int64_t r0 = (int64_t)cd[2 * KP], nr0 = (int64_t)cd[2 * KP + 1];
            if (rr[a] < 0) x = 0.0;
            else if (rr[a] >= r0 && rr[a] < r0 + nr0) x = cd[KP + (rr[a] - r0)];
            else x = -dot / ((drow[a] - cd[2 * KP + 3]) - cd[2 * KP + 2]);
          } else {  // unit column of an unchanged pair
            x = (kind == 1 && i == co[qh]) ? 1.0 : 0.0;
          }
          if (c < c1 && i < n) __stcs(xt + (c - c0) * n + i, x);
          s2[qq + h] = fma(x, x, s2[qq + h]);
        }
      }
    }
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) sb[qq][t] = s2[qq];
    __syncthreads();
    {
      double v = 0.0;
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) v += sb[warp][lane * 8 + k2];
      v = warp_sum(v);
      if (lane == 0) red[q0 + warp] = v;
    }
    __syncthreads();
  }
  if (t < kXt2) {
    const int64_t c = cb + t;
    if (c < c1) part[(c - c0) * gridDim.x + blockIdx.x] = red[t];
  }
}

// K4 v4 (plans without compressed runs, KP >= 4): the dot products
// P[c][i] = y_c . u_r(i) on the FP64 tensor pipe. One CTA = 128 columns
// (16 m-tiles of 8 columns, two per warp) x 256 original rows (32 n-tiles);
// A fragments (y of the warp's columns) stay in registers, B fragments come
// from the CTA's U rows staged in shared memory (rows padded to KP + 4
// doubles: conflict-free fragment loads). A lane holds P for column
// 8 m + lane / 4 and rows 8 nt + 2 (lane % 4) + {0, 1}: the epilogue divides
// by (d_r - d_o) - delta (or applies the bordered / unit rules of special
// columns, as xt_rows_kernel) and stores the row pair as one 16-byte store
// (a warp store fills 8 columns x 64 contiguous bytes). Column sums of
// squares: per lane, then over the 4 lanes of a column (butterfly), one
// partial per (column, CTA row block) reduced in order by xt_norm_kernel.
constexpr int kXtmCols = 128, kXtmRows = 256;

template <int KP>
struct XtmSmem {
  static constexpr int LDU = KP + 4;
  double ut[kXtmRows * LDU];
  double yt[kXtmCols * LDU];
  double drow[kXtmRows];
  int64_t rr[kXtmRows];
  double cdob[kXtmCols], cdel[kXtmCols];
  int64_t co[kXtmCols], cj[kXtmCols];
  int ck[kXtmCols], cm[kXtmCols];
};

template <int KP>
__global__ void __launch_bounds__(256, 3) xt_mma_kernel(
    ReducedView rp, int64_t n, const int* __restrict__ ckind, const int64_t* __restrict__ cpay,
    const int64_t* __restrict__ origin, const double* __restrict__ delta,
    const int* __restrict__ flags, const double* __restrict__ yall,
    const double* __restrict__ colldir, const int* __restrict__ collok,
    const int64_t* __restrict__ orig_map, const int64_t* __restrict__ dec_src, int64_t c0,
    int64_t c1, int64_t ldx, double* __restrict__ xt, double* __restrict__ part) {
  // Compact mode (orig_map == nullptr, ckind == nullptr): rows are the n
  // reduced rows themselves and columns c are roots (payload j = c); the
  // back-transform multiplies by the gathered Q~ of the reduced rows.
  using SM = XtmSmem<KP>;
  constexpr int LDU = SM::LDU, KC = KP / 4;
  extern __shared__ __align__(16) double xsm[];
  SM& sm = *reinterpret_cast<SM*>(xsm);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int t4 = lane & 3, g8 = lane >> 2;
  const int64_t cb = c0 + (int64_t)blockIdx.y * kXtmCols;
  const int64_t ib = (int64_t)blockIdx.x * kXtmRows;
  // column parameters (as xt_rows_kernel)
  if (t < kXtmCols) {
    const int64_t c = cb + t;
    int kind = -1, mode = 0;
    int64_t o = 0, jr = 0;
    double dob = 0.0, del = 0.0;
    double* y = sm.yt + t * LDU;
    for (int q = 0; q < KP; ++q) y[q] = 0.0;
    if (c < c1) {
      kind = ckind ? ckind[c] : 0;
      const int64_t pay = ckind ? cpay[c] : c;
      if (kind == 0) {
        const int64_t j = pay;
        jr = j;
        o = origin[j];
        dob = rp.d[o];
        del = delta[j];
        const bool coll = (flags[j] & 1) != 0;
        mode = (collok[j] == 1) ? 1 : ((collok[j] == 2 && coll) ? 2 : 0);
        const double* src = (mode == 1) ? colldir + j * kCollStride<KP> : yall + j * KP;
        for (int q = 0; q < KP; ++q) y[q] = src[q];
      } else if (kind == 1) {
        o = dec_src[pay];
      }
    }
    sm.ck[t] = kind;
    sm.cm[t] = mode;
    sm.co[t] = o;
    sm.cj[t] = jr;
    sm.cdob[t] = dob;
    sm.cdel[t] = del;
  }
  // rows: reduced index, pole value, u row (zero outside the reduced problem)
  for (int q = t; q < kXtmRows; q += 256) {
    const int64_t i = ib + q;
    const int64_t r = (i < n) ? (orig_map ? orig_map[i] : i) : -1;
    sm.rr[q] = r;
    sm.drow[q] = (r >= 0) ? rp.d[r] : 0.0;
  }
  __syncthreads();
  for (int q = t; q < kXtmRows * (KP / 2); q += 256) {
    const int row = q / (KP / 2), c2 = q % (KP / 2);
    const int64_t r = sm.rr[row];
    const double2 v = (r >= 0) ? __ldg(reinterpret_cast<const double2*>(rp.u + r * KP) + c2)
                               : make_double2(0.0, 0.0);
    *reinterpret_cast<double2*>(sm.ut + row * LDU + 2 * c2) = v;
  }
  __syncthreads();
  // this lane's two columns (m-tiles 2 warp, 2 warp + 1)
  double af[2][KC];
  int qc[2];
  bool fast[2];
  double s2[2] = {0.0, 0.0};
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    qc[m] = 8 * (2 * warp + m) + g8;
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) af[m][kc] = sm.yt[qc[m] * LDU + 4 * kc + t4];
    fast[m] = sm.ck[qc[m]] == 0 && sm.cm[qc[m]] == 0;
  }
  const bool vec = (ldx % 2) == 0;
#pragma unroll 2
  for (int nt = 0; nt < kXtmRows / 8; ++nt) {
    double bf[KC];
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) bf[kc] = sm.ut[(8 * nt + g8) * LDU + 4 * kc + t4];
    const int q0 = 8 * nt + 2 * t4;  // this lane's rows q0, q0 + 1
    const double d0 = sm.drow[q0], d1 = sm.drow[q0 + 1];
    const int64_t r0 = sm.rr[q0], r1 = sm.rr[q0 + 1];
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      double p0 = 0.0, p1 = 0.0;
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) dmma(p0, p1, af[m][kc], bf[kc]);
      const int qm = qc[m];
      const int64_t c = cb + qm;
      double x0, x1;
      if (fast[m]) {
        const double dob = sm.cdob[qm], del = sm.cdel[qm];
        x0 = (r0 >= 0) ? p0 * rcp64((d0 - dob) - del) : 0.0;
        x1 = (r1 >= 0) ? p1 * rcp64((d1 - dob) - del) : 0.0;
      } else {
        const int kind = sm.ck[qm], mode = sm.cm[qm];
        const int64_t co = sm.co[qm];
        double xv[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t r = h ? r1 : r0;
          const int64_t i = ib + q0 + h;
          const double dot = h ? p1 : p0, dr = h ? d1 : d0;
          double x = 0.0;
          if (kind == 0 && mode == 2) {  // collided fallback e_o
            x = (r >= 0 && r == co) ? 1.0 : 0.0;
          } else if (kind == 0) {  // bordered system; dot = u_r . z
            const double* cd = colldir + sm.cj[qm] * kCollStride<KP>;
            const int64_t rb0 = (int64_t)cd[2 * KP], nr0 = (int64_t)cd[2 * KP + 1];
            if (r < 0) x = 0.0;
            else if (r >= rb0 && r < rb0 + nr0) x = cd[KP + (r - rb0)];
            else x = -dot / ((dr - cd[2 * KP + 3]) - cd[2 * KP + 2]);
          } else if (kind == 1) {  // unit column of an unchanged pair
            x = (i == co) ? 1.0 : 0.0;
          }
          xv[h] = x;
        }
        x0 = xv[0];
        x1 = xv[1];
      }
      const int64_t i = ib + q0;
      if (c < c1) {
        double* dst = xt + (c - c0) * ldx + i;
        if (vec && i + 1 < n) {
          __stcs(reinterpret_cast<double2*>(dst), make_double2(x0, x1));
        } else {
          if (i < n) __stcs(dst, x0);
          if (i + 1 < n) __stcs(dst + 1, x1);
        }
      }
      s2[m] = fma(x0, x0, s2[m]);
      s2[m] = fma(x1, x1, s2[m]);
    }
  }
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    s2[m] += __shfl_xor_sync(0xffffffffu, s2[m], 1);
    s2[m] += __shfl_xor_sync(0xffffffffu, s2[m], 2);
    const int64_t c = cb + qc[m];
    if (t4 == 0 && c < c1) part[(c - c0) * gridDim.x + blockIdx.x] = s2[m];
  }
}

template <int KP>
void launch_xt(const Plan& p, const RootRecords& roots, const Columns& cols, const double* colldir,
               const int* collok, bool general, int64_t c0, int64_t c1, double* xt,
               double* colscale, int* cmode, DeviceScratch& ws, cudaStream_t st) {
  const double gap = kPoleMergeRelGap * p.scale;
  static int v1 = -1;  // EIGMOD_B200_XT=v1 selects the one-row-per-thread kernel
  if (v1 < 0) {
    const char* e = std::getenv("EIGMOD_B200_XT");
    v1 = (e && std::string(e) == "v1");
  }
  static int v2 = -1;  // EIGMOD_B200_XT=v2 selects the 64 x 64 smem-tile kernel
  if (v2 < 0) {
    const char* e = std::getenv("EIGMOD_B200_XT");
    v2 = (e && std::string(e) == "v2");
  }
  static int v3 = -1;  // EIGMOD_B200_XT=v3 selects the DFMA row kernel
  if (v3 < 0) {
    const char* e = std::getenv("EIGMOD_B200_XT");
    v3 = (e && std::string(e) == "v3");
  }
  if constexpr (KP >= 4) {
    if (!v1 && !v2 && !v3 && p.nmulti == 0) {
      const int64_t nchunks = cdiv(p.n, kXtmRows);
      double* part = ws.get_f64("xt_part", (size_t)nchunks * (c1 - c0));
      dim3 grid((unsigned)nchunks, (unsigned)cdiv(c1 - c0, kXtmCols));
      const size_t sm = sizeof(XtmSmem<KP>);
      EIGB_CUDA(cudaFuncSetAttribute(xt_mma_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sm));
      xt_mma_kernel<KP><<<grid, 256, sm, st>>>(p.view(), p.n, cols.kind, cols.payload,
                                               roots.origin, roots.delta, roots.flags, roots.y,
                                               colldir, collok, p.orig_map, p.dec_src, c0, c1,
                                               p.n, xt, part);
      EIGB_LAUNCH_CHECK();
      xt_norm_kernel<<<(unsigned)cdiv(c1 - c0, 128), 128, 0, st>>>(part, nchunks, c0, c1,
                                                                   cols.kind, colscale, cmode);
      EIGB_LAUNCH_CHECK();
      return;
    }
  }
  if (!v1 && !v2 && p.nmulti == 0) {
    using RC = XtRowsCfg<KP>;
    const int64_t nchunks = cdiv(p.n, RC::ROWS);
    double* part = ws.get_f64("xt_part", (size_t)nchunks * (c1 - c0));
    dim3 grid((unsigned)nchunks, (unsigned)cdiv(c1 - c0, kXt2));
    xt_rows_kernel<KP><<<grid, 256, 0, st>>>(
        p.view(), p.n, cols.kind, cols.payload, roots.origin, roots.delta, roots.flags, roots.y,
        colldir, collok, p.orig_map, p.dec_src, p.gstart, p.glen, p.hoff, p.hbuf, p.rank,
        p.off_red, gap, c0, c1, xt, part);
    EIGB_LAUNCH_CHECK();
    xt_norm_kernel<<<(unsigned)cdiv(c1 - c0, 128), 128, 0, st>>>(part, nchunks, c0, c1,
                                                                 cols.kind, colscale, cmode);
    EIGB_LAUNCH_CHECK();
    return;
  }
  if (!v1) {
    // CTAs keep their 64 columns and sweep a contiguous share of the row
    // tiles: the column setup is paid once per CTA, not once per tile. The
    // split depends on n and the column count only (deterministic sums).
    const int64_t ntiles = cdiv(p.n, kXt2), ctiles = cdiv(c1 - c0, kXt2);
    const int64_t splits = std::max<int64_t>(1, std::min<int64_t>(ntiles, cdiv(2368, ctiles)));
    const int64_t per = cdiv(ntiles, splits);
    const int64_t nchunks = cdiv(ntiles, per);
    double* part = ws.get_f64("xt_part", (size_t)nchunks * (c1 - c0));
    dim3 grid((unsigned)nchunks, (unsigned)ctiles);
    const size_t sm = sizeof(Xt2Smem<KP>);
    EIGB_CUDA(cudaFuncSetAttribute(xt_tile64_kernel<KP>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    xt_tile64_kernel<KP><<<grid, 256, sm, st>>>(
        p.view(), p.n, cols.kind, cols.payload, roots.origin, roots.delta, roots.flags, roots.y,
        colldir, collok, p.orig_map, p.dec_src, p.gstart, p.glen, p.hoff, p.hbuf, p.rank,
        p.off_red, gap, c0, c1, per, xt, part);
    EIGB_LAUNCH_CHECK();
    xt_norm_kernel<<<(unsigned)cdiv(c1 - c0, 128), 128, 0, st>>>(part, nchunks, c0, c1,
                                                                 cols.kind, colscale, cmode);
    EIGB_LAUNCH_CHECK();
    return;
  }
  const int64_t nchunks = cdiv(p.n, kXtThreads);
  double* part = ws.get_f64("xt_part", (size_t)nchunks * (c1 - c0));
  dim3 grid((unsigned)nchunks, (unsigned)cdiv(c1 - c0, kXtCols));
  xt_tile_kernel<KP><<<grid, kXtThreads, 0, st>>>(
      p.view(), p.n, cols.kind, cols.payload, roots.origin, roots.delta, roots.flags, roots.y,
      colldir, collok, p.orig_map, p.dec_src, p.gstart, p.glen, p.hoff, p.hbuf, p.rank, p.off_red,
      gap, c0, c1, xt, part);
  EIGB_LAUNCH_CHECK();
  xt_norm_kernel<<<(unsigned)cdiv(c1 - c0, 128), 128, 0, st>>>(part, nchunks, c0, c1, cols.kind,
                                                               colscale, cmode);
  EIGB_LAUNCH_CHECK();
}

template <int KP>
void launch_collisions(const Plan& p, const RootRecords& roots, const int64_t* list, int64_t cnt,
                       const int* mark, const int* which, double* colldir, int* collok,
                       DeviceScratch& ws, cudaStream_t st) {
  using C = PassCfg<KP>;
  const int grid = (int)cdiv(cnt, 32);
  double* scratch = ws.get_f64("coll_scratch", (size_t)grid * 32 * 4 * (2 * KP) * (2 * KP));
  const size_t sm = sizeof(double) * C::SMEM_DOUBLES;
  const double gap = kPoleMergeRelGap * p.scale;
  // few batches: split each batch's pole pass over slices of >= 256 poles so
  // that about two CTAs per SM run it
  int dev = 0, sms = 148;
  EIGB_CUDA(cudaGetDevice(&dev));
  EIGB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int splits = (int)std::max<int64_t>(
      1, std::min<int64_t>(cdiv(p.nred, 256), (2 * sms) / grid));
  double* partial = nullptr;
  if (splits > 1) {
    partial = ws.get_f64("coll_partial", (size_t)grid * splits * C::RED_DOUBLES);
    EIGB_CUDA(cudaFuncSetAttribute(collision_pass_kernel<KP>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    collision_pass_kernel<KP><<<dim3(grid, splits), kPassThreads, sm, st>>>(
        p.view(), list, cnt, roots.origin, roots.delta, mark, gap, partial);
    EIGB_LAUNCH_CHECK();
  }
  EIGB_CUDA(cudaFuncSetAttribute(collision_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm));
  collision_kernel<KP><<<grid, kPassThreads, sm, st>>>(p.view(), list, cnt, roots.origin,
                                                       roots.delta, mark, which, gap, colldir,
                                                       collok, scratch, roots.y, partial, splits);
  EIGB_LAUNCH_CHECK();
}

}  // namespace

namespace {
// EIGMOD_B200_BORDERED_MULTI=0: collided roots only (diagnostics)
int bordered_multi() {
  static int allow_multi = -1;
  if (allow_multi < 0) {
    const char* e = std::getenv("EIGMOD_B200_BORDERED_MULTI");
    allow_multi = !(e && std::string(e) == "0");
  }
  return allow_multi;
}

__global__ void any_mark_kernel(const int* __restrict__ mark, int64_t nr, int* __restrict__ any) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < nr && mark[j]) atomicOr(any, 1);
}
}  // namespace

void merge_columns_dev(const Plan& p, const RootRecords& roots, Columns& cols, DeviceScratch& ws,
                       cudaStream_t st) {
  const int64_t nr = p.nred, nd = p.ndec, n = p.n;
  cols.kind = ws.get_i32("col_kind", n);
  cols.payload = ws.get_i64("col_payload", n);
  cols.value = ws.get_f64("col_value", n);
  const double* rv = roots.value;
  const int64_t* perm = nullptr;
  cols.nmarked = -1;
  if (nr > 0) {
    // Roots come out ascending from the count-certified brackets; ties within
    // an ulp can swap, so verify and fall back to a stable device sort. The
    // same round trip brings back how many roots need a bordered-system
    // vector (collision_vectors_dev skips its own when none do).
    int* bad = ws.get_i32("merge_bad", 2);
    EIGB_CUDA(cudaMemsetAsync(bad, 0, 8, st));
    if (nr > 1) {
      root_order_check_kernel<<<(unsigned)cdiv(nr, 256), 256, 0, st>>>(rv, nr, bad);
      EIGB_LAUNCH_CHECK();
    }
    int* mark = ws.get_i32("coll_mark", nr);
    int* which = ws.get_i32("coll_which", nr);
    int* collok = ws.get_i32("collok", nr);
    bordered_mark_kernel<<<(unsigned)cdiv(nr, 256), 256, 0, st>>>(
        p.d, p.ur, p.kp, nr, roots.origin, roots.delta, roots.flags, nr, mark, which, collok,
        bordered_multi());
    EIGB_LAUNCH_CHECK();
    any_mark_kernel<<<(unsigned)cdiv(nr, 256), 256, 0, st>>>(mark, nr, bad + 1);
    EIGB_LAUNCH_CHECK();
    int h[2] = {0, 0};
    EIGB_CUDA(cudaMemcpyAsync(h, bad, 8, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaStreamSynchronize(st));
    const int bad_h = h[0];
    cols.nmarked = h[1];
    if (bad_h) {
      double* sv = ws.get_f64("merge_sorted", nr);
      int64_t* pm = ws.get_i64("merge_perm", nr);
      EIGB_CUDA(cudaMemcpyAsync(sv, rv, 8 * nr, cudaMemcpyDeviceToDevice, st));
      thrust::sequence(thrust::cuda::par.on(st), thrust::device_ptr<int64_t>(pm),
                       thrust::device_ptr<int64_t>(pm + nr));
      thrust::stable_sort_by_key(thrust::cuda::par.on(st), thrust::device_ptr<double>(sv),
                                 thrust::device_ptr<double>(sv + nr),
                                 thrust::device_ptr<int64_t>(pm));
      rv = sv;
      perm = pm;
    }
  }
  merge_kernel<<<(unsigned)cdiv(nr + nd, 256), 256, 0, st>>>(rv, perm, nr, p.dec_val, p.dec_src,
                                                             nd, cols.kind, cols.payload,
                                                             cols.value);
  EIGB_LAUNCH_CHECK();
}

__global__ void column_roots_kernel(const int* __restrict__ ckind, const int64_t* __restrict__ cpay,
                                    int64_t c0, int64_t c1, int* __restrict__ need) {
  const int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < c1 && ckind[c] == 0) need[cpay[c]] = 1;
}

int64_t collision_vectors_dev(const Plan& p, const RootRecords& roots, const Columns& cols,
                              int64_t c0, int64_t c1, double* colldir, int* collok,
                              DeviceScratch& ws, cudaStream_t st) {
  const int64_t nr = p.nred;
  if (nr == 0) return 0;
  // only the roots whose columns [c0, c1) this call builds (a rank's block)
  int* need = ws.get_i32("coll_need", nr);
  EIGB_CUDA(cudaMemsetAsync(need, 0, 4 * nr, st));
  if (c1 > c0) {
    column_roots_kernel<<<(unsigned)cdiv(c1 - c0, 256), 256, 0, st>>>(cols.kind, cols.payload, c0,
                                                                      c1, need);
    EIGB_LAUNCH_CHECK();
  }
  int* mark = ws.get_i32("coll_mark", nr);
  int* which = ws.get_i32("coll_which", nr);
  if (cols.nmarked == 0) return 0;  // merge_columns_dev found no root to border (collok zeroed)
  bordered_mark_kernel<<<(unsigned)cdiv(nr, 256), 256, 0, st>>>(p.d, p.ur, p.kp, nr, roots.origin,
                                                                roots.delta, roots.flags, nr, mark,
                                                                which, collok, bordered_multi());
  EIGB_LAUNCH_CHECK();
  std::vector<int> mh(nr), nh(nr);
  EIGB_CUDA(cudaMemcpyAsync(mh.data(), mark, 4 * nr, cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaMemcpyAsync(nh.data(), need, 4 * nr, cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> list;
  for (int64_t j = 0; j < nr; ++j)
    if (mh[j] && nh[j]) list.push_back(j);
  if (list.empty()) return 0;
  int64_t* dl = ws.get_i64("coll_list", list.size());
  EIGB_CUDA(cudaMemcpyAsync(dl, list.data(), 8 * list.size(), cudaMemcpyHostToDevice, st));
  const int64_t cnt = (int64_t)list.size();
  switch (p.kp) {
    case 1: launch_collisions<1>(p, roots, dl, cnt, mark, which, colldir, collok, ws, st); break;
    case 2: launch_collisions<2>(p, roots, dl, cnt, mark, which, colldir, collok, ws, st); break;
    case 4: launch_collisions<4>(p, roots, dl, cnt, mark, which, colldir, collok, ws, st); break;
    case 8: launch_collisions<8>(p, roots, dl, cnt, mark, which, colldir, collok, ws, st); break;
    case 16: launch_collisions<16>(p, roots, dl, cnt, mark, which, colldir, collok, ws, st); break;
    case 32: launch_collisions<32>(p, roots, dl, cnt, mark, which, colldir, collok, ws, st); break;
  }
  return cnt;
}

void build_xt_dev(const Plan& p, const RootRecords& roots, const Columns& cols,
                  const double* colldir, const int* collok, int64_t ncollided, int64_t c0,
                  int64_t c1, double* xt, double* colscale, int* cmode, DeviceScratch& ws,
                  cudaStream_t st) {
  if (c1 <= c0) return;
  const bool general = p.nmulti > 0 || ncollided > 0;
  switch (p.kp) {
    case 1: launch_xt<1>(p, roots, cols, colldir, collok, general, c0, c1, xt, colscale, cmode, ws, st); break;
    case 2: launch_xt<2>(p, roots, cols, colldir, collok, general, c0, c1, xt, colscale, cmode, ws, st); break;
    case 4: launch_xt<4>(p, roots, cols, colldir, collok, general, c0, c1, xt, colscale, cmode, ws, st); break;
    case 8: launch_xt<8>(p, roots, cols, colldir, collok, general, c0, c1, xt, colscale, cmode, ws, st); break;
    case 16: launch_xt<16>(p, roots, cols, colldir, collok, general, c0, c1, xt, colscale, cmode, ws, st); break;
    case 32: launch_xt<32>(p, roots, cols, colldir, collok, general, c0, c1, xt, colscale, cmode, ws, st); break;
  }
}


// ---------------------------------------------------------------------------
// Compact back-transform (plans with decoupled columns). Every root column of
// X is zero on the unchanged rows and, on a compressed run, a combination of
// the run's rotated rows; so Q' = Q X splits into
//   Q'[:, decoupled e] = Q~[:, e]            (a copy or one run rotation)
//   Q'[:, roots]       = Q~_red X_red        (n x nred x nroot on DMMA)
// with Q~ = Q H (the runs' Householder rotations, eigvec.cpp:288-291 and the
// rotation rows of the plan) and X_red the root columns over the reduced
// rows. The reference multiplies by the dense n x n X (eigvec.cpp:285-339);
// the exact zeros it skips are 2 n (n^2 - nred^2) flops.

// Range of the roots / decoupled entries whose final columns lie in [c0, c1)
// (both contiguous: the merge is a stable merge by value), and each one's
// column relative to c0.
__global__ void compact_ranges_kernel(const int* __restrict__ ckind,
                                      const int64_t* __restrict__ cpay, int64_t c0, int64_t c1,
                                      unsigned long long* __restrict__ rng) {
  const int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c1) return;
  const int kind = ckind[c];
  const unsigned long long pay = (unsigned long long)cpay[c];
  const int slot = (kind == 0) ? 0 : 2;
  atomicMin(rng + slot, pay);
  atomicMax(rng + slot + 1, pay + 1);
}

__global__ void compact_pos_kernel(const int* __restrict__ ckind, const int64_t* __restrict__ cpay,
                                   int64_t c0, int64_t c1, int64_t j0, int64_t e0,
                                   int64_t* __restrict__ jpos, int64_t* __restrict__ epos,
                                   int* __restrict__ cmode) {
  const int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c1) return;
  const int kind = ckind[c];
  if (kind == 0) jpos[cpay[c] - j0] = c - c0;
  else epos[cpay[c] - e0] = c - c0;
  cmode[c - c0] = (kind != 1);  // sign rule on computed columns (eigvec.cpp:340-347)
}

// Q~ column of a source code: >= 0 the original column, <= -2 row t of group
// g's rotation (code = -(g * 65536 + t) - 2, deflate.cu assemble_reduced).
__device__ __forceinline__ double qtilde(const double* __restrict__ qrow, int64_t code,
                                         const int64_t* __restrict__ gstart,
                                         const int64_t* __restrict__ glen,
                                         const int64_t* __restrict__ hoff,
                                         const double* __restrict__ hbuf) {
  if (code >= 0) return qrow[code];
  const int64_t c2 = -(code + 2), g = c2 / 65536, t = c2 % 65536;
  const int64_t s0 = gstart[g], m = glen[g];
  const double* H = hbuf + hoff[g] + t * m;
  double v = 0.0;
  for (int64_t s = 0; s < m; ++s) v = fma(H[s], qrow[s0 + s], v);
  return v;
}

// One thread = one item (a reduced row -> column of Qa, or a decoupled entry
// -> its final column of Q') over the 128 rows of a row tile; consecutive
// items read consecutive columns of Q (coalesced) and write consecutive
// columns of Qa. Decoupled columns also leave their signed max per row tile
// (first row on ties) for sign_rule_dev, as the GEMM epilogue does.
constexpr int kGatherRows = 128;

__global__ void __launch_bounds__(256) gather_qtilde_kernel(
    const double* __restrict__ q, int64_t n, int64_t ldq_in, int64_t nred,
    const int64_t* __restrict__ red_src, int64_t ne, const int64_t* __restrict__ dec_src,
    int64_t e0, const int64_t* __restrict__ epos, const int64_t* __restrict__ gstart,
    const int64_t* __restrict__ glen, const int64_t* __restrict__ hoff,
    const double* __restrict__ hbuf, double* __restrict__ qa, int64_t lda,
    double* __restrict__ qout, int64_t ldo, double* __restrict__ tile_colmax, int64_t tcm_ld) {
  const int64_t item = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  if (item >= nred + ne) return;
  const int64_t tm = blockIdx.x, i0 = tm * kGatherRows;
  const int64_t i1 = (i0 + kGatherRows < n) ? i0 + kGatherRows : n;
  const bool red = item < nred;
  const int64_t code = red ? red_src[item] : dec_src[e0 + (item - nred)];
  double* dst = red ? qa + item : qout + epos[item - nred];
  const int64_t ldd = red ? lda : ldo;
  double best = 0.0;  // first row on ties: strict > in ascending row order
  if (code >= 0) {
    int64_t i = i0;
    for (; i + 4 <= i1; i += 4) {
      double v[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) v[h] = __ldcs(q + (i + h) * ldq_in + code);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        dst[(i + h) * ldd] = v[h];
        if (fabs(v[h]) > fabs(best)) best = v[h];
      }
    }
    for (; i < i1; ++i) {
      const double v = __ldcs(q + i * ldq_in + code);
      dst[i * ldd] = v;
      if (fabs(v) > fabs(best)) best = v;
    }
  } else {
    for (int64_t i = i0; i < i1; ++i) {
      const double v = qtilde(q + i * ldq_in, code, gstart, glen, hoff, hbuf);
      dst[i * ldd] = v;
      if (fabs(v) > fabs(best)) best = v;
    }
  }
  if (!red && tile_colmax) tile_colmax[tm * tcm_ld + epos[item - nred]] = best;
}

void compact_columns_dev(const Plan& p, const Columns& cols, int64_t c0, int64_t c1,
                         CompactCols& cc, DeviceScratch& ws, cudaStream_t st) {
  cc = CompactCols{};
  if (c1 <= c0) return;
  const int64_t nc = c1 - c0;
  auto* rng = reinterpret_cast<unsigned long long*>(ws.get_i64("cmp_rng", 4));
  const unsigned long long init[4] = {~0ull, 0ull, ~0ull, 0ull};
  EIGB_CUDA(cudaMemcpyAsync(rng, init, sizeof(init), cudaMemcpyHostToDevice, st));
  compact_ranges_kernel<<<(unsigned)cdiv(nc, 256), 256, 0, st>>>(cols.kind, cols.payload, c0, c1,
                                                                 rng);
  EIGB_LAUNCH_CHECK();
  unsigned long long h[4];
  EIGB_CUDA(cudaMemcpyAsync(h, rng, sizeof(h), cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaStreamSynchronize(st));
  cc.j0 = (h[1] > 0) ? (int64_t)h[0] : 0;
  cc.j1 = (h[1] > 0) ? (int64_t)h[1] : 0;
  cc.e0 = (h[3] > 0) ? (int64_t)h[2] : 0;
  cc.e1 = (h[3] > 0) ? (int64_t)h[3] : 0;
  if ((cc.j1 - cc.j0) + (cc.e1 - cc.e0) != nc)
    throw Error(2, "assemble", "compact columns: root / decoupled ranges are not contiguous");
  cc.jpos = ws.get_i64("cmp_jpos", std::max<int64_t>(cc.j1 - cc.j0, 1));
  cc.epos = ws.get_i64("cmp_epos", std::max<int64_t>(cc.e1 - cc.e0, 1));
  cc.cmode = ws.get_i32("cmp_cmode", nc);
  compact_pos_kernel<<<(unsigned)cdiv(nc, 256), 256, 0, st>>>(cols.kind, cols.payload, c0, c1,
                                                              cc.j0, cc.e0, cc.jpos, cc.epos,
                                                              cc.cmode);
  EIGB_LAUNCH_CHECK();
}

void gather_qtilde_dev(const Plan& p, const double* q, const CompactCols& cc, double* qa,
                       int64_t lda, double* q_out, int64_t ldq, double* tile_colmax,
                       int64_t tcm_ld, cudaStream_t st) {
  const int64_t ne = cc.e1 - cc.e0, items = p.nred + ne;
  if (items == 0) return;
  dim3 grid((unsigned)cdiv(p.n, kGatherRows), (unsigned)cdiv(items, 256));
  gather_qtilde_kernel<<<grid, 256, 0, st>>>(q, p.n, p.n, p.nred, p.red_src, ne, p.dec_src, cc.e0,
                                             cc.epos, p.gstart, p.glen, p.hoff, p.hbuf, qa, lda,
                                             q_out, ldq, tile_colmax, tcm_ld);
  EIGB_LAUNCH_CHECK();
}

template <int KP>
void launch_xt_compact(const Plan& p, const RootRecords& roots, const double* colldir,
                       const int* collok, int64_t j0, int64_t j1, double* xt, int64_t ldx,
                       double* colscale, DeviceScratch& ws, cudaStream_t st) {
  if constexpr (KP >= 4) {
    const int64_t nchunks = cdiv(p.nred, kXtmRows);
    double* part = ws.get_f64("xt_part", (size_t)nchunks * (j1 - j0));
    int* cm = ws.get_i32("cmp_rootmode", j1 - j0);
    int* kinds = ws.get_i32("cmp_rootkind", j1 - j0);
    EIGB_CUDA(cudaMemsetAsync(kinds, 0, 4 * (j1 - j0), st));
    dim3 grid((unsigned)nchunks, (unsigned)cdiv(j1 - j0, kXtmCols));
    const size_t sm = sizeof(XtmSmem<KP>);
    EIGB_CUDA(cudaFuncSetAttribute(xt_mma_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)sm));
    xt_mma_kernel<KP><<<grid, 256, sm, st>>>(p.view(), p.nred, nullptr, nullptr, roots.origin,
                                             roots.delta, roots.flags, roots.y, colldir, collok,
                                             nullptr, p.dec_src, j0, j1, ldx, xt, part);
    EIGB_LAUNCH_CHECK();
    // every column is a root (kind 0): scale 1/||x_red||
    xt_norm_kernel<<<(unsigned)cdiv(j1 - j0, 128), 128, 0, st>>>(part, nchunks, 0, j1 - j0,
                                                                 kinds, colscale, cm);
    EIGB_LAUNCH_CHECK();
  } else {
    (void)p, (void)roots, (void)colldir, (void)collok, (void)j0, (void)j1, (void)xt, (void)ldx,
        (void)colscale, (void)ws, (void)st;
    throw Error(2, "assemble", "compact back-transform needs kp >= 4");
  }
}

void build_xt_compact_dev(const Plan& p, const RootRecords& roots, const double* colldir,
                          const int* collok, int64_t j0, int64_t j1, double* xt, int64_t ldx,
                          double* colscale, DeviceScratch& ws, cudaStream_t st) {
  if (j1 <= j0) return;
  switch (p.kp) {
    case 4: launch_xt_compact<4>(p, roots, colldir, collok, j0, j1, xt, ldx, colscale, ws, st); break;
    case 8: launch_xt_compact<8>(p, roots, colldir, collok, j0, j1, xt, ldx, colscale, ws, st); break;
    case 16: launch_xt_compact<16>(p, roots, colldir, collok, j0, j1, xt, ldx, colscale, ws, st); break;
    case 32: launch_xt_compact<32>(p, roots, colldir, collok, j0, j1, xt, ldx, colscale, ws, st); break;
    default: throw Error(2, "assemble", "compact back-transform needs kp >= 4");
  }
}

}  // namespace eigb
