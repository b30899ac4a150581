// K2 deflation weights, the count sweep and K3 batched per-root solver (sm_100a).
//
// K2 (proj/src/secular.cpp:168-202 group_weights): one pole pass per batch of
//   32 pole groups evaluated at their representatives, then per group the
//   reference's adjugate route (cofactors k <= 3, LU det*inverse, cofactor
//   expansion fallback) on M_g = J S_g, alpha_g = sum_s w_s^T adj(M_g) J w_s.
//
// Count sweep (replaces the location stage, proj/src/locate.cpp:65-252 and
//   sturm.cpp): the exact eigenvalue count #eig < x = #{d_i < x} + m -
//   nu(S(x)) (nu from a Bunch-Kaufman LDL^T of S) at the two
//   points d_a -/+ theta * gap next to every pole. Between consecutive points
//   the counts bracket every root; a bracket that holds one root and no pole
//   is "isolated". Two S evaluations per root locate all n roots at once.
//
// K3 (replaces rootfind.cpp:89-229, 342-377): a persistent kernel whose CTAs
//   own 32 root slots. Each slot starts from its sweep bracket; phase A
//   bisects the count until the root is isolated, phase B works in the
//   shifted origin x = d_o + delta (d_o the pole nearest the iterate) with a
//   Newton step on g = -delta f(x) (f the scalar secular function with the K2
//   residues; a pole of f at d_o becomes a line) until |step| < 1e-6 |delta|,
//   then Newton on psi = -delta sigma (sigma the eigenvalue of S nearest zero,
//   from inverse iteration; sigma' = y^T S' y from the same pass) to a few ulps
//   of delta. Every step is confined to the count-certified bracket. A
//   converged slot writes its root record (value, origin, delta, y) and takes
//   the next root index from a global counter.
#include "secular.cuh"

#include <cfloat>

#include <cooperative_groups.h>

namespace eigb {

namespace {

constexpr int FLAG_COLLIDED = 1;   // bracket collapsed onto a pole
constexpr int FLAG_UNISOLATED = 2; // ulp bracket without pole-free isolation
constexpr double kSweepTheta = 1e-3;
constexpr double kFSwitchRel = 1e-6;  // f-Newton -> sigma-Newton

// Sweep points: 2a -> d_a - theta*gap_left, 2a+1 -> d_a + theta*gap_right,
// gaps to the nearest distinct neighbours (1 at the ends).
__device__ __forceinline__ double sweep_point(const double* d, int64_t N, int64_t q) {
  const int64_t a = q >> 1;
  const double da = d[a];
  if (q & 1) {
    int64_t b = a + 1;
    while (b < N && d[b] == da) ++b;
    const double g = (b < N) ? d[b] - da : 1.0;
    return da + kSweepTheta * g;
  }
  int64_t b = a - 1;
  while (b >= 0 && d[b] == da) --b;
  const double g = (b >= 0) ? da - d[b] : 1.0;
  return da - kSweepTheta * g;
}

template <int KP>
__device__ __forceinline__ void load_S(const double* rb, const int* sgn, int k, double* F, int es) {
  using C = PassCfg<KP>;
  for (int r = 0; r < KP; ++r)
    for (int c = r; c < KP; ++c) {
      double v = rb[C::pidx(r, c)];
      if (r == c) v += (r < k) ? (double)sgn[r] : 1.0;
      F[(r * KP + c) * es] = v;
      F[(c * KP + r) * es] = v;
    }
}

// ------------------------------------------------------------ sweep kernel
template <int KP>
__global__ void __launch_bounds__(kPassThreads, 1) count_sweep_kernel(ReducedView rp,
                                                                      int* __restrict__ counts,
                                                                      int64_t qbeg, int64_t qend,
                                                                      double* __restrict__ gscratch) {
  using C = PassCfg<KP>;
  extern __shared__ __align__(16) double smem[];
  // factor storage: interleaved [KP*KP][32] in shared memory for KP <= 16,
  // per-slot rows in global scratch above (32 x 32 x 32 doubles do not fit)
  constexpr bool kSmemF = KP <= 16;
  double* F = kSmemF ? smem + C::SMEM_DOUBLES
                     : gscratch + (size_t)blockIdx.x * 32 * KP * KP;
  constexpr int es = kSmemF ? 32 : 1;
  __shared__ double dob[32], delta[32];
  __shared__ int active[32], hit[32];
  const int t = threadIdx.x;
  const int64_t Q = qend;
  const int64_t q0 = qbeg + (int64_t)blockIdx.x * 32;
  if (t < 32) {
    const int64_t q = q0 + t;
    active[t] = q < Q;
    dob[t] = 0.0;
    delta[t] = (q < Q) ? sweep_point(rp.d, rp.n, q) : 0.0;
    hit[t] = 0;
  }
  __syncthreads();
  PassSlots sl{dob, delta, nullptr, active, hit};
  PassOpts o;
  secular_pass<KP>(rp.d, rp.u, rp.n, sl, o, smem);
  if (t < 32 && active[t]) {
    const double* rb = pass_result<KP>(smem) + t * C::OUT;
    double* Ft = kSmemF ? F + t : F + (size_t)t * KP * KP;
    load_S<KP>(rb, rp.sgn, rp.k, Ft, es);
    int piv[KP], zero;
    const int neg = bk_factor(Ft, KP, KP, piv, &zero, es);
    const double x = delta[t];
    // a hit (x on a pole, duplicates) gives an unusable point: -1
    counts[q0 + t] = hit[t] ? -1 : (int)(dev_n_less(rp.d, rp.n, x) + rp.m_neg - neg);
  }
}

// ------------------------------------------------------------ solver
struct SolveSmem {
  double dob[32], delta[32], lo[32], hi[32], step_prev[32];
  int64_t j[32], o[32], below[32];
  int active[32], hit[32], phase[32], lo_ok[32], hi_ok[32], iters[32], itersA[32], fmode[32];
  unsigned long long jnext[32];  // root handed out by cluster rank 0
};

template <int KP>
struct SolveArgs {
  ReducedView rp;
  const double* alpha;     // residues of the reduced poles (nullptr: no f-Newton)
  const double* br_lo;     // initial brackets of roots [j0, j1) (bracket_kernel); nullptr:
  const double* br_hi;     //   Weyl windows
  const int* br_ok;        // bit 0: lo certified (count == j), bit 1: hi (count == j + 1)
  int64_t j0;
  int64_t j_end;
  unsigned long long* next_root;
  RootRecords out;
  int m_neg, p_pos;
  double lo_clip, hi_clip;
  double step_tol;
  int max_iters;
  int writer;  // writes root records (cluster rank 0)
  unsigned long long* prof;  // [0] passes, [1] active slot-passes, [2] slot batches
  double fexit_rel, floor_rel, floor_ulps, stall_ratio;
  int geo_bisect;
  int64_t trace_j;           // diagnostics (-1: off)
  double* trace;             // [kTraceRows][kTraceCols]
};

// Sweep bracket of root j: the last usable point with count <= j and the
// first with count > j, over the sequence d_a - theta g, d_a (the limit count
// at the pole itself, taken for poles with roots next to them), d_a + theta g
// (outer clips count 0 and N).
__device__ __forceinline__ int comb_count(const int* counts, const int* pcounts, int64_t q3) {
  const int64_t a = q3 / 3;
  const int r = (int)(q3 - 3 * a);
  if (r == 1) return pcounts ? pcounts[a] : -1;
  return counts[2 * a + (r == 2)];
}

__device__ __forceinline__ double comb_point(const double* d, int64_t N, int64_t q3) {
  const int64_t a = q3 / 3;
  const int r = (int)(q3 - 3 * a);
  if (r == 1) return d[a];
  return sweep_point(d, N, 2 * a + (r == 2));
}

// Initial brackets of roots [j0, j1): the last usable point with count <= j
// and the first with count > j over the sequence d_a - theta g, d_a (the
// limit count at the pole itself, where taken), d_a + theta g for the swept
// poles [pbeg, pend); outside them the Weyl window bound (proj/src/locate.cpp:
// 159-171), uncertified; outer clips count 0 and N.
__global__ void bracket_kernel(const double* __restrict__ d, int64_t N, const int* __restrict__ counts,
                               const int* __restrict__ pcounts, int64_t pbeg, int64_t pend,
                               int64_t j0, int64_t j1, int m_neg, int p_pos, double lo_clip,
                               double hi_clip, double* __restrict__ br_lo,
                               double* __restrict__ br_hi, int* __restrict__ br_ok) {
  const int64_t j = j0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= j1) return;
  const int64_t QB = 3 * pbeg, QE = 3 * pend;
  int64_t L = QB, R = QE;  // first usable q3 with count > j
  while (L < R) {
    const int64_t mid = (L + R) >> 1;
    int64_t q = mid;
    while (q < R && comb_count(counts, pcounts, q) < 0) ++q;
    if (q == R) { R = mid; continue; }
    if (comb_count(counts, pcounts, q) > j) R = mid; else L = q + 1;
  }
  int64_t qh = L;
  while (qh < QE && comb_count(counts, pcounts, qh) < 0) ++qh;
  int64_t ql = L - 1;
  while (ql >= QB && comb_count(counts, pcounts, ql) < 0) --ql;
  double lo, hi;
  int lok, hok;
  if (ql >= QB) {
    lo = comb_point(d, N, ql);
    lok = (comb_count(counts, pcounts, ql) == j);
  } else if (QB == 0) {
    lo = lo_clip;
    lok = (j == 0);
  } else {
    lo = (j - m_neg >= 0) ? d[j - m_neg] : lo_clip;
    lok = 0;
  }
  if (qh < QE) {
    hi = comb_point(d, N, qh);
    hok = (comb_count(counts, pcounts, qh) == j + 1);
  } else if (QE == 3 * N) {
    hi = hi_clip;
    hok = (j + 1 == N);
  } else {
    hi = (j + p_pos <= N - 1) ? d[j + p_pos] : hi_clip;
    hok = 0;
  }
  br_lo[j - j0] = lo;
  br_hi[j - j0] = hi;
  br_ok[j - j0] = lok | (hok << 1);
}

template <int KP>
__device__ void enter_phase_b(SolveSmem& s, int b, const SolveArgs<KP>& a, double xstart) {
  const double* d = a.rp.d;
  const int64_t N = a.rp.n;
  const double lo = s.lo[b], hi = s.hi[b];
  const int64_t pa = dev_n_leq(d, N, lo) - 1, pb = pa + 1;
  int64_t o;
  if (pa < 0) o = pb;
  else if (pb >= N) o = pa;
  else o = (xstart - d[pa] <= d[pb] - xstart) ? pa : pb;
  const double dob = d[o];
  s.o[b] = o;
  s.below[b] = pa + 1;
  s.dob[b] = dob;
  s.lo[b] = lo - dob;
  s.hi[b] = hi - dob;
  s.phase[b] = 1;
  s.itersA[b] = s.iters[b];
  s.fmode[b] = (a.alpha != nullptr);
  s.step_prev[b] = s.hi[b] - s.lo[b];
  s.delta[b] = xstart - dob;
}

template <int KP>
__device__ void slot_init(SolveSmem& s, double* y, int b, int64_t j, const SolveArgs<KP>& a) {
  const double* d = a.rp.d;
  const int64_t N = a.rp.n;
  s.j[b] = j;
  s.iters[b] = 0;
  s.itersA[b] = 0;
  s.hit[b] = 0;
  s.phase[b] = 0;
  s.active[b] = 1;
  s.dob[b] = 0.0;
  const double y0 = rsqrt((double)a.rp.k);
  for (int c = 0; c < KP; ++c) y[b * KP + c] = (c < a.rp.k) ? y0 : 0.0;
  double lo, hi;
  int lok, hok;
  if (a.br_lo) {
    lo = a.br_lo[j - a.j0];
    hi = a.br_hi[j - a.j0];
    lok = a.br_ok[j - a.j0] & 1;
    hok = (a.br_ok[j - a.j0] >> 1) & 1;
  } else {  // Weyl window (proj/src/locate.cpp:159-171)
    lo = (j - a.m_neg >= 0) ? d[j - a.m_neg] : a.lo_clip;
    hi = (j + a.p_pos <= N - 1) ? d[j + a.p_pos] : a.hi_clip;
    lok = hok = 0;
  }
  s.lo[b] = lo;
  s.hi[b] = hi;
  s.lo_ok[b] = lok;
  s.hi_ok[b] = hok;
  if (lok && hok && dev_n_less(d, N, hi) == dev_n_leq(d, N, lo)) {
    enter_phase_b<KP>(s, b, a, 0.5 * (lo + hi));
  } else {
    s.delta[b] = 0.5 * (lo + hi);
  }
}

template <int KP>
__device__ void slot_finish(SolveSmem& s, const double* y, int b, const SolveArgs<KP>& a,
                            int64_t o, double delta, double value, int flags, double* ynext) {
  const int64_t j = s.j[b];
  if (a.writer) {  // cluster rank 0 (every CTA of a cluster holds the same state)
    a.out.value[j] = value;
    a.out.origin[j] = o;
    a.out.delta[j] = delta;
    const int ia = s.phase[b] ? (s.itersA[b] < 255 ? s.itersA[b] : 255) : 255;
    a.out.flags[j] = flags | (ia << 8);
    a.out.evals[j] = s.iters[b];
    for (int c = 0; c < KP; ++c) a.out.y[j * KP + c] = y[c];
  }
  (void)ynext;
  s.active[b] = 2;  // refilled from the root queue by the kernel loop
}

// Phase A ended at ulp width without isolation: a pole inside [lo, hi] means
// the root sits on that pole (collision, proj/src/eigvec.cpp:303-323).
template <int KP>
__device__ void slot_finish_unisolated(SolveSmem& s, double* y, int b, const SolveArgs<KP>& a) {
  const double* d = a.rp.d;
  const int64_t N = a.rp.n;
  const double lo = s.lo[b], hi = s.hi[b], mid = 0.5 * (lo + hi);
  double yc[KP];
  for (int c = 0; c < KP; ++c) yc[c] = y[b * KP + c];
  int64_t p = dev_n_less(d, N, lo);
  if (p < N && d[p] <= hi) {
    int64_t o = p;
    for (int64_t q = p + 1; q < N && d[q] <= hi; ++q)
      if (fabs(d[q] - mid) < fabs(d[o] - mid)) o = q;
    slot_finish<KP>(s, yc, b, a, o, 0.0, d[o], FLAG_COLLIDED, y);
    return;
  }
  int64_t o = p < N ? p : N - 1;
  if (o > 0 && fabs(d[o - 1] - mid) < fabs(d[o] - mid)) o -= 1;
  slot_finish<KP>(s, yc, b, a, o, mid - d[o], mid, FLAG_UNISOLATED, y);
}

template <int KP>
__device__ void slot_step(SolveSmem& s, double* y, int b, const double* red, double* F, int es,
                          const SolveArgs<KP>& a) {
  using C = PassCfg<KP>;
  const double* d = a.rp.d;
  const int64_t N = a.rp.n;
  s.iters[b] += 1;
  if (s.hit[b]) {  // evaluation landed exactly on a pole: nudge and retry
    s.hit[b] = 0;
    const double cur = s.delta[b], lo = s.lo[b], hi = s.hi[b];
    double alt = nextafter(cur, hi);
    if (!(alt < hi)) alt = nextafter(cur, lo);
    if (!(alt > lo && alt < hi) || s.iters[b] > a.max_iters) {
      if (s.phase[b] == 0) {
        slot_finish_unisolated<KP>(s, y, b, a);
      } else {
        double yc[KP];
        for (int c = 0; c < KP; ++c) yc[c] = y[b * KP + c];
        slot_finish<KP>(s, yc, b, a, s.o[b], cur, s.dob[b] + cur, FLAG_UNISOLATED, y);
      }
      return;
    }
    s.delta[b] = alt;
    return;
  }
  const double* rb = red + b * C::OUT;
  load_S<KP>(rb, a.rp.sgn, a.rp.k, F, es);
  const double gp = rb[C::IG];
  const double fv = 1.0 + rb[C::IF], fpv = rb[C::IFP];
  int piv[KP], zero = 0;
  const int neg = bk_factor(F, KP, KP, piv, &zero, es);
  double pscale = 0.0;
  for (int c = 0; c < KP; ++c) pscale = fmax(pscale, fabs(F[(c * KP + c) * es]));
  // an exactly zero pivot (x is a root to working precision) is replaced by a
  // tiny multiple of the pivot scale: inverse iteration then still returns
  // the null vector instead of overflowing
  const double tiny = 1e-4 * DBL_EPSILON * fmax(pscale, 1e-300);
  double yv[KP], z[KP];
  for (int c = 0; c < KP; ++c) yv[c] = y[b * KP + c];
  for (int c = 0; c < KP; ++c) z[c] = yv[c];
  bk_solve(F, KP, KP, piv, z, tiny, es);
  double zz = 0.0, zy = 0.0;
  for (int c = 0; c < KP; ++c) zz += z[c] * z[c], zy += z[c] * yv[c];
  double sigma = 0.0;
  if (zz > 0.0 && isfinite(zz)) {
    sigma = zy / zz;  // Rayleigh quotient of S at z
    const double inv = rsqrt(zz);
    for (int c = 0; c < KP; ++c) yv[c] = z[c] * inv;
  }
  for (int c = 0; c < KP; ++c) y[b * KP + c] = yv[c];
  const int64_t j = s.j[b];

  if (s.phase[b] == 0) {
    const double x = s.delta[b];
    const int64_t cnt = dev_n_less(d, N, x) + a.m_neg - neg;
    if (j == a.trace_j && a.writer && s.iters[b] <= kTraceRows) {
      double* tr = a.trace + (s.iters[b] - 1) * kTraceCols;
      const double v[kTraceCols] = {(double)s.iters[b], 0.0, (double)cnt, x, s.lo[b], s.hi[b],
                                    fv, fpv, sigma, gp, 0.0, -1.0};
      for (int c = 0; c < kTraceCols; ++c) tr[c] = v[c];
    }
    if (cnt >= j + 1) { s.hi[b] = x; s.hi_ok[b] = (cnt == j + 1); }
    else { s.lo[b] = x; s.lo_ok[b] = (cnt == j); }
    const double lo = s.lo[b], hi = s.hi[b];
    if (s.lo_ok[b] && s.hi_ok[b] && dev_n_less(d, N, hi) == dev_n_leq(d, N, lo)) {
      enter_phase_b<KP>(s, b, a, 0.5 * (lo + hi));
      return;
    }
    const double xm = 0.5 * (lo + hi);
    if (!(xm > lo && xm < hi) || s.iters[b] > a.max_iters) {
      slot_finish_unisolated<KP>(s, y, b, a);
      return;
    }
    s.delta[b] = xm;
    return;
  }
  // ---- phase B (delta domain)
  const double dl = s.delta[b];
  const int64_t cnt = s.below[b] + a.m_neg - neg;
  if (cnt >= j + 1) s.hi[b] = dl; else s.lo[b] = dl;
  const double lo = s.lo[b], hi = s.hi[b];
  double step = NAN;
  if (s.fmode[b]) {  // Newton on g = -delta f: g' = -f - delta f'
    const double den = fv + dl * fpv;
    step = (den != 0.0) ? -dl * fv / den : NAN;
    // f resolved, or its root contradicts the certified bracket (residues of
    // poles next to a root are the least accurate): continue on S
    const double dt = dl + step;
    if (!(fabs(step) > kFSwitchRel * fabs(dl)) ||
        (!(dt > lo && dt < hi) && fabs(step) <= a.fexit_rel * fabs(dl))) {
      s.fmode[b] = 0;
      // the first S step corrects the error of the residues, not a
      // continuation of the f steps: do not judge it against them
      s.step_prev[b] = hi - lo;
    }
  }
  if (!s.fmode[b]) {  // Newton on psi = -delta sigma: psi' = -sigma - delta sigma'
    const double den = sigma + dl * gp;
    step = (gp > 0.0 && den != 0.0) ? -dl * sigma / den : NAN;
  }
  const double w = hi - lo;
  const double tol = 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi));
  if (j == a.trace_j && a.writer && s.iters[b] <= kTraceRows) {
    double* tr = a.trace + (s.iters[b] - 1) * kTraceCols;
    const double v[kTraceCols] = {(double)s.iters[b], 1.0, (double)s.fmode[b], dl, lo, hi,
                                  fv, fpv, sigma, gp, step, (double)s.o[b]};
    for (int c = 0; c < kTraceCols; ++c) tr[c] = v[c];
  }
  // converged: S-Newton correction below step_tol ulps, or stalled at the
  // rounding floor of sigma (no longer shrinking while already tiny)
  // (the S evaluation near a pole resolves delta only to ~eps * |S| / g in
  // absolute terms: a stalled step below a few ulps of the root x itself is
  // that floor, and further steps only bounce)
  // -- but only while the other poles are far: the vector's entries on a
  // pole s are 1/((d_s - d_o) - delta), so a neighbour within 1e10 steps
  // (clustered poles) needs delta to its own ulps
  const bool stalled = fabs(step) >= a.stall_ratio * fabs(s.step_prev[b]);
  bool far = false;
  if (stalled) {
    const int64_t o = s.o[b];
    double gn = INFINITY;
    if (o > 0) gn = fmin(gn, fabs((d[o - 1] - s.dob[b]) - dl));
    if (o + 1 < N) gn = fmin(gn, fabs((d[o + 1] - s.dob[b]) - dl));
    far = fabs(step) <= 1e-10 * gn;
  }
  const bool sdone =
      !s.fmode[b] && ((fabs(step) <= a.step_tol * DBL_EPSILON * fabs(dl)) ||
                      (stalled && (fabs(step) <= a.floor_rel * fabs(dl) ||
                                   (far && fabs(step) <= a.floor_ulps * DBL_EPSILON *
                                                             fabs(s.dob[b] + dl)))));
  if (sdone || w <= tol || zero || s.iters[b] > a.max_iters) {
    // two more inverse-iteration steps on the same factorization: the
    // eigenvector formula needs y to the accuracy of the root
    for (int it = 0; it < 2; ++it) {
      for (int c = 0; c < KP; ++c) z[c] = yv[c];
      bk_solve(F, KP, KP, piv, z, tiny, es);
      double z2 = 0.0;
      for (int c = 0; c < KP; ++c) z2 += z[c] * z[c];
      if (!(z2 > 0.0 && isfinite(z2))) break;
      const double inv = rsqrt(z2);
      for (int c = 0; c < KP; ++c) yv[c] = z[c] * inv;
    }
    slot_finish<KP>(s, yv, b, a, s.o[b], dl, s.dob[b] + dl, 0, y);
    return;
  }
  double dn = dl + step;
  // safeguard: bisect when the step leaves the certified bracket or stops
  // shrinking
  if (!(dn > lo && dn < hi) || !(fabs(step) < fabs(s.step_prev[b]))) {
    // a bracket spanning orders of magnitude of delta (root next to the
    // origin pole) is split geometrically
    const double alo = fabs(lo), ahi = fabs(hi);
    if (a.geo_bisect && lo * hi > 0.0 && fmax(alo, ahi) > 8.0 * fmin(alo, ahi))
      dn = copysign(sqrt(alo * ahi), lo);
    else
      dn = 0.5 * (lo + hi);
    s.step_prev[b] = w;
  } else {
    s.step_prev[b] = step;
  }
  // re-origin at the pole nearest the new iterate (keeps relative accuracy
  // of delta when the root sits next to the far end of the interval)
  const int64_t pa = s.below[b] - 1, pb = s.below[b];
  if (pa >= 0 && pb < N) {
    const double xn = s.dob[b] + dn;
    const int64_t want = (xn - d[pa] <= d[pb] - xn) ? pa : pb;
    if (want != s.o[b]) {
      const double sh = s.dob[b] - d[want];
      s.o[b] = want;
      s.dob[b] = d[want];
      s.lo[b] = lo + sh;
      s.hi[b] = hi + sh;
      dn = dn + sh;
      if (!(dn > s.lo[b] && dn < s.hi[b])) dn = 0.5 * (s.lo[b] + s.hi[b]);
    }
  }
  s.delta[b] = dn;
}

template <int KP>
constexpr bool kFactorInSmem = (KP <= 16);

// CL CTAs (a thread-block cluster on CL SMs) share one batch of 32 slots: CTA
// r runs the pole pass over pole slice r, the partial sums are combined over
// distributed shared memory in rank order, and every CTA then advances the
// (replicated, identical) slot state. Rank 0 alone talks to the root queue
// and writes records. Splitting the pole sum shortens an iteration by CL, so
// the tail of the last roots (lockstep slots idle while a few finish) costs
// CL times less wall time.
template <int KP, int CL>
__global__ void __launch_bounds__(kPassThreads, KP <= 4 ? 2 : 1) solve_roots_kernel(SolveArgs<KP> a,
                                                                      double* gscratch) {
  using C = PassCfg<KP>;
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) double smem[];
  double* y = smem + C::SMEM_DOUBLES;                      // [32][KP]
  double* Fs = y + 32 * KP;                                // [KP*KP][32] (KP <= 16)
  double* fullred = Fs + (kFactorInSmem<KP> ? 32 * KP * KP : 0);  // [32][OUT] (CL > 1)
  SolveSmem& s = *reinterpret_cast<SolveSmem*>(fullred + (CL > 1 ? C::RED_DOUBLES : 0));
  __shared__ int any;
  const int t = threadIdx.x;
  int rank = 0;
  if constexpr (CL > 1) rank = (int)cg::this_cluster().block_rank();
  a.writer = (rank == 0);
  const int64_t N = a.rp.n;
  const int64_t chunk = (N + CL - 1) / CL;
  const int64_t plo = (rank * chunk < N) ? rank * chunk : N;
  const int64_t pcnt = ((plo + chunk < N) ? plo + chunk : N) - plo;
  double* F;
  int es;
  if constexpr (kFactorInSmem<KP>) {
    F = Fs + (t & 31);
    es = 32;
  } else {
    F = gscratch + ((size_t)blockIdx.x * 32 + (t & 31)) * KP * KP;
    es = 1;
  }
  if (t < 32) s.active[t] = 2;
  __syncthreads();
  PassOpts o;
  o.alpha = a.alpha ? a.alpha + plo : nullptr;
  o.want_sigma = true;
  unsigned long long npass = 0, nact = 0;
  for (;;) {
    // ---- refill finished slots from the root queue
    if constexpr (CL == 1) {
      if (t < 32 && s.active[t] == 2) {
        const unsigned long long nj = atomicAdd(a.next_root, 1ull);
        if ((int64_t)nj < a.j_end) slot_init<KP>(s, y, t, (int64_t)nj, a);
        else s.active[t] = 0;
      }
    } else {
      cg::cluster_group cl = cg::this_cluster();
      if (rank == 0 && t < 32 && s.active[t] == 2) {
        const unsigned long long nj = atomicAdd(a.next_root, 1ull);
        for (int r = 0; r < CL; ++r) cl.map_shared_rank(&s, r)->jnext[t] = nj;
      }
      cl.sync();
      if (t < 32 && s.active[t] == 2) {
        const unsigned long long nj = s.jnext[t];
        if ((int64_t)nj < a.j_end) slot_init<KP>(s, y, t, (int64_t)nj, a);
        else s.active[t] = 0;
      }
    }
    if (t == 0) {
      int v = 0, c = 0;
      for (int b = 0; b < 32; ++b) {
        v |= s.active[b];
        c += (s.active[b] == 1);
      }
      any = v;
      npass += (v != 0);
      nact += c;
    }
    __syncthreads();
    if (!any) break;
    // ---- pole pass over this CTA's slice
    PassSlots sl{s.dob, s.delta, y, s.active, s.hit};
    secular_pass<KP>(a.rp.d + plo, a.rp.u + plo * KP, pcnt, sl, o, smem);
    const double* red = pass_result<KP>(smem);
    if constexpr (CL > 1) {
      cg::cluster_group cl = cg::this_cluster();
      cl.sync();  // all partial sums of this iteration are in place
      for (int idx = t; idx < C::RED_DOUBLES; idx += kPassThreads) {
        double v = 0.0;
        for (int r = 0; r < CL; ++r) v += cl.map_shared_rank(red, r)[idx];
        fullred[idx] = v;
      }
      if (t < 32) {
        int h = 0;
        for (int r = 0; r < CL; ++r) h |= cl.map_shared_rank(&s, r)->hit[t];
        s.hit[t] = h;  // OR is idempotent: safe while others still read it
      }
      cl.sync();  // partials no longer read remotely
      red = fullred;
    }
    if (t < 32 && s.active[t] == 1) slot_step<KP>(s, y, t, red, F, es, a);
    __syncthreads();
  }
  if (t == 0 && rank == 0 && a.prof) {
    atomicAdd(a.prof, npass);
    atomicAdd(a.prof + 1, nact);
    atomicAdd(a.prof + 2, 1ull);
  }
}

// ------------------------------------------------------------------ K2
template <int KP>
struct WeightArgs {
  const double* rep;     // pole value of every row (its group representative)
  const double* u;       // rows, padded [n][KP]
  int64_t n;
  const int64_t* gstart; // group start row
  const int64_t* glen;   // group length
  const double* gval;    // group representative
  int64_t ng;
  const int* sgn;        // [KP] (pads +1)
  int k;                 // effective rank (unpadded)
  double* alpha;         // [ng]
  double* scratch;       // gridDim.x * 32 * 4 * KP * KP
};

template <int KP>
__global__ void __launch_bounds__(kPassThreads, 1) group_weights_kernel(WeightArgs<KP> a) {
  using C = PassCfg<KP>;
  extern __shared__ __align__(16) double smem[];
  __shared__ double dob[32], delta[32];
  __shared__ int active[32], hit[32];
  const int t = threadIdx.x;
  const int64_t g0 = (int64_t)blockIdx.x * 32;
  if (t < 32) {
    const int64_t g = g0 + t;
    active[t] = g < a.ng;
    dob[t] = 0.0;
    delta[t] = (g < a.ng) ? a.gval[g] : 0.0;
    hit[t] = 0;
  }
  __syncthreads();
  PassSlots sl{dob, delta, nullptr, active, hit};
  PassOpts o;
  o.exclude_zero = true;
  secular_pass<KP>(a.rep, a.u, a.n, sl, o, smem);
  if (t < 32 && active[t]) {
    const int64_t g = g0 + t;
    const int k = a.k;
    double* M = a.scratch + ((size_t)blockIdx.x * 32 + t) * 4 * KP * KP;
    double* adj = M + KP * KP;
    double* work = adj + KP * KP;
    const double* rb = pass_result<KP>(smem) + t * C::OUT;
    // M = I + J T (proj/src/secular.cpp:176-188): row r scaled by sign r.
    for (int r = 0; r < k; ++r)
      for (int c = 0; c < k; ++c) {
        const double tv = (r <= c) ? rb[C::pidx(r, c)] : rb[C::pidx(c, r)];
        M[r * KP + c] = (r == c ? 1.0 : 0.0) + (double)a.sgn[r] * tv;
      }
    adjugate_dev(M, k, KP, adj, work);
    double al = 0.0;
    for (int64_t s = a.gstart[g]; s < a.gstart[g] + a.glen[g]; ++s) {
      const double* ws = a.u + s * KP;
      for (int r = 0; r < k; ++r) {
        double tt = 0.0;
        for (int c = 0; c < k; ++c) tt += adj[r * KP + c] * (double)a.sgn[c] * ws[c];
        al += ws[r] * tt;
      }
    }
    a.alpha[g] = al;
  }
}

template <int KP, int CL>
size_t solve_smem_bytes() {
  using C = PassCfg<KP>;
  return sizeof(double) * (C::SMEM_DOUBLES + 32 * KP + (kFactorInSmem<KP> ? 32 * KP * KP : 0) +
                           (CL > 1 ? C::RED_DOUBLES : 0)) +
         sizeof(SolveSmem);
}

template <int KP>
void launch_sweep(const ReducedView& rp, int* counts, int64_t qbeg, int64_t qend,
                  DeviceScratch& ws, cudaStream_t st) {
  using C = PassCfg<KP>;
  constexpr bool kSmemF = KP <= 16;
  const size_t sm = sizeof(double) * (C::SMEM_DOUBLES + (kSmemF ? 32 * KP * KP : 0));
  EIGB_CUDA(cudaFuncSetAttribute(count_sweep_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm));
  if (qend <= qbeg) return;
  const int64_t grid = cdiv(qend - qbeg, 32);
  double* gs = kSmemF ? nullptr : ws.get_f64("sweep_scratch", (size_t)grid * 32 * KP * KP);
  count_sweep_kernel<KP><<<(unsigned)grid, kPassThreads, sm, st>>>(rp, counts, qbeg, qend, gs);
  EIGB_LAUNCH_CHECK();
}

// Launches the solver on thread-block clusters of CL CTAs; false when the
// device cannot co-schedule such clusters (caller falls back to CL = 1).
template <int KP, int CL>
bool launch_solve_cluster(const SolveArgs<KP>& a, int64_t nroots, int sms, cudaStream_t st) {
  if constexpr (!kFactorInSmem<KP>) {
    return false;
  } else {
    const size_t sm = solve_smem_bytes<KP, CL>();
    auto kern = solve_roots_kernel<KP, CL>;
    EIGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kPassThreads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(CL * std::max(1, sms / CL));
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess || nclusters <= 0) {
      (void)cudaGetLastError();
      return false;
    }
    const int64_t want = cdiv(nroots, 32);
    cfg.gridDim = dim3((unsigned)(CL * std::min<int64_t>(nclusters, want)));
    EIGB_CUDA(cudaLaunchKernelEx(&cfg, kern, a, (double*)nullptr));
    EIGB_LAUNCH_CHECK();
    return true;
  }
}

template <int KP>
void launch_solve(const ReducedView& rp, const double* alpha, const double* br_lo,
                  const double* br_hi, const int* br_ok, int64_t j0, int64_t j1,
                  const RootRecords& out, const SolveOptions& opt, DeviceScratch& ws, int sms,
                  cudaStream_t st) {
  SolveArgs<KP> a;
  a.rp = rp;
  a.alpha = alpha;
  a.br_lo = br_lo;
  a.br_hi = br_hi;
  a.br_ok = br_ok;
  a.j0 = j0;
  a.j_end = j1;
  a.out = out;
  a.m_neg = rp.m_neg;
  a.p_pos = rp.k - rp.m_neg;
  a.lo_clip = rp.lo_clip;
  a.hi_clip = rp.hi_clip;
  a.step_tol = opt.step_tol;
  a.max_iters = opt.max_iters;
  a.writer = 1;
  const int64_t nroots = j1 - j0;
  a.next_root = reinterpret_cast<unsigned long long*>(ws.get_i64("solve_counter", 1));
  a.prof = reinterpret_cast<unsigned long long*>(ws.get_i64("solve_prof", 4));
  a.trace_j = opt.trace_root;
  a.fexit_rel = opt.fexit_rel;
  a.floor_rel = opt.floor_rel;
  a.floor_ulps = opt.floor_ulps;
  a.stall_ratio = opt.stall_ratio;
  a.geo_bisect = opt.geo_bisect;
  a.trace = ws.get_f64("solve_trace", (size_t)kTraceRows * kTraceCols);
  if (opt.trace_root >= 0)
    EIGB_CUDA(cudaMemsetAsync(a.trace, 0, sizeof(double) * kTraceRows * kTraceCols, st));
  EIGB_CUDA(cudaMemsetAsync(a.prof, 0, 4 * sizeof(unsigned long long), st));
  const unsigned long long start = (unsigned long long)j0;
  EIGB_CUDA(cudaMemcpyAsync(a.next_root, &start, sizeof(start), cudaMemcpyHostToDevice, st));
  // Size-based choice (tools/exp_cluster.py, cfg 2/4 at n = 8192/32768):
  // with many roots per SM the GPC-aligned pairs keep all 148 SMs busy (4-
  // and 8-CTA clusters leave GPC remainders idle); with few, the shorter
  // per-iteration pass of larger clusters shrinks the tail of the last roots.
  int cl = opt.cluster;
  if (cl < 0) {
    const int64_t per_sm = nroots / std::max(1, sms);
    cl = per_sm >= 160 ? 2 : (per_sm >= 20 ? 4 : 8);
  }
  if (!kFactorInSmem<KP> || cl <= 1 || nroots <= 32) cl = 1;
  if (cl >= 8 && launch_solve_cluster<KP, 8>(a, nroots, sms, st)) return;
  if (cl >= 4 && cl < 8 && launch_solve_cluster<KP, 4>(a, nroots, sms, st)) return;
  if (cl >= 2 && cl < 4 && launch_solve_cluster<KP, 2>(a, nroots, sms, st)) return;
  const int grid = (int)std::min<int64_t>(sms, cdiv(nroots, 32));
  double* gscratch = kFactorInSmem<KP> ? nullptr
                                       : ws.get_f64("solve_scratch", (size_t)grid * 32 * KP * KP);
  const size_t sm = solve_smem_bytes<KP, 1>();
  EIGB_CUDA(cudaFuncSetAttribute(solve_roots_kernel<KP, 1>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  solve_roots_kernel<KP, 1><<<grid, kPassThreads, sm, st>>>(a, gscratch);
  EIGB_LAUNCH_CHECK();
}

template <int KP>
void launch_weights(const double* rep, const double* u, int64_t n, const int64_t* gstart,
                    const int64_t* glen, const double* gval, int64_t ng, const int* sgn, int k,
                    double* alpha, DeviceScratch& ws, cudaStream_t st) {
  using C = PassCfg<KP>;
  WeightArgs<KP> a{rep, u, n, gstart, glen, gval, ng, sgn, k, alpha, nullptr};
  const int grid = (int)cdiv(ng, 32);
  a.scratch = ws.get_f64("weights_scratch", (size_t)grid * 32 * 4 * KP * KP);
  const size_t sm = sizeof(double) * C::SMEM_DOUBLES;
  EIGB_CUDA(cudaFuncSetAttribute(group_weights_kernel<KP>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  group_weights_kernel<KP><<<grid, kPassThreads, sm, st>>>(a);
  EIGB_LAUNCH_CHECK();
}

// ------------------------------------------------------- pole inertia (locate)
// For the location vector (proj/include/eigmod/locate.hpp:13-50; SURVEY.md
// §8(f)3): at a reduced pole value v with rows R (the pole's own rows of U),
// S(x) = T + sum_{r in R} u_r u_r^T / (v - x) with T = J + sum over the other
// rows. As x -> v from below the R-terms add |R| positive eigenvalues, so
// nu(S(v-)) = nu(T restricted to span(R)^perp), and the eigenvalue count below
// v is #{d < v} + m - that inertia. One pole pass per batch of 32 poles (the
// pole's own rows excluded as exact zero differences), then per pole the
// Householder reflections that map span(R) onto the leading coordinates and a
// Bunch-Kaufman inertia of the trailing block.
template <int KP>
struct InertiaArgs {
  ReducedView rp;
  const double* bval;   // pole value per boundary
  const int64_t* brow;  // first reduced row of the pole
  const int* bcnt;      // number of rows at the pole
  int64_t nb;
  int* nu;              // out: inertia of the projected T
  double* scratch;      // gridDim.x * 32 * (2 * KP * KP + KP)
};

template <int KP>
__global__ void __launch_bounds__(kPassThreads, 1) pole_inertia_kernel(InertiaArgs<KP> a) {
  using C = PassCfg<KP>;
  extern __shared__ __align__(16) double smem[];
  __shared__ double dob[32], delta[32];
  __shared__ int active[32], hit[32];
  const int t = threadIdx.x;
  const int64_t g0 = (int64_t)blockIdx.x * 32;
  if (t < 32) {
    const int64_t g = g0 + t;
    active[t] = g < a.nb;
    dob[t] = 0.0;
    delta[t] = (g < a.nb) ? a.bval[g] : 0.0;
    hit[t] = 0;
  }
  __syncthreads();
  PassSlots sl{dob, delta, nullptr, active, hit};
  PassOpts o;
  o.exclude_zero = true;
  secular_pass<KP>(a.rp.d, a.rp.u, a.rp.n, sl, o, smem);
  if (t >= 32 || !active[t]) return;
  const int64_t g = g0 + t;
  const int k = a.rp.k;
  double* T = a.scratch + ((size_t)blockIdx.x * 32 + t) * (2 * KP * KP + KP);
  double* W = T + KP * KP;   // reflectors, one per row of R
  double* x = W + KP * KP;
  const double* rb = pass_result<KP>(smem) + t * C::OUT;
  load_S<KP>(rb, a.rp.sgn, k, T, 1);
  // Householder vectors of span(R): reflector q acts on coordinates q..k-1
  int q = 0;
  const int64_t r0 = a.brow[g];
  for (int r = 0; r < a.bcnt[g] && q < k; ++r) {
    const double* v = a.rp.u + (r0 + r) * KP;
    double vn = 0.0;
    for (int c = 0; c < k; ++c) x[c] = v[c], vn += v[c] * v[c];
    for (int p = 0; p < q; ++p) {  // apply earlier reflectors
      const double* w = W + p * KP;
      double dw = 0.0;
      for (int c = p; c < k; ++c) dw += w[c] * x[c];
      for (int c = p; c < k; ++c) x[c] -= 2.0 * dw * w[c];
    }
    double tn = 0.0;
    for (int c = q; c < k; ++c) tn += x[c] * x[c];
    if (!(tn > 1e-28 * vn)) continue;  // dependent row: span unchanged
    const double al = (x[q] >= 0.0) ? -sqrt(tn) : sqrt(tn);
    double* w = W + q * KP;
    for (int c = 0; c < q; ++c) w[c] = 0.0;
    for (int c = q; c < k; ++c) w[c] = x[c];
    w[q] -= al;
    double wn = 0.0;
    for (int c = q; c < k; ++c) wn += w[c] * w[c];
    const double inv = rsqrt(wn);
    for (int c = q; c < k; ++c) w[c] *= inv;
    // T <- H T H, H = I - 2 w w^T
    for (int rr = 0; rr < k; ++rr) {  // T <- T H (rows)
      double dw = 0.0;
      for (int c = q; c < k; ++c) dw += T[rr * KP + c] * w[c];
      for (int c = q; c < k; ++c) T[rr * KP + c] -= 2.0 * dw * w[c];
    }
    for (int cc = 0; cc < k; ++cc) {  // T <- H T (columns)
      double dw = 0.0;
      for (int c = q; c < k; ++c) dw += w[c] * T[c * KP + cc];
      for (int c = q; c < k; ++c) T[c * KP + cc] -= 2.0 * dw * w[c];
    }
    ++q;
  }
  int neg = 0;
  if (q < k) {
    int piv[KP], zero;
    neg = bk_factor(T + q * KP + q, k - q, KP, piv, &zero, 1);
  }
  a.nu[g] = neg;
}

template <int KP>
void launch_inertia(const ReducedView& rp, const double* bval, const int64_t* brow,
                    const int* bcnt, int64_t nb, int* nu, DeviceScratch& ws, cudaStream_t st) {
  using C = PassCfg<KP>;
  const int grid = (int)cdiv(nb, 32);
  InertiaArgs<KP> a{rp, bval, brow, bcnt, nb, nu, nullptr};
  a.scratch = ws.get_f64("inertia_scratch", (size_t)grid * 32 * (2 * KP * KP + KP));
  const size_t sm = sizeof(double) * C::SMEM_DOUBLES;
  EIGB_CUDA(cudaFuncSetAttribute(pole_inertia_kernel<KP>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  pole_inertia_kernel<KP><<<grid, kPassThreads, sm, st>>>(a);
  EIGB_LAUNCH_CHECK();
}

// Poles with roots next to them (the sweep points d_a -/+ theta g count
// differently, or one of them is unusable) that are multiple (rows of a
// compressed run) or lost a point: their limit counts split those brackets
// at the pole itself. Rows at the pole value: [brow, brow + bcnt).
__global__ void pole_select_kernel(const double* __restrict__ d, int64_t N, int64_t pbeg,
                                   int64_t pend, const int* __restrict__ counts,
                                   int* __restrict__ pcounts, int64_t* __restrict__ list,
                                   double* __restrict__ bval, int64_t* __restrict__ brow,
                                   int* __restrict__ bcnt, unsigned long long* nsel) {
  const int64_t a = pbeg + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= pend) return;
  pcounts[a] = -1;
  const int c0 = counts[2 * a], c1 = counts[2 * a + 1];
  if (c0 >= 0 && c1 >= 0 && c0 == c1) return;
  const double v = d[a];
  if (a > 0 && d[a - 1] == v) return;  // one evaluation per pole value
  // simple poles with usable points are resolved by phase A bisection; the
  // limit count is needed where rows coincide (a compressed run) or a point
  // was unusable
  const bool multi = a + 1 < N && d[a + 1] == v;
  if (c0 >= 0 && c1 >= 0 && !multi) return;
  const int64_t r1 = dev_n_leq(d, N, v);
  const unsigned long long i = atomicAdd(nsel, 1ull);
  list[i] = a;
  bval[i] = v;
  brow[i] = a;
  bcnt[i] = (int)(r1 - a);
}

__global__ void pole_scatter_kernel(const int64_t* __restrict__ list, const int64_t* __restrict__ brow,
                                    const int* __restrict__ bcnt, const int* __restrict__ nu,
                                    int64_t nsel, int m_neg, int* __restrict__ pcounts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nsel) return;
  const int c = (int)(brow[i] + m_neg - nu[i]);
  for (int t = 0; t < bcnt[i]; ++t) pcounts[list[i] + t] = c;
}

}  // namespace

void solve_roots(const ReducedView& rp, const double* alpha, int64_t j0, int64_t j1,
                 const RootRecords& out, const SolveOptions& opt, DeviceScratch& ws, int sms,
                 cudaStream_t st) {
  if (j1 <= j0) return;
  int* counts = nullptr;
  // points next to the poles of every Weyl window of roots [j0, j1)
  // (multi-GPU ranks sweep only their share)
  const int64_t pb = std::max<int64_t>(0, j0 - rp.m_neg - 1);
  const int64_t pe = std::min<int64_t>(rp.n, j1 + (rp.k - rp.m_neg) + 1);
  const int64_t qbeg = 2 * pb, qend = 2 * pe;
  if (opt.sweep) {
    counts = ws.get_i32("sweep_counts", 2 * rp.n);
    switch (rp.kp) {
      case 1: launch_sweep<1>(rp, counts, qbeg, qend, ws, st); break;
      case 2: launch_sweep<2>(rp, counts, qbeg, qend, ws, st); break;
      case 4: launch_sweep<4>(rp, counts, qbeg, qend, ws, st); break;
      case 8: launch_sweep<8>(rp, counts, qbeg, qend, ws, st); break;
      case 16: launch_sweep<16>(rp, counts, qbeg, qend, ws, st); break;
      case 32: launch_sweep<32>(rp, counts, qbeg, qend, ws, st); break;
      default: throw Error(1, "", "solve_roots: unsupported padded rank");
    }
  }
  int* pcounts = nullptr;
  if (opt.sweep && opt.pole_split && pe > pb) {
    pcounts = ws.get_i32("sweep_pole_counts", rp.n);
    const int64_t np = pe - pb;
    int64_t* list = ws.get_i64("psel_list", np);
    double* bval = ws.get_f64("psel_val", np);
    int64_t* brow = ws.get_i64("psel_row", np);
    int* bcnt = ws.get_i32("psel_cnt", np);
    int* nu = ws.get_i32("psel_nu", np);
    auto* nsel = reinterpret_cast<unsigned long long*>(ws.get_i64("psel_n", 1));
    EIGB_CUDA(cudaMemsetAsync(nsel, 0, 8, st));
    pole_select_kernel<<<(unsigned)cdiv(np, 256), 256, 0, st>>>(rp.d, rp.n, pb, pe, counts, pcounts,
                                                                 list, bval, brow, bcnt, nsel);
    EIGB_LAUNCH_CHECK();
    unsigned long long nh = 0;
    EIGB_CUDA(cudaMemcpyAsync(&nh, nsel, 8, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaStreamSynchronize(st));
    if (nh > 0) {
      pole_inertia(rp, bval, brow, bcnt, (int64_t)nh, nu, ws, st);
      pole_scatter_kernel<<<(unsigned)cdiv((int64_t)nh, 256), 256, 0, st>>>(list, brow, bcnt, nu,
                                                                           (int64_t)nh, rp.m_neg,
                                                                           pcounts);
      EIGB_LAUNCH_CHECK();
    }
  }
  double *br_lo = nullptr, *br_hi = nullptr;
  int* br_ok = nullptr;
  if (opt.sweep) {
    const int64_t nr = j1 - j0;
    br_lo = ws.get_f64("br_lo", nr);
    br_hi = ws.get_f64("br_hi", nr);
    br_ok = ws.get_i32("br_ok", nr);
    bracket_kernel<<<(unsigned)cdiv(nr, 256), 256, 0, st>>>(
        rp.d, rp.n, counts, pcounts, pb, pe, j0, j1, rp.m_neg, rp.k - rp.m_neg, rp.lo_clip,
        rp.hi_clip, br_lo, br_hi, br_ok);
    EIGB_LAUNCH_CHECK();
  }
  if (!opt.fnewton) alpha = nullptr;
#define EIGB_SOLVE(K) \
  launch_solve<K>(rp, alpha, br_lo, br_hi, br_ok, j0, j1, out, opt, ws, sms, st)
  switch (rp.kp) {
    case 1: EIGB_SOLVE(1); break;
    case 2: EIGB_SOLVE(2); break;
    case 4: EIGB_SOLVE(4); break;
    case 8: EIGB_SOLVE(8); break;
    case 16: EIGB_SOLVE(16); break;
    case 32: EIGB_SOLVE(32); break;
    default: throw Error(1, "", "solve_roots: unsupported padded rank");
  }
#undef EIGB_SOLVE
}

void group_weights(int kp, const double* rep, const double* u, int64_t n, const int64_t* gstart,
                   const int64_t* glen, const double* gval, int64_t ng, const int* sgn, int k,
                   double* alpha, DeviceScratch& ws, cudaStream_t st) {
  if (ng <= 0) return;
  switch (kp) {
    case 1: launch_weights<1>(rep, u, n, gstart, glen, gval, ng, sgn, k, alpha, ws, st); break;
    case 2: launch_weights<2>(rep, u, n, gstart, glen, gval, ng, sgn, k, alpha, ws, st); break;
    case 4: launch_weights<4>(rep, u, n, gstart, glen, gval, ng, sgn, k, alpha, ws, st); break;
    case 8: launch_weights<8>(rep, u, n, gstart, glen, gval, ng, sgn, k, alpha, ws, st); break;
    case 16: launch_weights<16>(rep, u, n, gstart, glen, gval, ng, sgn, k, alpha, ws, st); break;
    case 32: launch_weights<32>(rep, u, n, gstart, glen, gval, ng, sgn, k, alpha, ws, st); break;
    default: throw Error(1, "", "group_weights: unsupported padded rank");
  }
}

void pole_inertia(const ReducedView& rp, const double* bval, const int64_t* brow, const int* bcnt,
                  int64_t nb, int* nu, DeviceScratch& ws, cudaStream_t st) {
  if (nb <= 0) return;
  switch (rp.kp) {
    case 1: launch_inertia<1>(rp, bval, brow, bcnt, nb, nu, ws, st); break;
    case 2: launch_inertia<2>(rp, bval, brow, bcnt, nb, nu, ws, st); break;
    case 4: launch_inertia<4>(rp, bval, brow, bcnt, nb, nu, ws, st); break;
    case 8: launch_inertia<8>(rp, bval, brow, bcnt, nb, nu, ws, st); break;
    case 16: launch_inertia<16>(rp, bval, brow, bcnt, nb, nu, ws, st); break;
    case 32: launch_inertia<32>(rp, bval, brow, bcnt, nb, nu, ws, st); break;
    default: throw Error(1, "", "pole_inertia: unsupported padded rank");
  }
}

}  // namespace eigb
