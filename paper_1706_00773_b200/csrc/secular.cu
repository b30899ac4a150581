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

// The compile-time factorization (bkl_*) for KP <= 16; KP = 32 (global
// scratch) keeps the generic one.
template <int KP>
constexpr bool kBkl = (KP <= 16);

template <int KP>
__device__ __forceinline__ void load_S(const double* rb, const int* sgn, int k, double* F, int es,
                                       bool full = false) {
  using C = PassCfg<KP>;
  for (int r = 0; r < KP; ++r)
    for (int c = r; c < KP; ++c) {
      double v = rb[C::pidx(r, c)];
      if (r == c) v += (r < k) ? (double)sgn[r] : 1.0;
      F[(c * KP + r) * es] = v;
      if (full || !kBkl<KP>) F[(r * KP + c) * es] = v;  // bkl_* reads the lower triangle only
    }
}

template <int KP>
__device__ __forceinline__ int slot_factor(double* F, int es, int* piv, int* zero) {
  if constexpr (kBkl<KP>) return bkl_factor<KP>(F, es, piv, zero);
  else return bk_factor(F, KP, KP, piv, zero, es);
}

template <int KP>
__device__ __forceinline__ void slot_solve(const double* F, int es, const int* piv, double* z,
                                           double tiny) {
  if constexpr (kBkl<KP>) bkl_solve<KP>(F, es, piv, z, tiny);
  else bk_solve(F, KP, KP, piv, z, tiny, es);
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
    const int neg = slot_factor<KP>(Ft, es, piv, &zero);
    const double x = delta[t];
    // a hit (x on a pole, duplicates) gives an unusable point: -1
    counts[q0 + t] = hit[t] ? -1 : (int)(dev_n_less(rp.d, rp.n, x) + rp.m_neg - neg);
  }
}

// ------------------------------------------------------------ solver
struct SolveSmem {
  double dob[32], delta[32], lo[32], hi[32], step_prev[32];
  int64_t j[32], o[32], below[32];
  int64_t pl[32], ph[32];  // pole window of the bracket: #{d <= lo}, #{d < hi}
  int active[32], hit[32], phase[32], lo_ok[32], hi_ok[32], iters[32], itersA[32], fmode[32];
  int warm[32];  // next evaluation only refreshes y (start at the f presolve's root)
  unsigned long long jnext[32];  // root handed out by cluster rank 0
};

template <int KP>
struct SolveArgs {
  ReducedView rp;
  const double* alpha;     // residues of the reduced poles (nullptr: no f-Newton)
  const double* br_lo;     // initial brackets of roots [j0, j1) (bracket_kernel); nullptr:
  const double* br_hi;     //   Weyl windows
  const int* br_ok;        // bit 0: lo certified (count == j), bit 1: hi (count == j + 1)
  const int64_t* br_pl;    // #{d <= lo} and #{d < hi} of those brackets
  const int64_t* br_ph;
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
  const int64_t* f_o;        // f presolve per root [j0, j1) (nullptr: none): origin,
  const double* f_delta;     //   delta of the f-root, state 0 none / 1 converged /
  const int* f_state;        //   2 stopped early (continue f-Newton on S)
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
                               double* __restrict__ br_hi, int* __restrict__ br_ok,
                               int64_t* __restrict__ br_pl, int64_t* __restrict__ br_ph) {
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
  br_pl[j - j0] = dev_n_leq(d, N, lo);
  br_ph[j - j0] = dev_n_less(d, N, hi);
}

// ------------------------------------------------------------ f presolve
// Scalar Newton on g(delta) = -delta f(d_o + delta), f(x) = 1 + sum_i alpha_i
// / (d_i - x) with the K2 residues, for every isolated root, before the S
// solver. One f evaluation costs ~8 flops per pole against ~KP^2/2 for an S
// evaluation, so the f phase of K3 (about half its evaluations) moves here
// and K3 starts psi-Newton next to the root. f(x) = det(I + J U^T (D - x)^-1
// U) = prod(lambda'_i - x) / prod(d_i - x), so inside an isolated bracket f
// changes sign only at the root and is (-1)^(j + #{d < x}) to its left: sign
// bisection safeguards the Newton steps. The residues carry rounding, so the
// result is only a starting point: K3 keeps the count-certified bracket.
struct FPreArgs {
  const double* d;
  const double* alpha;
  int64_t N;
  const double* br_lo;
  const double* br_hi;
  const int* br_ok;
  const int64_t* br_pl;
  const int64_t* br_ph;
  int64_t j0, j1;
  int64_t* f_o;
  double* f_delta;
  int* f_state;
  unsigned long long* next_root;
  int max_iters;
  unsigned long long* prof;  // [0] converged, [1] unconverged, [2] evaluations, [3] max
};

constexpr int kFPreWarps = 8;
constexpr int kFPreTile = 1024;  // poles per shared-memory tile (d, alpha pairs)

struct FPreSmem {
  double dob[32], del[32], lo[32], hi[32], stepp[32];
  int64_t j[32], o[32], below[32];
  int act[32], it[32], hit[32];
  double pf[kFPreWarps][32], pfp[kFPreWarps][32];
};

__device__ __forceinline__ void fpre_finish(FPreSmem& s, int b, const FPreArgs& a, int state,
                                            double delta) {
  const int64_t r = s.j[b] - a.j0;
  a.f_o[r] = s.o[b];
  a.f_delta[r] = delta;
  a.f_state[r] = state;
  s.act[b] = 2;
  if (state) atomicAdd(a.prof + (state == 1 ? 0 : 1), 1ull);
  atomicAdd(a.prof + 2, (unsigned long long)s.it[b]);
  atomicMax(a.prof + 3, (unsigned long long)s.it[b]);
}

__device__ void fpre_step(FPreSmem& s, int b, const FPreArgs& a) {
  const double* d = a.d;
  const int64_t N = a.N;
  const int it = ++s.it[b];
  double f = 1.0, fp = 0.0;
  for (int w = 0; w < kFPreWarps; ++w) f += s.pf[w][b], fp += s.pfp[w][b];
  const double dl = s.del[b];
  double lo = s.lo[b], hi = s.hi[b];
  if (s.hit[b]) {  // on a pole (cannot happen inside an isolated bracket but at its ends)
    s.hit[b] = 0;
    double alt = nextafter(dl, hi);
    if (!(alt < hi)) alt = nextafter(dl, lo);
    if (!(alt > lo && alt < hi) || it > a.max_iters) fpre_finish(s, b, a, 0, dl);
    else s.del[b] = alt;
    return;
  }
  if (!isfinite(f) || !isfinite(fp)) { fpre_finish(s, b, a, 0, dl); return; }
  if (f == 0.0) { fpre_finish(s, b, a, 1, dl); return; }
  const bool pos_left = ((s.j[b] + s.below[b]) & 1) == 0;
  if ((f > 0.0) == pos_left) lo = dl; else hi = dl;
  const double den = f + dl * fp;
  const double step = (den != 0.0) ? -dl * f / den : NAN;
  const double dn0 = dl + step;
  const bool inside = dn0 > lo && dn0 < hi;
  // converged: a few ulps, or no longer shrinking at the rounding floor of f
  if (inside && (fabs(step) <= 4.0 * DBL_EPSILON * fabs(dl) ||
                 (fabs(step) >= 0.5 * fabs(s.stepp[b]) && fabs(step) <= 1e-11 * fabs(dl)))) {
    fpre_finish(s, b, a, 1, dn0);
    return;
  }
  if (hi - lo <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi))) {
    fpre_finish(s, b, a, 1, 0.5 * (lo + hi));
    return;
  }
  if (it >= a.max_iters) { fpre_finish(s, b, a, 2, dl); return; }
  double dn = dn0;
  if (!inside || !(fabs(step) < fabs(s.stepp[b]))) {
    const double alo = fabs(lo), ahi = fabs(hi);
    if (lo * hi > 0.0 && fmax(alo, ahi) > 8.0 * fmin(alo, ahi)) dn = copysign(sqrt(alo * ahi), lo);
    else dn = 0.5 * (lo + hi);
    s.stepp[b] = hi - lo;
  } else {
    s.stepp[b] = step;
  }
  // re-origin at the pole nearest the new iterate (as K3)
  const int64_t pa = s.below[b] - 1, pb = s.below[b];
  if (pa >= 0 && pb < N) {
    const double xn = s.dob[b] + dn;
    const int64_t want = (xn - d[pa] <= d[pb] - xn) ? pa : pb;
    if (want != s.o[b]) {
      const double sh = s.dob[b] - d[want];
      s.o[b] = want;
      s.dob[b] = d[want];
      lo += sh;
      hi += sh;
      dn += sh;
      if (!(dn > lo && dn < hi)) dn = 0.5 * (lo + hi);
    }
  }
  s.lo[b] = lo;
  s.hi[b] = hi;
  s.del[b] = dn;
}

__global__ void __launch_bounds__(kFPreWarps * 32) fpresolve_kernel(FPreArgs a) {
  constexpr int NT = kFPreWarps * 32;
  constexpr int PER = kFPreTile / NT;  // tile entries loaded per thread
  __shared__ FPreSmem s;
  __shared__ double2 tile[kFPreTile];
  __shared__ int any;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const double* __restrict__ d = a.d;
  const double* __restrict__ al = a.alpha;
  const int64_t N = a.N;
  const int64_t ntiles = (N + kFPreTile - 1) / kFPreTile;
  if (t < 32) s.act[t] = 2;
  __syncthreads();
  for (;;) {
    if (t < 32 && s.act[t] == 2) {
      s.act[t] = 0;
      for (;;) {
        const unsigned long long nj = atomicAdd(a.next_root, 1ull);
        if ((int64_t)nj >= a.j1) break;
        const int64_t j = (int64_t)nj, r = j - a.j0;
        a.f_state[r] = 0;
        if (a.br_ok[r] != 3) continue;
        const double lo = a.br_lo[r], hi = a.br_hi[r];
        const int64_t below = a.br_pl[r];
        if (a.br_ph[r] != below) continue;  // not isolated: phase A in K3
        const double mid = 0.5 * (lo + hi);
        const int64_t pa = below - 1, pb = below;
        const int64_t o = (pa < 0) ? pb : (pb >= N ? pa : ((mid - d[pa] <= d[pb] - mid) ? pa : pb));
        const double dob = d[o];
        s.j[t] = j;
        s.o[t] = o;
        s.below[t] = below;
        s.dob[t] = dob;
        s.lo[t] = lo - dob;
        s.hi[t] = hi - dob;
        s.del[t] = mid - dob;
        s.stepp[t] = s.hi[t] - s.lo[t];
        s.it[t] = 0;
        s.hit[t] = 0;
        s.act[t] = 1;
        break;
      }
    }
    __syncthreads();
    if (t == 0) {
      int v = 0;
      for (int b = 0; b < 32; ++b) v |= s.act[b];
      any = v;
    }
    __syncthreads();
    if (!any) break;
    // one f evaluation of the 32 slots: tiles of (d, alpha) in shared memory,
    // poles of a tile split over the warps, slots over the lanes
    const bool act = s.act[lane] == 1;
    const double dob = s.dob[lane], del = s.del[lane];
    double f = 0.0, fp = 0.0;
    int hit = 0;
    double2 nxt[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int64_t i = e * NT + t;
      nxt[e] = (i < N) ? make_double2(__ldg(d + i), __ldg(al + i)) : make_double2(NAN, 0.0);
    }
    for (int64_t tt = 0; tt < ntiles; ++tt) {
#pragma unroll
      for (int e = 0; e < PER; ++e) tile[e * NT + t] = nxt[e];
      __syncthreads();
      if (tt + 1 < ntiles) {
        const int64_t base = (tt + 1) * kFPreTile;
#pragma unroll
        for (int e = 0; e < PER; ++e) {
          const int64_t i = base + e * NT + t;
          nxt[e] = (i < N) ? make_double2(__ldg(d + i), __ldg(al + i)) : make_double2(NAN, 0.0);
        }
      }
      if (act) {
#pragma unroll 4
        for (int i = warp; i < kFPreTile; i += kFPreWarps) {
          const double2 p = tile[i];
          const double diff = (p.x - dob) - del;
          hit |= (diff == 0.0);
          const double D = (diff == 0.0 || diff != diff) ? 0.0 : rcp64(diff);
          const double aD = p.y * D;
          f += aD;
          fp = fma(aD, D, fp);
        }
      }
      __syncthreads();
    }
    if (hit) s.hit[lane] = 1;
    s.pf[warp][lane] = f;
    s.pfp[warp][lane] = fp;
    __syncthreads();
    if (t < 32 && s.act[t] == 1) fpre_step(s, t, a);
    __syncthreads();
  }
}

template <int KP>
__device__ void enter_phase_b_at(SolveSmem& s, int b, const SolveArgs<KP>& a, int64_t o,
                                 double delta, int fmode) {
  const double* d = a.rp.d;
  const double lo = s.lo[b], hi = s.hi[b];
  const double dob = d[o];
  s.o[b] = o;
  s.below[b] = s.pl[b];
  s.dob[b] = dob;
  s.lo[b] = lo - dob;
  s.hi[b] = hi - dob;
  s.phase[b] = 1;
  s.itersA[b] = s.iters[b];
  s.fmode[b] = fmode && (a.alpha != nullptr);
  s.warm[b] = !s.fmode[b];
  s.step_prev[b] = s.hi[b] - s.lo[b];
  s.delta[b] = (delta > s.lo[b] && delta < s.hi[b]) ? delta : 0.5 * (s.lo[b] + s.hi[b]);
}

template <int KP>
__device__ void enter_phase_b(SolveSmem& s, int b, const SolveArgs<KP>& a, double xstart) {
  const double* d = a.rp.d;
  const int64_t N = a.rp.n;
  const double lo = s.lo[b], hi = s.hi[b];
  const int64_t pa = s.pl[b] - 1, pb = pa + 1;
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
  s.warm[b] = 0;
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
  s.warm[b] = 0;
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
    s.pl[b] = a.br_pl[j - a.j0];
    s.ph[b] = a.br_ph[j - a.j0];
  } else {  // Weyl window (proj/src/locate.cpp:159-171)
    lo = (j - a.m_neg >= 0) ? d[j - a.m_neg] : a.lo_clip;
    hi = (j + a.p_pos <= N - 1) ? d[j + a.p_pos] : a.hi_clip;
    lok = hok = 0;
    s.pl[b] = dev_n_leq(d, N, lo);
    s.ph[b] = dev_n_less(d, N, hi);
  }
  s.lo[b] = lo;
  s.hi[b] = hi;
  s.lo_ok[b] = lok;
  s.hi_ok[b] = hok;
  if (lok && hok && s.ph[b] == s.pl[b]) {
    const int fs = a.f_state ? a.f_state[j - a.j0] : 0;
    if (fs != 0) enter_phase_b_at<KP>(s, b, a, a.f_o[j - a.j0], a.f_delta[j - a.j0], fs == 2);
    else enter_phase_b<KP>(s, b, a, 0.5 * (lo + hi));
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
__device__ __noinline__ void slot_step(SolveSmem& s, double* y, int b, const double* red, double* F, int es,
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
  const int neg = slot_factor<KP>(F, es, piv, &zero);
  double pscale = 0.0;
  for (int c = 0; c < KP; ++c) pscale = fmax(pscale, fabs(F[(c * KP + c) * es]));
  // an exactly zero pivot (x is a root to working precision) is replaced by a
  // tiny multiple of the pivot scale: inverse iteration then still returns
  // the null vector instead of overflowing
  const double tiny = 1e-4 * DBL_EPSILON * fmax(pscale, 1e-300);
  double yv[KP], z[KP];
  for (int c = 0; c < KP; ++c) yv[c] = y[b * KP + c];
  // a slot started at the f presolve's root has no y from earlier
  // evaluations: its first evaluation takes three inverse-iteration steps on
  // this factorization and makes no Newton step (the pass computed sigma'
  // with the unconverged y), the second repeats the point with the new y
  const int ninv = s.warm[b] ? 3 : 1;
  double sigma = 0.0;
  for (int it = 0; it < ninv; ++it) {
    for (int c = 0; c < KP; ++c) z[c] = yv[c];
    slot_solve<KP>(F, es, piv, z, tiny);
    double zz = 0.0, zy = 0.0;
    for (int c = 0; c < KP; ++c) zz += z[c] * z[c], zy += z[c] * yv[c];
    if (!(zz > 0.0 && isfinite(zz))) break;
    sigma = zy / zz;  // Rayleigh quotient of S at z
    const double inv = rsqrt(zz);
    for (int c = 0; c < KP; ++c) yv[c] = z[c] * inv;
  }
  for (int c = 0; c < KP; ++c) y[b * KP + c] = yv[c];
  const int64_t j = s.j[b];

  if (s.phase[b] == 0) {
    const double x = s.delta[b];
    // x strictly inside (lo, hi): the count lies in the bracket's pole window
    const bool inside = x > s.lo[b] && x < s.hi[b] && s.pl[b] <= s.ph[b];
    const int64_t nl = inside ? dev_n_less_in(d, s.pl[b], s.ph[b], x) : dev_n_less(d, N, x);
    const int64_t cnt = nl + a.m_neg - neg;
    if (j == a.trace_j && a.writer && s.iters[b] <= kTraceRows) {
      double* tr = a.trace + (s.iters[b] - 1) * kTraceCols;
      const double v[kTraceCols] = {(double)s.iters[b], 0.0, (double)cnt, x, s.lo[b], s.hi[b],
                                    fv, fpv, sigma, gp, 0.0, -1.0};
      for (int c = 0; c < kTraceCols; ++c) tr[c] = v[c];
    }
    if (cnt >= j + 1) {
      s.hi[b] = x;
      s.hi_ok[b] = (cnt == j + 1);
      s.ph[b] = nl;  // #{d < x}
    } else {
      s.lo[b] = x;
      s.lo_ok[b] = (cnt == j);
      s.pl[b] = inside ? dev_n_leq_in(d, nl, s.ph[b], x) : dev_n_leq(d, N, x);
    }
    const double lo = s.lo[b], hi = s.hi[b];
    if (s.lo_ok[b] && s.hi_ok[b] && s.ph[b] == s.pl[b]) {
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
  if (s.warm[b]) {
    s.warm[b] = 0;
    s.step_prev[b] = hi - lo;
    return;  // same point again (it is now a bracket end)
  }
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
      slot_solve<KP>(F, es, piv, z, tiny);
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
  long long c_refill = 0, c_pass = 0, c_red = 0, c_step = 0;  // SM cycles (thread 0)
  for (;;) {
    const long long t0 = clock64();
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
    const long long t1 = clock64();
    // ---- pole pass over this CTA's slice
    PassSlots sl{s.dob, s.delta, y, s.active, s.hit};
    secular_pass<KP>(a.rp.d + plo, a.rp.u + plo * KP, pcnt, sl, o, smem);
    const double* red = pass_result<KP>(smem);
    const long long t2 = clock64();
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
    const long long t3 = clock64();
    if (t < 32 && s.active[t] == 1) slot_step<KP>(s, y, t, red, F, es, a);
    __syncthreads();
    const long long t4 = clock64();
    c_refill += t1 - t0;
    c_pass += t2 - t1;
    c_red += t3 - t2;
    c_step += t4 - t3;
  }
  if (t == 0 && rank == 0 && a.prof) {
    atomicAdd(a.prof, npass);
    atomicAdd(a.prof + 1, nact);
    atomicAdd(a.prof + 2, 1ull);
    atomicAdd(a.prof + 3, (unsigned long long)c_refill);
    atomicAdd(a.prof + 4, (unsigned long long)c_pass);
    atomicAdd(a.prof + 5, (unsigned long long)c_red);
    atomicAdd(a.prof + 6, (unsigned long long)c_step);
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
                  const double* br_hi, const int* br_ok, const int64_t* br_pl,
                  const int64_t* br_ph, const int64_t* f_o,
                  const double* f_delta, const int* f_state, int64_t j0, int64_t j1,
                  const RootRecords& out, const SolveOptions& opt, DeviceScratch& ws, int sms,
                  cudaStream_t st) {
  SolveArgs<KP> a;
  a.f_o = f_o;
  a.f_delta = f_delta;
  a.f_state = f_state;
  a.rp = rp;
  a.alpha = alpha;
  a.br_lo = br_lo;
  a.br_hi = br_hi;
  a.br_ok = br_ok;
  a.br_pl = br_pl;
  a.br_ph = br_ph;
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
  a.prof = reinterpret_cast<unsigned long long*>(ws.get_i64("solve_prof", 8));
  a.trace_j = opt.trace_root;
  a.fexit_rel = opt.fexit_rel;
  a.floor_rel = opt.floor_rel;
  a.floor_ulps = opt.floor_ulps;
  a.stall_ratio = opt.stall_ratio;
  a.geo_bisect = opt.geo_bisect;
  a.trace = ws.get_f64("solve_trace", (size_t)kTraceRows * kTraceCols);
  if (opt.trace_root >= 0)
    EIGB_CUDA(cudaMemsetAsync(a.trace, 0, sizeof(double) * kTraceRows * kTraceCols, st));
  EIGB_CUDA(cudaMemsetAsync(a.prof, 0, 8 * sizeof(unsigned long long), st));
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
  load_S<KP>(rb, a.rp.sgn, k, T, 1, true);
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
  int64_t *br_pl = nullptr, *br_ph = nullptr;
  if (opt.sweep) {
    const int64_t nr = j1 - j0;
    br_lo = ws.get_f64("br_lo", nr);
    br_hi = ws.get_f64("br_hi", nr);
    br_ok = ws.get_i32("br_ok", nr);
    br_pl = ws.get_i64("br_pl", nr);
    br_ph = ws.get_i64("br_ph", nr);
    bracket_kernel<<<(unsigned)cdiv(nr, 256), 256, 0, st>>>(
        rp.d, rp.n, counts, pcounts, pb, pe, j0, j1, rp.m_neg, rp.k - rp.m_neg, rp.lo_clip,
        rp.hi_clip, br_lo, br_hi, br_ok, br_pl, br_ph);
    EIGB_LAUNCH_CHECK();
  }
  if (!opt.fnewton) alpha = nullptr;
  int64_t* f_o = nullptr;
  double* f_delta = nullptr;
  int* f_state = nullptr;
  if (alpha && br_lo && opt.fpre) {
    const int64_t nr = j1 - j0;
    f_o = ws.get_i64("fpre_o", nr);
    f_delta = ws.get_f64("fpre_delta", nr);
    f_state = ws.get_i32("fpre_state", nr);
    FPreArgs fa{rp.d, alpha, rp.n, br_lo, br_hi, br_ok, br_pl, br_ph, j0, j1, f_o, f_delta, f_state,
                reinterpret_cast<unsigned long long*>(ws.get_i64("fpre_counter", 1)),
                opt.fpre_iters,
                reinterpret_cast<unsigned long long*>(ws.get_i64("fpre_prof", 4))};
    EIGB_CUDA(cudaMemsetAsync(fa.prof, 0, 4 * sizeof(unsigned long long), st));
    const unsigned long long start = (unsigned long long)j0;
    EIGB_CUDA(cudaMemcpyAsync(fa.next_root, &start, sizeof(start), cudaMemcpyHostToDevice, st));
    int per_sm = 0;
    EIGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fpresolve_kernel,
                                                            kFPreWarps * 32, 0));
    const int64_t grid = std::min<int64_t>((int64_t)std::max(1, per_sm) * sms, cdiv(nr, 32));
    fpresolve_kernel<<<(unsigned)grid, kFPreWarps * 32, 0, st>>>(fa);
    EIGB_LAUNCH_CHECK();
  }
#define EIGB_SOLVE(K)                                                                          \
  launch_solve<K>(rp, alpha, br_lo, br_hi, br_ok, br_pl, br_ph, f_o, f_delta, f_state, j0, j1, \
                  out, opt, ws, sms, st)
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
