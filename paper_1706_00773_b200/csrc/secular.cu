// K2 deflation weights, the count sweep and K3 batched per-root solver (sm_100a).
//
// K2 (proj/src/secular.cpp:168-202 group_weights): one pole pass per batch of
//   32 pole groups evaluated at their representatives; M_g = J S_g, so
//   alpha_g = sum_s w_s^T adj(M_g) J w_s = det(J) det(S_g) sum_s w_s^T S_g^-1
//   w_s from one Bunch-Kaufman factorization of S_g (all warps); groups whose
//   pivots span more than 1e8 take the reference's adjugate route (cofactors
//   k <= 3, LU det*inverse, cofactor expansion fallback).
//
// Count sweep (replaces the location stage, proj/src/locate.cpp:65-252 and
//   sturm.cpp): the exact eigenvalue count #eig < x = #{d_i < x} + m -
//   nu(S(x)) (nu from a Bunch-Kaufman LDL^T of S) at the two
//   points d_a -/+ theta * gap next to every pole. Between consecutive points
//   the counts bracket every root; a bracket that holds one root and no pole
//   is "isolated". Two S evaluations per root locate all n roots at once.
//
// f presolve (k >= 16): the f-root of every isolated root from the scalar
//   secular function alone (two-pole "middle way" model, sign-safeguarded),
//   a start for K3 that costs ~14 flops per pole per evaluation.
//
// K3 (replaces rootfind.cpp:89-229, 342-377): a persistent kernel whose CTAs
//   own 32 root slots. Each slot starts from its sweep bracket; phase A
//   bisects the count until the root is isolated, phase B works in the
//   shifted origin x = d_o + delta (d_o the pole nearest the iterate) with a
//   Newton step on g = -delta f(x) (f the scalar secular function with the K2
//   residues; a pole of f at d_o becomes a line) until |step| < 1e-6 |delta|,
//   then Newton on psi = -delta sigma (sigma the eigenvalue of S nearest zero,
//   from inverse iteration; sigma' = y^T S' y from the same pass) to a few ulps
//   of delta. Every step is confined to the count-certified bracket. After
//   each pass the 32 matrices S are factored and solved by all warps of the
//   CTA (par_factor / par_solve). A converged slot writes its root record
//   (value, origin, delta, y) and takes the next root index from a global
//   counter.
#include "secular.cuh"

#include <cfloat>
#include <cstdlib>

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

// S = J + (pass result) into a full KP x KP matrix (padded diagonal 1).
template <int KP>
__device__ __forceinline__ void load_S(const double* rb, const int* sgn, int k, double* F, int es) {
  using C = PassCfg<KP>;
  for (int r = 0; r < KP; ++r)
    for (int c = r; c < KP; ++c) {
      double v = rb[C::pidx(r, c)];
      if (r == c) v += (r < k) ? (double)sgn[r] : 1.0;
      F[(c * KP + r) * es] = v;
      F[(r * KP + c) * es] = v;
    }
}

// ------------------------------------------------------------ solver
struct SolveSmem {
  double dob[32], delta[32], lo[32], hi[32], step_prev[32];
  int64_t j[32], o[32], below[32];
  int64_t pl[32], ph[32];  // pole window of the bracket: #{d <= lo}, #{d < hi}
  int active[32], hit[32], phase[32], lo_ok[32], hi_ok[32], iters[32], itersA[32], fmode[32];
  int warm[32];  // next evaluation only refreshes y (start at the f presolve's root)
  int psi_new[32];  // the next psi step is the first after the f -> psi switch
  // a converged slot: record fields, written after the final inverse iterations
  int64_t fin_o[32];
  double fin_delta[32], fin_value[32];
  unsigned long long jnext[32];  // root handed out by cluster rank 0
};

template <int KP>
struct SolveArgs {
  ReducedView rp;
  const double* alpha;     // residues of the reduced poles (nullptr: no f-Newton)
  double* br_lo;           // initial brackets of roots [j0, j1) (bracket_kernel); nullptr:
  double* br_hi;           //   Weyl windows
  int* br_ok;              // bit 0: lo certified (count == j), bit 1: hi (count == j + 1),
                           //   bit 2: root finished (record written) by the phase-A stage
  int64_t* br_pl;          // #{d <= lo} and #{d < hi} of those brackets
  int64_t* br_ph;
  int phase_a_only;        // stage 1 of a split solve: stop each root once isolated and
  int* pa_evals;           //   store its bracket and evaluations (seed of stage 2)
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
  int compact;               // pack the slots of drained batches (tail passes on fewer m-tiles)
  const double* un2;         // |u_i|^2 of the reduced rows (noise-floor stopping; nullptr: off)
  double noise_c;            // converged when |sigma| <= noise_c eps (1 + sum |u_i|^2 |D_i|)
  int64_t trace_j;           // diagnostics (-1: off)
  double* trace;             // [kTraceRows][kTraceCols]
  const int64_t* f_o;        // f presolve per root [j0, j1) (nullptr: none): origin,
  const double* f_delta;     //   delta of the f-root, state 0 none / 1 converged /
  const int* f_state;        //   2 stopped early (continue f-Newton on S)
  const int64_t* order;      // queue position -> root (hard roots first), nullptr: identity
};

// Sweep bracket of root j: the last usable point with count <= j and the
// first with count > j, over the sequence d_a - theta g, d_a (the limit count
// at the pole itself, taken for poles with roots next to them), d_a + theta g
// (outer clips count 0 and N).
__device__ __forceinline__ int comb_count(const int* counts, const int* pcounts, int64_t q3) {
  const int64_t a = q3 / 3;
  const int r = (int)(q3 - 3 * a);
  if (r == 1) return pcounts ? pcounts[a] : -1;
  return counts ? counts[2 * a + (r == 2)] : -1;
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
  double rel;                // converged: |step| <= rel |delta| (the solver refines)
};

constexpr int kFPreWarps = 32;
constexpr int kFPreTile = 1024;  // poles per shared-memory tile (d, alpha pairs)

struct FPreSmem {
  double dob[32], del[32], lo[32], hi[32], stepp[32];
  int64_t j[32], o[32], below[32];
  int act[32], it[32], hit[32];
  // f split at the bracket: psi over the poles left of it, phi right of it
  double ps[kFPreWarps][32], psp[kFPreWarps][32], ph[kFPreWarps][32], php[kFPreWarps][32];
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
  double psi = 0.0, psip = 0.0, phi = 0.0, phip = 0.0;
  for (int w = 0; w < kFPreWarps; ++w) {
    psi += s.ps[w][b], psip += s.psp[w][b];
    phi += s.ph[w][b], phip += s.php[w][b];
  }
  const double f = 1.0 + psi + phi, fp = psip + phip;
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
  double step = (den != 0.0) ? -dl * f / den : NAN;
  // the two-pole model of the bracket (psi ~ a1 + b1 / (d_A - x), phi ~ a2 +
  // b2 / (d_B - x), value and slope matched at the iterate; the classical
  // "middle way" of rank-one secular solvers): its root in the bracket
  const int64_t pa = s.below[b] - 1, pb = s.below[b];
  if (pa >= 0 && pb < N) {
    const double dA = d[pa] - s.dob[b], dB = d[pb] - s.dob[b];
    const double eA = dA - dl, eB = dB - dl;
    const double b1 = psip * eA * eA, b2 = phip * eB * eB;
    const double cc = 1.0 + (psi - b1 / eA) + (phi - b2 / eB);
    // cc (dA - t)(dB - t) + b1 (dB - t) + b2 (dA - t) = 0
    const double qa = cc, qb = -(cc * (dA + dB) + b1 + b2), qc = cc * dA * dB + b1 * dB + b2 * dA;
    const double disc = qb * qb - 4.0 * qa * qc;
    if (disc >= 0.0 && qa != 0.0) {
      const double q = -0.5 * (qb + copysign(sqrt(disc), qb));
      const double r1 = q / qa, r2 = (q != 0.0) ? qc / q : r1;
      const bool in1 = r1 > lo && r1 < hi, in2 = r2 > lo && r2 < hi;
      if (in1 != in2) step = (in1 ? r1 : r2) - dl;
      else if (in1) step = ((fabs(r1 - dl) <= fabs(r2 - dl)) ? r1 : r2) - dl;
    }
  }
  const double dn0 = dl + step;
  const bool inside = dn0 > lo && dn0 < hi;
  // converged: a few ulps, or no longer shrinking at the rounding floor of f
  if (inside && (fabs(step) <= fmax(4.0 * DBL_EPSILON, a.rel) * fabs(dl) ||
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
  extern __shared__ __align__(16) double fpre_smem[];
  FPreSmem& s = *reinterpret_cast<FPreSmem*>(fpre_smem);
  double2* tile = reinterpret_cast<double2*>(fpre_smem + (sizeof(FPreSmem) + 15) / 16 * 2);
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
    const int64_t below = s.below[lane];
    double ps = 0.0, psp = 0.0, ph = 0.0, php = 0.0;
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
        const int64_t t0 = tt * kFPreTile;
        if (t0 + kFPreTile <= below || t0 >= below) {
          // the whole tile on one side of the slot's bracket: one accumulator
          // pair, added to psi or phi after the tile (same terms, same order)
          double fa = 0.0, fpa = 0.0;
#pragma unroll 4
          for (int i = warp; i < kFPreTile; i += kFPreWarps) {
            const double2 p = tile[i];
            const double diff = (p.x - dob) - del;
            hit |= (diff == 0.0);
            const double D = (diff == 0.0 || diff != diff) ? 0.0 : rcp64_fast(diff);
            const double aD = p.y * D;
            fa += aD;
            fpa = fma(aD, D, fpa);
          }
          if (t0 >= below) ph += fa, php += fpa;
          else ps += fa, psp += fpa;
        } else {
#pragma unroll 4
          for (int i = warp; i < kFPreTile; i += kFPreWarps) {
            const double2 p = tile[i];
            const double diff = (p.x - dob) - del;
            hit |= (diff == 0.0);
            const double D = (diff == 0.0 || diff != diff) ? 0.0 : rcp64_fast(diff);
            const double aD = p.y * D;
            const double aL = (t0 + i < below) ? aD : 0.0, aR = aD - aL;
            ps += aL;
            psp = fma(aL, D, psp);
            ph += aR;
            php = fma(aR, D, php);
          }
        }
      }
      __syncthreads();
    }
    if (hit) s.hit[lane] = 1;
    s.ps[warp][lane] = ps;
    s.psp[warp][lane] = psp;
    s.ph[warp][lane] = ph;
    s.php[warp][lane] = php;
    __syncthreads();
    if (t < 32 && s.act[t] == 1) fpre_step(s, t, a);
    __syncthreads();
  }
}

__global__ void row_norm2_kernel(const double* __restrict__ u, int64_t n, int kp,
                                 double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = 0.0;
  for (int c = 0; c < kp; ++c) v = fma(u[i * kp + c], u[i * kp + c], v);
  out[i] = v;
}

// A root-queue counter set on the stream (a pageable host-to-device copy of
// the start would synchronise the host with the stream).
__global__ void set_u64_kernel(unsigned long long* p, unsigned long long v) { *p = v; }

// Root queue order: the roots expected to need the most evaluations first
// (brackets without isolation, then presolve not converged, then the rest),
// so the last batches of a solve drain short roots (longest-first).
__device__ __forceinline__ int root_class(const int* br_ok, const int64_t* br_pl,
                                          const int64_t* br_ph, const int* f_state, int64_t r) {
  if (br_ok[r] & 4) return 3;  // finished by the phase-A stage: last (skipped)
  if (br_ok[r] != 3 || br_pl[r] != br_ph[r]) return 0;
  if (!f_state || f_state[r] != 1) return 1;
  return 2;
}

__global__ void order_count_kernel(const int* __restrict__ br_ok, const int64_t* __restrict__ br_pl,
                                   const int64_t* __restrict__ br_ph, const int* __restrict__ f_state,
                                   int64_t nr, unsigned long long* __restrict__ cnt) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nr) atomicAdd(cnt + root_class(br_ok, br_pl, br_ph, f_state, r), 1ull);
}

__global__ void order_scatter_kernel(const int* __restrict__ br_ok, const int64_t* __restrict__ br_pl,
                                     const int64_t* __restrict__ br_ph, const int* __restrict__ f_state,
                                     int64_t nr, int64_t j0, unsigned long long* __restrict__ cnt,
                                     int64_t* __restrict__ order) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nr) return;
  const int c = root_class(br_ok, br_pl, br_ph, f_state, r);
  unsigned long long base = 0;
  for (int q = 0; q < c; ++q) base += cnt[q];
  const unsigned long long pos = base + atomicAdd(cnt + 4 + c, 1ull);
  order[pos] = j0 + r;
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
  // the first evaluation only refreshes y (also for an unconverged presolve:
  // an immediate switch to psi-Newton would take its first step with the
  // sigma' of the initial y, and the must-shrink safeguard would then reject
  // the correct second step and bisect)
  s.warm[b] = 1;
  s.psi_new[b] = 0;
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
  s.psi_new[b] = 0;
  s.step_prev[b] = s.hi[b] - s.lo[b];
  s.delta[b] = xstart - dob;
}

template <int KP>
__device__ void slot_init(SolveSmem& s, double* y, int b, int64_t j, const SolveArgs<KP>& a) {
  const double* d = a.rp.d;
  const int64_t N = a.rp.n;
  s.j[b] = j;
  s.iters[b] = a.pa_evals ? a.pa_evals[j - a.j0] : 0;  // phase-A evaluations of a split solve
  s.itersA[b] = 0;
  if (a.br_ok && (a.br_ok[j - a.j0] & 4)) {  // finished by the phase-A stage
    s.active[b] = 2;
    return;
  }
  s.hit[b] = 0;
  s.phase[b] = 0;
  s.warm[b] = 0;
  s.psi_new[b] = 0;
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
    int fs = a.f_state ? a.f_state[j - a.j0] : 0;
    if (fs != 0) {
      // The presolved point is only trusted away from the bracket's ends: the
      // scalar f (residues with rounding; values of 1e20 on spectra graded over
      // many decades) can send its sign bisection into a pole, and an S
      // evaluation at 1e-20 of the interval from a pole has no meaningful
      // inertia (the pole's own term swamps the rest), so its count would
      // collapse the bracket onto the pole (stress seeds 7306, 7477, 7666).
      const double dob = d[a.f_o[j - a.j0]], fd = a.f_delta[j - a.j0];
      const double margin = 1e-9 * (hi - lo);
      if (!((dob - lo) + fd >= margin && (hi - dob) - fd >= margin)) fs = 0;
    }
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
    if (a.phase_a_only) a.br_ok[j - a.j0] |= 4;
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

// ---- the per-slot step, spread over the CTA's 8 warps
// After each pass the 32 slots' k x k matrices S are factored and solved by
// all 256 threads: thread (warp w, lane b) works on slot b's rows r with
// r % 8 == w (the Bunch-Kaufman pivot decisions and the permutations by warp
// 0). The same pivots and operations as bk_factor / bk_solve, with the
// column-oriented form of the L^T solve. A serial per-lane factorization
// left seven warps idle at a barrier and ran its dependent shared-memory
// chain without latency hiding (up to ~30% of the kernel at 4096 poles per
// CTA).
template <int KP>
struct ParSmem {
  double z[KP][32];             // right-hand side / solution per slot
  int piv[KP][32];
  int bs[KP][32];               // 0: 1x1 pivot, 1: first row of a 2x2, 2: its second row
  double redv[kPassWarps][32];  // pivot search partials
  int redi[kPassWarps][32];
  int dkp[32], dstep[32], dskip[32], neg[32], zero[32], ev[32], fin[32], ninv[32];
  double tiny[32], sigma[32];
  double ldet[32];  // log2 |det S| of the factored matrix (warm evaluations)
  int dsgn[32];     // its sign
};

constexpr size_t kSolveSmemPad = (sizeof(SolveSmem) + 15) / 16 * 16;

// element (i, j), i >= j, of slot b's matrix
// (lower triangle, packed by rows: every access has i >= j)
#define FA(i, j) F[(size_t)b * esl + ((i) * ((i) + 1) / 2 + (j)) * es]
// Warps sharing the rows of a slot: one row per warp up to 8 (KP = 1, 2, 4
// use KP warps, synchronised by a named barrier over those warps).
template <int KP>
constexpr int kParWarps = (KP >= kPassWarps) ? kPassWarps : KP;
constexpr int kRowsPer(int kp) { return (kp + kPassWarps - 1) / kPassWarps; }
template <int KP>
__device__ __forceinline__ void par_sync() {
  if constexpr (kParWarps<KP> == kPassWarps) __syncthreads();
  else if constexpr (kParWarps<KP> == 1) __syncwarp();
  else asm volatile("bar.sync 1, %0;" ::"r"(kParWarps<KP> * 32) : "memory");
}

template <int KP>
__device__ __forceinline__ void par_load_S(const double* red, const int* sgn, int k, double* F,
                                           size_t esl, int es, const ParSmem<KP>& P) {
  using C = PassCfg<KP>;
  const int b = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (w >= kParWarps<KP> || !P.ev[b]) return;
  const double* rb = red + b * C::OUT;
#pragma unroll
  for (int m = 0; m < kRowsPer(KP); ++m) {
    const int i = w + kParWarps<KP> * m;
    if (i >= KP) break;
    for (int c = 0; c <= i; ++c) {
      double v = rb[C::pidx(c, i)];
      if (c == i) v += (i < k) ? (double)sgn[i] : 1.0;
      FA(i, c) = v;
    }
  }
}

template <int KP>
__device__ void par_factor(double* F, size_t esl, int es, ParSmem<KP>& P) {
  const double alpha = 0.6403882032022076;
  const int b = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int RP = kRowsPer(KP);
  if (w >= kParWarps<KP>) return;
  for (int k = 0; k < KP; ++k) {
    const bool on = P.ev[b] && !P.dskip[b];
    // 1. column maximum below the diagonal over this thread's rows
    double cm = 0.0;
    int ci = k;
#pragma unroll
    for (int m = 0; m < RP; ++m) {
      const int i = w + kParWarps<KP> * m;
      if (on && i > k && i < KP) {
        const double v = fabs(FA(i, k));
        if (v > cm) cm = v, ci = i;
      }
    }
    P.redv[w][b] = cm;
    P.redi[w][b] = ci;
    par_sync<KP>();
    // 2. pivot decision (warp 0)
    if (w == 0) {
      int step = 0;
      if (P.ev[b] && P.dskip[b]) {
        P.dskip[b] = 0;  // second row of a 2x2 pivot
      } else if (P.ev[b]) {
        double colmax = 0.0;
        int imax = k;
        for (int ww = 0; ww < kParWarps<KP>; ++ww) {  // first maximum in row order
          const double v = P.redv[ww][b];
          const int i = P.redi[ww][b];
          if (v > colmax || (v == colmax && v > 0.0 && i < imax)) colmax = v, imax = i;
        }
        const double absakk = fabs(FA(k, k));
        if (fmax(absakk, colmax) == 0.0) {
          P.piv[k][b] = k;
          P.bs[k][b] = 0;
          P.zero[b] = 1;
        } else {
          int kp = k;
          step = 1;
          if (!(absakk >= alpha * colmax)) {
            double rowmax = 0.0;
            for (int j = k; j < KP; ++j) {
              if (j == imax) continue;
              rowmax = fmax(rowmax, fabs(j < imax ? FA(imax, j) : FA(j, imax)));
            }
            if (absakk >= alpha * colmax * (colmax / rowmax)) {
              kp = k;
            } else if (fabs(FA(imax, imax)) >= alpha * rowmax) {
              kp = imax;
            } else {
              kp = imax;
              step = 2;
            }
          }
          if (k + 1 >= KP) step = 1;
          P.dkp[b] = kp;
          if (step == 1) {
            P.piv[k][b] = kp;
            P.bs[k][b] = 0;
          } else {
            P.piv[k][b] = P.piv[k + 1][b] = -kp - 1;
            P.bs[k][b] = 1;
            P.bs[k + 1][b] = 2;
            P.dskip[b] = 1;
          }
        }
      }
      P.dstep[b] = step;
    }
    par_sync<KP>();
    const int step = P.dstep[b];
    // 3. symmetric interchange of kk < kp on the lower triangle (entry sets
    //    indexed by c, thread = owner of c)
    if (step) {
      const int kk = k + step - 1, kp = P.dkp[b];
      if (kp != kk) {
#pragma unroll
        for (int m = 0; m < RP; ++m) {
          const int c = w + kParWarps<KP> * m;
          if (c >= KP) break;
          if (c < kk) {
            const double t = FA(kk, c); FA(kk, c) = FA(kp, c); FA(kp, c) = t;
          } else if (c == kk) {
            const double t = FA(kk, kk); FA(kk, kk) = FA(kp, kp); FA(kp, kp) = t;
          } else if (c < kp) {
            const double t = FA(c, kk); FA(c, kk) = FA(kp, c); FA(kp, c) = t;
          } else if (c > kp) {
            const double t = FA(c, kk); FA(c, kk) = FA(c, kp); FA(c, kp) = t;
          }
        }
      }
    }
    par_sync<KP>();
    // 4. rank-1 / rank-2 update of this thread's trailing rows (reads the
    //    pivot columns, writes columns beyond them); multipliers kept
    double m1[RP], m2[RP];
    double dk = 0.0, det = 0.0;
    if (step == 1) {
      dk = FA(k, k);
      if (dk != 0.0) {
        const double r1 = 1.0 / dk;
#pragma unroll
        for (int m = 0; m < RP; ++m) {
          const int i = w + kParWarps<KP> * m;
          if (i > k && i < KP) {
            const double li = FA(i, k) * r1;
            for (int j = k + 1; j <= i; ++j) FA(i, j) -= li * FA(j, k);
            m1[m] = li;
          }
        }
      }
    } else if (step == 2) {
      const double a = FA(k, k), bb = FA(k + 1, k), c = FA(k + 1, k + 1);
      det = a * c - bb * bb;
      if (det != 0.0) {
        const double id = 1.0 / det;
#pragma unroll
        for (int m = 0; m < RP; ++m) {
          const int i = w + kParWarps<KP> * m;
          if (i >= k + 2 && i < KP) {
            const double x1 = FA(i, k), x2 = FA(i, k + 1);
            const double w1 = (c * x1 - bb * x2) * id;
            const double w2 = (a * x2 - bb * x1) * id;
            for (int j = k + 2; j <= i; ++j) FA(i, j) -= w1 * FA(j, k) + w2 * FA(j, k + 1);
            m1[m] = w1;
            m2[m] = w2;
          }
        }
      }
      if (w == 0) {
        if (det < 0.0) P.neg[b] += 1;
        else if (a + c < 0.0) P.neg[b] += 2;
        if (det == 0.0) P.zero[b] = 1;
      }
    }
    if (step == 1 && w == 0) {
      if (dk < 0.0) P.neg[b] += 1;
      if (dk == 0.0) P.zero[b] = 1;
    }
    par_sync<KP>();
    // 5. multipliers into the pivot columns (read by nobody until after the
    //    next barrier)
    if (step == 1 && dk != 0.0) {
#pragma unroll
      for (int m = 0; m < RP; ++m) {
        const int i = w + kParWarps<KP> * m;
        if (i > k && i < KP) FA(i, k) = m1[m];
      }
    } else if (step == 2 && det != 0.0) {
#pragma unroll
      for (int m = 0; m < RP; ++m) {
        const int i = w + kParWarps<KP> * m;
        if (i >= k + 2 && i < KP) FA(i, k) = m1[m], FA(i, k + 1) = m2[m];
      }
    }
  }
  par_sync<KP>();
}

// z[.][b] <- S^-1 z for the slots with sel (zero pivots replaced by tiny[b]).
template <int KP>
__device__ void par_solve(const double* F, size_t esl, int es, ParSmem<KP>& P, bool sel) {
  const int b = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int RP = kRowsPer(KP);
  if (w >= kParWarps<KP>) return;
  if (w == 0 && sel) {  // z <- P z
    for (int k = 0; k < KP; ++k) {
      const int t = P.bs[k][b];
      int r = -1, kp = 0;
      if (t == 0) r = k, kp = P.piv[k][b];
      else if (t == 1) r = k + 1, kp = -P.piv[k][b] - 1;
      if (r >= 0 && kp != r) { const double v = P.z[r][b]; P.z[r][b] = P.z[kp][b]; P.z[kp][b] = v; }
    }
  }
  par_sync<KP>();
  for (int k = 0; k < KP; ++k) {  // L y = z
    if (sel) {
      const int t = P.bs[k][b];
      if (t == 0) {
        const double zk = P.z[k][b];
#pragma unroll
        for (int m = 0; m < RP; ++m) {
          const int i = w + kParWarps<KP> * m;
          if (i > k && i < KP) P.z[i][b] -= FA(i, k) * zk;
        }
      } else if (t == 1) {
        const double zk = P.z[k][b], zk1 = P.z[k + 1][b];
#pragma unroll
        for (int m = 0; m < RP; ++m) {
          const int i = w + kParWarps<KP> * m;
          if (i >= k + 2 && i < KP) P.z[i][b] -= FA(i, k) * zk + FA(i, k + 1) * zk1;
        }
      }
    }
    par_sync<KP>();
  }
  if (sel) {  // D w = y
#pragma unroll
    for (int m = 0; m < RP; ++m) {
      const int i = w + kParWarps<KP> * m;
      if (i >= KP) break;
      const int t = P.bs[i][b];
      if (t == 0) {
        double dk = FA(i, i);
        if (dk == 0.0) dk = P.tiny[b];
        P.z[i][b] /= dk;
      } else if (t == 1) {
        const double a = FA(i, i), bb = FA(i + 1, i), c = FA(i + 1, i + 1);
        double det = a * c - bb * bb;
        if (det == 0.0) det = P.tiny[b];
        const double z1 = P.z[i][b], z2 = P.z[i + 1][b];
        P.z[i][b] = (c * z1 - bb * z2) / det;
        P.z[i + 1][b] = (a * z2 - bb * z1) / det;
      }
    }
  }
  par_sync<KP>();
  for (int i = KP - 1; i >= 0; --i) {  // L^T z = w, column-oriented
    if (sel) {
      const int t = P.bs[i][b];
      if (t == 0) {
        const double zi = P.z[i][b];
#pragma unroll
        for (int m = 0; m < RP; ++m) {
          const int k = w + kParWarps<KP> * m;
          if (k < i) P.z[k][b] -= FA(i, k) * zi;
        }
      } else if (t == 2) {
        const double zi = P.z[i][b], zi1 = P.z[i - 1][b];
#pragma unroll
        for (int m = 0; m < RP; ++m) {
          const int k = w + kParWarps<KP> * m;
          if (k < i - 1) P.z[k][b] -= FA(i, k) * zi + FA(i - 1, k) * zi1;
        }
      }
    }
    par_sync<KP>();
  }
  if (w == 0 && sel) {  // z <- P^T z
    for (int k = KP - 1; k >= 0; --k) {
      const int t = P.bs[k][b];
      int kp = -1;
      if (t == 0) kp = P.piv[k][b];
      else if (t == 2) kp = -P.piv[k][b] - 1;
      if (kp >= 0 && kp != k) { const double v = P.z[k][b]; P.z[k][b] = P.z[kp][b]; P.z[kp][b] = v; }
    }
  }
  par_sync<KP>();
}

// ------------------------------------------------------------ sweep kernel
template <int KP>
__global__ void __launch_bounds__(kPassThreads, KP <= 16 ? 2 : 1) count_sweep_kernel(ReducedView rp,
                                                                      int* __restrict__ counts,
                                                                      int64_t qbeg, int64_t qend,
                                                                      double* __restrict__ gscratch) {
  using C = PassCfg<KP>;
  extern __shared__ __align__(16) double smem[];
  // factor storage: interleaved [KP(KP+1)/2][32] in shared memory for KP <= 16,
  // per-slot matrices in global scratch above (32 x 32 x 32 doubles do not fit)
  // (KP <= 16: overlays the pass's tiles and D buffer, dead after the pass;
  // the pass result lies beyond them)
  constexpr bool kSmemF = KP <= 16;
  static_assert(!kSmemF || C::FACT <= 2 * C::TILE_DOUBLES + C::DBUF_DOUBLES,
                "factor storage must fit in the pass tiles");
  double* F = kSmemF ? smem : gscratch + (size_t)blockIdx.x * 32 * KP * KP;
  const size_t esl = kSmemF ? 1 : (size_t)KP * KP;
  constexpr int es = kSmemF ? 32 : 1;
  ParSmem<KP>& P = *reinterpret_cast<ParSmem<KP>*>(smem + C::SMEM_DOUBLES);
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
  // inertia of the 32 S(x) by the CTA's warps (par_factor)
  if (t < 32) {
    P.ev[t] = active[t] && !hit[t];
    P.neg[t] = 0;
    P.zero[t] = 0;
    P.dskip[t] = 0;
  }
  __syncthreads();
  par_load_S<KP>(pass_result<KP>(smem), rp.sgn, rp.k, F, esl, es, P);
  __syncthreads();
  par_factor<KP>(F, esl, es, P);
  if (t < 32 && active[t]) {
    const double x = delta[t];
    // a hit (x on a pole, duplicates) gives an unusable point: -1
    counts[q0 + t] = hit[t] ? -1 : (int)(dev_n_less(rp.d, rp.n, x) + rp.m_neg - P.neg[t]);
  }
}

// Warp 0, before the factorization: the evaluation count, and a pass that
// landed exactly on a pole (nudge and retry without factoring).
template <int KP>
__device__ void slot_pre(SolveSmem& s, ParSmem<KP>& P, double* y, int b, const SolveArgs<KP>& a) {
  P.ev[b] = 0;
  P.fin[b] = 0;
  P.ninv[b] = 0;
  if (s.active[b] != 1) return;
  s.iters[b] += 1;
  if (s.hit[b]) {
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
  P.ev[b] = 1;
  P.neg[b] = 0;
  P.zero[b] = 0;
  P.dskip[b] = 0;
  // a slot started at the f presolve's root has no y from earlier
  // evaluations: its first evaluation takes three inverse-iteration steps on
  // this factorization and makes no Newton step (the pass computed sigma'
  // with the unconverged y), the second repeats the point with the new y
  P.ninv[b] = s.warm[b] ? 3 : 1;
}

// Warp 0, after the factorization and inverse iteration: the count, bracket
// update and Newton step of the slot (y already holds the new vector).
// A converged slot gets fin = 1 (two more inverse-iteration steps, then its
// record).
template <int KP>
__device__ void slot_post(SolveSmem& s, ParSmem<KP>& P, double* y, int b, const double* red,
                          const SolveArgs<KP>& a) {
  using C = PassCfg<KP>;
  const double* d = a.rp.d;
  const int64_t N = a.rp.n;
  const double* rb = red + b * C::OUT;
  const double gp = rb[C::IG];
  const double fv = 1.0 + rb[C::IF], fpv = rb[C::IFP];
  const int neg = P.neg[b], zero = P.zero[b];
  const double sigma = P.sigma[b];
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
      if (a.phase_a_only) {  // isolated: hand the bracket to the presolve and stage 2
        if (a.writer) {
          const int64_t r = j - a.j0;
          a.br_lo[r] = lo;
          a.br_hi[r] = hi;
          a.br_ok[r] = 3;
          a.br_pl[r] = s.pl[b];
          a.br_ph[r] = s.ph[b];
          a.pa_evals[r] = s.iters[b];
        }
        s.active[b] = 2;
        return;
      }
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
    // sigma' from the scalar secular function instead of the stale y: f =
    // det(J) det S and sigma = det S / P with P the product of S's other
    // eigenvalues, so sigma' = det(J) f' / P - sigma P'/P ~ det(J) f' sigma
    // / det S (sigma is tiny at the presolved root). One psi-Newton step
    // with it replaces a second evaluation at the same point.
    double sj = 1.0;
    for (int r = 0; r < a.rp.k; ++r) sj *= (double)a.rp.sgn[r];
    if (sigma != 0.0 && isfinite(fpv) && P.ldet[b] == P.ldet[b]) {
      const double ratio = (double)P.dsgn[b] * copysign(exp2(log2(fabs(sigma)) - P.ldet[b]), sigma);
      const double gest = sj * fpv * ratio;
      if (gest > 0.0 && isfinite(gest)) {
        const double den = sigma + dl * gest;
        const double st = (den != 0.0) ? -dl * sigma / den : NAN;
        // (never a convergence verdict: sigma' is an estimate; the next
        // evaluation, with the refreshed y, judges the step)
        const double dn = dl + st;
        if (dn > lo && dn < hi) {
          s.delta[b] = dn;
          s.psi_new[b] = 1;  // do not judge the next step by this estimate
        }
      }
    }
    return;  // (else the same point again, now a bracket end)
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
      s.psi_new[b] = 1;
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
  // at the rounding floor of the S evaluation: |sigma| within the rounding
  // error of the pole sum (LAPACK dlaed4's |f| <= eps erretm for S) -- the
  // iterate is a root to working precision unless a neighbouring pole is
  // within 1e10 times the implied uncertainty (clustered poles, where the
  // vector needs delta to its own ulps)
  bool nfloor = false;
  if (!s.fmode[b] && a.noise_c > 0.0 && a.un2 && gp > 0.0) {
    const double gnv = rb[C::IGN];
    if (fabs(sigma) <= a.noise_c * DBL_EPSILON * (1.0 + gnv)) {
      const int64_t o = s.o[b];
      double gd = INFINITY;
      if (o > 0) gd = fmin(gd, fabs((d[o - 1] - s.dob[b]) - dl));
      if (o + 1 < N) gd = fmin(gd, fabs((d[o + 1] - s.dob[b]) - dl));
      nfloor = fabs(sigma) / gp <= 1e-10 * gd;
    }
  }
  const bool sdone =
      !s.fmode[b] && (nfloor || (fabs(step) <= a.step_tol * DBL_EPSILON * fabs(dl)) ||
                      (stalled && (fabs(step) <= a.floor_rel * fabs(dl) ||
                                   (far && fabs(step) <= a.floor_ulps * DBL_EPSILON *
                                                             fabs(s.dob[b] + dl)))));
  if (sdone || w <= tol || zero || s.iters[b] > a.max_iters) {
    // two more inverse-iteration steps on the same factorization follow (the
    // eigenvector formula needs y to the accuracy of the root)
    P.fin[b] = 1;
    s.fin_o[b] = s.o[b];
    s.fin_delta[b] = dl;
    s.fin_value[b] = s.dob[b] + dl;
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
  } else if (s.psi_new[b]) {
    // the first psi step after the switch used sigma' along the y of the
    // previous (f-Newton) iterate: too inaccurate to judge the next one by
    s.step_prev[b] = w;
  } else {
    s.step_prev[b] = step;
  }
  s.psi_new[b] = 0;
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


// Tail compaction (warp 0): once the root queue is drained, the active slots
// move to the lowest positions so the pass runs only the m-tiles that hold
// them (secular_pass mt < 4). A slot's arithmetic does not depend on its
// position, so this changes only the cost of the tail passes. Returns the
// number of active slots.
template <int KP>
__device__ int compact_slots(SolveSmem& s, double* y) {
  const int b = threadIdx.x & 31;
  const bool on = s.active[b] == 1;
  const unsigned mask = __ballot_sync(0xffffffffu, on);
  const int dst = __popc(mask & ((1u << b) - 1u));
  const int na = __popc(mask);
  if (mask == ((na == 32) ? 0xffffffffu : ((1u << na) - 1u))) return na;  // already packed
  double dv[5];
  int64_t iv[5];
  int nv[10];
  double yv[KP];
  if (on) {
    dv[0] = s.dob[b], dv[1] = s.delta[b], dv[2] = s.lo[b], dv[3] = s.hi[b], dv[4] = s.step_prev[b];
    iv[0] = s.j[b], iv[1] = s.o[b], iv[2] = s.below[b], iv[3] = s.pl[b], iv[4] = s.ph[b];
    nv[0] = s.hit[b], nv[1] = s.phase[b], nv[2] = s.lo_ok[b], nv[3] = s.hi_ok[b];
    nv[4] = s.iters[b], nv[5] = s.itersA[b], nv[6] = s.fmode[b], nv[7] = s.warm[b];
    nv[8] = s.psi_new[b];
    for (int c = 0; c < KP; ++c) yv[c] = y[b * KP + c];
  }
  __syncwarp();
  s.active[b] = (b < na) ? 1 : 0;
  if (on) {
    const int d = dst;
    s.dob[d] = dv[0], s.delta[d] = dv[1], s.lo[d] = dv[2], s.hi[d] = dv[3], s.step_prev[d] = dv[4];
    s.j[d] = iv[0], s.o[d] = iv[1], s.below[d] = iv[2], s.pl[d] = iv[3], s.ph[d] = iv[4];
    s.hit[d] = nv[0], s.phase[d] = nv[1], s.lo_ok[d] = nv[2], s.hi_ok[d] = nv[3];
    s.iters[d] = nv[4], s.itersA[d] = nv[5], s.fmode[d] = nv[6], s.warm[d] = nv[7];
    s.psi_new[d] = nv[8];
    for (int c = 0; c < KP; ++c) y[d * KP + c] = yv[c];
  }
  __syncwarp();
  return na;
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
__global__ void __launch_bounds__(kPassThreads, KP <= 16 ? 2 : 1) solve_roots_kernel(SolveArgs<KP> a,
                                                                      double* gscratch) {
  using C = PassCfg<KP>;
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) double smem[];
  double* y = smem + C::SMEM_DOUBLES;                      // [32][KP]
  // [KP(KP+1)/2][32] (KP <= 16): overlays the pass's tiles and D buffer, which are
  // dead while the step runs (the pass result it reads lies beyond them)
  double* Fs = smem;
  static_assert(!kFactorInSmem<KP> || C::FACT <= 2 * C::TILE_DOUBLES + C::DBUF_DOUBLES,
                "factor storage must fit in the pass tiles");
  SolveSmem& s = *reinterpret_cast<SolveSmem*>(y + 32 * KP);
  ParSmem<KP>& P = *reinterpret_cast<ParSmem<KP>*>(reinterpret_cast<char*>(&s) + kSolveSmemPad);
  __shared__ int any, mt_sh, need_f;
  __shared__ int drained;
  const int t = threadIdx.x;
  int rank = 0;
  if constexpr (CL > 1) rank = (int)cg::this_cluster().block_rank();
  a.writer = (rank == 0);
  const int64_t N = a.rp.n;
  const int64_t chunk = (N + CL - 1) / CL;
  const int64_t plo = (rank * chunk < N) ? rank * chunk : N;
  const int64_t pcnt = ((plo + chunk < N) ? plo + chunk : N) - plo;
  // slot b's matrix: element (i, j), i >= j, at F[b * esl + (i (i + 1) / 2 + j) * es]
  double* F;
  size_t esl;
  int es;
  if constexpr (kFactorInSmem<KP>) {
    F = Fs;
    esl = 1;
    es = 32;
  } else {
    F = gscratch + (size_t)blockIdx.x * 32 * KP * KP;
    esl = (size_t)KP * KP;
    es = 1;
  }
  const int lane = t & 31;
  if (t < 32) s.active[t] = 2;
  if (t == 0) drained = 0;
  __syncthreads();
  PassOpts o;
  // a phase-A stage bisects on the count alone: no sigma' (g) and no f
  const double* alpha_pass = (a.alpha && !a.phase_a_only) ? a.alpha + plo : nullptr;
  o.alpha = alpha_pass;
  o.un2 = (a.un2 && !a.phase_a_only && a.noise_c > 0.0) ? a.un2 + plo : nullptr;
  o.want_sigma = !a.phase_a_only;
  unsigned long long npass = 0, nact = 0;
  long long c_refill = 0, c_pass = 0, c_red = 0, c_step = 0;  // SM cycles (thread 0)
  long long c_load = 0, c_fact = 0, c_solve = 0;
  for (;;) {
    const long long t0 = clock64();
    // ---- refill finished slots from the root queue
    if constexpr (CL == 1) {
      if (t < 32 && s.active[t] == 2) {
        const unsigned long long nj = atomicAdd(a.next_root, 1ull);
        if ((int64_t)nj < a.j_end) slot_init<KP>(s, y, t, a.order ? a.order[nj - a.j0] : (int64_t)nj, a);
        else s.active[t] = 0, drained = 1;
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
        if ((int64_t)nj < a.j_end) slot_init<KP>(s, y, t, a.order ? a.order[nj - a.j0] : (int64_t)nj, a);
        else s.active[t] = 0, drained = 1;
      }
    }
    // the queue is drained: pack the remaining slots (every CTA of a cluster
    // holds the same state and packs it the same way)
    if (t < 32) {
      __syncwarp();
      int mt = 4;
      if (C::MMA && a.compact && drained) {
        const int na = compact_slots<KP>(s, y);
        mt = (na <= 8) ? 1 : (na <= 16 ? 2 : 4);
      }
      if (t == 0) mt_sh = mt;
    }
    if (t == 0) {
      int v = 0, c = 0, nf = 0;
      for (int b = 0; b < 32; ++b) {
        v |= s.active[b];
        c += (s.active[b] == 1);
        // f, f' are read by the f-Newton phase and by the first (warm)
        // evaluation of a presolved root (its sigma' estimate)
        nf |= (s.active[b] == 1 && s.phase[b] == 1 && (s.fmode[b] || s.warm[b]));
      }
      any = v;
      need_f = nf;
      npass += (v != 0);
      nact += c;
    }
    __syncthreads();
    if (!any) break;
    const long long t1 = clock64();
    // ---- pole pass over this CTA's slice
    PassSlots sl{s.dob, s.delta, y, s.active, s.hit};
    o.alpha = need_f ? alpha_pass : nullptr;
    secular_pass<KP>(a.rp.d + plo, a.rp.u + plo * KP, pcnt, sl, o, smem, mt_sh);
    const double* red = pass_result<KP>(smem);
    const long long t2 = clock64();
    if constexpr (CL > 1) {
      // in place, in two phases: rank r sums its slice of the partials over
      // the ranks in rank order, then stores the sums into every rank's copy
      cg::cluster_group cl = cg::this_cluster();
      constexpr int SL = (C::RED_DOUBLES + CL - 1) / CL;
      constexpr int PER = (SL + kPassThreads - 1) / kPassThreads;
      double* redw = const_cast<double*>(red);
      cl.sync();  // all partial sums of this iteration are in place
      double v[PER];
#pragma unroll
      for (int m = 0; m < PER; ++m) {
        const int idx = rank * SL + m * kPassThreads + t;
        v[m] = 0.0;
        if (m * kPassThreads + t < SL && idx < C::RED_DOUBLES)
          for (int r = 0; r < CL; ++r) v[m] += cl.map_shared_rank(redw, r)[idx];
      }
      int h = 0;
      if (t < 32)
        for (int r = 0; r < CL; ++r) h |= cl.map_shared_rank(&s, r)->hit[t];
      cl.sync();  // partials no longer read remotely
#pragma unroll
      for (int m = 0; m < PER; ++m) {
        const int idx = rank * SL + m * kPassThreads + t;
        if (m * kPassThreads + t < SL && idx < C::RED_DOUBLES)
          for (int r = 0; r < CL; ++r) cl.map_shared_rank(redw, r)[idx] = v[m];
      }
      if (t < 32) s.hit[t] = h;
      cl.sync();  // sums in place everywhere
    }
    const long long t3 = clock64();
    // ---- per-slot step (all warps): factor S, inverse iteration, Newton
    if (t < 32) slot_pre<KP>(s, P, y, t, a);
    __syncthreads();
    par_load_S<KP>(red, a.rp.sgn, a.rp.k, F, esl, es, P);
    __syncthreads();
    const long long t3a = clock64();
    par_factor<KP>(F, esl, es, P);
    const long long t3b = clock64();
    if (t < 32 && P.ev[t]) {
      const int b = t;
      double pscale = 0.0;
      for (int c = 0; c < KP; ++c) pscale = fmax(pscale, fabs(FA(c, c)));
      // an exactly zero pivot (x is a root to working precision) is replaced
      // by a tiny multiple of the pivot scale: inverse iteration then still
      // returns the null vector instead of overflowing
      P.tiny[b] = 1e-4 * DBL_EPSILON * fmax(pscale, 1e-300);
      P.sigma[b] = 0.0;
      for (int c = 0; c < KP; ++c) P.z[c][b] = y[b * KP + c];
      if (s.warm[b]) {  // det S from the pivots (log scale: k pivots may over/underflow)
        double l2 = 0.0;
        int sg = 1;
        for (int k = 0; k < KP; ++k) {
          const int bt = P.bs[k][b];
          double v;
          if (bt == 0) v = FA(k, k);
          else if (bt == 1) v = FA(k, k) * FA(k + 1, k + 1) - FA(k + 1, k) * FA(k + 1, k);
          else continue;
          if (v < 0.0) sg = -sg;
          l2 += log2(fabs(v));
        }
        P.ldet[b] = l2;
        P.dsgn[b] = sg;
      }
    }
    // Inverse iteration y <- S^-1 y / |.| (sigma: Rayleigh quotient). Every
    // evaluated slot takes one step, then the slots without a warm start take
    // their Newton step (slot_post); the warm slots' second and third steps
    // and the two final steps of the slots that just converged share the same
    // two solves (at most three solves per pass instead of five; the
    // arithmetic of every slot is unchanged).
    for (int it = 0; it < 3; ++it) {
      const bool selw = P.ev[lane] && P.ninv[lane] > it;         // refresh y (+ sigma)
      const bool self = it > 0 && P.fin[lane] == 1;               // converged: final steps
      if (!__syncthreads_or(selw || self)) break;
      if (t < 32 && self) {
        for (int c = 0; c < KP; ++c) P.z[c][t] = y[t * KP + c];
      }
      __syncthreads();
      par_solve<KP>(F, esl, es, P, selw || self);
      if (t < 32 && selw) {
        double zz = 0.0, zy = 0.0;
        for (int c = 0; c < KP; ++c) zz += P.z[c][t] * P.z[c][t], zy += P.z[c][t] * y[t * KP + c];
        if (!(zz > 0.0 && isfinite(zz))) {
          P.ninv[t] = 0;
        } else {
          P.sigma[t] = zy / zz;
          const double inv = rsqrt(zz);
          for (int c = 0; c < KP; ++c) {
            const double v = P.z[c][t] * inv;
            y[t * KP + c] = v;
            P.z[c][t] = v;
          }
        }
      }
      if (t < 32 && self) {
        double z2 = 0.0;
        for (int c = 0; c < KP; ++c) z2 += P.z[c][t] * P.z[c][t];
        if (!(z2 > 0.0 && isfinite(z2))) {
          P.fin[t] = 2;
        } else {
          const double inv = rsqrt(z2);
          for (int c = 0; c < KP; ++c) y[t * KP + c] = P.z[c][t] * inv;
        }
      }
      if (it == 0 && t < 32 && P.ev[t] && !s.warm[t]) slot_post<KP>(s, P, y, t, red, a);
    }
    const long long t3c = clock64();
    if (t < 32 && P.ev[t] && s.warm[t]) slot_post<KP>(s, P, y, t, red, a);
    __syncthreads();
    if (t < 32 && P.fin[t]) {
      double yc[KP];
      for (int c = 0; c < KP; ++c) yc[c] = y[t * KP + c];
      slot_finish<KP>(s, yc, t, a, s.fin_o[t], s.fin_delta[t], s.fin_value[t], 0, y);
    }
    __syncthreads();
    const long long t4 = clock64();
    c_load += t3a - t3;
    c_fact += t3b - t3a;
    c_solve += t3c - t3b;
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
    atomicAdd(a.prof + 7, (unsigned long long)c_load);
    atomicAdd(a.prof + 8, (unsigned long long)c_fact);
    atomicAdd(a.prof + 9, (unsigned long long)c_solve);
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

// alpha_g = sum_s w_s^T adj(M_g) J w_s with M_g = I + J T_g = J S_g (S_g = J +
// T_g symmetric, J^2 = I), so adj(M_g) J = det(M_g) S_g^-1 and alpha_g =
// det(J) det(S_g) sum_s w_s^T S_g^-1 w_s: one Bunch-Kaufman factorization of
// S_g (par_factor, all warps) and one solve per row of the group. Groups
// whose pivots span more than 1e8 (the reference's switch to cofactor
// expansion, secular.cpp:49-124) take the reference's adjugate route.
template <int KP>
__global__ void __launch_bounds__(kPassThreads, KP <= 16 ? 2 : 1) group_weights_kernel(WeightArgs<KP> a) {
  using C = PassCfg<KP>;
  extern __shared__ __align__(16) double smem[];
  __shared__ double dob[32], delta[32], acc[32];
  __shared__ int active[32], hit[32], route[32];
  __shared__ int64_t maxlen;
  const int t = threadIdx.x, lane = t & 31;
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
  const double* red = pass_result<KP>(smem);
  // (KP <= 16: overlays the pass's tiles and D buffer, dead after the pass)
  constexpr bool kSmemF = KP <= 16;
  static_assert(!kSmemF || C::FACT <= 2 * C::TILE_DOUBLES + C::DBUF_DOUBLES,
                "factor storage must fit in the pass tiles");
  double* F = kSmemF ? smem : a.scratch + (size_t)blockIdx.x * 32 * 4 * KP * KP;
  const size_t esl = kSmemF ? 1 : (size_t)4 * KP * KP;
  constexpr int es = kSmemF ? 32 : 1;
  ParSmem<KP>& P = *reinterpret_cast<ParSmem<KP>*>(smem + C::SMEM_DOUBLES);
  if (t < 32) {
    P.ev[t] = active[t];
    P.neg[t] = 0;
    P.zero[t] = 0;
    P.dskip[t] = 0;
  }
  if (t == 0) {
    int64_t m = 0;
    for (int b = 0; b < 32; ++b)
      if (g0 + b < a.ng) m = (a.glen[g0 + b] > m) ? a.glen[g0 + b] : m;
    maxlen = m;
  }
  __syncthreads();
  par_load_S<KP>(red, a.sgn, a.k, F, esl, es, P);
  __syncthreads();
  par_factor<KP>(F, esl, es, P);
  __syncthreads();
  if (t < 32 && active[t]) {
    const int b = t;
    double det = 1.0, pmax = 0.0, pmin = INFINITY;
    for (int k = 0; k < KP; ++k) {
      const int bt = P.bs[k][b];
      double pv;
      if (bt == 0) {
        pv = FA(k, k);
        det *= pv;
        pv = fabs(pv);
      } else if (bt == 1) {
        const double d2 = FA(k, k) * FA(k + 1, k + 1) - FA(k + 1, k) * FA(k + 1, k);
        det *= d2;
        pv = sqrt(fabs(d2));
      } else {
        continue;
      }
      pmax = fmax(pmax, pv);
      pmin = fmin(pmin, pv);
    }
    double sj = 1.0;
    for (int r = 0; r < a.k; ++r) sj *= (double)a.sgn[r];
    route[b] = (!P.zero[b] && pmin > 1e-8 * pmax && isfinite(det)) ? 1 : 0;
    P.sigma[b] = sj * det;
    acc[b] = 0.0;
  }
  __syncthreads();
  for (int64_t si = 0; si < maxlen; ++si) {
    const int64_t g = g0 + lane;
    const bool sel = active[lane] && route[lane] && si < a.glen[g];
    if (t < 32 && sel) {
      const double* w = a.u + (a.gstart[g] + si) * KP;
      for (int c = 0; c < KP; ++c) P.z[c][t] = w[c];
    }
    __syncthreads();
    par_solve<KP>(F, esl, es, P, sel);
    __syncthreads();
    if (t < 32 && sel) {
      const double* w = a.u + (a.gstart[g] + si) * KP;
      double v = 0.0;
      for (int c = 0; c < KP; ++c) v += w[c] * P.z[c][t];
      acc[t] += v;
    }
  }
  __syncthreads();
  if (t < 32 && active[t]) {
    const int64_t g = g0 + t;
    if (route[t]) {
      a.alpha[g] = P.sigma[t] * acc[t];
    } else {  // the reference's adjugate route (ill-conditioned M_g)
      const int k = a.k;
      double* M = a.scratch + ((size_t)blockIdx.x * 32 + t) * 4 * KP * KP;
      double* adj = M + KP * KP;
      double* work = adj + KP * KP;
      const double* rb = red + t * C::OUT;
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
}

template <int KP, int CL>
size_t solve_smem_bytes() {
  using C = PassCfg<KP>;
  return sizeof(double) * (C::SMEM_DOUBLES + 32 * KP) +
         kSolveSmemPad + sizeof(ParSmem<KP>);
}

template <int KP>
void launch_sweep(const ReducedView& rp, int* counts, int64_t qbeg, int64_t qend,
                  DeviceScratch& ws, cudaStream_t st) {
  using C = PassCfg<KP>;
  const size_t sm = sizeof(double) * C::SMEM_DOUBLES + sizeof(ParSmem<KP>);
  EIGB_CUDA(cudaFuncSetAttribute(count_sweep_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm));
  if (qend <= qbeg) return;
  const int64_t grid = cdiv(qend - qbeg, 32);
  double* gs = KP <= 16 ? nullptr : ws.get_f64("sweep_scratch", (size_t)grid * 32 * KP * KP);
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
void launch_solve(const ReducedView& rp, const double* alpha, double* br_lo, double* br_hi,
                  int* br_ok, int64_t* br_pl, int64_t* br_ph, const int64_t* f_o,
                  const double* f_delta, const int* f_state, const int64_t* order, int64_t j0,
                  int64_t j1, int64_t q_end, int phase_a_only, int* pa_evals, bool first_stage,
                  const RootRecords& out, const SolveOptions& opt, DeviceScratch& ws, int sms,
                  cudaStream_t st, const double* un2) {
  SolveArgs<KP> a;
  a.phase_a_only = phase_a_only;
  a.pa_evals = pa_evals;
  a.f_o = f_o;
  a.f_delta = f_delta;
  a.f_state = f_state;
  a.order = order;
  a.rp = rp;
  a.alpha = alpha;
  a.br_lo = br_lo;
  a.br_hi = br_hi;
  a.br_ok = br_ok;
  a.br_pl = br_pl;
  a.br_ph = br_ph;
  a.j0 = j0;
  a.j_end = q_end;  // queue positions [j0, q_end) (order maps them to roots)
  a.out = out;
  a.m_neg = rp.m_neg;
  a.p_pos = rp.k - rp.m_neg;
  a.lo_clip = rp.lo_clip;
  a.hi_clip = rp.hi_clip;
  a.step_tol = opt.step_tol;
  a.max_iters = opt.max_iters;
  a.writer = 1;
  const int64_t nroots = q_end - j0;
  (void)j1;
  a.next_root = reinterpret_cast<unsigned long long*>(ws.get_i64("solve_counter", 1));
  a.prof = reinterpret_cast<unsigned long long*>(ws.get_i64("solve_prof", 12));
  a.trace_j = opt.trace_root;
  a.fexit_rel = opt.fexit_rel;
  a.floor_rel = opt.floor_rel;
  a.floor_ulps = opt.floor_ulps;
  a.stall_ratio = opt.stall_ratio;
  a.geo_bisect = opt.geo_bisect;
  a.compact = opt.compact;
  a.noise_c = opt.noise_c;
  a.un2 = un2;
  a.trace = ws.get_f64("solve_trace", (size_t)kTraceRows * kTraceCols);
  if (first_stage) {  // a split solve's second stage keeps the first stage's trace and profile
    if (opt.trace_root >= 0)
      EIGB_CUDA(cudaMemsetAsync(a.trace, 0, sizeof(double) * kTraceRows * kTraceCols, st));
    EIGB_CUDA(cudaMemsetAsync(a.prof, 0, 12 * sizeof(unsigned long long), st));
  }
  set_u64_kernel<<<1, 1, 0, st>>>(a.next_root, (unsigned long long)j0);
  EIGB_LAUNCH_CHECK();
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
  const size_t sm = sizeof(double) * C::SMEM_DOUBLES + sizeof(ParSmem<KP>);
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
  double* scratch;      // gridDim.x * 32 * kInertiaScratch<KP>
  double* alpha_out;    // != nullptr: residue of every simple pole (at its row)
  const unsigned long long* nb_dev;  // != nullptr: the count on the device (nb: upper bound)
};

template <int KP>
constexpr int kInertiaScratch = 6 * KP * KP + KP;

// Residue of the simple pole v with row w (proj/src/secular.cpp:168-202, as
// group_weights_kernel): S = J + T(v) over the other rows, M = J S, alpha =
// w^T adj(M) J w = det(J) det(S) w^T S^-1 w from a Bunch-Kaufman
// factorization of S; pivots spanning more than 1e8 take the reference's
// adjugate route. S: full k x k (ld KP); rb: the pass result (packed T).
template <int KP>
__device__ double pole_residue(const double* S, const double* rb, const int* sgn, int k,
                               const double* w, double* work) {
  using C = PassCfg<KP>;
  double* A = work;  // KP * KP
  for (int r = 0; r < k; ++r)
    for (int c = 0; c < k; ++c) A[r * KP + c] = S[r * KP + c];
  int piv[KP], zero = 0;
  bk_factor(A, k, KP, piv, &zero, 1);
  double det = 1.0, pmax = 0.0, pmin = INFINITY;
  for (int q = 0; q < k;) {
    double pv;
    if (piv[q] >= 0) {
      pv = A[q * KP + q];
      det *= pv;
      pv = fabs(pv);
      q += 1;
    } else {
      const double d2 = A[q * KP + q] * A[(q + 1) * KP + q + 1] - A[(q + 1) * KP + q] * A[(q + 1) * KP + q];
      det *= d2;
      pv = sqrt(fabs(d2));
      q += 2;
    }
    pmax = fmax(pmax, pv);
    pmin = fmin(pmin, pv);
  }
  double sj = 1.0;
  for (int r = 0; r < k; ++r) sj *= (double)sgn[r];
  if (!zero && pmin > 1e-8 * pmax && isfinite(det)) {
    double z[KP];
    for (int r = 0; r < k; ++r) z[r] = w[r];
    bk_solve(A, k, KP, piv, z, 0.0, 1);
    double v = 0.0;
    for (int r = 0; r < k; ++r) v += w[r] * z[r];
    return sj * det * v;
  }
  // the reference's adjugate route (ill-conditioned M)
  double* M = work;  // KP * KP (A is dead)
  double* adj = M + KP * KP;
  double* aw = adj + KP * KP;  // 2 KP * KP
  for (int r = 0; r < k; ++r)
    for (int c = 0; c < k; ++c) {
      const double tv = (r <= c) ? rb[C::pidx(r, c)] : rb[C::pidx(c, r)];
      M[r * KP + c] = (r == c ? 1.0 : 0.0) + (double)sgn[r] * tv;
    }
  adjugate_dev(M, k, KP, adj, aw);
  double al = 0.0;
  for (int r = 0; r < k; ++r) {
    double tt = 0.0;
    for (int c = 0; c < k; ++c) tt += adj[r * KP + c] * (double)sgn[c] * w[c];
    al += w[r] * tt;
  }
  return al;
}

// CL > 1: a thread-block cluster of CL CTAs per batch of 32 pole values,
// CTA r passing over pole slice r (so the 1024 batches of n = 32768 fill the
// GPU's CTA slots in 7-14 waves instead of 3.5 -- less idle last wave); rank
// 0 sums the partials in rank order over distributed shared memory and does
// the per-pole work.
template <int KP, int CL>
__global__ void __launch_bounds__(kPassThreads, KP <= 16 ? 2 : 1) pole_inertia_kernel(InertiaArgs<KP> a) {
  using C = PassCfg<KP>;
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) double smem[];
  __shared__ double dob[32], delta[32];
  __shared__ int active[32], hit[32];
  const int t = threadIdx.x;
  int rank = 0;
  if constexpr (CL > 1) rank = (int)cg::this_cluster().block_rank();
  const int64_t g0 = (int64_t)(blockIdx.x / CL) * 32;
  if (a.nb_dev) {  // launched for an upper bound of the pole values
    a.nb = (int64_t)*a.nb_dev;
    if (g0 >= a.nb) return;  // (whole clusters exit together: g0 is per cluster)
  }
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
  const int64_t N = a.rp.n, chunk = (N + CL - 1) / CL;
  const int64_t plo = (rank * chunk < N) ? rank * chunk : N;
  const int64_t pcnt = ((plo + chunk < N) ? plo + chunk : N) - plo;
  secular_pass<KP>(a.rp.d + plo, a.rp.u + plo * KP, pcnt, sl, o, smem);
  if constexpr (CL > 1) {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();  // every slice's partial sums in place
    if (rank == 0) {
      double* red = const_cast<double*>(pass_result<KP>(smem));
      for (int idx = t; idx < C::RED_DOUBLES; idx += kPassThreads) {
        double v = red[idx];
        for (int r = 1; r < CL; ++r) v += cl.map_shared_rank(red, r)[idx];
        red[idx] = v;
      }
    }
    cl.sync();  // remote partials read: the other ranks may exit
    if (rank != 0) return;
    __syncthreads();
  }
  // Simple poles (one row w at v), all warps (par_factor / par_solve on the
  // shared-memory factor storage, as K2): one Bunch-Kaufman factorization of
  // T = S(v) without w's term gives nu(T) and z = T^-1 w; the bordered matrix
  // [[T, w], [w^T, 0]] has inertia In(T) + In(-w^T z) = In(T restricted to
  // w-perp) + (1, 1), so nu(T|w-perp) = nu(T) - [w^T z < 0], and the residue
  // is alpha = det(J) det(T) w^T z. Ill-conditioned T (pivots spanning more
  // than 1e8, a zero pivot, w^T z = 0) and multiple poles take the per-slot
  // path below (Householder projection, the reference's adjugate route).
  __shared__ int slow[32];
  if constexpr (kFactorInSmem<KP>) {
    ParSmem<KP>& P = *reinterpret_cast<ParSmem<KP>*>(smem + C::SMEM_DOUBLES);
    double* F = smem;
    constexpr size_t esl = 1;
    constexpr int es = 32;
    const double* red = pass_result<KP>(smem);
    if (t < 32) {
      P.ev[t] = active[t] && a.bcnt[g0 + t] == 1;
      P.neg[t] = 0;
      P.zero[t] = 0;
      P.dskip[t] = 0;
      slow[t] = active[t];
    }
    __syncthreads();
    par_load_S<KP>(red, a.rp.sgn, a.rp.k, F, esl, es, P);
    __syncthreads();
    par_factor<KP>(F, esl, es, P);
    if (t < 32 && P.ev[t]) {
      const double* w = a.rp.u + a.brow[g0 + t] * KP;
      for (int c = 0; c < KP; ++c) P.z[c][t] = (c < a.rp.k) ? w[c] : 0.0;
      P.tiny[t] = 0.0;
    }
    __syncthreads();
    par_solve<KP>(F, esl, es, P, P.ev[t & 31] != 0);
    if (t < 32 && P.ev[t]) {
      const int b = t;
      const double* w = a.rp.u + a.brow[g0 + b] * KP;
      double wz = 0.0;
      for (int c = 0; c < a.rp.k; ++c) wz += w[c] * P.z[c][b];
      double det = 1.0, pmax = 0.0, pmin = INFINITY;
      for (int q = 0; q < KP; ++q) {
        const int bt = P.bs[q][b];
        double pv;
        if (bt == 0) {
          pv = FA(q, q);
          det *= pv;
          pv = fabs(pv);
        } else if (bt == 1) {
          const double d2 = FA(q, q) * FA(q + 1, q + 1) - FA(q + 1, q) * FA(q + 1, q);
          det *= d2;
          pv = sqrt(fabs(d2));
        } else {
          continue;
        }
        pmax = fmax(pmax, pv);
        pmin = fmin(pmin, pv);
      }
      if (!P.zero[b] && pmin > 1e-8 * pmax && isfinite(det) && wz != 0.0 && isfinite(wz)) {
        a.nu[g0 + b] = P.neg[b] - (wz < 0.0 ? 1 : 0);
        if (a.alpha_out) {
          double sj = 1.0;
          for (int r = 0; r < a.rp.k; ++r) sj *= (double)a.rp.sgn[r];
          a.alpha_out[a.brow[g0 + b]] = sj * det * wz;
        }
        slow[b] = 0;
      }
    }
    __syncthreads();
  } else {
    if (t < 32) slow[t] = active[t];
    __syncthreads();
  }
  if (t >= 32 || !slow[t]) return;
  const int64_t g = g0 + t;
  const int k = a.rp.k;
  double* T = a.scratch + ((size_t)(blockIdx.x / CL) * 32 + t) * kInertiaScratch<KP>;
  double* W = T + KP * KP;   // reflectors, one per row of R
  double* x = W + KP * KP;
  const double* rb = pass_result<KP>(smem) + t * C::OUT;
  load_S<KP>(rb, a.rp.sgn, k, T, 1);
  if (a.alpha_out) {
    const int64_t r0 = a.brow[g];
    if (a.bcnt[g] == 1)
      a.alpha_out[r0] = pole_residue<KP>(T, rb, a.rp.sgn, k, a.rp.u + r0 * KP, x + KP);
    else
      for (int r = 0; r < a.bcnt[g]; ++r) a.alpha_out[r0 + r] = 0.0;  // not a simple pole
  }
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
                    const int* bcnt, int64_t nb, int* nu, double* alpha_out,
                    const unsigned long long* nb_dev, DeviceScratch& ws, cudaStream_t st) {
  using C = PassCfg<KP>;
  const int grid = (int)cdiv(nb, 32);
  InertiaArgs<KP> a{rp, bval, brow, bcnt, nb, nu, nullptr, alpha_out, nb_dev};
  a.scratch = ws.get_f64("inertia_scratch", (size_t)grid * 32 * kInertiaScratch<KP>);
  const size_t sm = sizeof(double) * C::SMEM_DOUBLES + (kFactorInSmem<KP> ? sizeof(ParSmem<KP>) : 0);
  // pole slices of >= 4096 per CTA; pairs for the MMA ranks (two CTAs per SM)
  static int count_cl = -1;  // EIGMOD_B200_COUNT_CL=2: pole slices on CTA pairs (experiment)
  if (count_cl < 0) {
    const char* e = std::getenv("EIGMOD_B200_COUNT_CL");
    count_cl = e ? std::atoi(e) : 1;
  }
  if constexpr (PassCfg<KP>::MMA) {
    if (count_cl == 2 && rp.n >= 8192) {
      constexpr int CL = 2;
      auto kern = pole_inertia_kernel<KP, CL>;
      EIGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = CL;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3((unsigned)(grid * CL));
      cfg.blockDim = dim3(kPassThreads);
      cfg.dynamicSmemBytes = sm;
      cfg.stream = st;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      EIGB_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
      EIGB_LAUNCH_CHECK();
      return;
    }
  }
  EIGB_CUDA(cudaFuncSetAttribute(pole_inertia_kernel<KP, 1>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  pole_inertia_kernel<KP, 1><<<grid, kPassThreads, sm, st>>>(a);
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
  // one evaluation per pole value: at the first row of its run, or at pbeg
  // when the run starts before this slice (a sharded rank)
  if (a > pbeg && d[a - 1] == v) return;
  // simple poles with usable points are resolved by phase A bisection; the
  // limit count is needed where rows coincide (a compressed run) or a point
  // was unusable
  const bool multi = (a + 1 < N && d[a + 1] == v) || (a > 0 && d[a - 1] == v);
  if (c0 >= 0 && c1 >= 0 && !multi) return;
  const int64_t r0 = dev_n_less(d, N, v), r1 = dev_n_leq(d, N, v);
  const unsigned long long i = atomicAdd(nsel, 1ull);
  list[i] = a;   // first row of the slice whose count is written
  bval[i] = v;
  brow[i] = r0;  // the whole run [r0, r1): excluded rows and #{d < v}
  bcnt[i] = (int)(r1 - r0);
}

// Every distinct pole value of [pbeg, pend) (first row of its run): the
// pole-limit counts alone bracket the roots (sweep_poles mode).
__global__ void pole_all_kernel(const double* __restrict__ d, int64_t N, int64_t pbeg, int64_t pend,
                                int* __restrict__ pcounts, int64_t* __restrict__ list,
                                double* __restrict__ bval, int64_t* __restrict__ brow,
                                int* __restrict__ bcnt, unsigned long long* nsel) {
  const int64_t a = pbeg + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= pend) return;
  const double v = d[a];
  // one evaluation per pole value: at the first row of its run, or at pbeg
  // when the run starts before this slice (a sharded rank)
  if (a > pbeg && d[a - 1] == v) return;
  const int64_t r0 = dev_n_less(d, N, v), r1 = dev_n_leq(d, N, v);
  const unsigned long long i = atomicAdd(nsel, 1ull);
  list[i] = a;   // first row of the slice whose count is written
  bval[i] = v;
  brow[i] = r0;  // the whole run [r0, r1): excluded rows and #{d < v}
  bcnt[i] = (int)(r1 - r0);
}

__global__ void fill_i32_kernel(int* __restrict__ p, int64_t n, int v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void pole_scatter_kernel(const int64_t* __restrict__ list, const int64_t* __restrict__ brow,
                                    const int* __restrict__ bcnt, const int* __restrict__ nu,
                                    int64_t nsel, int m_neg, int* __restrict__ pcounts,
                                    const unsigned long long* nsel_dev = nullptr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (nsel_dev) nsel = (int64_t)*nsel_dev;
  if (i >= nsel) return;
  const int c = (int)(brow[i] + m_neg - nu[i]);
  for (int64_t a = list[i]; a < brow[i] + bcnt[i]; ++a) pcounts[a] = c;
}

// Brackets from the counts (sweep points and / or pole-limit counts), then the
// presolve and the solver stages.
void solve_after_counts(const ReducedView& rp, const double* alpha, int64_t j0, int64_t j1,
                        const RootRecords& out, const SolveOptions& opt, DeviceScratch& ws,
                        int sms, cudaStream_t st, int* counts, int* pcounts, int64_t pb,
                        int64_t pe) {
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
  const int64_t nr = j1 - j0;
  int64_t* f_o = nullptr;
  double* f_delta = nullptr;
  int* f_state = nullptr;
  const bool pre = alpha && br_lo && opt.fpre && rp.kp >= opt.fpre_min_kp;
  // the presolve profile describes this solve even when no presolve runs
  EIGB_CUDA(cudaMemsetAsync(ws.get_i64("fpre_prof", 4), 0, 4 * sizeof(int64_t), st));
  auto run_presolve = [&]() {
    f_o = ws.get_i64("fpre_o", nr);
    f_delta = ws.get_f64("fpre_delta", nr);
    f_state = ws.get_i32("fpre_state", nr);
    FPreArgs fa{rp.d, alpha, rp.n, br_lo, br_hi, br_ok, br_pl, br_ph, j0, j1, f_o, f_delta, f_state,
                reinterpret_cast<unsigned long long*>(ws.get_i64("fpre_counter", 1)),
                opt.fpre_iters,
                reinterpret_cast<unsigned long long*>(ws.get_i64("fpre_prof", 4)), opt.fpre_rel};
    EIGB_CUDA(cudaMemsetAsync(fa.prof, 0, 4 * sizeof(unsigned long long), st));
    set_u64_kernel<<<1, 1, 0, st>>>(fa.next_root, (unsigned long long)j0);
    EIGB_LAUNCH_CHECK();
    const size_t fsm = (sizeof(FPreSmem) + 15) / 16 * 16 + sizeof(double2) * kFPreTile;
    EIGB_CUDA(cudaFuncSetAttribute(fpresolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)fsm));
    int per_sm = 0;
    EIGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fpresolve_kernel,
                                                            kFPreWarps * 32, fsm));
    // few CTAs per SM so that each refills its slots from the root queue many
    // times (iteration counts vary; a one-batch CTA runs as long as its
    // slowest root)
    const int64_t grid = std::min<int64_t>((int64_t)std::min(2, std::max(1, per_sm)) * sms, cdiv(nr, 32));
    fpresolve_kernel<<<(unsigned)grid, kFPreWarps * 32, fsm, st>>>(fa);
    EIGB_LAUNCH_CHECK();
  };
  int64_t* order = nullptr;
  unsigned long long* cnt = nullptr;
  auto build_order = [&]() {
    order = ws.get_i64("root_order", nr);
    cnt = reinterpret_cast<unsigned long long*>(ws.get_i64("root_order_cnt", 8));
    EIGB_CUDA(cudaMemsetAsync(cnt, 0, 8 * sizeof(unsigned long long), st));
    order_count_kernel<<<(unsigned)cdiv(nr, 256), 256, 0, st>>>(br_ok, br_pl, br_ph, f_state, nr, cnt);
    EIGB_LAUNCH_CHECK();
    order_scatter_kernel<<<(unsigned)cdiv(nr, 256), 256, 0, st>>>(br_ok, br_pl, br_ph, f_state, nr,
                                                                  j0, cnt, order);
    EIGB_LAUNCH_CHECK();
  };
  double* un2 = nullptr;  // |u_i|^2 per reduced row (noise-floor stopping)
  if (opt.noise_c > 0.0 && rp.n > 0) {
    un2 = ws.get_f64("solve_un2", rp.n);
    row_norm2_kernel<<<(unsigned)cdiv(rp.n, 256), 256, 0, st>>>(rp.u, rp.n, rp.kp, un2);
    EIGB_LAUNCH_CHECK();
  }
#define EIGB_SOLVE(K)                                                                          \
  launch_solve<K>(rp, alpha, br_lo, br_hi, br_ok, br_pl, br_ph, f_o, f_delta, f_state, order,   \
                  j0, j1, q_end, phase_a_only, pa_evals, first_stage, out, opt, ws, sms, st, un2)
  auto solve = [&](int64_t q_end, int phase_a_only, int* pa_evals, bool first_stage) {
    switch (rp.kp) {
      case 1: EIGB_SOLVE(1); break;
      case 2: EIGB_SOLVE(2); break;
      case 4: EIGB_SOLVE(4); break;
      case 8: EIGB_SOLVE(8); break;
      case 16: EIGB_SOLVE(16); break;
      case 32: EIGB_SOLVE(32); break;
      default: throw Error(1, "", "solve_roots: unsupported padded rank");
    }
  };
#undef EIGB_SOLVE
  if (pre && opt.split_phase_a) {
    // stage 1: the roots whose sweep bracket holds other roots or poles are
    // bisected on the count until isolated (their bracket is stored); then
    // every isolated root gets the scalar presolve, and stage 2 finishes all
    build_order();  // unisolated roots first
    unsigned long long c0 = 0;
    EIGB_CUDA(cudaMemcpyAsync(&c0, cnt, sizeof(c0), cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaStreamSynchronize(st));
    int* pa_evals = ws.get_i32("pa_evals", nr);
    EIGB_CUDA(cudaMemsetAsync(pa_evals, 0, 4 * nr, st));
    if (c0 > 0) solve(j0 + (int64_t)c0, 1, pa_evals, true);
    run_presolve();
    build_order();
    solve(j1, 0, pa_evals, c0 == 0);
    return;
  }
  if (pre) run_presolve();
  if (br_lo) build_order();
  solve(j1, 0, nullptr, true);
}

}  // namespace

void solve_roots(const ReducedView& rp, const double* alpha, int64_t j0, int64_t j1,
                 const RootRecords& out, const SolveOptions& opt, DeviceScratch& ws, int sms,
                 cudaStream_t st, double* alpha_fill) {
  if (j1 <= j0) return;
  int* counts = nullptr;
  // points next to the poles of every Weyl window of roots [j0, j1)
  // (multi-GPU ranks sweep only their share)
  const int64_t pb = std::max<int64_t>(0, j0 - rp.m_neg - 1);
  const int64_t pe = std::min<int64_t>(rp.n, j1 + (rp.k - rp.m_neg) + 1);
  const int64_t qbeg = 2 * pb, qend = 2 * pe;
  if (opt.sweep && opt.sweep_poles && pe > pb) {
    // brackets from the pole-limit counts alone: one evaluation per distinct
    // pole value (the projected inertia at the pole) instead of two points
    int* pcounts = ws.get_i32("sweep_pole_counts", rp.n);
    const int64_t np = pe - pb;
    int64_t* list = ws.get_i64("psel_list", np);
    double* bval = ws.get_f64("psel_val", np);
    int64_t* brow = ws.get_i64("psel_row", np);
    int* bcnt = ws.get_i32("psel_cnt", np);
    int* nu = ws.get_i32("psel_nu", np);
    auto* nsel = reinterpret_cast<unsigned long long*>(ws.get_i64("psel_n", 1));
    EIGB_CUDA(cudaMemsetAsync(nsel, 0, 8, st));
    fill_i32_kernel<<<(unsigned)cdiv(rp.n, 256), 256, 0, st>>>(pcounts, rp.n, -1);
    EIGB_LAUNCH_CHECK();
    pole_all_kernel<<<(unsigned)cdiv(np, 256), 256, 0, st>>>(rp.d, rp.n, pb, pe, pcounts, list, bval,
                                                              brow, bcnt, nsel);
    EIGB_LAUNCH_CHECK();
    // the residues need every pole value of the problem in the window
    if (alpha_fill && !(pb == 0 && pe == rp.n))
      throw Error(1, "", "solve_roots: fused residues need all poles");
    // launched for all np pole positions; the kernels read the number of
    // distinct pole values from the device (no host round trip)
    pole_inertia(rp, bval, brow, bcnt, np, nu, ws, st, alpha_fill, nsel);
    pole_scatter_kernel<<<(unsigned)cdiv(np, 256), 256, 0, st>>>(list, brow, bcnt, nu, np, rp.m_neg,
                                                                 pcounts, nsel);
    EIGB_LAUNCH_CHECK();
    if (alpha_fill) alpha = alpha_fill;
    solve_after_counts(rp, alpha, j0, j1, out, opt, ws, sms, st, nullptr, pcounts, pb, pe);
    return;
  }
  if (alpha_fill) throw Error(1, "", "solve_roots: fused residues need the pole-limit counts");
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
      pole_inertia(rp, bval, brow, bcnt, (int64_t)nh, nu, ws, st, nullptr);
      pole_scatter_kernel<<<(unsigned)cdiv((int64_t)nh, 256), 256, 0, st>>>(list, brow, bcnt, nu,
                                                                           (int64_t)nh, rp.m_neg,
                                                                           pcounts);
      EIGB_LAUNCH_CHECK();
    }
  }
  solve_after_counts(rp, alpha, j0, j1, out, opt, ws, sms, st, counts, pcounts, pb, pe);
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
                  int64_t nb, int* nu, DeviceScratch& ws, cudaStream_t st, double* alpha_out,
                  const unsigned long long* nb_dev) {
  if (nb <= 0) return;
  switch (rp.kp) {
    case 1: launch_inertia<1>(rp, bval, brow, bcnt, nb, nu, alpha_out, nb_dev, ws, st); break;
    case 2: launch_inertia<2>(rp, bval, brow, bcnt, nb, nu, alpha_out, nb_dev, ws, st); break;
    case 4: launch_inertia<4>(rp, bval, brow, bcnt, nb, nu, alpha_out, nb_dev, ws, st); break;
    case 8: launch_inertia<8>(rp, bval, brow, bcnt, nb, nu, alpha_out, nb_dev, ws, st); break;
    case 16: launch_inertia<16>(rp, bval, brow, bcnt, nb, nu, alpha_out, nb_dev, ws, st); break;
    case 32: launch_inertia<32>(rp, bval, brow, bcnt, nb, nu, alpha_out, nb_dev, ws, st); break;
    default: throw Error(1, "", "pole_inertia: unsupported padded rank");
  }
}

}  // namespace eigb
