// K2 deflation weights and K3 batched per-root solver (sm_100a).
//
// K2 (proj/src/secular.cpp:168-202 group_weights): one pole pass per batch of
//   32 pole groups evaluated at their representatives, then per group the
//   reference's adjugate route (cofactors k <= 3, LU det*inverse, cofactor
//   expansion fallback) on M_g = J S_g, alpha_g = sum_s w_s^T adj(M_g) J w_s.
// K3 (replaces locate.cpp / sturm.cpp / rootfind.cpp:89-229, 342-377): a
//   persistent kernel whose CTAs own 32 root slots each. Every iteration one
//   pole pass evaluates S(x_b) = J + U^T (D - x_b)^-1 U for all slots; a
//   Bunch-Kaufman LDL^T gives the inertia, hence the exact eigenvalue count
//   #eig < x_b = #{d_i < x_b} + m - nu(S(x_b)), and one
//   inverse-iteration step gives the eigenvalue sigma of S nearest zero with
//   its vector y. Phase A bisects the count inside the Weyl window
//   [d_{j-m}, d_{j+p}] (proj/src/locate.cpp:159-171) until root j is alone in
//   a pole-free bracket; phase B runs Newton on sigma (sigma' = y^T S' y from
//   the same pass) in the shifted origin x = d_o + delta, safeguarded by the
//   count-certified bracket, to ~1 ulp of delta. A converged slot writes its
//   root record (value, origin, delta, y) and takes the next root index from
//   a global counter, so the batch stays full until the queue drains.
#include "secular.cuh"

#include <cfloat>

namespace eigb {

namespace {

constexpr int FLAG_COLLIDED = 1;   // bracket collapsed onto a pole
constexpr int FLAG_UNISOLATED = 2; // ulp bracket without pole-free isolation

struct SolveSmem {
  double dob[32], delta[32], lo[32], hi[32], xlast[32], sig_last[32], gp_last[32], step_prev[32];
  int64_t j[32], o[32], below[32];
  int active[32], hit[32], phase[32], lo_ok[32], hi_ok[32], iters[32];
};

template <int KP>
struct SolveArgs {
  ReducedView rp;
  int64_t j_end;
  unsigned long long* next_root;
  RootRecords out;
  double* scratch;  // gridDim.x * 32 * KP * KP
  int m_neg, p_pos;
  double lo_clip, hi_clip;
  double step_tol;
  int max_iters;
};

template <int KP>
__device__ void slot_init(SolveSmem& s, double* y, int b, int64_t j, const SolveArgs<KP>& a) {
  const int64_t N = a.rp.n;
  s.j[b] = j;
  s.lo[b] = (j - a.m_neg >= 0) ? a.rp.d[j - a.m_neg] : a.lo_clip;
  s.hi[b] = (j + a.p_pos <= N - 1) ? a.rp.d[j + a.p_pos] : a.hi_clip;
  s.lo_ok[b] = s.hi_ok[b] = 0;
  s.phase[b] = 0;
  s.iters[b] = 0;
  s.hit[b] = 0;
  s.step_prev[b] = 0.0;
  s.dob[b] = 0.0;
  s.delta[b] = 0.5 * (s.lo[b] + s.hi[b]);
  s.active[b] = 1;
  const double y0 = rsqrt((double)a.rp.k);
  for (int c = 0; c < KP; ++c) y[b * KP + c] = (c < a.rp.k) ? y0 : 0.0;
}

template <int KP>
__device__ void slot_finish(SolveSmem& s, double* y, int b, const SolveArgs<KP>& a, int64_t o,
                            double delta, double value, int flags) {
  const int64_t j = s.j[b];
  a.out.value[j] = value;
  a.out.origin[j] = o;
  a.out.delta[j] = delta;
  a.out.flags[j] = flags;
  a.out.evals[j] = s.iters[b];
  for (int c = 0; c < KP; ++c) a.out.y[j * KP + c] = y[b * KP + c];
  const unsigned long long nj = atomicAdd(a.next_root, 1ull);
  if ((int64_t)nj < a.j_end) slot_init<KP>(s, y, b, (int64_t)nj, a);
  else s.active[b] = 0;
}

// Phase A ended at ulp width without isolation: a pole inside [lo, hi] means
// the root sits on that pole (collision, proj/src/eigvec.cpp:303-323).
template <int KP>
__device__ void slot_finish_unisolated(SolveSmem& s, double* y, int b, const SolveArgs<KP>& a) {
  const double* d = a.rp.d;
  const int64_t N = a.rp.n;
  const double lo = s.lo[b], hi = s.hi[b], mid = 0.5 * (lo + hi);
  int64_t p = dev_n_less(d, N, lo);
  if (p < N && d[p] <= hi) {
    int64_t o = p;
    for (int64_t q = p + 1; q < N && d[q] <= hi; ++q)
      if (fabs(d[q] - mid) < fabs(d[o] - mid)) o = q;
    slot_finish<KP>(s, y, b, a, o, 0.0, d[o], FLAG_COLLIDED);
    return;
  }
  int64_t o = p < N ? p : N - 1;
  if (o > 0 && fabs(d[o - 1] - mid) < fabs(d[o] - mid)) o -= 1;
  slot_finish<KP>(s, y, b, a, o, mid - d[o], mid, FLAG_UNISOLATED);
}

template <int KP>
__device__ void slot_step(SolveSmem& s, double* y, int b, const double* red, double* F, int* piv,
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
      if (s.phase[b] == 0) slot_finish_unisolated<KP>(s, y, b, a);
      else slot_finish<KP>(s, y, b, a, s.o[b], cur, s.dob[b] + cur, FLAG_UNISOLATED);
      return;
    }
    s.delta[b] = alt;
    return;
  }
  // S = J + packed sum, full storage in F (ld KP)
  const double* rb = red + b * (C::P + 1);
  for (int r = 0; r < KP; ++r)
    for (int c = r; c < KP; ++c) {
      double v = rb[C::pidx(r, c)];
      if (r == c) v += (r < a.rp.k) ? (double)a.rp.sgn[r] : 1.0;
      F[r * KP + c] = v;
      F[c * KP + r] = v;
    }
  const double gp = rb[C::P];
  int zero = 0;
  const int neg = bk_factor(F, KP, KP, piv, &zero);
  double z[KP];
  for (int c = 0; c < KP; ++c) z[c] = y[b * KP + c];
  // an exactly zero pivot (x is a root to working precision) is replaced by a
  // tiny multiple of the pivot scale, so inverse iteration still returns the
  // null vector instead of overflowing
  double pscale = 0.0;
  for (int c = 0; c < KP; ++c) pscale = fmax(pscale, fabs(F[c * KP + c]));
  const double tiny = 1e-4 * DBL_EPSILON * fmax(pscale, 1e-300);
  bk_solve(F, KP, KP, piv, z, tiny);
  double zz = 0.0, zy = 0.0;
  for (int c = 0; c < KP; ++c) zz += z[c] * z[c], zy += z[c] * y[b * KP + c];
  double sigma = 0.0;
  if (zz > 0.0 && isfinite(zz)) {
    sigma = zy / zz;
    const double inv = rsqrt(zz);
    for (int c = 0; c < KP; ++c) y[b * KP + c] = z[c] * inv;
  }
  const int64_t j = s.j[b];

  if (s.phase[b] == 0) {
    const double x = s.delta[b];
    const int64_t below = dev_n_less(d, N, x);
    const int64_t cnt = below + a.m_neg - neg;
    if (cnt >= j + 1) { s.hi[b] = x; s.hi_ok[b] = (cnt == j + 1); }
    else { s.lo[b] = x; s.lo_ok[b] = (cnt == j); }
    const double lo = s.lo[b], hi = s.hi[b];
    if (s.lo_ok[b] && s.hi_ok[b] && dev_n_less(d, N, hi) == dev_n_leq(d, N, lo)) {
      // isolated: shifted origin at the nearer bracketing pole
      const int64_t pa = dev_n_leq(d, N, lo) - 1, pb = pa + 1;
      const double mid = 0.5 * (lo + hi);
      int64_t o;
      if (pa < 0) o = pb;
      else if (pb >= N) o = pa;
      else o = (mid - d[pa] <= d[pb] - mid) ? pa : pb;
      const double dob = d[o];
      s.o[b] = o;
      s.below[b] = pa + 1;
      s.dob[b] = dob;
      s.lo[b] = lo - dob;
      s.hi[b] = hi - dob;
      s.phase[b] = 1;
      const double dl = x - dob;
      const double step = (gp > 0.0) ? -sigma / gp : NAN;
      double dn = dl + step;
      if (!(dn > s.lo[b] && dn < s.hi[b])) dn = 0.5 * (s.lo[b] + s.hi[b]);
      s.step_prev[b] = s.hi[b] - s.lo[b];
      s.delta[b] = dn;
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
  // phase B (delta domain)
  const double dl = s.delta[b];
  const int64_t cnt = s.below[b] + a.m_neg - neg;
  if (cnt >= j + 1) s.hi[b] = dl; else s.lo[b] = dl;
  const double lo = s.lo[b], hi = s.hi[b];
  const double step = (gp > 0.0) ? -sigma / gp : NAN;
  const double w = hi - lo;
  const double tol = 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi));
  if ((fabs(step) <= a.step_tol * DBL_EPSILON * fabs(dl)) || w <= tol || zero ||
      s.iters[b] > a.max_iters) {
    // two more inverse-iteration steps on the same factorization: the
    // eigenvector formula needs y to the accuracy of the root
    for (int it = 0; it < 2; ++it) {
      for (int c = 0; c < KP; ++c) z[c] = y[b * KP + c];
      bk_solve(F, KP, KP, piv, z, tiny);
      double z2 = 0.0;
      for (int c = 0; c < KP; ++c) z2 += z[c] * z[c];
      if (!(z2 > 0.0 && isfinite(z2))) break;
      const double inv = rsqrt(z2);
      for (int c = 0; c < KP; ++c) y[b * KP + c] = z[c] * inv;
    }
    slot_finish<KP>(s, y, b, a, s.o[b], dl, s.dob[b] + dl, 0);
    return;
  }
  double dn = dl + step;
  if (!(dn > lo && dn < hi) || !(fabs(step) <= 0.5 * fabs(s.step_prev[b]))) {
    dn = 0.5 * (lo + hi);
    s.step_prev[b] = w;
  } else {
    s.step_prev[b] = step;
  }
  s.delta[b] = dn;
}

template <int KP>
__global__ void __launch_bounds__(kPassThreads, 1) solve_roots_kernel(SolveArgs<KP> a) {
  using C = PassCfg<KP>;
  extern __shared__ __align__(16) double smem[];
  double* tiles = smem;
  double* red = tiles + 2 * C::TILE_DOUBLES;
  double* y = red + C::RED_DOUBLES;                       // [32][KP]
  SolveSmem& s = *reinterpret_cast<SolveSmem*>(y + 32 * KP);
  __shared__ int any;
  const int t = threadIdx.x;
  double* F = a.scratch + ((size_t)blockIdx.x * 32 + (t & 31)) * KP * KP;
  int piv[KP];

  if (t < 32) {
    const unsigned long long nj = atomicAdd(a.next_root, 1ull);
    if ((int64_t)nj < a.j_end) slot_init<KP>(s, y, t, (int64_t)nj, a);
    else s.active[t] = 0;
  }
  __syncthreads();
  for (;;) {
    if (t == 0) {
      int v = 0;
      for (int b = 0; b < 32; ++b) v |= s.active[b];
      any = v;
    }
    __syncthreads();
    if (!any) break;
    PassSlots sl{s.dob, s.delta, y, s.active, s.hit};
    secular_pass<KP>(a.rp.d, a.rp.u, a.rp.n, sl, true, false, 0.0, tiles, red);
    if (t < 32 && s.active[t]) slot_step<KP>(s, y, t, red, F, piv, a);
    __syncthreads();
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
  double* tiles = smem;
  double* red = tiles + 2 * C::TILE_DOUBLES;
  __shared__ double dob[32], delta[32], yy[32 * KP];
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
  PassSlots sl{dob, delta, yy, active, hit};
  secular_pass<KP>(a.rep, a.u, a.n, sl, false, true, 0.0, tiles, red);
  if (t < 32 && active[t]) {
    const int64_t g = g0 + t;
    const int k = a.k;
    double* M = a.scratch + ((size_t)blockIdx.x * 32 + t) * 4 * KP * KP;
    double* adj = M + KP * KP;
    double* work = adj + KP * KP;
    const double* rb = red + t * (C::P + 1);
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

template <int KP>
size_t solve_smem_bytes() {
  using C = PassCfg<KP>;
  return sizeof(double) * (2 * C::TILE_DOUBLES + C::RED_DOUBLES + 32 * KP) + sizeof(SolveSmem);
}

template <int KP>
size_t weights_smem_bytes() {
  using C = PassCfg<KP>;
  return sizeof(double) * (2 * C::TILE_DOUBLES + C::RED_DOUBLES);
}

template <int KP>
void launch_solve(const ReducedView& rp, int64_t j0, int64_t j1, const RootRecords& out,
                  const SolveOptions& opt, DeviceScratch& ws, int sms, cudaStream_t st) {
  SolveArgs<KP> a;
  a.rp = rp;
  a.j_end = j1;
  a.out = out;
  a.m_neg = rp.m_neg;
  a.p_pos = rp.k - rp.m_neg;
  a.lo_clip = rp.lo_clip;
  a.hi_clip = rp.hi_clip;
  a.step_tol = opt.step_tol;
  a.max_iters = opt.max_iters;
  const int64_t nroots = j1 - j0;
  const int grid = (int)std::min<int64_t>(sms, cdiv(nroots, 32));
  a.scratch = ws.get_f64("solve_scratch", (size_t)grid * 32 * KP * KP);
  a.next_root = reinterpret_cast<unsigned long long*>(ws.get_i64("solve_counter", 1));
  const unsigned long long start = (unsigned long long)j0;
  EIGB_CUDA(cudaMemcpyAsync(a.next_root, &start, sizeof(start), cudaMemcpyHostToDevice, st));
  const size_t sm = solve_smem_bytes<KP>();
  EIGB_CUDA(cudaFuncSetAttribute(solve_roots_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm));
  solve_roots_kernel<KP><<<grid, kPassThreads, sm, st>>>(a);
  EIGB_LAUNCH_CHECK();
}

template <int KP>
void launch_weights(const double* rep, const double* u, int64_t n, const int64_t* gstart,
                    const int64_t* glen, const double* gval, int64_t ng, const int* sgn, int k,
                    double* alpha, DeviceScratch& ws, cudaStream_t st) {
  WeightArgs<KP> a{rep, u, n, gstart, glen, gval, ng, sgn, k, alpha, nullptr};
  const int grid = (int)cdiv(ng, 32);
  a.scratch = ws.get_f64("weights_scratch", (size_t)grid * 32 * 4 * KP * KP);
  const size_t sm = weights_smem_bytes<KP>();
  EIGB_CUDA(cudaFuncSetAttribute(group_weights_kernel<KP>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  group_weights_kernel<KP><<<grid, kPassThreads, sm, st>>>(a);
  EIGB_LAUNCH_CHECK();
}

}  // namespace

void solve_roots(const ReducedView& rp, int64_t j0, int64_t j1, const RootRecords& out,
                 const SolveOptions& opt, DeviceScratch& ws, int sms, cudaStream_t st) {
  if (j1 <= j0) return;
  switch (rp.kp) {
    case 1: launch_solve<1>(rp, j0, j1, out, opt, ws, sms, st); break;
    case 2: launch_solve<2>(rp, j0, j1, out, opt, ws, sms, st); break;
    case 4: launch_solve<4>(rp, j0, j1, out, opt, ws, sms, st); break;
    case 8: launch_solve<8>(rp, j0, j1, out, opt, ws, sms, st); break;
    case 16: launch_solve<16>(rp, j0, j1, out, opt, ws, sms, st); break;
    case 32: launch_solve<32>(rp, j0, j1, out, opt, ws, sms, st); break;
    default: throw Error(1, "", "solve_roots: unsupported padded rank");
  }
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

}  // namespace eigb
