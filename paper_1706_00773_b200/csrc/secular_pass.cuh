// The secular "pole pass": for a batch of 32 evaluation points x_b (one per
// lane, "slots") accumulate, over all poles i with D_ib = 1/(d_i - x_b),
//     S_b  = J + sum_i D_ib u_i u_i^T                    (k x k, symmetric)
//     g_b  = sum_i (u_i . y_b)^2 D_ib^2                  (= y_b^T S'(x_b) y_b)
//     f_b  = 1 + sum_i alpha_i D_ib,  f'_b = sum_i alpha_i D_ib^2
// (f is the reference's scalar secular function, proj/src/secular.cpp:223-243,
// with the residues alpha from K2). This contraction is the inner loop of
//   * the deflation weights  (x_b = representative of pole group b; the
//     excluded self term is the diff == 0 case; proj/src/secular.cpp:168-202),
//   * the count sweep and the root solver,
//   * the collision vectors  (proj/src/eigvec.cpp:75-119).
//
// One CTA = 8 warps, lane = slot. Per tile of kPoleTile poles (staged in
// shared memory by cp.async, double-buffered):
//   D phase:   warp w takes poles w, w+8, ...; each lane forms its
//              difference (d_i - dob_b) - delta_b (shifted origin), one
//              MUFU.RCP64H + 4 DFMA reciprocal, writes D to shared memory and
//              accumulates g_b, f_b, f'_b. Each reciprocal is computed once.
//   FMA phase: warp w = (entry group g, pole split p) accumulates its share
//              of the packed upper triangle: per pole one D load, the row u_i
//              as warp-wide broadcasts, then (KP - r) DFMA per row r.
// Entry groups are balanced (KP = 16: rows 0-4 = 70 entries, rows 5-15 =
// 66), so no warp idles at the tile barriers.
#pragma once

#include "common.cuh"

#include <utility>

namespace eigb {

constexpr int kPassWarps = 8;
constexpr int kPassThreads = kPassWarps * 32;
constexpr int kPoleTile = 64;

template <int KP>
struct PassCfg {
  static constexpr int P = KP * (KP + 1) / 2;
  // KP = 8, 16: the FMA phase on the FP64 tensor pipe (DMMA.8x8x4, see
  // pass_body_mma); other ranks: DFMA with compile-time entries
  static constexpr bool MMA = (KP == 8 || KP == 16);
  static constexpr int EG = (KP <= 8) ? 1 : (KP == 16 ? 2 : 8);
  static constexpr int PS = kPassWarps / EG;
  // MMA layout: S (32 slots x P entries) = D (32 x poles) W (poles x P),
  // W[i][e] = u_i[r_e] u_i[c_e]: 4 m-tiles of 8 slots, n-tiles of 8 entries in
  // NG groups (MmaMap), warps = 2 m-halves x NG groups x MPS pole splits.
  static constexpr int NG = (KP == 16) ? 2 : 1;
  static constexpr int MPS = kPassWarps / (2 * NG);
  // u rows in the tile: KP + 4 doubles (20 / 12), so the fragment loads of
  // both MMA phases (rows by lane / 4 or by lane % 4) fall into distinct bank
  // pairs (two wavefronts per warp load)
  static constexpr int LDU = MMA ? KP + 4 : KP;
  // D buffer stride per k-step: 4 m-tiles x 32 A-fragment elements + 1, so
  // the D phase's stores (two k-steps per warp store) hit distinct bank pairs
  static constexpr int DKS = 4 * 32 + 1;
  // Entry group g = packed entries [e_lo(g), e_lo(g+1)): an even split of the
  // packed triangle (a row may straddle two groups), so no warp waits for the
  // other group at the tile barriers.
  __host__ __device__ static constexpr int e_lo(int g) { return (P * g) / EG; }
  // row and column of packed entry e
  __host__ __device__ static constexpr int row_of(int e) {
    int r = 0;
    while (r + 1 < KP && (r + 1) * KP - (r + 1) * r / 2 <= e) ++r;
    return r;
  }
  __host__ __device__ static constexpr int col_of(int e) {
    return row_of(e) + (e - (row_of(e) * KP - row_of(e) * (row_of(e) - 1) / 2));
  }
  // packed index of (r, c), r <= c
  __host__ __device__ static constexpr int pidx(int r, int c) {
    return r * KP - r * (r - 1) / 2 + (c - r);
  }
  // reduced output per slot: P packed entries, then g, f, f', and the
  // rounding scale sum_i |u_i|^2 |D_i| of the S evaluation (noise bound)
  static constexpr int OUT = P + 4;
  static constexpr int IG = P, IF = P + 1, IFP = P + 2, IGN = P + 3;
  // shared memory (doubles): tile = d, alpha, u rows
  // poles per tile: 128 (64 for KP = 32, whose reduction buffer is 136 KB;
  // 64 in MMA mode, 16 k-steps of 4 poles)
  static constexpr int T = MMA ? kPoleTile : ((KP >= 32) ? kPoleTile : 2 * kPoleTile);
  // tile: d, alpha, |u|^2 (noise bound), then the u rows
  static constexpr int TILE_DOUBLES = T * (LDU + 3);
  // D buffer: lane = slot order (DFMA), or A fragments per k-step (MMA)
  static constexpr int DBUF_MIN = MMA ? (T / 4) * DKS : T * 32;
  // the solver and K2 overlay their k x k factors (lower triangles, packed:
  // 32 KP (KP + 1) / 2 doubles for KP <= 16) on the tiles and the D buffer
  static constexpr int FACT = (KP <= 16) ? 32 * P : 0;
  static constexpr int DBUF_DOUBLES =
      (2 * TILE_DOUBLES + DBUF_MIN >= FACT) ? DBUF_MIN : FACT - 2 * TILE_DOUBLES;
  static constexpr int RED_DOUBLES = 32 * OUT;
  static constexpr int SMEM_DOUBLES = 2 * TILE_DOUBLES + DBUF_DOUBLES + RED_DOUBLES;
};

// Per-slot evaluation point: x_b = dob[b] + delta[b]; the difference to pole i
// is formed as (d_i - dob[b]) - delta[b] so a shifted origin keeps relative
// accuracy near d_o. active[b] == 0 disables the slot (its terms are zero).
struct PassSlots {
  double* dob;     // [32]
  double* delta;   // [32]
  double* y;       // [32][KP]  direction for g_b
  int* active;     // [32]
  int* hit;        // [32]  set when some d_i - x_b == 0 (solver: pole hit)
  const int64_t* excl_row = nullptr;  // [32] with excl_gap: exclude this row only (>= 0)
};

struct PassOpts {
  const double* alpha = nullptr;  // residues for f (nullptr: f not needed)
  const double* un2 = nullptr;    // |u_i|^2 (nullptr: no rounding-scale sum)
  bool want_sigma = false;        // accumulate g_b along y_b
  bool exclude_zero = false;      // diff == 0 drops the term (no hit flag)
  double excl_gap = 0.0;          // > 0: drop poles with |d_i - dob| < excl_gap
};

template <int KP>
__device__ __forceinline__ void load_pole_tile(double* tile, const double* __restrict__ d,
                                               const double* __restrict__ alpha,
                                               const double* __restrict__ u, int64_t i0,
                                               int64_t n, const double* __restrict__ un2 = nullptr) {
  // tile layout: [T] d, [T] alpha, [T] |u|^2, then [T][LDU] rows. Rows beyond
  // n are zero with d = NaN (NaN difference => term skipped).
  constexpr int T = PassCfg<KP>::T, LDU = PassCfg<KP>::LDU;
  double* td = tile;
  double* ta = tile + T;
  double* tn = tile + 2 * T;
  double* tu = tile + 3 * T;
  const int tid = threadIdx.x;
  const int64_t cnt = (n - i0) < T ? (n - i0) : T;
  for (int t = tid; t < T; t += kPassThreads) {
    td[t] = (t < cnt) ? d[i0 + t] : __longlong_as_double(0x7ff8000000000000ll);
    ta[t] = (t < cnt && alpha) ? alpha[i0 + t] : 0.0;
    tn[t] = (t < cnt && un2) ? un2[i0 + t] : 0.0;
  }
  if constexpr (KP >= 2) {
    constexpr int CH = KP / 2;  // 16-byte chunks per row
    const double2* src = reinterpret_cast<const double2*>(u + i0 * KP);
    for (int t = tid; t < T * CH; t += kPassThreads) {
      double2* dst = reinterpret_cast<double2*>(tu + (t / CH) * LDU) + (t % CH);
      if (t < cnt * CH) {
        const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(dst));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(src + t));
      } else {
        *dst = make_double2(0.0, 0.0);
      }
    }
  } else {
    for (int t = tid; t < T; t += kPassThreads) tu[t] = (t < cnt) ? u[i0 + t] : 0.0;
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// One packed entry E of group offset E0: compile-time row and column.
template <int KP, int E, int E0, int RLO>
__device__ __forceinline__ void fma_entry(double* acc, const double* v, const double* ur) {
  constexpr int r = PassCfg<KP>::row_of(E), c = PassCfg<KP>::col_of(E);
  acc[E - E0] = fma(v[r - RLO], ur[c], acc[E - E0]);
}

template <int KP, int E0, int RLO, int... Es>
__device__ __forceinline__ void fma_entries(double* acc, const double* v, const double* ur,
                                            std::integer_sequence<int, Es...>) {
  (fma_entry<KP, E0 + Es, E0, RLO>(acc, v, ur), ...);
}

// FMA phase of entry group G on one tile (compile-time entries, so only this
// group's accumulators are live).
template <int KP, int G>
__device__ __forceinline__ void fma_tile(const double* __restrict__ tu, const double* __restrict__ db,
                                         int p, int lane, double* acc) {
  using C = PassCfg<KP>;
  constexpr int E0 = C::e_lo(G), E1 = C::e_lo(G + 1);
  constexpr int RLO = C::row_of(E0), RHI = C::row_of(E1 - 1) + 1;
  constexpr int CLO = RLO;  // v needs ur[r] of every row touched
  constexpr int per = C::T / C::PS;
#pragma unroll 2
  for (int ii = 0; ii < per; ++ii) {
    const int i = p * per + ii;
    const double D = db[i * 32 + lane];
    double ur[KP];
    if constexpr (KP >= 2) {
#pragma unroll
      for (int c = CLO & ~1; c < KP; c += 2) {
        const double2 v = *reinterpret_cast<const double2*>(tu + i * KP + c);
        ur[c] = v.x;
        ur[c + 1] = v.y;
      }
    } else {
      ur[0] = tu[i];
    }
    // all row scales first: the DFMAs then never wait on the DMUL latency
    double v[RHI - RLO];
#pragma unroll
    for (int r = RLO; r < RHI; ++r) v[r - RLO] = D * ur[r];
    fma_entries<KP, E0, RLO>(acc, v, ur, std::make_integer_sequence<int, E1 - E0>{});
  }
}

template <int KP, int G>
__device__ __forceinline__ void pass_body(const double* __restrict__ d, const double* __restrict__ u,
                                          int64_t n, const PassSlots& slots, const PassOpts& o,
                                          double* tiles, double* dbuf, double* red, int p) {
  using C = PassCfg<KP>;
  constexpr int E = C::e_lo(G + 1) - C::e_lo(G);
  constexpr int E0 = C::e_lo(G);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const double dob = slots.dob[lane];
  const double del = slots.delta[lane];
  const bool act = slots.active[lane] != 0;
  const bool sig = o.want_sigma;
  const bool wf = o.alpha != nullptr;
  const bool wn = o.un2 != nullptr;
  double yv[KP];
#pragma unroll
  for (int c = 0; c < KP; ++c) yv[c] = sig ? slots.y[lane * KP + c] : 0.0;
  double acc[E > 0 ? E : 1];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.0;
  double gs = 0.0, fs = 0.0, fps = 0.0, gn = 0.0;
  int hit = 0;

  const int64_t ntiles = (n + C::T - 1) / C::T;
  if (ntiles > 0) load_pole_tile<KP>(tiles, d, o.alpha, u, 0, n, o.un2);
  for (int64_t t = 0; t < ntiles; ++t) {
    const double* cur = tiles + (t & 1) * C::TILE_DOUBLES;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // tile t landed; previous FMA phase done with dbuf
    if (t + 1 < ntiles)
      load_pole_tile<KP>(tiles + ((t + 1) & 1) * C::TILE_DOUBLES, d, o.alpha, u,
                         (t + 1) * C::T, n, o.un2);
    const double* td = cur;
    const double* ta = cur + C::T;
    const double* tn = cur + 2 * C::T;
    const double* tu = cur + 3 * C::T;
    // ---- D phase
#pragma unroll 8
    for (int i = warp; i < C::T; i += kPassWarps) {
      const double diff = (td[i] - dob) - del;
      double D;
      if (o.excl_gap > 0.0) {  // the bordered block: rows within excl_gap of dob, or one row
        const int64_t xr = slots.excl_row ? slots.excl_row[lane] : -1;
        const bool ex = (xr >= 0) ? (t * C::T + i == xr) : (fabs(td[i] - dob) < o.excl_gap);
        D = (act && !ex && diff == diff) ? rcp64(diff) : 0.0;
      } else if (diff == 0.0) {
        hit |= !o.exclude_zero;
        D = 0.0;
      } else {
        D = (act && diff == diff) ? rcp64(diff) : 0.0;
      }
      dbuf[i * 32 + lane] = D;
      if (sig) {
        double tt = 0.0;
        if constexpr (KP >= 2) {
          // two partial dot products: half the dependent DFMA chain
          double t0 = 0.0, t1 = 0.0;
#pragma unroll
          for (int c = 0; c < KP; c += 2) {
            const double2 v = *reinterpret_cast<const double2*>(tu + i * KP + c);
            t0 = fma(v.x, yv[c], t0);
            t1 = fma(v.y, yv[c + 1], t1);
          }
          tt = t0 + t1;
        } else {
          tt = tu[i] * yv[0];
        }
        const double td2 = tt * D;
        gs = fma(td2, td2, gs);
      }
      if (wf) {
        const double aD = ta[i] * D;
        fs += aD;
        fps = fma(aD, D, fps);
      }
      if (wn) gn = fma(tn[i], fabs(D), gn);
    }
    __syncthreads();  // D of this tile visible
    // ---- FMA phase
    fma_tile<KP, G>(tu, dbuf, p, lane, acc);
  }
  __syncthreads();

  // Deterministic reduction: FMA partials over pole splits p = 0.. in order,
  // D-phase partials (g, f, f') over warps 0..7 in order.
  constexpr int OUT = C::OUT;
  for (int q = 0; q < C::PS; ++q) {
    if (p == q) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (q == 0) red[lane * OUT + E0 + e] = acc[e];
        else red[lane * OUT + E0 + e] += acc[e];
      }
    }
    __syncthreads();
  }
  for (int q = 0; q < kPassWarps; ++q) {
    if (warp == q) {
      if (q == 0) {
        red[lane * OUT + C::IG] = gs;
        red[lane * OUT + C::IF] = fs;
        red[lane * OUT + C::IFP] = fps;
        red[lane * OUT + C::IGN] = gn;
      } else {
        red[lane * OUT + C::IG] += gs;
        red[lane * OUT + C::IF] += fs;
        red[lane * OUT + C::IFP] += fps;
        red[lane * OUT + C::IGN] += gn;
      }
    }
    __syncthreads();
  }
  if (hit) atomicOr(&slots.hit[lane], 1);
}

// The pass with its FMA phase on the FP64 tensor pipe (KP = 8, 16):
//   S[b][e] = sum_i D[i][b] W[i][e],  W[i][e] = u_i[r_e] u_i[c_e]
// as mma.sync.m8n8k4.f64 tiles (M = 32 slots in 4 m-tiles, N = P packed
// entries in n-tiles of 8, K = the poles of the tile in k-steps of 4). One DMMA
// replaces 16 warp-wide DFMAs (512 flops per issue), so the FP64 budget, which
// DFMA and DMMA share on B200 (profiles/coissue_dmma_dfma_r02.json), goes to
// the contraction instead of instruction issue.
//
// Round 2 layout (two CTAs per SM: <= 128 registers, <= ~100 KB of shared
// memory per CTA, so one CTA's D phase overlaps the other's MMA phase):
//  * D phase in C-fragment layout: warp w owns m-tile w & 3 (lane -> slot
//    8 (w & 3) + lane / 4) and the pole n-tiles (w >> 2) + 2 j. With sigma,
//    P = Y U^T (the projections u_i . y_b) is itself a DMMA (A = Y fragments
//    held in registers, B = the u rows of the tile), then per element the
//    reciprocal D, g += (P D)^2, f, f'. D is stored in A-fragment order.
//  * MMA phase: warp = (m-half, n-group, pole split): 2 m-tiles x 8-9 n-tiles
//    of accumulators (36 doubles). The packed entries are ordered by lane
//    pattern (mma_entry): within an n-tile the entry of B column n is
//    (n, 8 + nt) (the off-diagonal 8 x 8 block), (n, (n + s) & 7) or
//    (8 + n, 8 + ((n + s) & 7)) (the diagonal blocks by cyclic distance s),
//    so a lane forms its B elements from 2-8 loads of its pole row instead of
//    two per element.
// The k x k matrix entries come out in any order: the reduction writes them
// at their packed index.
template <int KP>
struct MmaMap {
  // global n-tiles: KP = 16: group 0 = tiles 0..8, group 1 = 9..16; KP = 8: 0..4
  static constexpr int NTILES = (KP == 16) ? 17 : 5;
  __host__ __device__ static constexpr int nt_lo(int g) { return (KP == 16) ? (g == 0 ? 0 : 9) : 0; }
  __host__ __device__ static constexpr int nt_cnt(int g) { return (KP == 16) ? (g == 0 ? 9 : 8) : 5; }
  // (row, column) of B column n of n-tile nt, or -1 (unused)
  __host__ __device__ static inline void entry(int nt, int n, int& r, int& c) {
    if constexpr (KP == 16) {
      if (nt < 8) { r = n; c = 8 + nt; return; }
      if (nt == 8) { r = (n < 4) ? n : n + 4; c = r + 4; return; }
      if (nt < 13) { r = n; c = (n + (nt - 9)) & 7; return; }
      r = 8 + n; c = 8 + ((n + (nt - 13)) & 7);
      return;
    } else {
      if (nt < 4) { r = n; c = (n + nt) & 7; return; }
      if (n < 4) { r = n; c = n + 4; return; }
      r = c = -1;
    }
  }
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// B elements of one k-step for n-group G: ur = this lane's pole row
template <int KP, int G>
__device__ __forceinline__ void mma_bvals(const double* __restrict__ ur, int g8, double* b) {
  if constexpr (KP == 16 && G == 0) {
    const double r0 = ur[g8];
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      const double2 v = *reinterpret_cast<const double2*>(ur + 8 + j);
      b[j] = r0 * v.x;
      b[j + 1] = r0 * v.y;
    }
    const int rm = (g8 < 4) ? g8 : g8 + 4;
    b[8] = ur[rm] * ur[rm + 4];
  } else {
    constexpr int OFF = (KP == 16) ? 8 : 0;  // G == 1 of KP = 16: the lower block too
    const double x0 = ur[g8], x1 = ur[(g8 + 1) & 7], x2 = ur[(g8 + 2) & 7], x3 = ur[(g8 + 3) & 7];
    b[0] = x0 * x0;
    b[1] = x0 * x1;
    b[2] = x0 * x2;
    b[3] = x0 * x3;
    if constexpr (KP == 16) {
      const double y0 = ur[OFF + g8], y1 = ur[OFF + ((g8 + 1) & 7)], y2 = ur[OFF + ((g8 + 2) & 7)],
                   y3 = ur[OFF + ((g8 + 3) & 7)];
      b[4] = y0 * y0;
      b[5] = y0 * y1;
      b[6] = y0 * y2;
      b[7] = y0 * y3;
    } else {
      b[4] = (g8 < 4) ? x0 * ur[g8 + 4] : 0.0;
    }
  }
}

// MT = active m-tiles (4, 2 or 1: the solver's compacted tail batches hold
// slots 0 .. 8 MT - 1 only). The warps' shares change with MT, the
// arithmetic of a slot does not: every (slot, entry) sum runs the same DMMA
// chain over the same pole split (p), and the D-phase partials of a slot
// stay with the same (m-tile, pole n-tile set) -- results are independent of
// MT, so compaction keeps the solver deterministic.
//   MT = 4: warp (sel = m-half, g, p): m-tiles 2 sel, 2 sel + 1, all n-tiles
//   MT = 2: warp (sel = m-tile, g, p): one m-tile, all n-tiles
//   MT = 1: warp (sel = n-half, g, p): m-tile 0, half the n-tiles
template <int KP, int G, int MT>
__device__ __forceinline__ void pass_body_mma(const double* __restrict__ d,
                                              const double* __restrict__ u, int64_t n,
                                              const PassSlots& slots, const PassOpts& o,
                                              double* tiles, double* dbuf, double* red, int sel,
                                              int p) {
  using C = PassCfg<KP>;
  using MM = MmaMap<KP>;
  constexpr int NTL = MM::nt_cnt(G);
  constexpr int MW = (MT == 4) ? 2 : 1;  // m-tiles per warp
  const int m0 = (MT == 4) ? 2 * sel : (MT == 2 ? sel : 0);
  // n-tiles [j_lo, j_hi) of the group (MT = 1 splits them)
  const int j_lo = (MT == 1) ? sel * ((NTL + 1) / 2) : 0;
  const int j_hi = (MT == 1) ? (sel ? NTL : (NTL + 1) / 2) : NTL;
  constexpr int KSW = (C::T / 4) / C::MPS;  // k-steps per warp per tile
  constexpr int LDU = C::LDU;
  constexpr int KC = KP / 4;                // k-steps of P = Y U^T
  constexpr int DKS = C::DKS;               // D buffer stride per k-step
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int t4 = lane & 3, g8 = lane >> 2;
  // ---- D-phase role: m-tile md, lane -> slot
  const int md = warp & 3;
  const int slot = 8 * md + g8;
  const double dob = slots.dob[slot];
  const double del = slots.delta[slot];
  const bool act = slots.active[slot] != 0;
  const bool sig = o.want_sigma;
  const bool wf = o.alpha != nullptr;
  const bool wn = o.un2 != nullptr;
  const bool exg = o.excl_gap > 0.0;
  const int64_t xr = (exg && slots.excl_row) ? slots.excl_row[slot] : -1;
  double yf[KC];
#pragma unroll
  for (int kc = 0; kc < KC; ++kc) yf[kc] = sig ? slots.y[slot * KP + 4 * kc + t4] : 0.0;
  double acc[2][NTL][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int j = 0; j < NTL; ++j) acc[m][j][0] = acc[m][j][1] = 0.0;
  double gs = 0.0, fs = 0.0, fps = 0.0, gn = 0.0;
  int hit = 0;

  const int64_t ntiles = (n + C::T - 1) / C::T;
  if (ntiles > 0) load_pole_tile<KP>(tiles, d, o.alpha, u, 0, n, o.un2);
  for (int64_t t = 0; t < ntiles; ++t) {
    const double* cur = tiles + (t & 1) * C::TILE_DOUBLES;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // tile t landed; previous MMA phase done with dbuf
    if (t + 1 < ntiles)
      load_pole_tile<KP>(tiles + ((t + 1) & 1) * C::TILE_DOUBLES, d, o.alpha, u,
                         (t + 1) * C::T, n, o.un2);
    const double* td = cur;
    const double* ta = cur + C::T;
    const double* tn = cur + 2 * C::T;
    const double* tu = cur + 3 * C::T;
    // ---- D phase (C-fragment layout: slot row g8, poles 8 nd + 2 t4 + h)
#pragma unroll
    for (int jn = 0; jn < C::T / 16; ++jn) {
      if (md >= MT) break;  // slots of this m-tile are empty (compacted batch)
      const int nd = (warp >> 2) + 2 * jn;
      double pv0 = 0.0, pv1 = 0.0;
      if (sig) {
        const double* ub = tu + (8 * nd + g8) * LDU + t4;
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) dmma(pv0, pv1, yf[kc], ub[4 * kc]);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = 8 * nd + 2 * t4 + h;
        const double diff = (td[i] - dob) - del;
        double D;
        if (exg) {  // the bordered block: rows within excl_gap of dob, or one row
          const bool ex = (xr >= 0) ? (t * C::T + i == xr) : (fabs(td[i] - dob) < o.excl_gap);
          D = (act && !ex && diff == diff) ? rcp64(diff) : 0.0;
        } else if (diff == 0.0) {
          hit |= !o.exclude_zero;
          D = 0.0;
        } else {
          D = (act && diff == diff) ? rcp64(diff) : 0.0;
        }
        dbuf[(i >> 2) * DKS + md * 32 + g8 * 4 + (i & 3)] = D;
        if (sig) {
          const double td2 = (h ? pv1 : pv0) * D;
          gs = fma(td2, td2, gs);
        }
        if (wf) {
          const double aD = ta[i] * D;
          fs += aD;
          fps = fma(aD, D, fps);
        }
        if (wn) gn = fma(tn[i], fabs(D), gn);
      }
    }
    __syncthreads();  // D of this tile visible
    // ---- MMA phase: k-steps p * KSW .. of this tile, m-tiles 2 mh, 2 mh + 1
#pragma unroll 2
    for (int kk = 0; kk < KSW; ++kk) {
      const int ks = p * KSW + kk;
      const double a0 = dbuf[ks * DKS + m0 * 32 + lane];
      const double a1 = (MW > 1) ? dbuf[ks * DKS + (m0 + 1) * 32 + lane] : 0.0;
      double b[NTL];
      mma_bvals<KP, G>(tu + (4 * ks + t4) * LDU, g8, b);
#pragma unroll
      for (int j = 0; j < NTL; ++j) {
        if (MT == 1 && (j < j_lo || j >= j_hi)) continue;
        dmma(acc[0][j][0], acc[0][j][1], a0, b[j]);
        if constexpr (MW > 1) dmma(acc[1][j][0], acc[1][j][1], a1, b[j]);
      }
    }
  }
  __syncthreads();

  // Deterministic reduction: the C fragments (slot 8 m + lane / 4, B columns
  // 2 (lane % 4) + h) over pole splits p = 0.. in order; the D-phase partials
  // (g, f, f') over the 4 lanes of a slot (butterfly: every lane the same
  // sum), then over the two warps of an m-tile in order.
  constexpr int OUT = C::OUT;
  for (int q = 0; q < C::MPS; ++q) {
    if (p == q) {
#pragma unroll
      for (int m = 0; m < MW; ++m)
#pragma unroll
        for (int j = 0; j < NTL; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (MT == 1 && (j < j_lo || j >= j_hi)) continue;
            int r, c;
            MM::entry(MM::nt_lo(G) + j, 2 * t4 + h, r, c);
            if (r >= 0) {
              const int e = (r <= c) ? C::pidx(r, c) : C::pidx(c, r);
              double* rr = red + (8 * (m0 + m) + g8) * OUT + e;
              *rr = (q == 0) ? acc[m][j][h] : *rr + acc[m][j][h];
            }
          }
    }
    __syncthreads();
  }
#pragma unroll
  for (int o2 = 1; o2 <= 2; o2 <<= 1) {
    gs += __shfl_xor_sync(0xffffffffu, gs, o2);
    fs += __shfl_xor_sync(0xffffffffu, fs, o2);
    fps += __shfl_xor_sync(0xffffffffu, fps, o2);
    gn += __shfl_xor_sync(0xffffffffu, gn, o2);
  }
  for (int q = 0; q < 2; ++q) {
    if ((warp >> 2) == q && t4 == 0) {
      double* rb = red + slot * OUT;
      if (q == 0) {
        rb[C::IG] = gs;
        rb[C::IF] = fs;
        rb[C::IFP] = fps;
        rb[C::IGN] = gn;
      } else {
        rb[C::IG] += gs;
        rb[C::IF] += fs;
        rb[C::IFP] += fps;
        rb[C::IGN] += gn;
      }
    }
    __syncthreads();
  }
  if (hit) atomicOr(&slots.hit[slot], 1);
}

// Runs the pass. On return (after __syncthreads) red[b * OUT + e] holds the
// packed S_b (without J) and red[b*OUT + P..P+2] = g_b, f_b - 1, f'_b.
// smem: SMEM_DOUBLES doubles (tiles, D buffer, reduction).
template <int KP, int MT>
__device__ __forceinline__ void pass_mma_dispatch(const double* __restrict__ d,
                                                  const double* __restrict__ u, int64_t n,
                                                  const PassSlots& slots, const PassOpts& o,
                                                  double* tiles, double* dbuf, double* red) {
  using C = PassCfg<KP>;
  const int warp = threadIdx.x >> 5;
  const int sel = warp & 1;
  const int g = (warp >> 1) % C::NG;
  const int p = warp / (2 * C::NG);
  if (g == 0) pass_body_mma<KP, 0, MT>(d, u, n, slots, o, tiles, dbuf, red, sel, p);
  if constexpr (C::NG > 1) {
    if (g == 1) pass_body_mma<KP, 1, MT>(d, u, n, slots, o, tiles, dbuf, red, sel, p);
  }
}

// mt: active m-tiles (4: all 32 slots; 2 or 1: only slots < 8 mt are active,
// the solver's compacted tail batches; MMA ranks only, others ignore it)
template <int KP>
__device__ void secular_pass(const double* __restrict__ d, const double* __restrict__ u, int64_t n,
                             const PassSlots& slots, const PassOpts& o, double* smem_pass,
                             int mt = 4) {
  using C = PassCfg<KP>;
  double* tiles = smem_pass;
  double* dbuf = tiles + 2 * C::TILE_DOUBLES;
  double* red = dbuf + C::DBUF_DOUBLES;
  const int warp = threadIdx.x >> 5;
  if constexpr (C::MMA) {
    if (mt >= 4) pass_mma_dispatch<KP, 4>(d, u, n, slots, o, tiles, dbuf, red);
    else if (mt == 2) pass_mma_dispatch<KP, 2>(d, u, n, slots, o, tiles, dbuf, red);
    else pass_mma_dispatch<KP, 1>(d, u, n, slots, o, tiles, dbuf, red);
    __syncthreads();
    return;
  }
  const int g = warp % C::EG;
  const int p = warp / C::EG;
#define EIGB_PASS_CASE(GG)                                                     \
  case GG:                                                                    \
    if constexpr (GG < C::EG) pass_body<KP, GG>(d, u, n, slots, o, tiles, dbuf, red, p); \
    break;
  switch (g) {
    EIGB_PASS_CASE(0)
    EIGB_PASS_CASE(1)
    EIGB_PASS_CASE(2)
    EIGB_PASS_CASE(3)
    EIGB_PASS_CASE(4)
    EIGB_PASS_CASE(5)
    EIGB_PASS_CASE(6)
    EIGB_PASS_CASE(7)
  }
#undef EIGB_PASS_CASE
  __syncthreads();
}

template <int KP>
__device__ __forceinline__ const double* pass_result(const double* smem_pass) {
  using C = PassCfg<KP>;
  return smem_pass + 2 * C::TILE_DOUBLES + C::DBUF_DOUBLES;
}

// ------------------------------------------------------------ small k x k
// Bunch-Kaufman LDL^T (partial pivoting, alpha = (1+sqrt(17))/8) of the full
// symmetric n x n matrix A (row-major, leading dimension ld), in place.
// piv[k] encodes the interchange of step k (>= 0: 1x1 with row piv[k];
// < 0: 2x2 block with row -piv[k]-1). Returns the number of negative
// eigenvalues (inertia); *zero is set when an exactly zero pivot occurred.
__host__ __device__ inline int bk_factor(double* A, int n, int ld, int* piv, int* zero, int es = 1) {
  const double alpha = 0.6403882032022076;
  int neg = 0;
  *zero = 0;
  int k = 0;
  while (k < n) {
    const double absakk = fabs(A[(k * ld + k) * es]);
    int imax = k;
    double colmax = 0.0;
    for (int i = k + 1; i < n; ++i) {
      const double v = fabs(A[(i * ld + k) * es]);
      if (v > colmax) colmax = v, imax = i;
    }
    int kstep = 1, kp = k;
    if (fmax(absakk, colmax) == 0.0) {
      piv[k] = k;
      *zero = 1;
      ++k;
      continue;
    }
    if (absakk >= alpha * colmax) {
      kp = k;
    } else {
      double rowmax = 0.0;
      for (int j = k; j < n; ++j)
        if (j != imax) rowmax = fmax(rowmax, fabs(A[(imax * ld + j) * es]));
      if (absakk >= alpha * colmax * (colmax / rowmax)) {
        kp = k;
      } else if (fabs(A[(imax * ld + imax) * es]) >= alpha * rowmax) {
        kp = imax;
      } else {
        kp = imax;
        kstep = 2;
      }
    }
    const int kk = k + kstep - 1;
    if (kp != kk) {  // symmetric interchange of kk and kp (whole rows/cols)
      for (int j = 0; j < n; ++j) {
        const double t = A[(kk * ld + j) * es];
        A[(kk * ld + j) * es] = A[(kp * ld + j) * es];
        A[(kp * ld + j) * es] = t;
      }
      for (int i = 0; i < n; ++i) {
        const double t = A[(i * ld + kk) * es];
        A[(i * ld + kk) * es] = A[(i * ld + kp) * es];
        A[(i * ld + kp) * es] = t;
      }
    }
    if (kstep == 1) {
      const double dk = A[(k * ld + k) * es];
      piv[k] = kp;
      if (dk < 0.0) ++neg;
      if (dk == 0.0) {
        *zero = 1;
      } else {
        const double r1 = 1.0 / dk;
        for (int i = k + 1; i < n; ++i) {
          const double li = A[(i * ld + k) * es] * r1;
          for (int j = k + 1; j <= i; ++j) A[(i * ld + j) * es] -= li * A[(j * ld + k) * es];
        }
        for (int i = k + 1; i < n; ++i) A[(i * ld + k) * es] *= r1;
        for (int i = k + 1; i < n; ++i)
          for (int j = k + 1; j < i; ++j) A[(j * ld + i) * es] = A[(i * ld + j) * es];
      }
    } else {
      const double a = A[(k * ld + k) * es], b = A[((k + 1) * ld + k) * es], c = A[((k + 1) * ld + k + 1) * es];
      const double det = a * c - b * b;
      piv[k] = -kp - 1;
      piv[k + 1] = -kp - 1;
      if (det < 0.0) neg += 1;
      else if (a + c < 0.0) neg += 2;
      if (det == 0.0) {
        *zero = 1;
      } else {
        const double id = 1.0 / det;
        // D^-1 = id * [[c, -b], [-b, a]]
        // rows in decreasing order: row i reads columns k, k+1 of rows j <= i
        // before they are overwritten by their L entries
        for (int i = n - 1; i >= k + 2; --i) {
          const double x1 = A[(i * ld + k) * es], x2 = A[(i * ld + k + 1) * es];
          const double w1 = (c * x1 - b * x2) * id;
          const double w2 = (a * x2 - b * x1) * id;
          for (int j = k + 2; j <= i; ++j)
            A[(i * ld + j) * es] -= w1 * A[(j * ld + k) * es] + w2 * A[(j * ld + k + 1) * es];
          A[(i * ld + k) * es] = w1;
          A[(i * ld + k + 1) * es] = w2;
        }
        for (int i = k + 2; i < n; ++i)
          for (int j = k + 2; j < i; ++j) A[(j * ld + i) * es] = A[(i * ld + j) * es];
      }
    }
    k += kstep;
  }
  return neg;
}

// Solves A z = b with the factorization of bk_factor. bk_factor applies
// every interchange to whole rows and columns (including the finished L
// columns), so P A P^T = L D L^T with one permutation P: permute b, solve
// L, D (1x1 / 2x2 blocks), L^T, permute back. Zero pivots are replaced by
// `tiny` (inverse iteration on a singular matrix).
__host__ __device__ inline void bk_solve(const double* A, int n, int ld, const int* piv, double* b,
                                         double tiny, int es = 1) {
  int k = 0;
  while (k < n) {  // b <- P b (interchanges in factorization order)
    if (piv[k] >= 0) {
      const int kp = piv[k];
      if (kp != k) { const double t = b[k]; b[k] = b[kp]; b[kp] = t; }
      k += 1;
    } else {
      const int kp = -piv[k] - 1;
      if (kp != k + 1) { const double t = b[k + 1]; b[k + 1] = b[kp]; b[kp] = t; }
      k += 2;
    }
  }
  k = 0;
  while (k < n) {  // L y = b
    if (piv[k] >= 0) {
      for (int i = k + 1; i < n; ++i) b[i] -= A[(i * ld + k) * es] * b[k];
      k += 1;
    } else {
      for (int i = k + 2; i < n; ++i) b[i] -= A[(i * ld + k) * es] * b[k] + A[(i * ld + k + 1) * es] * b[k + 1];
      k += 2;
    }
  }
  k = 0;
  while (k < n) {  // D w = y
    if (piv[k] >= 0) {
      double dk = A[(k * ld + k) * es];
      if (dk == 0.0) dk = tiny;
      b[k] /= dk;
      k += 1;
    } else {
      const double a = A[(k * ld + k) * es], bb = A[((k + 1) * ld + k) * es], c = A[((k + 1) * ld + k + 1) * es];
      double det = a * c - bb * bb;
      if (det == 0.0) det = tiny;
      const double x1 = (c * b[k] - bb * b[k + 1]) / det;
      const double x2 = (a * b[k + 1] - bb * b[k]) / det;
      b[k] = x1;
      b[k + 1] = x2;
      k += 2;
    }
  }
  k = n - 1;
  while (k >= 0) {  // L^T z = w
    if (piv[k] >= 0) {
      for (int i = k + 1; i < n; ++i) b[k] -= A[(i * ld + k) * es] * b[i];
      k -= 1;
    } else {  // block (k-1, k)
      for (int i = k + 1; i < n; ++i) {
        b[k] -= A[(i * ld + k) * es] * b[i];
        b[k - 1] -= A[(i * ld + k - 1) * es] * b[i];
      }
      k -= 2;
    }
  }
  // z <- P^T z (interchanges in reverse order)
  k = n - 1;
  while (k >= 0) {
    if (piv[k] >= 0) {
      const int kp = piv[k];
      if (kp != k) { const double t = b[k]; b[k] = b[kp]; b[kp] = t; }
      k -= 1;
    } else {
      const int kp = -piv[k] - 1;  // second row of the block is k
      if (kp != k) { const double t = b[k]; b[k] = b[kp]; b[kp] = t; }
      k -= 2;
    }
  }
}

// proj/src/secular.cpp:14-38 (LU with partial pivoting, det on the fly).
__device__ inline int lu_factor_dev(double* m, int k, int ld, int* piv, double* det) {
  for (int i = 0; i < k; ++i) piv[i] = i;
  *det = 1.0;
  for (int col = 0; col < k; ++col) {
    int best = col;
    for (int i = col + 1; i < k; ++i)
      if (fabs(m[i * ld + col]) > fabs(m[best * ld + col])) best = i;
    if (best != col) {
      for (int j = 0; j < k; ++j) {
        const double t = m[col * ld + j];
        m[col * ld + j] = m[best * ld + j];
        m[best * ld + j] = t;
      }
      const int t = piv[col];
      piv[col] = piv[best];
      piv[best] = t;
      *det = -*det;
    }
    const double pivot = m[col * ld + col];
    *det *= pivot;
    if (pivot == 0.0) return 0;
    for (int i = col + 1; i < k; ++i) {
      const double f = m[i * ld + col] / pivot;
      m[i * ld + col] = f;
      for (int j = col + 1; j < k; ++j) m[i * ld + j] -= f * m[col * ld + j];
    }
  }
  return 1;
}

// Adjugate of the k x k matrix m (ld) into adj (ld), following
// proj/src/secular.cpp:49-124: cofactors for k <= 3, LU det*inverse when
// min pivot > 1e-8 max pivot, cofactor expansion with LU minors otherwise.
// `scratch` holds at least 2*k*k doubles.
__device__ inline void adjugate_dev(const double* m, int k, int ld, double* adj, double* scratch) {
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) adj[i * ld + j] = 0.0;
  if (k == 1) { adj[0] = 1.0; return; }
#define MM(i, j) m[(i) * ld + (j)]
  if (k == 2) {
    adj[0] = MM(1, 1); adj[1] = -MM(0, 1); adj[ld] = -MM(1, 0); adj[ld + 1] = MM(0, 0);
    return;
  }
  if (k == 3) {
    adj[0 * ld + 0] = MM(1, 1) * MM(2, 2) - MM(1, 2) * MM(2, 1);
    adj[0 * ld + 1] = MM(0, 2) * MM(2, 1) - MM(0, 1) * MM(2, 2);
    adj[0 * ld + 2] = MM(0, 1) * MM(1, 2) - MM(0, 2) * MM(1, 1);
    adj[1 * ld + 0] = MM(1, 2) * MM(2, 0) - MM(1, 0) * MM(2, 2);
    adj[1 * ld + 1] = MM(0, 0) * MM(2, 2) - MM(0, 2) * MM(2, 0);
    adj[1 * ld + 2] = MM(0, 2) * MM(1, 0) - MM(0, 0) * MM(1, 2);
    adj[2 * ld + 0] = MM(1, 0) * MM(2, 1) - MM(1, 1) * MM(2, 0);
    adj[2 * ld + 1] = MM(0, 1) * MM(2, 0) - MM(0, 0) * MM(2, 1);
    adj[2 * ld + 2] = MM(0, 0) * MM(1, 1) - MM(0, 1) * MM(1, 0);
    return;
  }
  double* lu = scratch;  // k x k, ld k
  int piv[kMaxRank];
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) lu[i * k + j] = MM(i, j);
  double det, maxpiv = 0.0, minpiv = 0.0;
  if (lu_factor_dev(lu, k, k, piv, &det)) {
    maxpiv = fabs(lu[0]);
    minpiv = maxpiv;
    for (int i = 1; i < k; ++i) {
      const double pv = fabs(lu[i * k + i]);
      maxpiv = fmax(maxpiv, pv);
      minpiv = fmin(minpiv, pv);
    }
  }
  if (minpiv > 1e-8 * maxpiv) {
    double x[kMaxRank];
    for (int j = 0; j < k; ++j) {
      for (int i = 0; i < k; ++i) x[i] = (piv[i] == j) ? det : 0.0;
      for (int i = 1; i < k; ++i)
        for (int l = 0; l < i; ++l) x[i] -= lu[i * k + l] * x[l];
      for (int ii = k; ii-- > 0;) {
        for (int l = ii + 1; l < k; ++l) x[ii] -= lu[ii * k + l] * x[l];
        x[ii] /= lu[ii * k + ii];
      }
      for (int i = 0; i < k; ++i) adj[i * ld + j] = x[i];
    }
    return;
  }
  double* minor = scratch + k * k;
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) {
      int mr = 0;
      for (int r = 0; r < k; ++r) {
        if (r == i) continue;
        int mc = 0;
        for (int c = 0; c < k; ++c) {
          if (c == j) continue;
          minor[mr * (k - 1) + mc] = MM(r, c);
          ++mc;
        }
        ++mr;
      }
      double dm;
      int pv[kMaxRank];
      lu_factor_dev(minor, k - 1, k - 1, pv, &dm);
      adj[j * ld + i] = (((i + j) % 2) ? -1.0 : 1.0) * dm;
    }
#undef MM
}

}  // namespace eigb
