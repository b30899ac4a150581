// K1 projection U = Q^T K and the deflation pre-pass (sm_100a).
//
// K1 (proj/src/secular.cpp:155-161 -> kernels.cpp:50-65): HBM-bound
//   streaming pass over Q (row-major, n x n): thread t of a CTA owns two
//   columns i of Q, reads Q[r, i] coalesced row by row, and accumulates
//   U[i, :] += Q[r, i] * K[r, :] with K rows broadcast from shared memory.
//   Rows are split across CTAs; the partial sums are reduced in a fixed
//   order (deterministic, independent of the launch geometry per split).
// Deflation (proj/src/secular.cpp:278-340): runs of near-equal poles
//   (lambda[i] - lambda[i-1] < rel * max(1, max|lambda|)) with the run mean as
//   representative, classification by the reference's alpha/row-mass rules,
//   and the reduced problem the solver works on. Multi-member runs are
//   compressed with a Householder QR of their U rows (exact mode):
//   rows beyond the numerical rank decouple at the representative.
#include "pipeline.cuh"

#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <string>

namespace eigb {

namespace {

constexpr int kTfThreads = 128;
constexpr int kTfCols = 2 * kTfThreads;
constexpr int kTfRows = 32;

template <int KP>
__global__ void __launch_bounds__(kTfThreads) transform_partial_kernel(
    const double* __restrict__ q, const double* __restrict__ kmat, int64_t n, int k,
    int64_t rows_per_split, int64_t col_lo, int64_t col_hi, double* __restrict__ part) {
  __shared__ __align__(16) double ks[kTfRows][KP];
  const int64_t c0 = col_lo + (int64_t)blockIdx.x * kTfCols + threadIdx.x;
  const int64_t c1 = c0 + kTfThreads;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split;
  const int64_t r1 = (r0 + rows_per_split < n) ? r0 + rows_per_split : n;
  double a0[KP], a1[KP];
#pragma unroll
  for (int c = 0; c < KP; ++c) a0[c] = a1[c] = 0.0;
  const bool v0 = c0 < col_hi, v1 = c1 < col_hi;
  for (int64_t rr = r0; rr < r1; rr += kTfRows) {
    __syncthreads();
    for (int t = threadIdx.x; t < kTfRows * KP; t += kTfThreads) {
      const int r = t / KP, c = t % KP;
      const int64_t row = rr + r;
      ks[r][c] = (row < r1 && c < k) ? kmat[row * k + c] : 0.0;
    }
    __syncthreads();
    const int cnt = (int)((r1 - rr < kTfRows) ? r1 - rr : kTfRows);
#pragma unroll 4
    for (int r = 0; r < cnt; ++r) {
      const double q0 = v0 ? __ldcs(q + (rr + r) * n + c0) : 0.0;
      const double q1 = v1 ? __ldcs(q + (rr + r) * n + c1) : 0.0;
#pragma unroll
      for (int c = 0; c < KP; ++c) {
        a0[c] = fma(q0, ks[r][c], a0[c]);
        a1[c] = fma(q1, ks[r][c], a1[c]);
      }
    }
  }
  const int64_t ncols = col_hi - col_lo;
  double* out = part + (int64_t)blockIdx.y * ncols * KP;
  if (v0)
    for (int c = 0; c < KP; ++c) out[(c0 - col_lo) * KP + c] = a0[c];
  if (v1)
    for (int c = 0; c < KP; ++c) out[(c1 - col_lo) * KP + c] = a1[c];
}

__global__ void transform_reduce_kernel(const double* __restrict__ part, int64_t cnt, int splits,
                                        double* __restrict__ u) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  double s = part[t];
  for (int p = 1; p < splits; ++p) s += part[(int64_t)p * cnt + t];
  u[t] = s;
}

// ---------------------------------------------------------------- K1 on DMMA
// U^T = K^T Q as a tall-skinny GEMM on the FP64 tensor pipe (m = KP rows of
// U^T in DMMA m-tiles of 8, n = Q columns, the reduction over Q rows). At
// k = 16 the projection needs 4 flops per byte of Q, ~0.7 of the FP64 peak
// at full HBM bandwidth, so the FMA issue must be cheap: one
// mma.sync.m8n8k4.f64 per 512 flops (DMMA.8x8x4), fragments from shared
// memory. Q arrives by 1D bulk copies (cp.async.bulk, one 2 KB row segment
// of a 256-column block each, rows padded by 64 B so the four rows of a B
// fragment fall into different bank halves) and K by one bulk copy per stage
// of 8 rows, into a 4-stage mbarrier ring. The grid is persistent: CTA b
// walks the flattened (column block, row stage) range [f0, f1) in order, so
// the ring never drains at a column-block boundary; when its column block
// changes it stores its partial U rows as one of at most two records, and a
// second kernel sums the records of each column block in CTA order
// (deterministic for a given grid).
constexpr int kK1Cols = 256;                  // Q columns per block
constexpr int kK1Rows = 8;                    // Q rows per stage (2 k-steps)
constexpr int kK1Ld = kK1Cols + 8;            // padded smem row (doubles)
constexpr int kK1Threads = 256;               // 8 warps x 32 columns

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(d), "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void k1_mbar_init(uint64_t* bar, unsigned count) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void k1_mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void k1_mbar_arrive(uint64_t* bar) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void k1_mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "K1WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra K1WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

struct K1Geom {
  int64_t n, ncols, col_lo;
  int k;
  int64_t ncb;   // 256-column blocks
  int64_t spc;   // row stages (8 rows) per column block
  int64_t cs;    // row stages per chunk (a function of n only)
  int64_t nch;   // chunks per column block
  int64_t items; // ncb * nch work items (column block, row chunk)
};

// Work item i = (column block i / nch, row chunk i % nch): its stages
// (32-bit: at most 2^31 / 8 rows, far beyond 180 GB of Q).
__device__ __forceinline__ void k1_item(const K1Geom& g, int i, int* cb, int* st0, int* st1) {
  *cb = i / (int)g.nch;
  const int m = i - *cb * (int)g.nch;
  *st0 = m * (int)g.cs;
  *st1 = min((int)g.spc, *st0 + (int)g.cs);
}

// The producer's position (thread 0 only): kept in shared memory, off the
// consumers' register budget.
struct K1Prod {
  int item, cb, st, end, slot;
};

template <int KP, int kK1Stages>
__global__ void __launch_bounds__(kK1Threads, (KP >= 32 ? 2 : 4)) transform_dmma_kernel(
    const double* __restrict__ q, const double* __restrict__ kmat, K1Geom g,
    double* __restrict__ part) {
  constexpr int MT = (KP + 7) / 8;  // m-tiles of 8 U columns
  constexpr int KSTAGE = kK1Rows * (KP < 2 ? 2 : KP);  // K doubles per stage (padded)
  extern __shared__ __align__(128) unsigned char smraw[];
  double* sq = reinterpret_cast<double*>(smraw);                          // [S][R][Ld]
  double* sk = sq + kK1Stages * kK1Rows * kK1Ld;                          // [S][R*k]
  uint64_t* full = reinterpret_cast<uint64_t*>(sk + kK1Stages * KSTAGE);
  uint64_t* empty = full + kK1Stages;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int i0 = (int)(g.items * b / G), i1 = (int)(g.items * (b + 1) / G);
  if (i1 <= i0) return;
  __shared__ K1Prod pp;
  if (tid == 0) {
    for (int s = 0; s < kK1Stages; ++s) {
      k1_mbar_init(&full[s], 1);
      k1_mbar_init(&empty[s], kK1Threads / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // stages of this CTA's items in order; iters = their total
  int iters = 0;
  for (int i = i0; i < i1; ++i) {
    int cb, a, e;
    k1_item(g, i, &cb, &a, &e);
    iters += e - a;
  }
  // producer position: the next stage to issue as a running (item, stage)
  // pair (no divisions per stage)
  if (tid == 0) {
    pp.item = i0;
    k1_item(g, i0, &pp.cb, &pp.st, &pp.end);
    pp.slot = 0;
  }
  auto issue = [&]() {
    const int s = pp.slot;
    const int64_t cb = pp.cb, st = pp.st;
    pp.slot = (pp.slot + 1 == kK1Stages) ? 0 : pp.slot + 1;
    if (++pp.st == pp.end && ++pp.item < i1) k1_item(g, pp.item, &pp.cb, &pp.st, &pp.end);
    const int64_t r0 = st * kK1Rows;
    const int rows = (int)min((int64_t)kK1Rows, g.n - r0);
    const int64_t c0 = g.col_lo + cb * kK1Cols;
    const int cols = (int)min((int64_t)kK1Cols, g.col_lo + g.ncols - c0);
    const unsigned qb = (unsigned)cols * 8u, kb = (unsigned)(rows * g.k) * 8u;
    k1_mbar_expect_tx(&full[s], qb * (unsigned)rows + kb);
    double* dq = sq + (size_t)s * kK1Rows * kK1Ld;
    for (int r = 0; r < rows; ++r) bulk_g2s(dq + r * kK1Ld, q + (r0 + r) * g.n + c0, qb, &full[s]);
    bulk_g2s(sk + (size_t)s * KSTAGE, kmat + r0 * g.k, kb, &full[s]);
  };
  if (tid == 0)
    for (int f = 0; f < iters && f < kK1Stages; ++f) issue();

  double acc[MT][4][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[m][j][0] = acc[m][j][1] = 0.0;
  const int t4 = lane & 3, g8 = lane >> 2;
  // the item's partial U rows: record `item` (summed over chunks in order)
  auto flush = [&](int item, int cb) {
    const int64_t c0 = cb * kK1Cols;  // relative to col_lo
    double* out = part + (size_t)item * kK1Cols * KP;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int col = warp * 32 + nt * 8 + 2 * t4 + j;
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          const int kc = m * 8 + g8;
          if (kc < KP && c0 + col < g.ncols) out[col * KP + kc] = acc[m][nt][j];
          acc[m][nt][j] = 0.0;
        }
      }
  };
  int c_item = i0, c_cb, c_st, c_end;
  k1_item(g, c_item, &c_cb, &c_st, &c_end);
  int s = 0;                  // ring slot of iteration it
  unsigned phase = 0;         // its mbarrier parity
  int ps = kK1Stages - 1;     // slot of the previous iteration
  unsigned pphase = 1;
  for (int it = 0; it < iters; ++it) {
    // refill the slot released in the previous iteration
    if (tid == 0 && it > 0 && it - 1 + kK1Stages < iters) {
      k1_mbar_wait(&empty[ps], pphase);
      issue();
    }
    k1_mbar_wait(&full[s], phase);
    const int64_t r0 = (int64_t)c_st * kK1Rows;
    const int rows = (int)min((int64_t)kK1Rows, g.n - r0);
    const double* dq = sq + (size_t)s * kK1Rows * kK1Ld + warp * 32;
    const double* dk = sk + (size_t)s * KSTAGE;
#pragma unroll
    for (int ks = 0; ks < kK1Rows / 4; ++ks) {
      const int r = ks * 4 + t4;
      const bool ok = r < rows;
      double a[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const int kc = m * 8 + g8;
        a[m] = (ok && kc < g.k) ? dk[r * g.k + kc] : 0.0;
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const double bq = ok ? dq[r * kK1Ld + nt * 8 + g8] : 0.0;
#pragma unroll
        for (int m = 0; m < MT; ++m)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
              : "+d"(acc[m][nt][0]), "+d"(acc[m][nt][1])
              : "d"(a[m]), "d"(bq));
      }
    }
    __syncwarp();
    if (lane == 0) k1_mbar_arrive(&empty[s]);
    ps = s;
    pphase = phase;
    if (++s == kK1Stages) s = 0, phase ^= 1u;
    if (++c_st == c_end) {
      flush(c_item, c_cb);
      if (++c_item < i1) k1_item(g, c_item, &c_cb, &c_st, &c_end);
    }
  }
}

// U[c, :] = the sum of the chunk records of c's column block, in row order:
// every column's sum runs over the same row chunks whatever the column range
// (a multi-GPU slice gives the one-shot bits).
template <int KP>
__global__ void transform_dmma_reduce_kernel(const double* __restrict__ part, K1Geom g,
                                             double* __restrict__ u) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.ncols * KP) return;
  const int64_t c = t / KP;
  const int kc = (int)(t % KP);
  const int64_t cb = c / kK1Cols;
  const int col = (int)(c % kK1Cols);
  const double* p = part + (size_t)cb * g.nch * kK1Cols * KP + col * KP + kc;
  double s = 0.0;
  for (int64_t m = 0; m < g.nch; ++m) s += p[(size_t)m * kK1Cols * KP];
  u[t] = s;
}

template <int KP, int kK1Stages>
void launch_transform_dmma_s(const double* q, const double* kmat, int64_t n, int k, int64_t col_lo,
                             int64_t col_hi, double* u, DeviceScratch& ws, int sms, cudaStream_t st) {
  constexpr int KSTAGE = kK1Rows * (KP < 2 ? 2 : KP);
  const size_t smem = (size_t)kK1Stages * kK1Rows * kK1Ld * 8 + (size_t)kK1Stages * KSTAGE * 8 +
                      2 * kK1Stages * 8;
  static bool attr = false;
  if (!attr) {
    EIGB_CUDA(cudaFuncSetAttribute(transform_dmma_kernel<KP, kK1Stages>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  int per_sm = 0;
  EIGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, transform_dmma_kernel<KP, kK1Stages>,
                                                          kK1Threads, smem));
  K1Geom g;
  g.n = n;
  g.ncols = col_hi - col_lo;
  g.col_lo = col_lo;
  g.k = k;
  g.ncb = cdiv(g.ncols, kK1Cols);
  g.spc = cdiv(n, kK1Rows);
  // row chunks of 32 .. 1024 rows (n / 32, a function of n alone: the same
  // summation order for any column range), at most 32 records per column
  const int64_t cr = std::min<int64_t>(1024, std::max<int64_t>(32, cdiv(cdiv(n, 32), kK1Rows) * kK1Rows));
  g.cs = cr / kK1Rows;
  g.nch = cdiv(g.spc, g.cs);
  g.items = g.ncb * g.nch;
  // persistent grid: every resident slot busy (items split evenly)
  const int64_t grid = std::min<int64_t>(g.items, (int64_t)std::max(1, per_sm) * sms);
  double* part = ws.get_f64("tf_dpart", (size_t)g.items * kK1Cols * KP);
  transform_dmma_kernel<KP, kK1Stages><<<(unsigned)grid, kK1Threads, smem, st>>>(q, kmat, g, part);
  EIGB_LAUNCH_CHECK();
  const int64_t cnt = g.ncols * KP;
  transform_dmma_reduce_kernel<KP><<<(unsigned)cdiv(cnt, 256), 256, 0, st>>>(part, g, u);
  EIGB_LAUNCH_CHECK();
}

// Ring depth: 3 stages (17 KB each at k = 16) let 4 CTAs share an SM: 32
// warps hide the DMMA latency better than 2 CTAs of 4 stages
// (EIGMOD_B200_K1_STAGES = 2..4 for experiments).
template <int KP>
void launch_transform_dmma(const double* q, const double* kmat, int64_t n, int k, int64_t col_lo,
                           int64_t col_hi, double* u, DeviceScratch& ws, int sms, cudaStream_t st) {
  static const char* env = std::getenv("EIGMOD_B200_K1_STAGES");
  const int stages = env ? std::atoi(env) : 3;
  if (stages == 2) launch_transform_dmma_s<KP, 2>(q, kmat, n, k, col_lo, col_hi, u, ws, sms, st);
  else if (stages == 4) launch_transform_dmma_s<KP, 4>(q, kmat, n, k, col_lo, col_hi, u, ws, sms, st);
  else launch_transform_dmma_s<KP, 3>(q, kmat, n, k, col_lo, col_hi, u, ws, sms, st);
}

template <int KP>
void launch_transform(const double* q, const double* kmat, int64_t n, int k, int64_t col_lo,
                      int64_t col_hi, double* u, DeviceScratch& ws, int sms, cudaStream_t st) {
  const int64_t ncols = col_hi - col_lo;
  // DMMA path: 16-byte aligned bulk copies need even n, column range and
  // 16-byte aligned Q and K (EIGMOD_B200_K1=fma selects the DFMA kernel)
  static const char* env = std::getenv("EIGMOD_B200_K1");
  const bool aligned = (n % 2 == 0) && (col_lo % 2 == 0) && (ncols % 2 == 0) &&
                       (reinterpret_cast<uintptr_t>(q) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(kmat) % 16 == 0);
  if (aligned && !(env && std::string(env) == "fma")) {
    launch_transform_dmma<KP>(q, kmat, n, k, col_lo, col_hi, u, ws, sms, st);
    return;
  }
  const int64_t gx = cdiv(ncols, kTfCols);
  int64_t splits = std::max<int64_t>(1, cdiv(4 * (int64_t)sms, gx));
  splits = std::min<int64_t>(splits, cdiv(n, kTfRows));
  const int64_t rps = cdiv(cdiv(n, splits), kTfRows) * kTfRows;
  splits = cdiv(n, rps);
  double* part = ws.get_f64("tf_part", (size_t)splits * ncols * KP);
  dim3 grid((unsigned)gx, (unsigned)splits);
  transform_partial_kernel<KP><<<grid, kTfThreads, 0, st>>>(q, kmat, n, k, rps, col_lo, col_hi, part);
  EIGB_LAUNCH_CHECK();
  const int64_t cnt = ncols * KP;
  transform_reduce_kernel<<<(unsigned)cdiv(cnt, 256), 256, 0, st>>>(part, cnt, (int)splits, u);
  EIGB_LAUNCH_CHECK();
}

// Column norms of U (first k columns), fixed-order block reduction.
__global__ void colnorm_kernel(const double* __restrict__ u, int64_t n, int kp, int k,
                               double* __restrict__ out) {
  __shared__ double red[32];
  const int c = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += u[i * kp + c] * u[i * kp + c];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    out[c] = t;
  }
}

// Repack the kept columns (host-chosen) into a fresh padded [n][kp2] array.
__global__ void repack_kernel(const double* __restrict__ u, int64_t n, int kp, const int* keep,
                              int k2, int kp2, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * kp2) return;
  const int64_t i = t / kp2;
  const int c = (int)(t % kp2);
  out[t] = (c < k2) ? u[i * kp + keep[c]] : 0.0;
}

// ---------------------------------------------------------------- runs
// Single-CTA planning kernel: scale, run boundaries, groups, representatives.
// groups are emitted in ascending order; rep_row[i] = representative of row i.
constexpr int kPlanThreads = 1024;
constexpr int64_t kPlanParMinN = 8192;  // parallel plan finish from here on (build_plan_finish)

__device__ double block_max(double v, double* red) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
    t = warp_max(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const double r = red[0];
  __syncthreads();
  return r;
}

// Deterministic block sum: per-thread strided partials, then fixed-order tree.
__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    red[0] = t;
  }
  __syncthreads();
  const double r = red[0];
  __syncthreads();
  return r;
}

// Exclusive scan of 0/1-ish int64 counts over n items by one CTA, in chunks.
__device__ void block_exclusive_scan(const int64_t* in, int64_t* out, int64_t n, int64_t* total,
                                     int64_t* sh) {
  int64_t carry = 0;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = (i < n) ? in[i] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < (int)blockDim.x; off <<= 1) {
      const int64_t t = (threadIdx.x >= (unsigned)off) ? sh[threadIdx.x - off] : 0;
      __syncthreads();
      sh[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < n) out[i] = carry + sh[threadIdx.x] - v;
    const int64_t chunk = sh[blockDim.x - 1];
    __syncthreads();
    carry += chunk;
  }
  if (total) *total = carry;
}

__global__ void __launch_bounds__(kPlanThreads) runs_kernel(const double* __restrict__ lam,
                                                            int64_t n, double rel, double ufro2,
                                                            const double* __restrict__ norms2,
                                                            int k, int exact,
                                                            int64_t* __restrict__ flag,
                                                            int64_t* __restrict__ gid,
                                                            int64_t* __restrict__ gstart,
                                                            int64_t* __restrict__ glen,
                                                            double* __restrict__ gval,
                                                            double* __restrict__ rep_row,
                                                            int64_t* __restrict__ counts,
                                                            double* __restrict__ scal) {
  __shared__ double red[32];
  __shared__ int64_t sh[kPlanThreads];
  // parity: the reference's scale max(1, max|lambda|) (secular.cpp:285-287);
  // exact: max(max|lambda|, max_r ||u_r||^2), the size of A', so every
  // threshold is relative to the problem (A -> c A gives c lambda')
  if (norms2) {
    // speculative plan: the column-drop rule of plan_groups (capi.cu,
    // proj/src/rootfind.cpp:318-340) on the device; any dropped column is
    // flagged in scal[7] (the host rebuilds the plan) and ufro2 is the max
    // over all columns
    double mx = 0.0;
    for (int c = 0; c < k; ++c) mx = fmax(mx, sqrt(norms2[c]));
    const double drop = kColumnDropRel * (exact ? mx : fmax(1.0, mx));
    int bad = 0;
    ufro2 = 0.0;
    for (int c = 0; c < k; ++c) {
      const double v = sqrt(norms2[c]);
      if (v > drop && v > 0.0) ufro2 = fmax(ufro2, v * v);
      else bad = 1;
    }
    if (threadIdx.x == 0) scal[7] = bad;
  }
  double m = exact ? 0.0 : 1.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, fabs(lam[i]));
  double scale = block_max(m, red);
  if (exact) {
    scale = fmax(scale, ufro2);
    if (!(scale > 0.0)) scale = 1.0;
  }
  const double gap = rel * scale;
  if (!exact) {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
      flag[i] = (i == 0 || !(lam[i] - lam[i - 1] < gap)) ? 1 : 0;
  } else {
    // exact mode: a run never spans more than the gap (merging moves every
    // member by less than the gap; the reference chains consecutive gaps).
    // Run starts are found sequentially over the (rare) chains of close
    // neighbours: thread 0 walks only positions whose left gap is small.
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
      flag[i] = (i == 0 || !(lam[i] - lam[i - 1] < gap)) ? 1 : 0;
    // Chains are independent: one thread per chain start (a start followed
    // by a close neighbour) walks its chain; candidates are marked first (in
    // gid, free until the scan) so no walk reads another chain's new starts.
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
      gid[i] = (flag[i] && i + 1 < n && !flag[i + 1]) ? 1 : 0;
    __syncthreads();
    for (int64_t i0 = threadIdx.x; i0 < n; i0 += blockDim.x) {
      if (!gid[i0]) continue;
      int64_t start = i0;
      for (int64_t i = i0 + 1; i < n && !flag[i]; ++i) {
        if (!(lam[i] - lam[start] < gap)) {
          flag[i] = 1;
          start = i;
        }
      }
    }
  }
  __syncthreads();
  __shared__ int64_t ng;
  block_exclusive_scan(flag, gid, n, &ng, sh);
  __syncthreads();
  // gid is exclusive scan of starts; group of row i = gid[i] + flag[i] - 1
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t g = gid[i] + flag[i] - 1;
    if (flag[i]) gstart[g] = i;
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) gid[i] = gid[i] + flag[i] - 1;
  __syncthreads();
  for (int64_t g = threadIdx.x; g < ng; g += blockDim.x) {
    const int64_t s0 = gstart[g];
    const int64_t s1 = (g + 1 < ng) ? gstart[g + 1] : n;
    glen[g] = s1 - s0;
    double s = 0.0;  // proj/src/secular.cpp:299-301 (sequential sum, then divide)
    for (int64_t i = s0; i < s1; ++i) s += lam[i];
    gval[g] = s / (double)(s1 - s0);
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) rep_row[i] = gval[gid[i]];
  int64_t nm = 0;  // multi-member runs (read back with ng: no separate round trip)
  for (int64_t g = threadIdx.x; g < ng; g += blockDim.x) nm += glen[g] > 1;
  nm = (int64_t)block_sum((double)nm, red);
  if (threadIdx.x == 0) {
    counts[0] = ng;
    counts[4] = nm;
    scal[0] = scale;
  }
}

// Classification (proj/src/secular.cpp:306-331): kind 0 survives, 1 unchanged
// (all members decouple at their own value), 2 collided (value kept; in the
// solve the row stays coupled and the root lands on the pole).
__global__ void __launch_bounds__(kPlanThreads) classify_kernel(
    const double* __restrict__ u, int64_t n, int kp, int k, const double* __restrict__ alpha,
    const int64_t* __restrict__ gstart, const int64_t* __restrict__ glen, const int64_t* counts,
    int exact, int* __restrict__ kind, double* __restrict__ scal) {
  __shared__ double red[32];
  const int64_t ng = counts[0];
  double am = 0.0;
  for (int64_t g = threadIdx.x; g < ng; g += blockDim.x) am += fabs(alpha[g]);
  const double alpha_mass = block_sum(am, red);
  double um = 0.0;
  for (int64_t t = threadIdx.x; t < n * kp; t += blockDim.x) {
    const int c = (int)(t % kp);
    if (c < k) um += u[t] * u[t];
  }
  const double fn = sqrt(block_sum(um, red));
  const double u_mass = fn * fn;
  const double drop = kWeightDeflationRel * (1.0 + alpha_mass);
  // exact mode: a group decouples unchanged when its rows couple to the rest
  // by less than 1e-13 of the problem scale (|u_g| ||U|| <= 1e-13 s: residual
  // of the unchanged pair below 1e-13 ||A'||); collided groups stay in the
  // reduced problem, where the solver finds their roots on the pole
  const double scale = scal[0];
  for (int64_t g = threadIdx.x; g < ng; g += blockDim.x) {
    int kd = 0;
    if (exact) {
      double row_mass = 0.0;
      for (int64_t i = gstart[g]; i < gstart[g] + glen[g]; ++i)
        for (int r = 0; r < k; ++r) row_mass += u[i * kp + r] * u[i * kp + r];
      kd = (sqrt(row_mass) * fn <= kExactCouplingRel * scale) ? 1 : 0;
    } else if (fabs(alpha[g]) <= drop) {
      double row_mass = 0.0;
      for (int64_t i = gstart[g]; i < gstart[g] + glen[g]; ++i)
        for (int r = 0; r < k; ++r) row_mass += u[i * kp + r] * u[i * kp + r];
      kd = (row_mass <= kRowMassRel * (1.0 + u_mass)) ? 1 : 2;
    }
    kind[g] = kd;
  }
  if (threadIdx.x == 0) {
    scal[1] = alpha_mass;
    scal[2] = u_mass;
    scal[3] = fn;
  }
}

// Householder QR of each multi-member run's rows (exact mode compression).
// One thread per multi group (rare: near-equal poles only). Writes R (m x kp,
// in place of a copy), H (m x m) and the numerical rank.
__global__ void compress_kernel(const double* __restrict__ u, int kp, int k,
                                const int64_t* __restrict__ gstart,
                                const int64_t* __restrict__ glen, const int* __restrict__ kind,
                                const int64_t* counts, const int64_t* __restrict__ hoff,
                                const int64_t* __restrict__ roff, double* __restrict__ hbuf,
                                double* __restrict__ rbuf, int64_t* __restrict__ rank,
                                const double* __restrict__ scal, int exact) {
  const int64_t ng = counts[0];
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int64_t m = glen[g];
  if (m < 2 || kind[g] == 1) {
    rank[g] = 0;
    return;
  }
  double* H = hbuf + hoff[g];
  double* B = rbuf + roff[g];
  const int64_t s0 = gstart[g];
  for (int64_t i = 0; i < m; ++i)
    for (int c = 0; c < kp; ++c) B[i * kp + c] = u[(s0 + i) * kp + c];
  for (int64_t i = 0; i < m * m; ++i) H[i] = 0.0;
  for (int64_t i = 0; i < m; ++i) H[i * m + i] = 1.0;
  const int64_t steps = m < k ? m : k;
  // Householder QR with column pivoting (largest remaining column): rank-
  // revealing, so a numerically dependent run row leaves a tiny residual row.
  unsigned long long used = 0ull;  // pivot columns (k <= 32)
  for (int64_t c = 0; c < steps; ++c) {
    int pc = -1;
    double best = 0.0;
    for (int jj = 0; jj < k; ++jj) {
      if ((used >> jj) & 1ull) continue;
      double s2 = 0.0;
      for (int64_t i = c; i < m; ++i) s2 += B[i * kp + jj] * B[i * kp + jj];
      if (s2 > best) best = s2, pc = jj;
    }
    if (pc < 0) break;
    used |= 1ull << pc;
    const double nrm = sqrt(best);
    const double al = B[c * kp + pc] >= 0.0 ? -nrm : nrm;
    const double v_c = B[c * kp + pc] - al;
    double vn = v_c * v_c;
    for (int64_t i = c + 1; i < m; ++i) vn += B[i * kp + pc] * B[i * kp + pc];
    if (vn == 0.0) continue;
    const double beta = 2.0 / vn;
    // H <- (I - beta v v^T) H, B <- (I - beta v v^T) B, v = (v_c, B[c+1.., pc]);
    // the pivot column is updated last (it holds v)
    for (int64_t j = 0; j < m; ++j) {
      double s = v_c * H[c * m + j];
      for (int64_t i = c + 1; i < m; ++i) s += B[i * kp + pc] * H[i * m + j];
      s *= beta;
      H[c * m + j] -= s * v_c;
      for (int64_t i = c + 1; i < m; ++i) H[i * m + j] -= s * B[i * kp + pc];
    }
    for (int j = 0; j < kp; ++j) {
      if (j == pc) continue;
      double s = v_c * B[c * kp + j];
      for (int64_t i = c + 1; i < m; ++i) s += B[i * kp + pc] * B[i * kp + j];
      s *= beta;
      B[c * kp + j] -= s * v_c;
      for (int64_t i = c + 1; i < m; ++i) B[i * kp + j] -= s * B[i * kp + pc];
    }
    B[c * kp + pc] = al;
    for (int64_t i = c + 1; i < m; ++i) B[i * kp + pc] = 0.0;
  }
  // numerical rank: leading rows with norm above eps * ||U||_F; in exact mode
  // also above the decoupling level of classify_kernel (a direction whose
  // coupling |r| ||U|| is below 1e-13 of the scale decouples at the run value)
  double thr = DBL_EPSILON * scal[3];
  if (exact && scal[3] > 0.0) thr = fmax(thr, kExactCouplingRel * scal[0] / scal[3]);
  int64_t r = 0;
  for (int64_t t = 0; t < steps; ++t) {
    double rn = 0.0;
    for (int c = 0; c < kp; ++c) rn += B[t * kp + c] * B[t * kp + c];
    if (sqrt(rn) > thr) r = t + 1;
  }
  rank[g] = r;
}

// Reduced-problem assembly (single CTA, scans over groups in order).
//   reduced rows: singleton non-unchanged groups (their row), multi groups
//   (their first rank[g] compressed rows at the representative);
//   decoupled entries (ascending by construction): unchanged members at
//   their own value (unit vectors), multi-group rows beyond the rank at the
//   representative (rotation vectors).
__global__ void __launch_bounds__(kPlanThreads) assemble_reduced_kernel(
    const double* __restrict__ lam, const double* __restrict__ u, int64_t n, int kp,
    const int64_t* __restrict__ gstart, const int64_t* __restrict__ glen,
    const double* __restrict__ gval, const int* __restrict__ kind,
    const int64_t* __restrict__ rank, const int64_t* __restrict__ roff,
    const double* __restrict__ rbuf, int64_t* counts, int64_t* __restrict__ tmp_a,
    int64_t* __restrict__ tmp_b, int64_t* __restrict__ off_red, int64_t* __restrict__ off_dec,
    const double* __restrict__ alpha, double* __restrict__ alpha_red,
    double* __restrict__ d, double* __restrict__ ur, int64_t* __restrict__ red_src,
    double* __restrict__ dec_val, int64_t* __restrict__ dec_src, int64_t* __restrict__ orig_map) {
  __shared__ int64_t sh[kPlanThreads];
  const int64_t ng = counts[0];
  for (int64_t g = threadIdx.x; g < ng; g += blockDim.x) {
    const int64_t m = glen[g];
    int64_t nr, nd;
    if (kind[g] == 1) nr = 0, nd = m;
    else if (m == 1) nr = 1, nd = 0;
    else nr = rank[g], nd = m - rank[g];
    tmp_a[g] = nr;
    tmp_b[g] = nd;
  }
  __syncthreads();
  __shared__ int64_t nred, ndec;
  block_exclusive_scan(tmp_a, off_red, ng, &nred, sh);
  __syncthreads();
  block_exclusive_scan(tmp_b, off_dec, ng, &ndec, sh);
  __syncthreads();
  for (int64_t g = threadIdx.x; g < ng; g += blockDim.x) {
    const int64_t m = glen[g], s0 = gstart[g];
    int64_t pr = off_red[g], pd = off_dec[g];
    if (kind[g] == 1) {
      for (int64_t i = 0; i < m; ++i) {
        dec_val[pd + i] = lam[s0 + i];
        dec_src[pd + i] = s0 + i;            // unit vector e_(s0+i)
        orig_map[s0 + i] = -1;               // decoupled coordinate
      }
    } else if (m == 1) {
      d[pr] = lam[s0];
      alpha_red[pr] = alpha[g];
      for (int c = 0; c < kp; ++c) ur[pr * kp + c] = u[s0 * kp + c];
      red_src[pr] = s0;
      orig_map[s0] = pr;
    } else {
      const int64_t r = rank[g];
      const double* B = rbuf + roff[g];
      for (int64_t t = 0; t < r; ++t) {
        d[pr + t] = gval[g];
        alpha_red[pr + t] = 0.0;  // not a simple pole: f-Newton is disabled
        for (int c = 0; c < kp; ++c) ur[(pr + t) * kp + c] = B[t * kp + c];
        red_src[pr + t] = -(g * 65536 + t) - 2;  // rotated row t of group g
      }
      for (int64_t t = r; t < m; ++t) {
        dec_val[pd + t - r] = gval[g];
        dec_src[pd + t - r] = -(g * 65536 + t) - 2;
      }
      for (int64_t i = 0; i < m; ++i) orig_map[s0 + i] = -2 - g;  // member of multi group g
    }
  }
  if (threadIdx.x == 0) {
    counts[1] = nred;
    counts[2] = ndec;
  }
}

__global__ void clips_kernel(const double* __restrict__ d, const double* __restrict__ ur,
                             const int64_t* __restrict__ counts, int kp, int k,
                             const int* __restrict__ sgn, double* __restrict__ scal) {
  __shared__ double red[32];
  const int64_t nr = counts[1];  // from assemble_reduced_kernel, no host round trip
  double pos = 0.0, neg = 0.0, m = 0.0;
  for (int64_t t = threadIdx.x; t < nr * kp; t += blockDim.x) {
    const int c = (int)(t % kp);
    if (c >= k) continue;
    const double v = ur[t] * ur[t];
    if (sgn[c] > 0) pos += v; else neg += v;
  }
  for (int64_t i = threadIdx.x; i < nr; i += blockDim.x) m = fmax(m, fabs(d[i]));
  pos = block_sum(pos, red);
  neg = block_sum(neg, red);
  m = block_max(m, red);
  if (threadIdx.x == 0) {
    m = fmax(m, pos + neg);
    const double pad = 1e-9 * (m > 0.0 ? m : 1.0);
    scal[4] = (nr > 0) ? d[0] - neg * (1.0 + 1e-12) - pad : 0.0;
    scal[5] = (nr > 0) ? d[nr - 1] + pos * (1.0 + 1e-12) + pad : 0.0;
  }
}


// ---- parallel plan finish (n >= kPlanParMinN): the single-CTA kernels above
// take 0.3-0.8 ms each at n = 32768 (one SM's worth of latency-bound loops),
// and every rank of a multi-GPU update repeats them. Same decisions per
// group; the three sums (|alpha|, ||U||_F^2, the signed column masses of the
// clips) are per-CTA partials over kPlanParBlocks fixed slices added in slice
// order, so they are deterministic for a given n but round differently from
// the single-CTA sums (they feed thresholds and the 1e-9-padded outer clips).
constexpr int kPlanParBlocks = 64;
constexpr int kPlanParThreads = 256;

__global__ void __launch_bounds__(kPlanParThreads) plan_sums_kernel(
    const double* __restrict__ u, int64_t n, int kp, int k, const double* __restrict__ alpha,
    const int64_t* __restrict__ counts, double* __restrict__ part) {
  __shared__ double red[32];
  const int64_t ng = counts[0];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double am = 0.0, um = 0.0;
  for (int64_t g = t0; g < ng; g += stride) am += fabs(alpha[g]);
  for (int64_t i = t0; i < n; i += stride)
    for (int r = 0; r < k; ++r) um = fma(u[i * kp + r], u[i * kp + r], um);
  am = block_sum(am, red);
  um = block_sum(um, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = am;
    part[2 * blockIdx.x + 1] = um;
  }
}

__global__ void __launch_bounds__(kPlanParThreads) classify_par_kernel(
    const double* __restrict__ u, int kp, int k, const double* __restrict__ alpha,
    const int64_t* __restrict__ gstart, const int64_t* __restrict__ glen,
    const int64_t* __restrict__ counts, int exact, const double* __restrict__ part, int nparts,
    int* __restrict__ kind, double* __restrict__ scal) {
  __shared__ double sums[2];
  if (threadIdx.x == 0) {
    double am = 0.0, um = 0.0;
    for (int b = 0; b < nparts; ++b) {
      am += part[2 * b];
      um += part[2 * b + 1];
    }
    sums[0] = am;
    sums[1] = um;
  }
  __syncthreads();
  const double alpha_mass = sums[0];
  const double fn = sqrt(sums[1]);
  const double u_mass = fn * fn;
  const double drop = kWeightDeflationRel * (1.0 + alpha_mass);
  const double scale = scal[0];
  const int64_t ng = counts[0];
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < ng) {  // the rules of classify_kernel
    int kd = 0;
    if (exact) {
      double row_mass = 0.0;
      for (int64_t i = gstart[g]; i < gstart[g] + glen[g]; ++i)
        for (int r = 0; r < k; ++r) row_mass += u[i * kp + r] * u[i * kp + r];
      kd = (sqrt(row_mass) * fn <= kExactCouplingRel * scale) ? 1 : 0;
    } else if (fabs(alpha[g]) <= drop) {
      double row_mass = 0.0;
      for (int64_t i = gstart[g]; i < gstart[g] + glen[g]; ++i)
        for (int r = 0; r < k; ++r) row_mass += u[i * kp + r] * u[i * kp + r];
      kd = (row_mass <= kRowMassRel * (1.0 + u_mass)) ? 1 : 2;
    }
    kind[g] = kd;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    scal[1] = alpha_mass;
    scal[2] = u_mass;
    scal[3] = fn;
  }
}

__global__ void __launch_bounds__(kPlanParThreads) assemble_count_kernel(
    const int64_t* __restrict__ glen, const int* __restrict__ kind,
    const int64_t* __restrict__ rank, const int64_t* __restrict__ counts,
    int64_t* __restrict__ tmp_a, int64_t* __restrict__ tmp_b) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= counts[0]) return;
  const int64_t m = glen[g];
  int64_t nr, nd;
  if (kind[g] == 1) nr = 0, nd = m;
  else if (m == 1) nr = 1, nd = 0;
  else nr = rank[g], nd = m - rank[g];
  tmp_a[g] = nr;
  tmp_b[g] = nd;
}

__global__ void __launch_bounds__(kPlanThreads) assemble_scan_kernel(
    const int64_t* __restrict__ tmp_a, const int64_t* __restrict__ tmp_b, int64_t* counts,
    int64_t* __restrict__ off_red, int64_t* __restrict__ off_dec) {
  __shared__ int64_t sh[kPlanThreads];
  __shared__ int64_t nred, ndec;
  const int64_t ng = counts[0];
  block_exclusive_scan(tmp_a, off_red, ng, &nred, sh);
  __syncthreads();
  block_exclusive_scan(tmp_b, off_dec, ng, &ndec, sh);
  __syncthreads();
  if (threadIdx.x == 0) {
    counts[1] = nred;
    counts[2] = ndec;
  }
}

// The scatter of assemble_reduced_kernel, one thread per group.
__global__ void __launch_bounds__(kPlanParThreads) assemble_scatter_kernel(
    const double* __restrict__ lam, const double* __restrict__ u, int kp,
    const int64_t* __restrict__ gstart, const int64_t* __restrict__ glen,
    const double* __restrict__ gval, const int* __restrict__ kind,
    const int64_t* __restrict__ rank, const int64_t* __restrict__ roff,
    const double* __restrict__ rbuf, const int64_t* __restrict__ counts,
    const int64_t* __restrict__ off_red, const int64_t* __restrict__ off_dec,
    const double* __restrict__ alpha, double* __restrict__ alpha_red, double* __restrict__ d,
    double* __restrict__ ur, int64_t* __restrict__ red_src, double* __restrict__ dec_val,
    int64_t* __restrict__ dec_src, int64_t* __restrict__ orig_map) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= counts[0]) return;
  const int64_t m = glen[g], s0 = gstart[g];
  const int64_t pr = off_red[g], pd = off_dec[g];
  if (kind[g] == 1) {
    for (int64_t i = 0; i < m; ++i) {
      dec_val[pd + i] = lam[s0 + i];
      dec_src[pd + i] = s0 + i;
      orig_map[s0 + i] = -1;
    }
  } else if (m == 1) {
    d[pr] = lam[s0];
    alpha_red[pr] = alpha[g];
    for (int c = 0; c < kp; ++c) ur[pr * kp + c] = u[s0 * kp + c];
    red_src[pr] = s0;
    orig_map[s0] = pr;
  } else {
    const int64_t r = rank[g];
    const double* B = rbuf + roff[g];
    for (int64_t t = 0; t < r; ++t) {
      d[pr + t] = gval[g];
      alpha_red[pr + t] = 0.0;
      for (int c = 0; c < kp; ++c) ur[(pr + t) * kp + c] = B[t * kp + c];
      red_src[pr + t] = -(g * 65536 + t) - 2;
    }
    for (int64_t t = r; t < m; ++t) {
      dec_val[pd + t - r] = gval[g];
      dec_src[pd + t - r] = -(g * 65536 + t) - 2;
    }
    for (int64_t i = 0; i < m; ++i) orig_map[s0 + i] = -2 - g;
  }
}

__global__ void __launch_bounds__(kPlanParThreads) clips_part_kernel(
    const double* __restrict__ d, const double* __restrict__ ur,
    const int64_t* __restrict__ counts, int kp, int k, const int* __restrict__ sgn,
    double* __restrict__ part) {
  __shared__ double red[32];
  const int64_t nr = counts[1];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double pos = 0.0, neg = 0.0, m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += stride) {
    for (int c = 0; c < k; ++c) {
      const double v = ur[i * kp + c] * ur[i * kp + c];
      if (sgn[c] > 0) pos += v; else neg += v;
    }
    m = fmax(m, fabs(d[i]));
  }
  pos = block_sum(pos, red);
  neg = block_sum(neg, red);
  m = block_max(m, red);
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x] = pos;
    part[3 * blockIdx.x + 1] = neg;
    part[3 * blockIdx.x + 2] = m;
  }
}

__global__ void clips_final_kernel(const double* __restrict__ d,
                                   const int64_t* __restrict__ counts,
                                   const double* __restrict__ part, int nparts,
                                   double* __restrict__ scal) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int64_t nr = counts[1];
  double pos = 0.0, neg = 0.0, m = 0.0;
  for (int b = 0; b < nparts; ++b) {
    pos += part[3 * b];
    neg += part[3 * b + 1];
    m = fmax(m, part[3 * b + 2]);
  }
  m = fmax(m, pos + neg);
  const double pad = 1e-9 * (m > 0.0 ? m : 1.0);
  scal[4] = (nr > 0) ? d[0] - neg * (1.0 + 1e-12) - pad : 0.0;
  scal[5] = (nr > 0) ? d[nr - 1] + pos * (1.0 + 1e-12) + pad : 0.0;
}

}  // namespace

// ------------------------------------------------------------------ host side
void transform_update_dev(const double* q, const double* kmat, int64_t n, int k, int kp,
                          int64_t col_lo, int64_t col_hi, double* u, DeviceScratch& ws, int sms,
                          cudaStream_t st) {
  switch (kp) {
    case 1: launch_transform<1>(q, kmat, n, k, col_lo, col_hi, u, ws, sms, st); break;
    case 2: launch_transform<2>(q, kmat, n, k, col_lo, col_hi, u, ws, sms, st); break;
    case 4: launch_transform<4>(q, kmat, n, k, col_lo, col_hi, u, ws, sms, st); break;
    case 8: launch_transform<8>(q, kmat, n, k, col_lo, col_hi, u, ws, sms, st); break;
    case 16: launch_transform<16>(q, kmat, n, k, col_lo, col_hi, u, ws, sms, st); break;
    case 32: launch_transform<32>(q, kmat, n, k, col_lo, col_hi, u, ws, sms, st); break;
    default: throw Error(1, "", "transform: unsupported padded rank");
  }
}

void column_norms2_dev(const double* u, int64_t n, int kp, int k, double* out, cudaStream_t st) {
  colnorm_kernel<<<k, 256, 0, st>>>(u, n, kp, k, out);
  EIGB_LAUNCH_CHECK();
}

void repack_columns_dev(const double* u, int64_t n, int kp, const int* keep, int k2, int kp2,
                        double* out, cudaStream_t st) {
  repack_kernel<<<(unsigned)cdiv(n * kp2, 256), 256, 0, st>>>(u, n, kp, keep, k2, kp2, out);
  EIGB_LAUNCH_CHECK();
}

// Runs / groups of the (kept-column) problem; sizes p.alpha for K2.
void build_plan_groups(Plan& p, const double* lam, int64_t n, double run_rel, DeviceScratch& ws,
                       cudaStream_t st) {
  p.n = n;
  p.exact = run_rel != kPoleMergeRelGap;
  int64_t* flag = ws.get_i64("pl_flag", n);
  p.gid = ws.get_i64("pl_gid", n);
  p.gstart = ws.get_i64("pl_gstart", n);
  p.glen = ws.get_i64("pl_glen", n);
  p.gval = ws.get_f64("pl_gval", n);
  p.rep_row = ws.get_f64("pl_rep_row", n);
  p.counts = ws.get_i64("pl_counts", 8);
  p.scal = ws.get_f64("pl_scal", 8);
  runs_kernel<<<1, kPlanThreads, 0, st>>>(lam, n, run_rel, p.ufro2, p.spec ? p.norms_dev : nullptr,
                                           p.k, p.exact ? 1 : 0, flag, p.gid, p.gstart, p.glen,
                                           p.gval, p.rep_row, p.counts, p.scal);
  EIGB_LAUNCH_CHECK();
  if (p.spec) {  // sizes read back by build_plan_finish; n bounds the group count
    p.ng = n;
    p.nmulti = 0;
    p.alpha = ws.get_f64("pl_alpha", n);
    return;
  }
  int64_t cnt[5] = {0, 0, 0, 0, 0};
  EIGB_CUDA(cudaMemcpyAsync(cnt, p.counts, sizeof(cnt), cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaStreamSynchronize(st));
  p.ng = cnt[0];
  p.nmulti = cnt[4];
  p.alpha = ws.get_f64("pl_alpha", p.ng);
}

// K2 for groups [g0, g1) into alpha_out (length g1 - g0); the full vector may
// be assembled from several ranks' slices before build_plan_finish.
void build_plan_weights(const Plan& p, int64_t g0, int64_t g1, double* alpha_out,
                        DeviceScratch& ws, cudaStream_t st) {
  if (g1 <= g0) return;
  group_weights(p.kp, p.rep_row, p.u, p.n, p.gstart + g0, p.glen + g0, p.gval + g0, g1 - g0,
                p.sgn, p.k, alpha_out, ws, st);
}

void build_plan_finish(Plan& p, const double* lam, DeviceScratch& ws, cudaStream_t st) {
  const int kp = p.kp, k = p.k;
  const int64_t n = p.n, ng = p.ng;
  p.kind = ws.get_i32("pl_kind", ng);
  const bool par = p.par_mode < 0 ? n >= kPlanParMinN : p.par_mode != 0;
  const unsigned gblocks = (unsigned)cdiv(std::max<int64_t>(ng, 1), kPlanParThreads);
  double* part = par ? ws.get_f64("pl_part", 3 * kPlanParBlocks) : nullptr;
  if (par) {
    plan_sums_kernel<<<kPlanParBlocks, kPlanParThreads, 0, st>>>(p.u, n, kp, k, p.alpha, p.counts,
                                                                 part);
    EIGB_LAUNCH_CHECK();
    classify_par_kernel<<<gblocks, kPlanParThreads, 0, st>>>(p.u, kp, k, p.alpha, p.gstart, p.glen,
                                                             p.counts, p.exact ? 1 : 0, part,
                                                             kPlanParBlocks, p.kind, p.scal);
  } else {
    classify_kernel<<<1, kPlanThreads, 0, st>>>(p.u, n, kp, k, p.alpha, p.gstart, p.glen, p.counts,
                                                 p.exact ? 1 : 0, p.kind, p.scal);
  }
  EIGB_LAUNCH_CHECK();

  // multi-member runs (their count came back with ng): host-side offsets,
  // since the lengths size the H/R storage; none (the common case): no trip
  const int64_t nmulti = p.nmulti;
  std::vector<int64_t> glen_h;
  p.hoff = ws.get_i64("pl_hoff", ng);
  p.roff = ws.get_i64("pl_roff", ng);
  p.rank = ws.get_i64("pl_rank", ng);
  int64_t hs = 0, rs = 0;
  if (nmulti > 0) {
    glen_h.resize(ng);
    EIGB_CUDA(cudaMemcpyAsync(glen_h.data(), p.glen, 8 * ng, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaStreamSynchronize(st));
    std::vector<int64_t> hoff(ng), roff(ng);
    for (int64_t g = 0; g < ng; ++g) {
      hoff[g] = hs;
      roff[g] = rs;
      if (glen_h[g] > 1) {
        hs += glen_h[g] * glen_h[g];
        rs += glen_h[g] * kp;
      }
    }
    EIGB_CUDA(cudaMemcpyAsync(p.hoff, hoff.data(), 8 * ng, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(p.roff, roff.data(), 8 * ng, cudaMemcpyHostToDevice, st));
    // the host vectors must outlive the copies
    EIGB_CUDA(cudaStreamSynchronize(st));
  } else {
    EIGB_CUDA(cudaMemsetAsync(p.hoff, 0, 8 * ng, st));
    EIGB_CUDA(cudaMemsetAsync(p.roff, 0, 8 * ng, st));
  }
  p.hbuf = ws.get_f64("pl_hbuf", hs);
  p.rbuf = ws.get_f64("pl_rbuf", rs);
  if (nmulti > 0) {
    compress_kernel<<<(unsigned)cdiv(ng, 64), 64, 0, st>>>(p.u, kp, k, p.gstart, p.glen, p.kind,
                                                         p.counts, p.hoff, p.roff, p.hbuf, p.rbuf,
                                                         p.rank, p.scal, p.exact ? 1 : 0);
    EIGB_LAUNCH_CHECK();
  } else {
    EIGB_CUDA(cudaMemsetAsync(p.rank, 0, 8 * ng, st));
  }
  p.d = ws.get_f64("pl_d", n);
  p.alpha_red = ws.get_f64("pl_alpha_red", n);
  p.ur = ws.get_f64("pl_ur", (size_t)n * kp);
  p.red_src = ws.get_i64("pl_red_src", n);
  p.dec_val = ws.get_f64("pl_dec_val", n);
  p.dec_src = ws.get_i64("pl_dec_src", n);
  p.orig_map = ws.get_i64("pl_orig_map", n);
  int64_t* ta = ws.get_i64("pl_tmpa", ng);
  int64_t* tb = ws.get_i64("pl_tmpb", ng);
  p.off_red = ws.get_i64("pl_off_red", ng);
  p.off_dec = ws.get_i64("pl_off_dec", ng);
  if (par) {
    assemble_count_kernel<<<gblocks, kPlanParThreads, 0, st>>>(p.glen, p.kind, p.rank, p.counts, ta,
                                                               tb);
    EIGB_LAUNCH_CHECK();
    assemble_scan_kernel<<<1, kPlanThreads, 0, st>>>(ta, tb, p.counts, p.off_red, p.off_dec);
    EIGB_LAUNCH_CHECK();
    assemble_scatter_kernel<<<gblocks, kPlanParThreads, 0, st>>>(
        lam, p.u, kp, p.gstart, p.glen, p.gval, p.kind, p.rank, p.roff, p.rbuf, p.counts, p.off_red,
        p.off_dec, p.alpha, p.alpha_red, p.d, p.ur, p.red_src, p.dec_val, p.dec_src, p.orig_map);
    EIGB_LAUNCH_CHECK();
    clips_part_kernel<<<kPlanParBlocks, kPlanParThreads, 0, st>>>(p.d, p.ur, p.counts, kp, k, p.sgn,
                                                                  part);
    EIGB_LAUNCH_CHECK();
    clips_final_kernel<<<1, 32, 0, st>>>(p.d, p.counts, part, kPlanParBlocks, p.scal);
    EIGB_LAUNCH_CHECK();
  } else {
    assemble_reduced_kernel<<<1, kPlanThreads, 0, st>>>(
        lam, p.u, n, kp, p.gstart, p.glen, p.gval, p.kind, p.rank, p.roff, p.rbuf, p.counts, ta, tb,
        p.off_red, p.off_dec, p.alpha, p.alpha_red, p.d, p.ur, p.red_src, p.dec_val, p.dec_src,
        p.orig_map);
    EIGB_LAUNCH_CHECK();
    clips_kernel<<<1, kPlanThreads, 0, st>>>(p.d, p.ur, p.counts, kp, k, p.sgn, p.scal);
    EIGB_LAUNCH_CHECK();
  }
  // one round trip for the sizes, the scales and (with multi-member runs) the
  // run ranks and kinds; a speculative plan also learns its group count and
  // whether its assumptions held
  int64_t cnt[5];
  double sc[8];
  std::vector<int64_t> rk(nmulti > 0 ? ng : 0);
  std::vector<int> kd(nmulti > 0 ? ng : 0);
  EIGB_CUDA(cudaMemcpyAsync(cnt, p.counts, 40, cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaMemcpyAsync(sc, p.scal, 64, cudaMemcpyDeviceToHost, st));
  if (nmulti > 0) {
    EIGB_CUDA(cudaMemcpyAsync(rk.data(), p.rank, 8 * ng, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaMemcpyAsync(kd.data(), p.kind, 4 * ng, cudaMemcpyDeviceToHost, st));
  }
  EIGB_CUDA(cudaStreamSynchronize(st));
  if (p.spec) {
    p.ng = cnt[0];
    p.nmulti = cnt[4];
    p.spec_failed = (p.nmulti > 0) || (sc[7] != 0.0);
    if (p.spec_failed) return;
  }
  p.nred = cnt[1];
  p.ndec = cnt[2];
  bool ok = true;  // rows of compressed runs are not simple poles of f
  for (int64_t g = 0; g < (nmulti > 0 ? ng : 0) && ok; ++g)
    if (glen_h[g] > 1 && kd[g] != 1 && rk[g] > 0) ok = false;
  p.alpha_red_ok = ok;
  if (p.nred + p.ndec != n) throw Error(2, "merge", "reduced problem does not account for n pairs");
  p.scale = sc[0];
  p.alpha_mass = sc[1];
  p.u_mass = sc[2];
  p.lo_clip = sc[4];
  p.hi_clip = sc[5];
}

void build_plan_dev(Plan& p, const double* lam, int64_t n, double run_rel, DeviceScratch& ws,
                    cudaStream_t st) {
  build_plan_groups(p, lam, n, run_rel, ws, st);
  build_plan_weights(p, 0, p.ng, p.alpha, ws, st);
  build_plan_finish(p, lam, ws, st);
}

}  // namespace eigb
