// K5: FP64 back-transform Q' = Q X on the DMMA tensor pipe (sm_100a).
//
// proj/src/eigvec.cpp:339 (kernels::gemm_nn, kernels.cpp:32-48). FP64 has no
// tcgen05 kind on sm_100a; the FP64 tensor path is mma.sync.m8n8k4.f64,
// which ptxas lowers to DMMA.8x8x4 (measured ceiling 37.0 TFLOP/s,
// profiles/fp64_peaks_r01.json). X is stored transposed (Xt, one row per
// eigenvector), so both operands are K-contiguous ("TN"):
//   C[i, c] = s_c * sum_l A[i, l] Xt[c, l]
// CTA tile 128 x 128, K-tile 16 doubles, 4-stage cp.async pipeline into
// 128-byte XOR-swizzled shared memory, 8 warps of 64 x 32. The K index inside
// a tile is permuted per lane (step s of lane t uses k = 4*(t%4) + s for both
// operands) so every fragment load is one conflict-free 16-byte LDS.128
// feeding two DMMA k-steps. The epilogue applies the column scale (the
// eigenvector norms from K4) and records, per 128-row tile and column, the
// signed entry of largest magnitude (first row on ties) for the reference's
// sign rule (eigvec.cpp:340-347), which a second pass applies.
#include "pipeline.cuh"

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <string>

namespace eigb {

namespace {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4;
constexpr int GEMM_THREADS = 256;
constexpr int STAGE_DOUBLES = (BM + BN) * BK;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Stage layout: A tile [BM][BK] then B tile [BN][BK]; row r holds 8 chunks of
// 2 doubles, logical chunk q at physical chunk q ^ (r & 7).
__device__ __forceinline__ void load_stage(double* st, const double* __restrict__ a,
                                           const double* __restrict__ b, int64_t m, int64_t nn,
                                           int64_t K, int64_t lda, int64_t ldb, int64_t m0,
                                           int64_t n0, int64_t k0) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int s = 0; s < (BM * BK / 2) / GEMM_THREADS; ++s) {
    const int id = tid + s * GEMM_THREADS;
    const int row = id >> 3, q = id & 7;
    const int64_t gr = m0 + row, gk = k0 + 2 * q;
    int bytes = 0;
    if (gr < m && gk < K) bytes = (K - gk >= 2) ? 16 : 8;
    const double* src = bytes ? a + gr * lda + gk : a;
    cp_async16(st + row * BK + 2 * (q ^ (row & 7)), src, bytes);
  }
  double* sb = st + BM * BK;
#pragma unroll
  for (int s = 0; s < (BN * BK / 2) / GEMM_THREADS; ++s) {
    const int id = tid + s * GEMM_THREADS;
    const int row = id >> 3, q = id & 7;
    const int64_t gr = n0 + row, gk = k0 + 2 * q;
    int bytes = 0;
    if (gr < nn && gk < K) bytes = (K - gk >= 2) ? 16 : 8;
    const double* src = bytes ? b + gr * ldb + gk : b;
    cp_async16(sb + row * BK + 2 * (q ^ (row & 7)), src, bytes);
  }
}

// Epilogue shared by both kernels: column scale (eigenvector norms from K4),
// row-major stores with leading dimension ldc, and per (row tile, column) the
// signed entry of largest magnitude, first row on ties (eigvec.cpp:340-347).
__device__ __forceinline__ void epilogue_store(double (&acc)[8][4][2], int64_t m, int64_t nn,
                                               double* __restrict__ c, int64_t ldc,
                                               const double* __restrict__ colscale,
                                               const int64_t* __restrict__ colmap, int64_t m0,
                                               int64_t n0, int wm, int wn, int g, int t4,
                                               double* colbest, int* colrow) {
#pragma unroll
  for (int nb = 0; nb < 4; ++nb) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int cl = wn * 32 + nb * 8 + 2 * t4 + e;
      const int64_t cg = n0 + cl;
      const double sc = (cg < nn) ? colscale[cg] : 0.0;
      double best = 0.0;
      int brow = 0x7fffffff;
#pragma unroll
      for (int mb = 0; mb < 8; ++mb) {
        const int rl = wm * 64 + mb * 8 + g;
        const double v = acc[mb][nb][e] * sc;
        acc[mb][nb][e] = v;
        if (m0 + rl < m && (fabs(v) > fabs(best) || (fabs(v) == fabs(best) && rl < brow))) {
          best = v;
          brow = rl;
        }
      }
      // reduce over the 8 lanes sharing this column (g = 0..7)
#pragma unroll
      for (int o = 4; o <= 16; o <<= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int orow = __shfl_xor_sync(0xffffffffu, brow, o);
        if (fabs(ob) > fabs(best) || (fabs(ob) == fabs(best) && orow < brow)) {
          best = ob;
          brow = orow;
        }
      }
      if (g == 0) {
        colbest[wm * BN + cl] = best;
        colrow[wm * BN + cl] = brow;
      }
    }
  }
  if (colmap) {  // scattered output columns (compact back-transform)
    int64_t oc[4][2];
#pragma unroll
    for (int nb = 0; nb < 4; ++nb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t col = n0 + wn * 32 + nb * 8 + 2 * t4 + e;
        oc[nb][e] = (col < nn) ? colmap[col] : -1;
      }
#pragma unroll
    for (int mb = 0; mb < 8; ++mb) {
      const int64_t row = m0 + wm * 64 + mb * 8 + g;
      if (row >= m) continue;
#pragma unroll
      for (int nb = 0; nb < 4; ++nb)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (oc[nb][e] >= 0) c[row * ldc + oc[nb][e]] = acc[mb][nb][e];
    }
    return;
  }
#pragma unroll
  for (int mb = 0; mb < 8; ++mb) {
    const int64_t row = m0 + wm * 64 + mb * 8 + g;
    if (row >= m) continue;
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
      const int64_t col = n0 + wn * 32 + nb * 8 + 2 * t4;
      double* dst = c + row * ldc + col;
      if (col + 1 < nn && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        *reinterpret_cast<double2*>(dst) = make_double2(acc[mb][nb][0], acc[mb][nb][1]);
      } else {
        if (col < nn) dst[0] = acc[mb][nb][0];
        if (col + 1 < nn) dst[1] = acc[mb][nb][1];
      }
    }
  }
}

__device__ __forceinline__ void tile_colmax_write(double* __restrict__ tile_colmax, int64_t tm,
                                                  int64_t nn, int64_t tcm_ld,
                                                  const int64_t* __restrict__ colmap, int64_t n0,
                                                  int tid, const double* colbest,
                                                  const int* colrow) {
  const int64_t cg = n0 + tid;
  if (cg >= nn) return;
  const double b0 = colbest[tid], b1 = colbest[BN + tid];
  const int r0 = colrow[tid], r1 = colrow[BN + tid];
  double best = b0;
  if (fabs(b1) > fabs(b0) || (fabs(b1) == fabs(b0) && r1 < r0)) best = b1;
  tile_colmax[tm * tcm_ld + (colmap ? colmap[cg] : cg)] = best;
}

__global__ void __launch_bounds__(GEMM_THREADS, 1)
    dmma_gemm_nt_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t m,
                        int64_t nn, int64_t K, int64_t lda, int64_t ldb, double* __restrict__ c,
                        int64_t ldc, const double* __restrict__ colscale,
                        const int64_t* __restrict__ colmap, double* __restrict__ tile_colmax,
                        int64_t tcm_ld) {
  extern __shared__ __align__(128) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps
  // grouped rasterization: 8 M-tiles share each run of N-tiles (L2 reuse)
  const int64_t tiles_m = cdiv_dev(m, BM), tiles_n = cdiv_dev(nn, BN);
  const int64_t pid = blockIdx.x;
  const int64_t group = 8;
  const int64_t per_group = group * tiles_n;
  const int64_t gidx = pid / per_group;
  const int64_t first_m = gidx * group;
  const int64_t gsize = (tiles_m - first_m) < group ? (tiles_m - first_m) : group;
  const int64_t tm = first_m + (pid % per_group) % gsize;
  const int64_t tn = (pid % per_group) / gsize;
  const int64_t m0 = tm * BM, n0 = tn * BN;

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int64_t KT = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT)
      load_stage(smem + s * STAGE_DOUBLES, a, b, m, nn, K, lda, ldb, m0, n0, (int64_t)s * BK);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  const int g = lane >> 2, t4 = lane & 3;
  for (int64_t kt = 0; kt < KT; ++kt) {
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 2) : "memory");
    __syncthreads();
    const int64_t nk = kt + STAGES - 1;
    if (nk < KT)
      load_stage(smem + (nk % STAGES) * STAGE_DOUBLES, a, b, m, nn, K, lda, ldb, m0, n0, nk * BK);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const double* sa = smem + (kt % STAGES) * STAGE_DOUBLES;
    const double* sb = sa + BM * BK;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = 2 * t4 + h;
      double2 af[8], bf[4];
#pragma unroll
      for (int mb = 0; mb < 8; ++mb) {
        const int row = wm * 64 + mb * 8 + g;
        af[mb] = *reinterpret_cast<const double2*>(sa + row * BK + 2 * (q ^ g));
      }
#pragma unroll
      for (int nb = 0; nb < 4; ++nb) {
        const int row = wn * 32 + nb * 8 + g;
        bf[nb] = *reinterpret_cast<const double2*>(sb + row * BK + 2 * (q ^ g));
      }
#pragma unroll
      for (int mb = 0; mb < 8; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) dmma(acc[mb][nb][0], acc[mb][nb][1], af[mb].x, bf[nb].x);
#pragma unroll
      for (int mb = 0; mb < 8; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) dmma(acc[mb][nb][0], acc[mb][nb][1], af[mb].y, bf[nb].y);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();

  // ---- epilogue: scale, store, per-tile column max for the sign rule
  double* colbest = smem;                               // [2][BN] signed value
  int* colrow = reinterpret_cast<int*>(smem + 2 * BN);  // [2][BN] row of best
  epilogue_store(acc, m, nn, c, ldc, colscale, colmap, m0, n0, wm, wn, g, t4, colbest, colrow);
  __syncthreads();
  if (tile_colmax && tid < BN)
    tile_colmax_write(tile_colmax, tm, nn, tcm_ld, colmap, n0, tid, colbest, colrow);
}

}  // namespace
}  // namespace eigb

#include "gemm_tma.cuh"

namespace eigb {
namespace {

// Sign rule across row tiles: first tile holding the maximal |entry| decides.
__global__ void colsign_kernel(const double* __restrict__ tile_colmax, int64_t tiles_m,
                               int64_t tcm_ld, int64_t nn, const int* __restrict__ mode,
                               double* __restrict__ flip) {
  const int64_t cidx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (cidx >= nn) return;
  double best = 0.0;
  for (int64_t t = 0; t < tiles_m; ++t) {
    const double v = tile_colmax[t * tcm_ld + cidx];
    if (fabs(v) > fabs(best)) best = v;
  }
  flip[cidx] = (mode[cidx] && best < 0.0) ? -1.0 : 1.0;
}

__global__ void apply_sign_kernel(double* __restrict__ c, int64_t m, int64_t nn, int64_t ldc,
                                  const double* __restrict__ flip, const int* any) {
  if (!*any) return;
  for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
    double* row = c + i * ldc;
    for (int64_t j = threadIdx.x; j < nn; j += blockDim.x)
      if (flip[j] < 0.0) row[j] = -row[j];
  }
}

__global__ void any_flip_kernel(const double* flip, int64_t nn, int* any) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < nn && flip[j] < 0.0) atomicOr(any, 1);
}

}  // namespace

void gemm_nt_dev(const double* a, const double* b, int64_t m, int64_t nn, int64_t kk, double* c,
                 int64_t ldc, const double* colscale, double* tile_colmax, cudaStream_t st) {
  gemm_nt_ex(a, kk, b, kk, m, nn, kk, c, ldc, colscale, nullptr, tile_colmax, nn, st);
}

void gemm_nt_ex(const double* a, int64_t lda, const double* b, int64_t ldb, int64_t m, int64_t nn,
                int64_t kk, double* c, int64_t ldc, const double* colscale, const int64_t* colmap,
                double* tile_colmax, int64_t tcm_ld, cudaStream_t st) {
  if (m <= 0 || nn <= 0) return;
  if ((lda & 1) || (ldb & 1) || (reinterpret_cast<uintptr_t>(a) & 15) ||
      (reinterpret_cast<uintptr_t>(b) & 15)) {
    // odd inner dimension (odd n) or unaligned operands: stage zero-padded
    // copies with an even, 16-byte aligned row pitch (stream-ordered pool)
    const int64_t kp2 = (kk + 1) & ~int64_t(1);
    double *ap = nullptr, *bp = nullptr;
    EIGB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ap), sizeof(double) * m * kp2, st));
    EIGB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&bp), sizeof(double) * nn * kp2, st));
    EIGB_CUDA(cudaMemsetAsync(ap, 0, sizeof(double) * m * kp2, st));
    EIGB_CUDA(cudaMemsetAsync(bp, 0, sizeof(double) * nn * kp2, st));
    EIGB_CUDA(cudaMemcpy2DAsync(ap, 8 * kp2, a, 8 * lda, 8 * kk, m, cudaMemcpyDeviceToDevice, st));
    EIGB_CUDA(cudaMemcpy2DAsync(bp, 8 * kp2, b, 8 * ldb, 8 * kk, nn, cudaMemcpyDeviceToDevice, st));
    gemm_nt_ex(ap, kp2, bp, kp2, m, nn, kp2, c, ldc, colscale, colmap, tile_colmax, tcm_ld, st);
    EIGB_CUDA(cudaFreeAsync(ap, st));
    EIGB_CUDA(cudaFreeAsync(bp, st));
    return;
  }
  const int64_t tiles = cdiv(m, BM) * cdiv(nn, BN);
  static int use_tma = -1;  // EIGMOD_B200_GEMM=cpasync selects the cp.async kernel
  if (use_tma < 0) {
    const char* e = std::getenv("EIGMOD_B200_GEMM");
    use_tma = !(e && std::string(e) == "cpasync");
  }
  CUtensorMap ma, mb;
  if (use_tma && kk <= INT32_MAX && m <= INT32_MAX && nn <= INT32_MAX &&
      make_map(&ma, a, m, kk, lda) && make_map(&mb, b, nn, kk, ldb)) {
    const size_t sm = sizeof(double) * TMA_STAGES * STAGE_DOUBLES + 2 * TMA_STAGES * 8 + 1024;
    EIGB_CUDA(cudaFuncSetAttribute(dmma_gemm_nt_tma_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    static int group = 0;  // EIGMOD_B200_GEMM_GROUP: row tiles per rasterization group
    if (group == 0) {
      const char* e = std::getenv("EIGMOD_B200_GEMM_GROUP");
      group = e ? std::max(1, std::atoi(e)) : 4;
    }
    dmma_gemm_nt_tma_kernel<<<(unsigned)tiles, TMA_THREADS, sm, st>>>(
        ma, mb, m, nn, kk, c, ldc, colscale, colmap, tile_colmax, tcm_ld, group);
    EIGB_LAUNCH_CHECK();
    return;
  }
  const size_t sm = sizeof(double) * STAGES * STAGE_DOUBLES;
  EIGB_CUDA(cudaFuncSetAttribute(dmma_gemm_nt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm));
  dmma_gemm_nt_kernel<<<(unsigned)tiles, GEMM_THREADS, sm, st>>>(
      a, b, m, nn, kk, lda, ldb, c, ldc, colscale, colmap, tile_colmax, tcm_ld);
  EIGB_LAUNCH_CHECK();
}

void sign_rule_dev(const double* tile_colmax, int64_t n, int64_t ncols, const int* mode, double* c,
                   int64_t ldc, DeviceScratch& ws, cudaStream_t st) {
  sign_rule_ld(tile_colmax, ncols, n, ncols, mode, c, ldc, ws, st);
}

void sign_rule_ld(const double* tile_colmax, int64_t tcm_ld, int64_t n, int64_t ncols,
                  const int* mode, double* c, int64_t ldc, DeviceScratch& ws, cudaStream_t st) {
  if (ncols <= 0) return;
  const int64_t tiles_m = cdiv(n, BM);
  double* flip = ws.get_f64("gemm_flip", ncols);
  int* any = ws.get_i32("gemm_any_flip", 1);
  colsign_kernel<<<(unsigned)cdiv(ncols, 256), 256, 0, st>>>(tile_colmax, tiles_m, tcm_ld, ncols,
                                                             mode, flip);
  EIGB_LAUNCH_CHECK();
  EIGB_CUDA(cudaMemsetAsync(any, 0, 4, st));
  any_flip_kernel<<<(unsigned)cdiv(ncols, 256), 256, 0, st>>>(flip, ncols, any);
  EIGB_LAUNCH_CHECK();
  apply_sign_kernel<<<148 * 8, 256, 0, st>>>(c, n, ncols, ldc, flip, any);
  EIGB_LAUNCH_CHECK();
}

double* tile_colmax_buffer(int64_t n, int64_t ncols, DeviceScratch& ws) {
  return ws.get_f64("gemm_tile_colmax", (size_t)cdiv(n, BM) * std::max<int64_t>(ncols, 1));
}

}  // namespace eigb

// ------------------------------------------------------------ FP64 ceilings
// Loop kernels that saturate the DMMA tensor pipe and the DFMA pipe; bench.py
// uses them as the live FP64 roofline denominators (MEASURED_PEAKS.json has
// no FP64 entry).
namespace eigb {
namespace {

__global__ void dmma_peak_kernel(double* out, int iters, double av, double bv) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  const double A = av + threadIdx.x, B = bv - threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], A, B);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dfma_peak_kernel(double* out, int iters, double a, double b) {
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

}  // namespace

void fp64_peaks_dev(int sms, double* dmma_tflops, double* dfma_tflops, DeviceScratch& ws,
                    cudaStream_t st) {
  double* out = ws.get_f64("peak_out", 1024);
  cudaEvent_t e0, e1;
  EIGB_CUDA(cudaEventCreate(&e0));
  EIGB_CUDA(cudaEventCreate(&e1));
  const int iters = 20000;
  auto timed = [&](auto launch) {
    launch();
    EIGB_LAUNCH_CHECK();
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      EIGB_CUDA(cudaEventRecord(e0, st));
      launch();
      EIGB_CUDA(cudaEventRecord(e1, st));
      EIGB_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      EIGB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      best = std::min(best, ms);
    }
    return (double)best;
  };
  const int bm = 8 * sms;
  const double ms_m = timed([&] { dmma_peak_kernel<<<bm, 128, 0, st>>>(out, iters / 4, 1e-3, 2e-3); });
  *dmma_tflops = 2.0 * 256 * 8 * (iters / 4) * 4.0 * bm / (ms_m * 1e-3) / 1e12;
  const int bf = 8 * sms;
  const double ms_f = timed([&] { dfma_peak_kernel<<<bf, 256, 0, st>>>(out, iters, 0.999, 1e-3); });
  *dfma_tflops = 2.0 * 8 * iters * 256.0 * bf / (ms_f * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

}  // namespace eigb
