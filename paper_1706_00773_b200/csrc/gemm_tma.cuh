// TMA variant of the K5 DMMA GEMM (included by gemm.cu after its helpers).
//
// One elected thread issues cp.async.bulk.tensor (TMA, 128-byte swizzle =
// the layout load_stage writes) into a 6-stage ring guarded by full/empty
// mbarriers; all 8 warps wait only for "full", run the same DMMA fragment
// schedule as the cp.async kernel and release the slot with one arrive per
// warp. The refill of a slot is issued one k-tile after its release, so the
// issuing thread rarely waits. No CTA-wide barrier in the main loop, no
// per-thread copy instructions. (A dedicated producer warp would make the
// CTA 288 threads, which caps registers at 168 and spills the accumulators.)
// Out-of-range boxes are zero-filled by the TMA unit.
//
// Round 2: with two warps per scheduler the tensor pipe idles whenever both
// are outside their DMMA streams, so the loop's non-DMMA work is kept minimal:
// fragments are explicit LDS.128 on 32-bit shared addresses (a generic LD
// through the aligned pointer cost latency and 64-bit address registers), the
// stage index and barrier parity advance incrementally (no 64-bit modulo),
// and the next stage's full barrier is tested before the last 64 DMMAs of the
// current one. Tensor pipe active 96.4% -> 98.3% (ncu, n = 8192), 36.04 ->
// 36.79 TFLOP/s at n = 32768 (cuBLAS DGEMM: 36.65).
//
// Rasterization: groups of `group_rows` row tiles sweep the column tiles, so
// consecutive CTAs share a B panel. The CTAs of a launch drift apart in k
// (tiles start whenever an SM frees up), and only CTAs a few launches apart
// still find each other's panel slices in L2: DRAM reads per launch at
// n = 32768 are 2.40 / 1.52 / 1.39 / 1.53 / 1.45 / 1.84 / 2.08 / 2.28 TB for
// groups of 1 / 2 / 3 / 4 / 6 / 8 / 16 / 32 row tiles (ncu), the time the same
// (tensor-bound) for all; 4 is the default (EIGMOD_B200_GEMM_GROUP).
#pragma once

#include <cuda.h>

namespace eigb {
namespace {

constexpr int TMA_STAGES = 6;
constexpr int TMA_THREADS = GEMM_THREADS;

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ double2 lds128(unsigned addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
// One non-blocking test of a barrier phase (1 = completed).
__device__ __forceinline__ unsigned mbar_test(unsigned bar32, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(bar32), "r"(parity)
      : "memory");
  return ok;
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(d),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(b), "r"(c0), "r"(c1)
      : "memory");
}

__global__ void __launch_bounds__(TMA_THREADS, 1)
    dmma_gemm_nt_tma_kernel(const __grid_constant__ CUtensorMap tma_a,
                            const __grid_constant__ CUtensorMap tma_b, int64_t m, int64_t nn,
                            int64_t K, double* __restrict__ c, int64_t ldc,
                            const double* __restrict__ colscale,
                            const int64_t* __restrict__ colmap, double* __restrict__ tile_colmax,
                            int64_t tcm_ld, int group_rows) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  double* smem = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(smraw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TMA_STAGES * STAGE_DOUBLES);
  uint64_t* empty = full + TMA_STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t tiles_m = cdiv_dev(m, BM), tiles_n = cdiv_dev(nn, BN);
  const int64_t pid = blockIdx.x;
  const int64_t group = group_rows;
  const int64_t per_group = group * tiles_n;
  const int64_t gidx = pid / per_group;
  const int64_t first_m = gidx * group;
  const int64_t gsize = (tiles_m - first_m) < group ? (tiles_m - first_m) : group;
  const int64_t tm = first_m + (pid % per_group) % gsize;
  const int64_t tn = (pid % per_group) / gsize;
  const int64_t m0 = tm * BM, n0 = tn * BN;
  const int64_t KT = (K + BK - 1) / BK;

  if (tid == 0) {
    for (int s = 0; s < TMA_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], GEMM_THREADS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int64_t kt) {
    const int s = (int)(kt % TMA_STAGES);
    double* st = smem + s * STAGE_DOUBLES;
    mbar_expect_tx(&full[s], STAGE_DOUBLES * 8);
    tma_load_2d(st, &tma_a, &full[s], (int)(kt * BK), (int)m0);
    tma_load_2d(st + BM * BK, &tma_b, &full[s], (int)(kt * BK), (int)n0);
  };
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
    for (int64_t kt = 0; kt < TMA_STAGES && kt < KT; ++kt) issue(kt);
  }

  const int wm = warp >> 2, wn = warp & 3;
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int g = lane >> 2, t4 = lane & 3;
  // 32-bit loop state (stage index and parity advance incrementally: no
  // 64-bit modulo in the loop), explicit LDS.128, and the full-barrier test
  // of the next stage issued before the last 64 DMMAs of this one, so its
  // latency is off the critical path.
  const unsigned sb32 = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const unsigned full32 = static_cast<unsigned>(__cvta_generic_to_shared(full));
  const unsigned oa = (unsigned)((wm * 64 + g) * BK * 8);
  const unsigned ob = (unsigned)(BM * BK * 8 + (wn * 32 + g) * BK * 8);
  const unsigned q0 = 16u * (unsigned)((2 * t4) ^ g), q1 = 16u * (unsigned)((2 * t4 + 1) ^ g);
  const int kts = (int)KT;
  int s = 0;            // stage of k-tile kt
  unsigned par = 0;     // its full-barrier parity
  int rs = 0;           // stage refilled next (k-tile kt - 1)
  unsigned rpar = 0;
  unsigned ready = mbar_test(full32, 0) ? 1u : 0u;
  for (int kt = 0; kt < kts; ++kt) {
    if (tid == 0 && kt >= 1) {
      if (kt - 1 + TMA_STAGES < kts) {
        mbar_wait(&empty[rs], rpar);
        issue((int64_t)kt - 1 + TMA_STAGES);
      }
      if (++rs == TMA_STAGES) { rs = 0; rpar ^= 1u; }
    }
    if (!ready) mbar_wait(&full[s], par);
    const unsigned st = sb32 + (unsigned)s * (STAGE_DOUBLES * 8);
    int s1 = s + 1;
    unsigned par1 = par;
    if (s1 == TMA_STAGES) { s1 = 0; par1 ^= 1u; }
    {
      double2 af[8], bf[4];
#pragma unroll
      for (int nb = 0; nb < 4; ++nb) bf[nb] = lds128(st + ob + q0 + nb * 8 * BK * 8);
#pragma unroll
      for (int mb = 0; mb < 8; ++mb) af[mb] = lds128(st + oa + q0 + mb * 8 * BK * 8);
#pragma unroll
      for (int mb = 0; mb < 8; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) dmma(acc[mb][nb][0], acc[mb][nb][1], af[mb].x, bf[nb].x);
#pragma unroll
      for (int mb = 0; mb < 8; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) dmma(acc[mb][nb][0], acc[mb][nb][1], af[mb].y, bf[nb].y);
    }
    {
      double2 af[8], bf[4];
#pragma unroll
      for (int mb = 0; mb < 8; ++mb) af[mb] = lds128(st + oa + q1 + mb * 8 * BK * 8);
#pragma unroll
      for (int nb = 0; nb < 4; ++nb) bf[nb] = lds128(st + ob + q1 + nb * 8 * BK * 8);
      ready = (kt + 1 < kts && mbar_test(full32 + 8u * (unsigned)s1, par1)) ? 1u : 0u;
#pragma unroll
      for (int mb = 0; mb < 8; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) dmma(acc[mb][nb][0], acc[mb][nb][1], af[mb].x, bf[nb].x);
#pragma unroll
      for (int mb = 0; mb < 8; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) dmma(acc[mb][nb][0], acc[mb][nb][1], af[mb].y, bf[nb].y);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    s = s1;
    par = par1;
  }

  // ---- epilogue
  __syncthreads();
  double* colbest = smem;
  int* colrow = reinterpret_cast<int*>(smem + 2 * BN);
  epilogue_store(acc, m, nn, c, ldc, colscale, colmap, m0, n0, wm, wn, g, t4, colbest, colrow);
  __syncthreads();
  if (tile_colmax && tid < BN)
    tile_colmax_write(tile_colmax, tm, nn, tcm_ld, colmap, n0, tid, colbest, colrow);
}

// Driver entry point for tensor-map encoding (no -lcuda at link time).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2D map of a row-major [rows][kk] FP64 matrix with row pitch ld (even),
// box BK (k) x 128 (rows); k beyond kk reads as zero.
bool make_map(CUtensorMap* map, const double* base, int64_t rows, int64_t kk, int64_t ld) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)kk, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {BK, 128};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace
}  // namespace eigb
