// Validation metrics of an update on the GPU (proj/src/eigvec.cpp:384-393):
//   residual_fro = || sym(Q' diag(l') Q'^T) - sym(sym(Q diag(l) Q^T) + K J K^T) ||_F
//   ortho_err    = max_ij |(Q'^T Q' - I)_ij|
// with the reference's symmetrization (kernels.cpp:123-131, applied by
// SymmetricDense::from at core.cpp:66-74). The three n^3 products run on the
// K5 DMMA GEMM; the reference does them on the CPU (outside its timer).
#include "pipeline.cuh"

namespace eigb {

namespace {

__global__ void scale_cols_kernel(const double* __restrict__ q, const double* __restrict__ lam,
                                  int64_t n, double* __restrict__ w) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x)
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) w[i * n + j] = q[i * n + j] * lam[j];
}

__global__ void transpose_kernel(const double* __restrict__ a, int64_t n, double* __restrict__ t) {
  __shared__ double tile[32][33];
  const int64_t bx = (int64_t)blockIdx.x * 32, by = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = by + r, j = bx + threadIdx.x;
    tile[r][threadIdx.x] = (i < n && j < n) ? a[i * n + j] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = bx + r, j = by + threadIdx.x;
    if (i < n && j < n) t[i * n + j] = tile[threadIdx.x][r];
  }
}

// Partial sums of squared residual entries (upper triangle + diagonal, both
// symmetrized exactly as the reference), one value per block.
__global__ void residual_kernel(const double* __restrict__ g1, const double* __restrict__ g2,
                                const double* __restrict__ kmat, const int* __restrict__ sgn,
                                int64_t n, int k, double* __restrict__ part) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
      // target = sym(sym(A) + K J K^T); got = sym(G1)
      const double a = 0.5 * (g2[i * n + j] + g2[j * n + i]);
      double kjk = 0.0;
      for (int r = 0; r < k; ++r) kjk += (double)sgn[r] * kmat[i * k + r] * kmat[j * k + r];
      const double tgt = a + kjk;  // kjk is symmetric; sym() leaves it unchanged
      const double got = 0.5 * (g1[i * n + j] + g1[j * n + i]);
      const double d = got - tgt;
      s += d * d;
    }
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

__global__ void ortho_kernel(const double* __restrict__ g, int64_t n, double* __restrict__ part) {
  __shared__ double red[32];
  double m = 0.0;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x)
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x)
      m = fmax(m, fabs(g[i * n + j] - (i == j ? 1.0 : 0.0)));
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
    part[blockIdx.x] = t;
  }
}

// In-place symmetrization a(i,j) = a(j,i) = 0.5 (a(i,j) + a(j,i))
// (kernels.cpp:123-131): one block per 32 x 32 tile pair above or on the
// diagonal; both tiles staged in shared memory so the transposed side is read
// and written coalesced.
__global__ void symmetrize_kernel(double* __restrict__ a, int64_t n) {
  const int64_t bi = blockIdx.y, bj = blockIdx.x;
  if (bj < bi) return;
  __shared__ double t1[32][33], t2[32][33];
  const int tx = threadIdx.x;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i1 = bi * 32 + r, j1 = bj * 32 + tx;  // tile (bi, bj)
    const int64_t i2 = bj * 32 + r, j2 = bi * 32 + tx;  // tile (bj, bi)
    t1[r][tx] = (i1 < n && j1 < n) ? a[i1 * n + j1] : 0.0;
    t2[r][tx] = (i2 < n && j2 < n) ? a[i2 * n + j2] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i1 = bi * 32 + r, j1 = bj * 32 + tx;
    const int64_t i2 = bj * 32 + r, j2 = bi * 32 + tx;
    // element (i1, j1) pairs with t2[tx][r] = a(j1, i1)
    if (i1 < n && j1 < n && (bi != bj || j1 > i1))
      a[i1 * n + j1] = __dmul_rn(0.5, __dadd_rn(t1[r][tx], t2[tx][r]));
    if (bi != bj && i2 < n && j2 < n)
      a[i2 * n + j2] = __dmul_rn(0.5, __dadd_rn(t2[r][tx], t1[tx][r]));
    else if (bi == bj && i1 < n && j1 < n && j1 < i1)
      a[i1 * n + j1] = __dmul_rn(0.5, __dadd_rn(t1[tx][r], t1[r][tx]));
  }
}

// out = a + sum_r s_r k_r k_r^T with the reference's rounding sequence
// (core.cpp:105-115 -> kernels.cpp:111-121: c = s_r k_ir rounded, then
// out_ij += c k_jr, r ascending, no contraction): bit-identical.
__global__ void rank_update_kernel(const double* __restrict__ a, const double* __restrict__ kmat,
                                   const int* __restrict__ sgn, int64_t n, int k,
                                   double* __restrict__ out) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const double* ki = kmat + i * k;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
      double v = a[i * n + j];
      for (int r = 0; r < k; ++r)
        v = __dadd_rn(v, __dmul_rn(__dmul_rn((double)sgn[r], ki[r]), kmat[j * k + r]));
      out[i * n + j] = v;
    }
  }
}

__global__ void transpose_rect_kernel(const double* __restrict__ a, int64_t rows, int64_t cols,
                                      double* __restrict__ t) {
  __shared__ double tile[32][33];
  const int64_t bx = (int64_t)blockIdx.x * 32, by = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = by + r, j = bx + threadIdx.x;
    tile[r][threadIdx.x] = (i < rows && j < cols) ? a[i * cols + j] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = bx + r, j = by + threadIdx.x;  // t is cols x rows
    if (i < cols && j < rows) t[i * rows + j] = tile[threadIdx.x][r];
  }
}

__global__ void ortho_rect_kernel(const double* __restrict__ g, int64_t m,
                                  double* __restrict__ part) {
  __shared__ double red[32];
  double v = 0.0;
  for (int64_t i = blockIdx.x; i < m; i += gridDim.x)
    for (int64_t j = threadIdx.x; j < m; j += blockDim.x)
      v = fmax(v, fabs(g[i * m + j] - (i == j ? 1.0 : 0.0)));
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
    part[blockIdx.x] = t;
  }
}

double* ones_buffer(int64_t n, DeviceScratch& ws, cudaStream_t st) {
  double* ones = ws.get_f64("met_ones", n);
  std::vector<double> h(n, 1.0);
  EIGB_CUDA(cudaMemcpyAsync(ones, h.data(), 8 * n, cudaMemcpyHostToDevice, st));
  EIGB_CUDA(cudaStreamSynchronize(st));
  return ones;
}

}  // namespace

void symmetrize_dev(double* a, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  dim3 tb(32, 8), tg((unsigned)cdiv(n, 32), (unsigned)cdiv(n, 32));
  symmetrize_kernel<<<tg, tb, 0, st>>>(a, n);
  EIGB_LAUNCH_CHECK();
}

// kernels.cpp:98-109: W = Q diag(lambda), A = W Q^T (K5 DMMA), symmetrized.
void reconstruct_dev(const double* q, const double* lam, int64_t n, double* out, DeviceScratch& ws,
                     cudaStream_t st) {
  double* w = ws.get_f64("met_w", (size_t)n * n);
  double* ones = ones_buffer(n, ws, st);
  const int blocks = (int)std::min<int64_t>(n, 4096);
  scale_cols_kernel<<<blocks, 256, 0, st>>>(q, lam, n, w);
  EIGB_LAUNCH_CHECK();
  gemm_nt_dev(w, q, n, n, n, out, n, ones, nullptr, st);
  symmetrize_dev(out, n, st);
}

// core.cpp:105-115 (bit-identical, including the final symmetrization).
void apply_update_dev(const double* a, const double* kmat, const int* sgn, int64_t n, int k,
                      double* out, cudaStream_t st) {
  const int blocks = (int)std::min<int64_t>(n, 8192);
  rank_update_kernel<<<blocks, 256, 0, st>>>(a, kmat, sgn, n, k, out);
  EIGB_LAUNCH_CHECK();
  symmetrize_dev(out, n, st);
}

// kernels.cpp:150-154: max |A^T A - I| for A rows x cols; A^T A = T T^T with
// T = A^T on the K5 DMMA GEMM.
double ortho_error_dev(const double* a, int64_t rows, int64_t cols, DeviceScratch& ws,
                       cudaStream_t st) {
  double* t = ws.get_f64("met_t", (size_t)rows * cols);
  double* g = ws.get_f64("met_g1", (size_t)cols * cols);
  double* ones = ones_buffer(cols, ws, st);
  dim3 tb(32, 8), tg((unsigned)cdiv(cols, 32), (unsigned)cdiv(rows, 32));
  transpose_rect_kernel<<<tg, tb, 0, st>>>(a, rows, cols, t);
  EIGB_LAUNCH_CHECK();
  gemm_nt_dev(t, t, cols, cols, rows, g, cols, ones, nullptr, st);
  const int blocks = (int)std::min<int64_t>(cols, 4096);
  double* part = ws.get_f64("met_part", blocks);
  ortho_rect_kernel<<<blocks, 256, 0, st>>>(g, cols, part);
  EIGB_LAUNCH_CHECK();
  std::vector<double> hp(blocks);
  EIGB_CUDA(cudaMemcpyAsync(hp.data(), part, 8 * blocks, cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaStreamSynchronize(st));
  double m = 0.0;
  for (double v : hp) m = std::max(m, v);
  return m;
}

void update_metrics_dev(const double* q, const double* lam, const double* kmat, const int* sgn,
                        int64_t n, int k, const double* qo, const double* lo, double* residual_fro,
                        double* ortho_err, DeviceScratch& ws, cudaStream_t st) {
  double* w = ws.get_f64("met_w", (size_t)n * n);
  double* g1 = ws.get_f64("met_g1", (size_t)n * n);
  double* g2 = ws.get_f64("met_g2", (size_t)n * n);
  double* ones = ws.get_f64("met_ones", n);
  {
    std::vector<double> h(n, 1.0);
    EIGB_CUDA(cudaMemcpyAsync(ones, h.data(), 8 * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaStreamSynchronize(st));
  }
  const int blocks = (int)std::min<int64_t>(n, 4096);
  scale_cols_kernel<<<blocks, 256, 0, st>>>(qo, lo, n, w);
  EIGB_LAUNCH_CHECK();
  gemm_nt_dev(w, qo, n, n, n, g1, n, ones, nullptr, st);
  scale_cols_kernel<<<blocks, 256, 0, st>>>(q, lam, n, w);
  EIGB_LAUNCH_CHECK();
  gemm_nt_dev(w, q, n, n, n, g2, n, ones, nullptr, st);
  double* part = ws.get_f64("met_part", blocks);
  residual_kernel<<<blocks, 256, 0, st>>>(g1, g2, kmat, sgn, n, k, part);
  EIGB_LAUNCH_CHECK();
  std::vector<double> hp(blocks);
  EIGB_CUDA(cudaMemcpyAsync(hp.data(), part, 8 * blocks, cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaStreamSynchronize(st));
  double s = 0.0;
  for (double v : hp) s += v;
  *residual_fro = std::sqrt(s);
  // Q'^T Q' = T T^T with T = Q'^T
  dim3 tb(32, 8), tg((unsigned)cdiv(n, 32), (unsigned)cdiv(n, 32));
  transpose_kernel<<<tg, tb, 0, st>>>(qo, n, w);
  EIGB_LAUNCH_CHECK();
  gemm_nt_dev(w, w, n, n, n, g1, n, ones, nullptr, st);
  ortho_kernel<<<blocks, 256, 0, st>>>(g1, n, part);
  EIGB_LAUNCH_CHECK();
  EIGB_CUDA(cudaMemcpyAsync(hp.data(), part, 8 * blocks, cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaStreamSynchronize(st));
  double m = 0.0;
  for (double v : hp) m = std::max(m, v);
  *ortho_err = m;
}

}  // namespace eigb
