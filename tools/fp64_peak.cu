// FP64 ceiling probe for B200 (sm_100a): DFMA pipe, DMMA.8x8x4 tensor pipe,
// MUFU.RCP64H-based reciprocal, and cuBLAS DGEMM. These numbers are the FP64
// roofline denominators DESIGN.md reports against (MEASURED_PEAKS.json has no
// FP64 entry). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lcublas
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cublas_v2.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int CH>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dmma_loop(double* out, int iters, double av, double bv) {
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double A = av + threadIdx.x, B = bv - threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(A), "d"(B));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

template <int CH>
__global__ void rcp_loop(double* out, int iters) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = 1.5 + threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = fast_rcp(acc[i]) + 1.25;
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void fill(double* p, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)i * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = (x & 0xffffff) * (1.0 / 16777216.0) - 0.5;
  }
}

template <class F>
float time_ms(F f, int reps = 5) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 1 << 20));
  const int iters = 20000;
  printf("{\"sms\": %d", sms);
  for (int bpsm : {2, 4, 8}) {
    const int threads = 256, blocks = sms * bpsm;
    float ms = time_ms([&] { dfma_loop<8><<<blocks, threads>>>(out, iters, 0.999, 1e-3); });
    double fl = 2.0 * 8 * iters * (double)threads * blocks;
    printf(", \"dfma_tflops_b%d\": %.2f", bpsm, fl / ms / 1e9);
  }
  for (int bpsm : {1, 2, 4, 8}) {
    const int threads = 128, blocks = sms * bpsm;
    float ms = time_ms([&] { dmma_loop<8><<<blocks, threads>>>(out, iters / 4, 1e-3, 2e-3); });
    double fl = 2.0 * 256 * 8 * (iters / 4) * (double)(threads / 32) * blocks;
    printf(", \"dmma_tflops_w%d\": %.2f", bpsm * 4, fl / ms / 1e9);
  }
  {
    const int threads = 256, blocks = sms * 4;
    float ms = time_ms([&] { rcp_loop<4><<<blocks, threads>>>(out, iters / 4); });
    double n = 4.0 * (iters / 4) * (double)threads * blocks;
    printf(", \"rcp_per_clk_sm_equiv_Grcp_s\": %.1f", n / ms / 1e6);
  }
  cublasHandle_t h;
  cublasCreate(&h);
  for (int n : {4096, 8192, 16384}) {
    double *A, *B, *C;
    size_t bytes = (size_t)n * n * sizeof(double);
    CK(cudaMalloc(&A, bytes));
    CK(cudaMalloc(&B, bytes));
    CK(cudaMalloc(&C, bytes));
    fill<<<1024, 256>>>(A, (size_t)n * n, 1u);
    fill<<<1024, 256>>>(B, (size_t)n * n, 2u);
    double one = 1.0, zero = 0.0;
    float ms = time_ms([&] {
      cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
    }, 3);
    printf(", \"cublas_dgemm_%d_tflops\": %.2f", n, 2.0 * n * (double)n * n / ms / 1e9);
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf(", \"clock_khz_attr\": %d}\n", clk);
  return 0;
}
