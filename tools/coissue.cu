// Do DMMA (FP64 tensor pipe) and DFMA (FP64 pipe) issue concurrently on
// B200 (sm_100a)? VERDICT r1 next #4 asks before moving the K3 pole pass's
// FMA phase onto mma.sync.m8n8k4.f64. Four measurements, all on every SM:
//   dfma     DFMA loop alone                      (FP64 pipe ceiling)
//   dmma     DMMA.8x8x4 loop alone                (tensor pipe ceiling)
//   split    half the warps DFMA, half DMMA       (pipes shared by the SM)
//   mixed    each warp interleaves both           (same warp, both pipes)
// If the pipes are separate, split/mixed reach ~ dfma + dmma.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/coissue tools/coissue.cu
#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);             \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// mode 0 dfma, 1 dmma, 2 split by warp parity, 3 mixed in every warp.
// Per iteration: FCH independent DFMA chains, MCH independent DMMA chains.
template <int FCH, int MCH, int MODE>
__global__ void loop(double* out, int iters, double a, double b) {
  constexpr int mode = MODE;
  double f[FCH], c[MCH][2];
#pragma unroll
  for (int i = 0; i < FCH; ++i) f[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < MCH; ++i) c[i][0] = c[i][1] = 0.0;
  const int warp = threadIdx.x >> 5;
  const double A = a + threadIdx.x, B = b - threadIdx.x;
  // mode 2: the warp's role is uniform, and each role has its own loop (no
  // predicated-off instructions of the other kind in either)
  const bool f_warp = mode == 0 || (mode == 2 && (warp & 1) == 0);
  const bool m_warp = mode == 1 || (mode == 2 && (warp & 1) == 1);
  if (mode == 3) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < MCH; ++i) dmma(c[i][0], c[i][1], A, B);
#pragma unroll
      for (int i = 0; i < FCH; ++i) f[i] = fma(f[i], a, b);
    }
  } else if (m_warp) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < MCH; ++i) dmma(c[i][0], c[i][1], A, B);
    }
  } else if (f_warp) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < FCH; ++i) f[i] = fma(f[i], a, b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < FCH; ++i) s += f[i];
#pragma unroll
  for (int i = 0; i < MCH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  constexpr int FCH = 8, MCH = 4;
  const int iters = 8000, threads = 256;
  printf("{\"sms\": %d", sms);
  const char* names[] = {"dfma", "dmma", "split", "mixed"};
  for (int bpsm : {2, 4, 8}) {
    const int blocks = sms * bpsm;
    for (int mode = 0; mode < 4; ++mode) {
      auto run = [&] {
        if (mode == 0) loop<FCH, MCH, 0><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
        if (mode == 1) loop<FCH, MCH, 1><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
        if (mode == 2) loop<FCH, MCH, 2><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
        if (mode == 3) loop<FCH, MCH, 3><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
      };
      run();
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0));
        run();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
      }
      const double warps = (double)blocks * threads / 32;
      const double fw = mode == 0 || mode == 3 ? warps : (mode == 2 ? warps / 2 : 0);
      const double mw = mode == 1 || mode == 3 ? warps : (mode == 2 ? warps / 2 : 0);
      const double ff = fw * 32 * 2.0 * FCH * iters;       // DFMA flops
      const double fm = mw * 2.0 * 8 * 8 * 4 * MCH * iters;  // DMMA flops
      printf(", \"%s_b%d\": {\"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"total\": %.2f}",
             names[mode], bpsm, ff / best / 1e9, fm / best / 1e9, (ff + fm) / best / 1e9);
    }
  }
  printf("}\n");
  return 0;
}
