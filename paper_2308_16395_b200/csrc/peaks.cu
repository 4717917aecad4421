// FP64 throughput microbenchmarks: the FP64 tensor pipe (DMMA via
// mma.sync.m8n8k4.f64) and the FP64 FMA pipe (DFMA). MEASURED_PEAKS.json
// carries only HBM and bf16 figures; the FP64 roofline denominator of the
// projection kernels is measured here on the same box.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace tsg {
namespace {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) dmma_peak_kernel(int iters, double* out) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma884(c[2 * i], c[2 * i + 1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;  // keep the work alive
}

__global__ void __launch_bounds__(256) dfma_peak_kernel(int iters, double* out) {
  double x[8];
  const double a = 1.0 + threadIdx.x * 1e-12, b = 1e-12;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

}  // namespace

// Returns TFLOP/s for the DMMA and DFMA pipes (best of 3 launches).
int measure_fp64_peaks(int device, double* dmma_tflops, double* dfma_tflops) {
  if (cudaSetDevice(device) != cudaSuccess) return 4;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  if (cudaMalloc(&out, 8) != cudaSuccess) return 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 256, iters = 4096;
  double best_m = 0.0, best_f = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    dmma_peak_kernel<<<blocks, threads>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 256.0 * 8.0 * iters * (blocks * threads / 32.0);
    if (rep > 0) best_m = fmax(best_m, flops / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0);
    dfma_peak_kernel<<<blocks, threads>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fflops = 2.0 * 8.0 * iters * (double)blocks * threads;
    if (rep > 0) best_f = fmax(best_f, fflops / (ms * 1e-3) / 1e12);
  }
  g_launches += 8;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  *dmma_tflops = best_m;
  *dfma_tflops = best_f;
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // namespace tsg
