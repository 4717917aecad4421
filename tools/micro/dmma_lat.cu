// DMMA (mma.sync.m8n8k4.f64) latency / throughput vs independent chains per warp and warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(int iters, double* out, long long* cyc) {
  double c[CH][2];
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int CH> void run(int warps, int blocks) {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8);
  const int iters = 2000;
  k<CH><<<blocks, 32 * warps>>>(iters, o, c);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<CH><<<blocks, 32 * warps>>>(iters, o, c);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  double dmmas = (double)iters * CH * warps * blocks;
  printf("chains/warp %2d warps/CTA %2d CTAs %4d : cycles per dependent DMMA (1 warp view) %.1f, TF/s %.1f\n",
         CH, warps, blocks, (double)cy / iters, dmmas * 512 / (ms * 1e-3) / 1e12);
}
int main() {
  run<1>(1, 1); run<2>(1, 1); run<4>(1, 1); run<8>(1, 1);
  run<1>(4, 148); run<2>(4, 148); run<4>(4, 148); run<8>(4, 148);
  run<1>(8, 148); run<2>(8, 148); run<4>(8, 148); run<8>(8, 148);
  run<4>(16, 148); run<2>(16, 148); run<1>(16, 148); run<1>(32, 148);
  return 0;
}
