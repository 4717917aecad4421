// Issue cost (cycles per warp instruction, 16 independent chains per lane)
// of FP64 reciprocal variants (tools/micro, not shipped).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp64h(double x) {
  double y;
  asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
template <int OP>
__global__ void k(double* out, long long* cyc) {
  double x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = 1.5 + threadIdx.x * 1e-6 + j * 1e-3;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (OP == 0) x[j] = rcp64h(x[j]) + 0.5;
      if (OP == 1) x[j] = (double)__frcp_rn((float)x[j]) + 0.5;
      if (OP == 2) x[j] = fma(x[j], 0.999, 0.001);
      if (OP == 3) x[j] = sqrt(x[j]) + 0.5;
      if (OP == 4) x[j] = 1.0 / x[j] + 0.5;
      if (OP == 5) x[j] = (double)((float)x[j]) + 0.5;
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += x[j];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[OP] = (t1 - t0);
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64 * 8);
  k<0><<<1, 32>>>(o, c); k<1><<<1, 32>>>(o, c); k<2><<<1, 32>>>(o, c);
  k<3><<<1, 32>>>(o, c); k<4><<<1, 32>>>(o, c); k<5><<<1, 32>>>(o, c);
  long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
  const char* n[6] = {"rcp.approx.f64+add", "f32 rcp via cvt +add", "dfma", "sqrt+add", "div+add", "cvt f64>f32>f64 +add"};
  for (int i = 0; i < 6; ++i) printf("%-22s %.1f cycles per (16 ops)/lane step -> %.2f per op\n", n[i], h[i] / 64.0, h[i] / 64.0 / 16);
  return 0;
}
