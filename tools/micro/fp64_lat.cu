// Dependent-chain latency of FP64 ops on this GPU (tools/micro, not shipped).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
template <int OP>
__global__ void k(double* out, long long* cyc, double seed) {
  double x = seed + threadIdx.x * 1e-9;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
    if (OP == 0) x = fma(x, 0.999999, 1e-7);
    if (OP == 1) x = x + 1e-9;
    if (OP == 2) x = sqrt(x) + 1.0;
    if (OP == 3) x = 1.0 / x + 1.0;
    if (OP == 4) x = rcp_nr(x) + 1.0;
    if (OP == 5) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-9;
    if (OP == 6) { double y; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y + 1.0; }
    if (OP == 7) x = __dmul_rn(x, 1.0000001);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[OP] = (t1 - t0) / 256;
  out[threadIdx.x] = x;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64 * 8);
  k<0><<<1, 32>>>(o, c, 1.5); k<1><<<1, 32>>>(o, c, 1.5); k<2><<<1, 32>>>(o, c, 1.5);
  k<3><<<1, 32>>>(o, c, 1.5); k<4><<<1, 32>>>(o, c, 1.5); k<5><<<1, 32>>>(o, c, 1.5);
  k<6><<<1, 32>>>(o, c, 1.5); k<7><<<1, 32>>>(o, c, 1.5);
  long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
  const char* n[8] = {"dfma", "dadd", "sqrt+add", "div+add", "rcp_nr+add", "shfl64+dadd", "rcp.approx+add", "dmul"};
  for (int i = 0; i < 8; ++i) printf("%-16s %lld cycles/iter\n", n[i], h[i]);
  return 0;
}
