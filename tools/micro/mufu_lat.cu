// Dependent latency (1 warp) of the FP64 special-function approximations and
// of the Newton-refined reciprocal used by the insertion kernels.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcpa(double x) { double y; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }
__device__ __forceinline__ double rsqa(double x) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }
__device__ __forceinline__ double rcpn(double x) { double y = rcpa(x); double e = fma(-x, y, 1.0); y = fma(y, e, y); e = fma(-x, y, 1.0); return fma(y, e, y); }
template <int mode>
__global__ void k(int iters, double* out, long long* cyc) {
  double x = 1.000001 + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode == 0) x = rcpa(x) + 0.5;
    else if (mode == 1) x = rsqa(x) + 0.5;
    else if (mode == 2) x = rcpn(x) + 0.5;
    else if (mode == 3) x = 1.0 / x + 0.5;
    else if (mode == 4) x = sqrt(x) + 0.5;
    else x = fma(x, 0.999, 0.5);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 32); cudaMalloc(&c, 8);
  const char* names[] = {"rcp.approx.f64 + add", "rsqrt.approx.f64 + add", "rcp (approx+2 Newton) + add", "IEEE 1/x + add", "IEEE sqrt + add", "DFMA"};
  for (int m = 0; m < 6; ++m) {
    auto go = [&] {
      switch (m) {
        case 0: k<0><<<1, 32>>>(1000, o, c); break;
        case 1: k<1><<<1, 32>>>(1000, o, c); break;
        case 2: k<2><<<1, 32>>>(1000, o, c); break;
        case 3: k<3><<<1, 32>>>(1000, o, c); break;
        case 4: k<4><<<1, 32>>>(1000, o, c); break;
        default: k<5><<<1, 32>>>(1000, o, c); break;
      }
    };
    go(); go();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-30s %.1f cycles per dependent step\n", names[m], h / 1000.0);
  }
  return 0;
}
