// DMMA (mma.sync.m8n8k4.f64) and DFMA co-issue: do the FP64 tensor pipe and
// the FP64 FMA pipe run concurrently? Prints TF/s for DMMA only, DFMA only and
// interleaved mixes (per warp: ND DMMAs and NF DFMA instructions per loop).
// Also the single-warp dependent latency of DMMA and DFMA.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int ND, int NF>
__global__ void k(int iters, double* out) {
  double c[ND > 0 ? ND : 1][2];
  double f[NF > 0 ? NF : 1];
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) c[i][0] = c[i][1] = 0;
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) f[i] = threadIdx.x * 1e-3 + i;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < (ND > NF ? ND : NF); ++i) {
      if (i < ND) dmma(c[i][0], c[i][1], a, b);
      if (i < NF) f[i] = fma(f[i], a, b);
    }
  }
  double s = 0;
  for (int i = 0; i < ND; ++i) s += c[i][0] + c[i][1];
  for (int i = 0; i < NF; ++i) s += f[i];
  if (s == 1.2345) out[0] = s;
}
template <int ND, int NF>
void run(int warps, int blocks) {
  double* o;
  cudaMalloc(&o, 8);
  const int iters = 4000;
  k<ND, NF><<<blocks, 32 * warps>>>(iters, o);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<ND, NF><<<blocks, 32 * warps>>>(iters, o);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double thr = (double)iters * warps * blocks;
  const double fd = thr * ND * 512, ff = thr * NF * 64;
  printf("DMMA/warp-iter %2d DFMA/warp-iter %2d warps %2d CTAs %4d : %.3f ms  DMMA %.1f TF  DFMA %.1f TF  total %.1f TF\n",
         ND, NF, warps, blocks, ms, fd / (ms * 1e-3) / 1e12, ff / (ms * 1e-3) / 1e12,
         (fd + ff) / (ms * 1e-3) / 1e12);
  cudaFree(o);
}
template <int CH>
__global__ void lat(int iters, double* out, long long* cyc, int mode) {
  double c[CH][2];
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = threadIdx.x;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0;
  long long t0 = clock64();
  if (mode == 0) {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], a, b);
  } else {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < CH; ++i) c[i][0] = fma(c[i][0], a, b);
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int CH>
void runlat(int mode) {
  double* o;
  long long* c;
  cudaMalloc(&o, 8);
  cudaMalloc(&c, 8);
  lat<CH><<<1, 32>>>(1000, o, c, mode);
  lat<CH><<<1, 32>>>(1000, o, c, mode);
  long long cy;
  cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  printf("%s chains %d: %.1f cycles per iteration (1 warp)\n", mode ? "DFMA" : "DMMA", CH, cy / 1000.0);
}

// DMMA with distinct A/B registers per instruction (no operand reuse)
template <int CH>
__global__ void kv(int iters, double* out) {
  double c[CH][2];
  double av[CH], bv[CH];
  for (int i = 0; i < CH; ++i) { c[i][0] = c[i][1] = 0; av[i] = 1.0 + threadIdx.x * 1e-9 * i; bv[i] = 1.0 - i * 1e-9; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], av[i], bv[(i + it) % CH]);
  }
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
// DMMA with B operands from shared memory (one LDS.64 per DMMA)
template <int CH>
__global__ void ks(int iters, double* out) {
  __shared__ double sb[64 * 32];
  for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) sb[i] = 1.0 + i * 1e-12;
  __syncthreads();
  double c[CH][2];
  double av[CH];
  for (int i = 0; i < CH; ++i) { c[i][0] = c[i][1] = 0; av[i] = 1.0 + threadIdx.x * 1e-9 * i; }
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], av[i], sb[((it * CH + i) & 63) * 32 + lane]);
  }
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
template <int CH, int V>
void runv(int warps, int blocks) {
  double* o;
  cudaMalloc(&o, 8);
  const int iters = 4000;
  auto go = [&] { if (V == 0) kv<CH><<<blocks, 32 * warps>>>(iters, o); else ks<CH><<<blocks, 32 * warps>>>(iters, o); };
  go();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  go();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fd = (double)iters * warps * blocks * CH * 512;
  printf("%s chains %d warps %2d: DMMA %.1f TF\n", V == 0 ? "distinct-reg" : "smem-B", CH, warps, fd / (ms * 1e-3) / 1e12);
  cudaFree(o);
}
int main2() {
  for (int w : {4, 8, 12, 16}) { runv<8, 0>(w, 148); runv<8, 1>(w, 148); runv<4, 1>(w, 148); }
  return 0;
}
int main() {
  main2();
  runlat<1>(0); runlat<2>(0); runlat<4>(0); runlat<8>(0);
  runlat<1>(1); runlat<4>(1); runlat<8>(1);
  for (int w : {4, 8, 16}) {
    run<8, 0>(w, 148);
    run<0, 8>(w, 148);
    run<8, 8>(w, 148);
    run<4, 8>(w, 148);
    run<2, 8>(w, 148);
    run<8, 16>(w, 148);
    run<4, 16>(w, 148);
  }
  return 0;
}
