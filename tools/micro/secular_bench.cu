// Latency of the warp secular solver on an 11x11 ISVD-like problem
// (tools/micro, not shipped).
#include <cstdio>
#include <cuda_runtime.h>
#define SEC_CLK(i) \
  do { if (threadIdx.x == 0) g_clk[i] = clock64(); } while (0)
__device__ long long g_clk[16];
#include "../../paper_2308_16395_b200/csrc/secular.cuh"
using namespace tsg;

template <int KM>
__global__ void run(const double* d, const double* z, int m, double* lam_out, long long* cyc, int* its) {
  __shared__ double sd[32], sz[32], sQ[32 * 33], sx[8 * 32], lam[33], W[33 * 33], sW[32 * 33];
  __shared__ int si[96];
  const int lane = threadIdx.x;
  if (lane < m) { sd[lane] = d[lane]; sz[lane] = z[lane]; }
  __syncwarp();
  secular::Scratch S;
  S.sQ = sQ; S.dK = sx; S.wK = sx + 32; S.zK = sx + 64; S.ls = sx + 96; S.lt = sx + 128;
  S.zh = sx + 160; S.lamall = sx + 192; S.idx = si; S.perm = si + 32; S.flag = si + 64;
  long long t0 = clock64();
  int it = secular::eig_rank_one_fast<KM>(m, sd, sz, S, lam, W, sW);
  long long t1 = clock64();
  const long long cold = t1 - t0;
  t0 = clock64();
  it = secular::eig_rank_one_fast<KM>(m, sd, sz, S, lam, W, sW);
  t1 = clock64();
  if (lane == 0) cyc[39] = cold;
  if (lane < m) lam_out[lane] = lam[lane];
  if (lane == 0) { cyc[0] = t1 - t0; *its = it; }
  // per-lane root solve timing
  double dK[KM], wK[KM];
  for (int i = 0; i < KM; ++i) { dK[i] = i < m ? sd[i] : 1e300; wK[i] = i < m ? sz[i] * sz[i] : 0.0; }
  double wsum = 0; for (int i = 0; i < m; ++i) wsum += sz[i] * sz[i];
  __shared__ double sdk[32], swk[32];
  if (lane < m) { sdk[lane] = sd[lane]; swk[lane] = sz[lane] * sz[lane]; }
  __syncwarp();
  long long a = clock64();
  int o; double tau; int n_it = 0;
  if (lane < m) n_it = secular::solve_root_reg<KM>(dK, wK, sdk, swk, m, wsum, lane, o, tau);
  long long b = clock64();
  if (lane < m) { cyc[1 + lane] = b - a; its[1 + lane] = n_it; }
}

int main() {
  const int m = 11;
  double hd[m], hz[m];
  for (int i = 0; i < m - 1; ++i) { double s = 100.0 / (1 + i); hd[i] = s * s; hz[i] = 0.3 * s * ((i % 3) - 1.0 + 0.37); }
  hd[m - 1] = 0; hz[m - 1] = 0.5;
  double *d, *z, *lo; long long* cyc; int* its;
  cudaMalloc(&d, 8 * 32); cudaMalloc(&z, 8 * 32); cudaMalloc(&lo, 8 * 32); cudaMalloc(&cyc, 8 * 40); cudaMalloc(&its, 4 * 40);
  cudaMemcpy(d, hd, 8 * m, cudaMemcpyHostToDevice); cudaMemcpy(z, hz, 8 * m, cudaMemcpyHostToDevice);
  run<13><<<1, 32>>>(d, z, m, lo, cyc, its);
  long long hc[40]; int hi[40];
  cudaMemcpy(hc, cyc, 8 * 40, cudaMemcpyDeviceToHost); cudaMemcpy(hi, its, 4 * 40, cudaMemcpyDeviceToHost);
  long long hk[16]; cudaMemcpyFromSymbol(hk, g_clk, sizeof hk);
  printf("eig_rank_one_fast cold %lld cycles, hot %lld cycles, iters %d\n", hc[39], hc[0], hi[0]);
  printf("phases: roots %lld zhat %lld sort %lld vectors-to-end\n", hk[11] - hk[10], hk[12] - hk[11], hk[13] - hk[12]);
  for (int l = 0; l < m; ++l) printf("root %2d: %lld cycles, %d iters\n", l, hc[1 + l], hi[1 + l]);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
