// Stand-alone timing of the fused tail kernel on C2-shaped inputs
// (tools/micro, not shipped): nvcc -I paper_2308_16395_b200/csrc ...
#include <cstdio>
#include <vector>

#include "../../paper_2308_16395_b200/csrc/tail.cu"

namespace tsg {
long long g_launches = 0;
}
using namespace tsg;

int main(int argc, char** argv) {
  const int N1 = 200, N2 = 200, R0 = 10, R1 = 10, R2 = 10;
  const long long xin = (long long)R0 * N1 * N2;
  double *x, *o1, *o2, *u1, *u2, *part, *pp;
  cudaMalloc(&x, xin * 8);
  cudaMalloc(&o1, xin * 8);
  cudaMalloc(&o2, xin * 8);
  cudaMalloc(&u1, N1 * R1 * 8);
  cudaMalloc(&u2, N2 * R2 * 8);
  cudaMalloc(&part, 4096 * 8);
  cudaMalloc(&pp, 4096 * 8);
  std::vector<double> h(xin);
  for (long long i = 0; i < xin; ++i) h[i] = (double)((i * 7919) % 1000) / 1000.0;
  cudaMemcpy(x, h.data(), xin * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(u1, h.data(), N1 * R1 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(u2, h.data() + 5000, N2 * R2 * 8, cudaMemcpyHostToDevice);
  cudaMemset(pp, 0, 4096 * 8);
  SliceCtl* slot;
  cudaMalloc(&slot, sizeof(SliceCtl) * 2);
  unsigned long long* clk;
  cudaMalloc(&clk, 17 * kMaxGrid * 8);
  cudaMemset(clk, 0, 17 * kMaxGrid * 8);
  TailArgs t;
  memset(&t, 0, sizeof t);
  t.x = x;
  t.out[1] = o1;
  t.out[2] = o2;
  t.u[1] = u1;
  t.u[2] = u2;
  t.N[1] = N1;
  t.N[2] = N2;
  t.R[1] = R1;
  t.R[2] = R2;
  t.left[1] = R0;
  t.right[1] = N2;
  t.left[2] = R0 * R1;
  t.right[2] = 1;
  t.m0 = 1;
  t.m1 = 3;
  t.part = part;
  unsigned* done;
  cudaMalloc(&done, 8);
  cudaMemset(done, 0, 8);
  t.done = done;
  t.da.slot = slot;
  t.da.partial = pp;
  t.da.off[0] = 0;
  t.da.cnt[0] = 296;
  t.da.nmodes = 3;
  t.da.first_mode = 0;
  t.da.tau = 1e-2;
  t.da.order = 4;
  cudaStream_t st;
  cudaStreamCreate(&st);
  int g = launch_tail(t, st);
  printf("grid %d status %s\n", g, cudaGetErrorString(cudaStreamSynchronize(st)));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 20; ++i) launch_tail(t, st);
  cudaEventRecord(a, st);
  for (int i = 0; i < 200; ++i) launch_tail(t, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("tail kernel back-to-back: %.2f us/launch\n", ms * 1000 / 200);
  t.clk = clk;
  launch_tail(t, st);
  cudaStreamSynchronize(st);
  std::vector<unsigned long long> c(16 * kMaxGrid);
  cudaMemcpy(c.data(), clk, c.size() * 8, cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ULL;
  for (int bb = 0; bb < g; ++bb) t0 = std::min(t0, c[bb * 16]);
  for (int i = 0; i < 16; ++i) {
    unsigned long long lo = ~0ULL, hi = 0;
    for (int bb = 0; bb < g; ++bb)
      if (c[bb * 16 + i] >= t0) {
        lo = std::min(lo, c[bb * 16 + i]);
        hi = std::max(hi, c[bb * 16 + i]);
      }
    if (hi) printf("stamp %2d: %7.2f .. %7.2f us\n", i, (lo - t0) * 1e-3, (hi - t0) * 1e-3);
  }
  std::vector<long long> cc(16);
  cudaMemcpy(cc.data(), clk + 16 * kMaxGrid, 128, cudaMemcpyDeviceToHost);
  printf("fibre cycles: load %lld  phase1 %lld  reduce %lld  phase2 %lld\n", cc[5] - cc[4], cc[6] - cc[5],
         cc[7] - cc[6], cc[8] - cc[7]);
  printf("last-CTA cycles: arrive %lld  reduce %lld  decide %lld\n", cc[1] - cc[0], cc[2] - cc[1],
         cc[3] - cc[2]);
  return 0;
}
