// Cost (cycles, one warp) of publishing a ~320-byte record to mapped host
// memory with different system-scope orderings before the `done` flag.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void pub(unsigned long long* rec, unsigned long long* done, long long* cyc, int reps) {
  const int lane = threadIdx.x;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int w = lane; w < 40; w += 32) rec[w] = r * 100 + w;
    if (MODE == 0) __threadfence_system();
    if (MODE == 1) asm volatile("fence.acq_rel.sys;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      if (MODE == 2)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(done), "l"((unsigned long long)r + 1) : "memory");
      else
        *reinterpret_cast<volatile unsigned long long*>(done) = r + 1;
    }
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) cyc[0] = (t1 - t0) / reps;
}
int main() {
  unsigned long long *h, *d;
  cudaHostAlloc(&h, 4096, cudaHostAllocMapped);
  cudaHostGetDevicePointer(&d, h, 0);
  long long* c;
  cudaMalloc(&c, 8);
  const char* nm[] = {"__threadfence_system (fence.sc.sys)", "fence.acq_rel.sys", "st.release.sys on done", "no fence"};
  for (int m = 0; m < 4; ++m) {
    for (int k = 0; k < 2; ++k) {
      if (m == 0) pub<0><<<1, 32>>>(d, d + 100, c, 50);
      if (m == 1) pub<1><<<1, 32>>>(d, d + 100, c, 50);
      if (m == 2) pub<2><<<1, 32>>>(d, d + 100, c, 50);
      if (m == 3) pub<3><<<1, 32>>>(d, d + 100, c, 50);
    }
    long long h2;
    cudaMemcpy(&h2, c, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %lld cycles per record\n", nm[m], h2);
  }
  return 0;
}
