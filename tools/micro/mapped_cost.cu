// Cost of publishing small records to host-mapped memory from a kernel, and
// of reading a host-mapped word from many CTAs (tools/micro, not shipped).
#include <cstdio>
#include <ctime>
int graph_costs();
#include <cuda_runtime.h>

struct Rec { double v[48]; };

__global__ void k_empty() {}
__global__ void k_scalar(Rec* h, int fence) {
  if (threadIdx.x) return;
  for (int i = 0; i < 48; ++i) h->v[i] = i;
  if (fence) __threadfence_system();
}
__global__ void k_vec(Rec* h, int fence) {
  if (threadIdx.x < 24) reinterpret_cast<double2*>(h->v)[threadIdx.x] = make_double2(1, 2);
  if (fence) __threadfence_system();
}
__global__ void k_release(Rec* h, unsigned long long* flag) {
  if (threadIdx.x < 24) reinterpret_cast<double2*>(h->v)[threadIdx.x] = make_double2(1, 2);
  __syncwarp();
  if (threadIdx.x == 0) {
    unsigned long long v = 1;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(v) : "memory");
  }
}
__global__ void k_dev_then_fence(Rec* d) {
  if (threadIdx.x < 24) reinterpret_cast<double2*>(d->v)[threadIdx.x] = make_double2(1, 2);
  __threadfence();
}
__global__ void k_read_volatile(const double* const* p, double* sink) {
  __shared__ const double* s;
  if (threadIdx.x == 0) s = *reinterpret_cast<const double* const volatile*>(p);
  __syncthreads();
  if (threadIdx.x == 0 && s == nullptr) sink[blockIdx.x] = 1;
}
__global__ void k_read_plain(const double* const* p, double* sink) {
  __shared__ const double* s;
  if (threadIdx.x == 0) s = *p;
  __syncthreads();
  if (threadIdx.x == 0 && s == nullptr) sink[blockIdx.x] = 1;
}

template <class F>
float timeit(F f, int n = 200) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 10; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < n; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return 1000.f * ms / n;
}

int main() {
  Rec* h;
  cudaHostAlloc(&h, sizeof(Rec) + 64, cudaHostAllocMapped);
  Rec* hd;
  cudaHostGetDevicePointer((void**)&hd, h, 0);
  unsigned long long* flag = reinterpret_cast<unsigned long long*>(hd + 1);
  Rec* dev;
  cudaMalloc(&dev, sizeof(Rec));
  const double** ph;
  cudaHostAlloc(&ph, 64, cudaHostAllocMapped);
  ph[0] = reinterpret_cast<const double*>(dev);
  const double* const* pd;
  cudaHostGetDevicePointer((void**)&pd, ph, 0);
  const double** pdev;
  cudaMalloc(&pdev, 64);
  cudaMemcpy(pdev, ph, 8, cudaMemcpyHostToDevice);
  double* sink;
  cudaMalloc(&sink, 4096 * 8);
  printf("empty                 %.2f us\n", timeit([&] { k_empty<<<1, 32>>>(); }));
  printf("scalar 48 no fence    %.2f us\n", timeit([&] { k_scalar<<<1, 32>>>(hd, 0); }));
  printf("scalar 48 + fence.sys %.2f us\n", timeit([&] { k_scalar<<<1, 32>>>(hd, 1); }));
  printf("vec 24x16B no fence   %.2f us\n", timeit([&] { k_vec<<<1, 32>>>(hd, 0); }));
  printf("vec 24x16B + fence    %.2f us\n", timeit([&] { k_vec<<<1, 32>>>(hd, 1); }));
  printf("vec + st.release.sys  %.2f us\n", timeit([&] { k_release<<<1, 32>>>(hd, flag); }));
  printf("device vec + fence.gpu%.2f us\n", timeit([&] { k_dev_then_fence<<<1, 32>>>(dev); }));
  for (int g : {1, 16, 148, 296}) {
    printf("read host volatile  grid %3d  %.2f us\n", g,
           timeit([&] { k_read_volatile<<<g, 256>>>(pd, sink); }));
    printf("read host plain     grid %3d  %.2f us\n", g,
           timeit([&] { k_read_plain<<<g, 256>>>(pd, sink); }));
    printf("read device volatile grid %3d %.2f us\n", g,
           timeit([&] { k_read_volatile<<<g, 256>>>(pdev, sink); }));
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return graph_costs();
}

// ---- host cost of graph launch and kernel-node parameter update
struct Big { const double* x; double pad[40]; };
__global__ void k_args(Big b, double* sink) { if (threadIdx.x == 0 && b.x == nullptr) sink[0] = 1; }

int graph_costs() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  double* sink;
  cudaMalloc(&sink, 64);
  Big b{};
  b.x = sink;
  cudaGraph_t g;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
  k_args<<<1, 32, 0, s>>>(b, sink);
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  cudaStreamGetCaptureInfo(s, &cs, nullptr, nullptr, &deps, &nd);
  cudaGraphNode_t node = nd ? deps[0] : nullptr;
  for (int i = 0; i < 5; ++i) k_args<<<1, 32, 0, s>>>(b, sink);
  cudaStreamEndCapture(s, &g);
  cudaGraphExec_t ex;
  cudaGraphInstantiate(&ex, g, 0);
  cudaKernelNodeParams kp;
  cudaGraphKernelNodeGetParams(node, &kp);
  auto now = [] { timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec * 1e6 + t.tv_nsec * 1e-3; };
  for (int i = 0; i < 50; ++i) cudaGraphLaunch(ex, s);
  cudaStreamSynchronize(s);
  double t0 = now();
  for (int i = 0; i < 1000; ++i) cudaGraphLaunch(ex, s);
  double t1 = now();
  cudaStreamSynchronize(s);
  printf("graph launch (6 kernels) host %.2f us\n", (t1 - t0) / 1000);
  Big nb = b;
  void* args[2] = {&nb, &sink};
  kp.kernelParams = args;
  t0 = now();
  for (int i = 0; i < 1000; ++i) {
    nb.x = sink + (i & 1);
    cudaGraphExecKernelNodeSetParams(ex, node, &kp);
  }
  t1 = now();
  printf("exec kernel node set params host %.2f us (node %p)\n", (t1 - t0) / 1000, (void*)node);
  t0 = now();
  for (int i = 0; i < 1000; ++i) {
    nb.x = sink + (i & 1);
    cudaGraphExecKernelNodeSetParams(ex, node, &kp);
    cudaGraphLaunch(ex, s);
  }
  t1 = now();
  cudaStreamSynchronize(s);
  printf("set params + launch host %.2f us\n", (t1 - t0) / 1000);
  t0 = now();
  for (int i = 0; i < 1000; ++i) k_args<<<1, 32, 0, s>>>(b, sink);
  t1 = now();
  cudaStreamSynchronize(s);
  printf("plain kernel launch host %.2f us\n", (t1 - t0) / 1000);
  cudaEvent_t e;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  t0 = now();
  for (int i = 0; i < 1000; ++i) cudaEventRecord(e, s);
  t1 = now();
  printf("event record host %.2f us\n", (t1 - t0) / 1000);
  t0 = now();
  for (int i = 0; i < 1000; ++i) cudaStreamQuery(s);
  t1 = now();
  printf("stream query host %.2f us\n", (t1 - t0) / 1000);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
