// Device reconstruction of streamed slices from the streaming state, and the
// relative reconstruction error against given slices (
// reference reconstruct / relative_error, sthosvd.cpp:135-160, applied to
// StreamingState::full_model(), streaming.hpp:48-49).
//
// Slices [t0, t0 + count) of the model are
//   X_t = C x_0 U_0 ... x_{d-2} U_{d-2} x_{d-1} left[t, :]
// computed as Z = C_mat (n x r) * left[t0 : t0+count, :]^T (n x count), then
// one mode product per spatial mode (out[l, i, q] = sum_j U[i, j] Z[l, j, q]).
// These are verification / export paths, not the per-slice hot path, so the
// kernels are plain FP64 (one output element per thread, operands from L2).
#include "kernels.cuh"

namespace tsg {

namespace {

__global__ void recon_core_kernel(const double* __restrict__ core, long long n, int r,
                                  const double* __restrict__ left, int capr, long long t0,
                                  long long count, double* __restrict__ z) {
  const long long total = n * count;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx % n, c = idx / n;
    const double* lrow = left + (t0 + c) * capr;
    double s = 0.0;
    for (int j = 0; j < r; ++j) s = fma(core[i + (long long)j * n], lrow[j], s);
    z[idx] = s;
  }
}

// out (left, N, right) = U (N x R, column-major) applied along the middle
// mode of z (left, R, right).
__global__ void recon_expand_kernel(const double* __restrict__ z, long long left, int R,
                                    long long right, const double* __restrict__ u, long long N,
                                    double* __restrict__ out) {
  const long long total = left * N * right;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long l = idx % left;
    const long long rest = idx / left;
    const long long i = rest % N, q = rest / N;
    const double* zc = z + l + left * R * q;
    double s = 0.0;
    for (int j = 0; j < R; ++j) s = fma(u[i + (long long)j * N], zc[left * j], s);
    out[idx] = s;
  }
}

// Per-CTA partials of ||x - y||^2 and ||x||^2 (fixed order reduction later).
__global__ void diff_sumsq_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                  long long n, double* __restrict__ part) {
  __shared__ double red[32];
  double a = 0.0, b = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double xv = x[i], d = xv - y[i];
    a = fma(d, d, a);
    b = fma(xv, xv, b);
  }
  a = block_sum(a, red);
  b = block_sum(b, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

__global__ void pair_sum_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double red[32];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    a += part[2 * i];
    b += part[2 * i + 1];
  }
  a = block_sum(a, red);
  b = block_sum(b, red);
  if (threadIdx.x == 0) {
    out[0] = a;
    out[1] = b;
  }
}

int grid_of(long long n) {
  long long g = (n + 255) / 256;
  if (g > 8LL * kNumSMs) g = 8LL * kNumSMs;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

void launch_recon_core(const double* core, long long n, int r, const double* left, int capr,
                       long long t0, long long count, double* z, cudaStream_t st) {
  recon_core_kernel<<<grid_of(n * count), 256, 0, st>>>(core, n, r, left, capr, t0, count, z);
  ++g_launches;
}

void launch_recon_expand(const double* z, long long left, int R, long long right, const double* u,
                         long long N, double* out, cudaStream_t st) {
  recon_expand_kernel<<<grid_of(left * N * right), 256, 0, st>>>(z, left, R, right, u, N, out);
  ++g_launches;
}

void launch_diff_sumsq(const double* x, const double* y, long long n, double* part, double* out,
                       cudaStream_t st) {
  const int nb = 2 * kNumSMs;
  diff_sumsq_kernel<<<nb, 256, 0, st>>>(x, y, n, part);
  pair_sum_kernel<<<1, 256, 0, st>>>(part, nb, out);
  g_launches += 2;
}

}  // namespace tsg
