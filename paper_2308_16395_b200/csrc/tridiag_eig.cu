// Leading eigenpairs of a symmetric Gram matrix through a tridiagonal form:
// the basis-growth / stream_init eigensolve for n >= 96 (mode_subspace,
// sthosvd.cpp:61-75, which calls sym_eig_desc, linalg.cpp:120-181).
//
// The reference runs cyclic Jacobi on the n x n Gram matrix and keeps the
// leading `rank` eigenvectors. The cooperative Jacobi here needs one grid
// barrier per rotation round, ~8 sweeps x (n-1) rounds: 23 ms at n = 384,
// the dominant term of every basis growth of configs 4 and 5. mode_subspace
// only consumes (a) all eigenvalues, for the truncation rule, and (b) the
// leading `rank` eigenvectors, so this route computes exactly that:
//
//   1. tridiag_coop_kernel   Householder tridiagonalisation T = Q^T G Q on a
//      cooperative grid: ONE grid barrier per column. The rank-2 update of
//      step k-1 is applied lazily inside the symmetric matrix-vector product
//      of step k (one pass over the L2-resident trailing block per step);
//      reflector and scalars are recomputed redundantly per CTA.
//   2. tri_bisect_kernel     all eigenvalues of T by Sturm-count multisection
//      (one warp per eigenvalue, 32 shifts per pass, ~12 passes).
//   3. tri_invit_kernel      eigenvectors of T for the leading `rank`
//      eigenvalues by inverse iteration (partial-pivoting tridiagonal LU,
//      random start, rescaled iterations); eigenvalues closer than
//      1e-3 ||T|| form a cluster handled by one CTA with modified
//      Gram-Schmidt against the cluster's earlier vectors (LAPACK dstein's
//      published scheme, restated).
//   4. tri_backtransform_kernel   z <- H_0 .. H_{n-3} z per retained vector,
//      then the reference's sign rule (linalg.cpp:170-178).
//
// Differences from the reference's Jacobi are rounding-level times the
// conditioning of the retained eigenvectors (backward error ~ eps ||G||, as
// for Jacobi stopped at off <= 1e-14 ||G||, linalg.cpp:13); eigenvalues are
// clamped at zero and sorted descending as sym_eig_desc does.
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "kernels.cuh"

namespace tsg {
namespace {

namespace cg = cooperative_groups;

constexpr int kTriThreads = 256;
constexpr double kEps = 2.220446049250313e-16;

// work layout (doubles): A n^2 | Vh n^2 | p 2n | d n | e n | beta n | lam n | Z n*rank
struct TriWork {
  double *A, *Vh, *p, *d, *e, *beta, *lam, *Z;
};
__host__ __device__ inline TriWork tri_work(double* w, int n) {
  TriWork t;
  const long long nn = (long long)n * n;
  t.A = w;
  t.Vh = w + nn;
  t.p = w + 2 * nn;
  t.d = t.p + 2 * n;
  t.e = t.d + n;
  t.beta = t.e + n;
  t.lam = t.beta + n;
  t.Z = t.lam + n;
  return t;
}

__global__ void __launch_bounds__(kTriThreads) tridiag_coop_kernel(const double* __restrict__ gin,
                                                                   int n, double* work) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  __shared__ double red[32];
  double* v = sm;
  double* w = sm + n;
  double* vp = sm + 2 * n;
  double* wp = sm + 3 * n;
  const TriWork W = tri_work(work, n);
  double* A = W.A;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nwarps = (int)gridDim.x * (kTriThreads / 32);
  const int gw = (int)blockIdx.x * (kTriThreads / 32) + wid;
  const long long nn = (long long)n * n;
  for (long long idx = blockIdx.x * (long long)kTriThreads + tid; idx < nn;
       idx += (long long)gridDim.x * kTriThreads) {
    A[idx] = gin[idx];
    W.Vh[idx] = 0.0;
  }
  for (int i = tid; i < n; i += kTriThreads) vp[i] = wp[i] = v[i] = w[i] = 0.0;
  grid.sync();
  for (int k = 0; k + 2 < n; ++k) {
    // true column k (pending rank-2 update of step k-1 applied), rows >= k
    const double vpk = vp[k], wpk = wp[k];
    double x2 = 0.0;
    for (int i = k + tid; i < n; i += kTriThreads) {
      const double a = A[i + (long long)k * n] - vp[i] * wpk - wp[i] * vpk;
      v[i] = a;
      if (i > k) x2 += a * a;
    }
    const double sigma2 = block_sum(x2, red);  // barriers inside publish v[]
    const double dk = v[k], x0 = v[k + 1];
    const double sigma = sqrt(sigma2);
    double alpha = 0.0, b = 0.0;
    if (sigma > 0.0) {
      alpha = x0 >= 0.0 ? -sigma : sigma;
      b = 1.0 / (sigma * (sigma + fabs(x0)));
    }
    __syncthreads();
    for (int i = tid; i <= k + 1; i += kTriThreads) v[i] = (i == k + 1) ? x0 - alpha : 0.0;
    __syncthreads();
    if (blockIdx.x == 0) {
      if (tid == 0) {
        W.d[k] = dk;
        W.e[k] = alpha;
        W.beta[k] = b;
      }
      for (int i = k + 1 + tid; i < n; i += kTriThreads) W.Vh[i + (long long)k * n] = v[i];
    }
    // owned columns of the trailing block: apply the pending update, store,
    // and accumulate p = b A v in the same pass
    double* pk = W.p + (k & 1) * n;
    for (int j = k + 1 + gw; j < n; j += nwarps) {
      const double vpj = vp[j], wpj = wp[j];
      double acc = 0.0;
      for (int i = k + 1 + lane; i < n; i += 32) {
        const double a = A[i + (long long)j * n] - vp[i] * wpj - wp[i] * vpj;
        A[i + (long long)j * n] = a;
        acc += a * v[i];
      }
      acc = warp_sum(acc);
      if (lane == 0) pk[j] = b * acc;
    }
    grid.sync();
    // w = p - (b p^T v / 2) v, redundantly per CTA
    double g = 0.0;
    for (int i = k + 1 + tid; i < n; i += kTriThreads) {
      const double pi = pk[i];
      w[i] = pi;
      g += pi * v[i];
    }
    const double gamma = block_sum(g, red);
    const double coef = 0.5 * b * gamma;
    for (int i = tid; i < n; i += kTriThreads) w[i] = i > k ? w[i] - coef * v[i] : 0.0;
    __syncthreads();
    double* t = v;
    v = vp;
    vp = t;
    t = w;
    w = wp;
    wp = t;
  }
  if (blockIdx.x == 0 && tid == 0) {
    if (n == 1) {
      W.d[0] = A[0];
    } else {
      const int i0 = n - 2, i1 = n - 1;
      auto at = [&](int i, int j) {
        return A[i + (long long)j * n] - vp[i] * wp[j] - wp[i] * vp[j];
      };
      W.d[i0] = at(i0, i0);
      W.e[i0] = at(i1, i0);
      W.d[i1] = at(i1, i1);
      W.beta[i0] = 0.0;
    }
    W.e[n - 1] = 0.0;
    W.beta[n - 1] = 0.0;
  }
}

// Eigenvalues below x of the tridiagonal (sd, se2 = e^2), Sturm count.
__device__ __forceinline__ int sturm_count(const double* sd, const double* se2, int n, double x,
                                           double pivmin) {
  double q = sd[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  int c = q < 0.0;
  for (int i = 1; i < n; ++i) {
    q = sd[i] - x - se2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    c += q < 0.0;
  }
  return c;
}

__global__ void __launch_bounds__(kTriThreads) tri_bisect_kernel(int n, double* work,
                                                                 double* __restrict__ evals) {
  extern __shared__ double sm[];
  __shared__ double red[64];
  double* sd = sm;
  double* se2 = sm + n;
  const TriWork W = tri_work(work, n);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double lo = DBL_MAX, hi = -DBL_MAX, emax = 0.0;
  for (int i = tid; i < n; i += kTriThreads) {
    const double di = W.d[i];
    const double el = i > 0 ? fabs(W.e[i - 1]) : 0.0;
    const double er = i + 1 < n ? fabs(W.e[i]) : 0.0;
    sd[i] = di;
    se2[i] = er * er;
    lo = fmin(lo, di - el - er);
    hi = fmax(hi, di + el + er);
    emax = fmax(emax, er * er);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  }
  if (lane == 0) {
    red[wid] = lo;
    red[8 + wid] = hi;
    red[16 + wid] = emax;
  }
  __syncthreads();
  for (int q = 0; q < kTriThreads / 32; ++q) {
    lo = fmin(lo, red[q]);
    hi = fmax(hi, red[8 + q]);
    emax = fmax(emax, red[16 + q]);
  }
  const double pivmin = DBL_MIN * fmax(1.0, emax);
  const double bnorm = fmax(fabs(lo), fabs(hi));
  lo -= 2.1 * bnorm * kEps * n + 4.2 * pivmin;
  hi += 2.1 * bnorm * kEps * n + 4.2 * pivmin;
  const int a = (int)blockIdx.x * (kTriThreads / 32) + wid;  // ascending index
  if (a >= n) return;
  for (int it = 0; it < 16; ++it) {
    const double width = hi - lo;
    if (width <= 2.0 * kEps * fmax(fabs(lo), fabs(hi)) + 2.0 * pivmin) break;
    const double x = lo + width * ((double)(lane + 1) / 33.0);
    const int cnt = sturm_count(sd, se2, n, x, pivmin);
    const unsigned above = __ballot_sync(0xffffffffu, cnt > a);
    const int first = above ? __ffs(above) - 1 : 32;
    const double xh = __shfl_sync(0xffffffffu, x, first < 32 ? first : 31);
    const double xl = __shfl_sync(0xffffffffu, x, first > 0 ? first - 1 : 0);
    if (first < 32) hi = xh;
    if (first > 0) lo = xl;
  }
  if (lane == 0) {
    const double lam = 0.5 * (lo + hi);
    const int j = n - 1 - a;  // descending
    W.lam[j] = lam;
    evals[j] = lam < 0.0 ? 0.0 : lam;  // clamp as sym_eig_desc (linalg.cpp:163-166)
  }
}

__device__ __forceinline__ double hash_uniform(unsigned a, unsigned b) {
  unsigned h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA6Bu;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  h *= 0x297A2D39u;
  h ^= h >> 15;
  return ((double)h + 0.5) * (2.0 / 4294967296.0) - 1.0;  // (-1, 1)
}

// One warp per cluster of the leading r eigenvalues (descending order).
__global__ void __launch_bounds__(32) tri_invit_kernel(int n, int r, double* work) {
  extern __shared__ double sm[];
  double* u = sm;            // U main diagonal
  double* s = sm + n;        // U first superdiagonal
  double* t = sm + 2 * n;    // U second superdiagonal
  double* l = sm + 3 * n;    // L multipliers
  double* z = sm + 4 * n;    // iterate
  int* piv = reinterpret_cast<int*>(sm + 5 * n);
  const TriWork W = tri_work(work, n);
  const int lane = threadIdx.x;
  // ||T||_1
  double onenrm = 0.0;
  for (int i = lane; i < n; i += 32) {
    const double el = i > 0 ? fabs(W.e[i - 1]) : 0.0;
    const double er = i + 1 < n ? fabs(W.e[i]) : 0.0;
    onenrm = fmax(onenrm, fabs(W.d[i]) + el + er);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) onenrm = fmax(onenrm, __shfl_xor_sync(0xffffffffu, onenrm, o));
  if (onenrm == 0.0) onenrm = 1.0;
  const double ortol = 1e-3 * onenrm;
  const double pertol = 10.0 * kEps * onenrm;
  const double pivtol = kEps * onenrm;
  const double stpcrt = sqrt(0.1 / n);
  const int j0 = blockIdx.x;
  if (j0 >= r) return;
  if (j0 > 0 && W.lam[j0 - 1] - W.lam[j0] <= ortol) return;  // not a cluster start
  double xprev = 0.0;
  for (int jj = j0; jj < r; ++jj) {
    if (jj > j0 && W.lam[jj - 1] - W.lam[jj] > ortol) break;
    double x = W.lam[jj];
    if (jj > j0 && xprev - x < pertol) x = xprev - pertol;  // keep shifts distinct
    xprev = x;
    // LU of T - x I with partial pivoting (lane 0)
    if (lane == 0) {
      double a = W.d[0] - x;
      double bsup = n > 1 ? W.e[0] : 0.0;
      for (int i = 0; i + 1 < n; ++i) {
        const double c = W.e[i];
        const double an = W.d[i + 1] - x;
        const double bn = i + 2 < n ? W.e[i + 1] : 0.0;
        if (fabs(a) >= fabs(c)) {
          if (fabs(a) < pivtol) a = a < 0.0 ? -pivtol : pivtol;
          const double m = c / a;
          u[i] = a;
          s[i] = bsup;
          t[i] = 0.0;
          l[i] = m;
          piv[i] = 0;
          a = an - m * bsup;
          bsup = bn;
        } else {
          const double m = a / c;
          u[i] = c;
          s[i] = an;
          t[i] = bn;
          l[i] = m;
          piv[i] = 1;
          a = bsup - m * an;
          bsup = -m * bn;
        }
      }
      if (fabs(a) < pivtol) a = a < 0.0 ? -pivtol : pivtol;
      u[n - 1] = a;
      s[n - 1] = 0.0;
      t[n - 1] = 0.0;
    }
    for (int i = lane; i < n; i += 32) z[i] = hash_uniform((unsigned)jj + 1u, (unsigned)i);
    __syncwarp();
    int its = 0, good = 0;
    while (true) {
      ++its;
      // scale the right-hand side (dstein): ||b||_1 = n ||T|| max(eps, |u_nn|)
      double b1 = 0.0;
      for (int i = lane; i < n; i += 32) b1 += fabs(z[i]);
      b1 = warp_sum(b1);
      const double scl = n * onenrm * fmax(kEps, fabs(u[n - 1])) / fmax(b1, DBL_MIN);
      for (int i = lane; i < n; i += 32) z[i] *= scl;
      __syncwarp();
      if (lane == 0) {
        for (int i = 0; i + 1 < n; ++i) {
          if (piv[i]) {
            const double zi = z[i];
            z[i] = z[i + 1];
            z[i + 1] = zi - l[i] * z[i];
          } else {
            z[i + 1] -= l[i] * z[i];
          }
        }
        z[n - 1] = z[n - 1] / u[n - 1];
        if (n > 1) z[n - 2] = (z[n - 2] - s[n - 2] * z[n - 1]) / u[n - 2];
        for (int i = n - 3; i >= 0; --i) z[i] = (z[i] - s[i] * z[i + 1] - t[i] * z[i + 2]) / u[i];
      }
      __syncwarp();
      // modified Gram-Schmidt against the cluster's earlier vectors
      for (int q = j0; q < jj; ++q) {
        const double* zq = W.Z + (long long)q * n;
        double dot = 0.0;
        for (int i = lane; i < n; i += 32) dot += zq[i] * z[i];
        dot = warp_sum(dot);
        for (int i = lane; i < n; i += 32) z[i] -= dot * zq[i];
        __syncwarp();
      }
      double mx = 0.0, n2 = 0.0;
      for (int i = lane; i < n; i += 32) {
        mx = fmax(mx, fabs(z[i]));
        n2 += z[i] * z[i];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      n2 = warp_sum(n2);
      const double inv = n2 > 0.0 ? 1.0 / sqrt(n2) : 0.0;
      for (int i = lane; i < n; i += 32) z[i] *= inv;
      __syncwarp();
      if (mx >= stpcrt) ++good;
      if (good >= 3 || its >= 8) break;
    }
    double* out = W.Z + (long long)jj * n;
    for (int i = lane; i < n; i += 32) out[i] = z[i];
    __threadfence_block();
    __syncwarp();
  }
}

// z <- H_0 H_1 .. H_{n-3} z for retained vector blockIdx.x, then the sign rule.
__global__ void __launch_bounds__(128) tri_backtransform_kernel(int n, double* work,
                                                                double* __restrict__ evecs) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  double* z = sm;
  const TriWork W = tri_work(work, n);
  const int j = blockIdx.x, tid = threadIdx.x;
  for (int i = tid; i < n; i += 128) z[i] = W.Z[(long long)j * n + i];
  __syncthreads();
  for (int k = n - 3; k >= 0; --k) {
    const double b = W.beta[k];
    const double* vk = W.Vh + (long long)k * n;
    double dot = 0.0;
    double vloc[8];
    int c = 0;
    // entries are owned by a FIXED thread (i mod 128 == tid) in every step:
    // a thread only ever reads and writes its own z[i], so the barriers inside
    // block_sum are the only ones needed (v_k is zero for i <= k)
    for (int i = tid; i < n; i += 128) {
      const double vi = i > k ? vk[i] : 0.0;
      if (c < 8) vloc[c] = vi;
      ++c;
      dot += vi * z[i];
    }
    dot = block_sum(dot, red) * b;
    c = 0;
    for (int i = tid; i < n; i += 128) {
      const double vi = c < 8 ? vloc[c] : (i > k ? vk[i] : 0.0);
      ++c;
      z[i] -= dot * vi;
    }
  }
  __syncthreads();
  // sign rule: the entry of largest magnitude (first index on ties) is positive
  if (tid < 32) {
    double best = -1.0;
    int arg = 0x7fffffff;
    for (int i = tid; i < n; i += 32) {
      const double a = fabs(z[i]);
      if (a > best) {
        best = a;
        arg = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
      if (ob > best || (ob == best && oa < arg)) {
        best = ob;
        arg = oa;
      }
    }
    if (tid == 0) red[0] = z[arg] < 0.0 ? -1.0 : 1.0;
  }
  __syncthreads();
  const double sgn = red[0];
  for (int i = tid; i < n; i += 128) evecs[i + (long long)j * n] = sgn * z[i];
}

}  // namespace

long long tri_eig_work_doubles(int n, int max_rank) {
  return 2LL * n * n + 6LL * n + (long long)n * std::max(max_rank, 1) + 64;
}

int tri_eig_max_rank(int n) { return std::min(n, std::max(64, n / 2)); }

bool tri_eig_applicable(int n) {
  static const int min_n = [] {  // TSG_EIG_TRI: smallest n for this route (0 = off)
    const char* e = std::getenv("TSG_EIG_TRI");
    return e ? std::atoi(e) : 96;
  }();
  return min_n > 0 && n >= min_n && n <= 2048;
}

// All eigenvalues (descending, clamped at zero) of the symmetric n x n matrix g;
// `work` (tri_eig_work_doubles) keeps the tridiagonal form for the vectors.
bool launch_tri_eigvals(const double* g, int n, double* evals, double* work, cudaStream_t st) {
  int dev = 0, coop = 0, sms = kNumSMs;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return false;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = sizeof(double) * 4 * (size_t)n;
  cudaFuncSetAttribute(tridiag_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tridiag_coop_kernel, kTriThreads, smem);
  if (per_sm < 1) return false;
  // one column per warp at the widest step; a smaller grid has a cheaper barrier
  int grid = std::min(sms, (n + kTriThreads / 32 - 1) / (kTriThreads / 32));
  grid = std::max(grid, 1);
  void* args[] = {(void*)&g, (void*)&n, (void*)&work};
  if (cudaLaunchCooperativeKernel((void*)tridiag_coop_kernel, grid, kTriThreads, args, smem, st) !=
      cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  const int bgrid = (n + kTriThreads / 32 - 1) / (kTriThreads / 32);
  tri_bisect_kernel<<<bgrid, kTriThreads, sizeof(double) * 2 * n, st>>>(n, work, evals);
  g_launches += 2;
  return true;
}

// The leading `rank` eigenvectors (n x rank, ld n) after launch_tri_eigvals.
void launch_tri_eigvecs(int n, int rank, double* work, double* evecs, cudaStream_t st) {
  if (rank <= 0) return;
  const size_t smem = sizeof(double) * 5 * (size_t)n + sizeof(int) * (size_t)n;
  cudaFuncSetAttribute(tri_invit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tri_invit_kernel<<<rank, 32, smem, st>>>(n, rank, work);
  tri_backtransform_kernel<<<rank, 128, sizeof(double) * n, st>>>(n, work, evecs);
  g_launches += 2;
}

}  // namespace tsg
