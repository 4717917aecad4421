// Incremental SVD row insertion and streaming-mode core update
// (reference proj/src/isvd.cpp:163-250 add_row, proj/src/streaming.cpp:196-224
// core rotation, :39-64 coupling check), entirely on the device.
//
// Two execution shapes:
//  * fused: one CTA performs the whole chain (p_gram, the two projection
//    passes, the inner SVD, the Q / core / left updates and the coupling
//    check) when the ISVD width n and rank are small (configs 1, 2, early 5):
//    one launch per slice, no inter-kernel latency;
//  * split: grid-wide projection passes and row updates around the same
//    inner SVD when n is large (configs 3, 4, late 5).
// The inner SVD of S' = [diag(s) 0; p^T k] follows small_svd_truncated
// (linalg.cpp:210-259): Gram route S'^T S', Jacobi eigensolve with the
// reference's stopping rule, stable descending sort, clamp and sign rule,
// sigma floor, truncation rank, U = S' V / sigma and one MGS pass. The
// cyclic sweep order is replaced by the round-robin parallel order (every
// pair once per sweep); for m = r+1 <= 32 it runs in a single warp with no
// block barriers.
#include <cstdio>
#include <cstdlib>
#include <cooperative_groups.h>

#include "kernels.cuh"
namespace tsg {
__device__ long long g_isvd_clk[32];  // debug phase clocks (thread 0)
__device__ long long g_isvd_acc[32];  // sums of (stamp - stamp 0) over insertions, [31] = count
}
#define SEC_CLK(i)                                         \
  do {                                                     \
    if (threadIdx.x == 0) ::tsg::g_isvd_clk[i] = clock64(); \
  } while (0)
#include "secular.cuh"

namespace tsg {


// Scratch layout of the inner SVD (all column-major, in the `inner` buffer).
struct InnerLayout {
  long long W, U, M, w, lam, G, V, p, perm, pg;
  long long total;
};
__host__ __device__ inline InnerLayout inner_layout(int capr) {
  const long long m = capr + 1;
  InnerLayout L;
  long long o = 0;
  L.W = o; o += m * m;     // eigenvectors of S'^T S' (kept columns = right factor Q')
  L.U = o; o += m * m;     // left factor P' of S'
  L.M = o; o += m * m;     // core rotation M = P'_top^T p_gram
  L.w = o; o += m;         // last row of P'
  L.lam = o; o += m;       // eigenvalues
  L.G = o; o += m * m;     // global fallback for large inner problems
  L.V = o; o += m * m;
  L.p = o; o += m;         // p = p1 + p2
  L.perm = o; o += m;      // int scratch (stored in doubles' space)
  L.pg = o; o += m * m;    // p_gram (r x r)
  L.total = o;
  return L;
}
int isvd_inner_scratch(int capr) { return (int)inner_layout(capr).total; }

int read_isvd_clocks(long long* out) {
  if (out[0] == -12345) return cudaMemcpyFromSymbol(out, g_isvd_acc, sizeof(long long) * 32) == cudaSuccess ? 0 : 4;
  return cudaMemcpyFromSymbol(out, g_isvd_clk, sizeof(long long) * 32) == cudaSuccess ? 0 : 4;
}

namespace {

constexpr unsigned FULL = 0xffffffffu;
#define TSG_CLK(i) \
  do {             \
    if (threadIdx.x == 0) g_isvd_clk[i] = clock64(); \
  } while (0)

struct InnerIO {
  Ctrl* ctrl;
  int r;
  const double* sigma;     // r
  const double* p;         // r (p1 + p2)
  double k;                // ||e||
  int deg;                 // degenerate: residual direction dropped
  double delta;
  const double* pgram;     // r x r
  double* inner;           // scratch (InnerLayout)
  double* sigma_new;
  int capr;
};

__device__ __forceinline__ double Sp(const InnerIO& io, int i, int j) {
  // S'(i,j): diag(s) stacked over [p^T k] (isvd.cpp:203-209)
  if (i < io.r) return (i == j) ? io.sigma[j] : 0.0;
  return (j < io.r) ? io.p[j] : io.k;
}

// Truncation on the sorted spectrum (linalg.cpp:224-240, isvd.cpp:210-215);
// single thread. Returns the rank.
__device__ int inner_truncate(const InnerIO& io, double* lam, int m, int sweeps) {
  Ctrl* c = io.ctrl;
  const double smax = sqrt(lam[0]);
  int rank = 0;
  double disc = 0.0, margin = 0.0;
  if (smax > 0.0) {
    const double fl = kSigmaZeroFactor * smax;
    for (int i = 0; i < m; ++i)
      if (sqrt(lam[i]) <= fl) lam[i] = 0.0;
    const double budget = io.delta * io.delta;
    double s = 0.0, prev_excess = -1.0;
    int rr = m;
    for (int i = m - 1; i >= 0; --i) {
      const double nx = s + lam[i];
      if (nx <= budget) {
        s = nx;
        rr = i;
      } else {
        prev_excess = nx;
        break;
      }
    }
    rank = rr < 1 ? 1 : rr;
    for (int j = m - 1; j >= rank; --j) disc += lam[j];
    if (budget > 0.0) {
      double mg = fabs(budget - s) / budget;
      if (prev_excess >= 0.0) mg = fmin(mg, fabs(prev_excess - budget) / budget);
      margin = mg;
    }
  } else {
    c->status = 3;  // S' == 0 cannot happen with r >= 1 and sigma > 0
  }
  double added = disc;
  if (io.deg) added += io.k * io.k;
  const double sq_err = c->squared_error;
  c->trunc_margin = margin;
  c->sweeps = sweeps;
  c->added_error_sq = added;
  c->squared_error = sq_err + added;  // isvd.cpp:212-215
  c->r_new = rank;
  c->degenerate = io.deg;
  return rank;
}

// Whole inner problem in one warp (m = columns of S' <= 32). RM >= r + 1
// bounds the rows of S' so that MGS columns live in registers. Shared-memory
// scratch: sG (sorted eigenvectors, pitch 33) and sU (left factor).
template <int RM>
__device__ void inner_solve_warp(const InnerIO& io, double* sG, double* sU) {
  const int lane = threadIdx.x & 31;
  const int r = io.r;
  const int m = io.deg ? r : r + 1;
  const int rows = r + 1;
  constexpr int P = 33;
  const InnerLayout L = inner_layout(io.capr);
  double* lam = io.inner + L.lam;
  double* W = io.inner + L.W;
  // S'^T S' = diag(s^2, 0) + z z^T, z = [p; k] (degenerate: diag(s^2) + p p^T)
  __shared__ double sd[32], sz[33], ssig[32], sQ[32 * 33], sx[8 * 32];
  __shared__ int si[3 * 32];
  if (lane < m) {
    const double sg = lane < r ? io.sigma[lane] : 0.0;
    ssig[lane] = sg;
    sd[lane] = sg * sg;
    sz[lane] = lane < r ? io.p[lane] : io.k;
  }
  __syncwarp();
  TSG_CLK(4);
  secular::Scratch S;
  S.sQ = sQ;
  S.dK = sx;
  S.wK = sx + 32;
  S.zK = sx + 64;
  S.ls = sx + 96;
  S.lt = sx + 128;
  S.zh = sx + 160;
  S.lamall = sx + 192;
  S.idx = si;
  S.perm = si + 32;
  S.flag = si + 64;
  const int iters = secular::eig_rank_one_fast<RM>(m, sd, sz, S, lam, W, sG);
  TSG_CLK(5);
  int rank = 0;
  if (lane == 0) rank = inner_truncate(io, lam, m, iters);
  rank = __shfl_sync(FULL, rank, 0);
  __syncwarp();
  TSG_CLK(6);
  // sigma_new and U = S' W / sigma, column `lane` in registers
  // (multiply, linalg.cpp:250-256; rows i < r of S' are diag(s))
  double u[RM];
#pragma unroll
  for (int l = 0; l < RM; ++l) u[l] = 0.0;
  if (lane < rank) {
    const double lj = lam[lane];
    io.sigma_new[lane] = sqrt(lj);
    const double inv = 1.0 / sqrt(lj);
    double s = 0.0;
    for (int l = 0; l < m; ++l) s += sz[l] * sG[l * P + lane];
#pragma unroll
    for (int l = 0; l < RM; ++l) {
      if (l < r) u[l] = ssig[l] * sG[l * P + lane] * inv;
      else if (l == r) u[l] = s * inv;
    }
  }
  // one MGS pass, right-looking (linalg.cpp:64-78); column i broadcast by shuffles
  for (int i = 0; i < rank; ++i) {
    if (lane == i) {
      double ss = 0.0;
#pragma unroll
      for (int l = 0; l < RM; ++l) ss += u[l] * u[l];
      const double nrm = sqrt(ss);
      if (nrm > 0.0) {
#pragma unroll
        for (int l = 0; l < RM; ++l) u[l] /= nrm;
      }
    }
    double dot = 0.0;
    double ui[RM];
#pragma unroll
    for (int l = 0; l < RM; ++l) {
      ui[l] = __shfl_sync(FULL, u[l], i);
      dot += ui[l] * u[l];
    }
    if (lane > i && lane < rank) {
#pragma unroll
      for (int l = 0; l < RM; ++l) u[l] -= dot * ui[l];
    }
  }
  TSG_CLK(7);
  // outputs: U (P'), M = P'_top^T p_gram, w = last row of P'
  double* U = io.inner + L.U;
  double* M = io.inner + L.M;
  double* w = io.inner + L.w;
  if (lane < rank) {
#pragma unroll
    for (int l = 0; l < RM; ++l)
      if (l < rows) {
        sU[l * P + lane] = u[l];
        U[l + lane * rows] = u[l];
      }
    w[lane] = sU[r * P + lane];
  }
  __syncwarp();
  for (int idx = lane; idx < rank * r; idx += 32) {
    const int jn = idx % rank, j = idx / rank;
    double s = 0.0;
    for (int l = 0; l < r; ++l) s += sU[l * P + jn] * io.pgram[l + j * r];
    M[jn + j * rank] = s;
  }
  __syncwarp();
}

// Block-wide version for m > 32 (G, V in smem when they fit, else global).
// `wide` (shared memory, kWideScratch doubles, may be null): for m <= 64 the
// spectrum comes from the one-warp secular solver (secular::eig_rank_one_wide)
// instead of block Jacobi on the explicit Gram matrix — ~15 us instead of
// ~430 us at m = 37 (config 5's last epochs, config 3's r = 32).
constexpr int kWideScratch = secular::ScratchWide::doubles() + 2 * secular::kWide;
__device__ void inner_solve_block(const InnerIO& io, double* G, double* V, double* wide = nullptr) {
  __shared__ double red[32];
  __shared__ int sh_rank;
  struct RotL {
    double c, s, t;
    int p, q;
  };
  __shared__ RotL rot[128];
  const InnerLayout L = inner_layout(io.capr);
  const int r = io.r;
  const int m = io.deg ? r : r + 1;
  const int rows = r + 1;
  const bool use_wide = wide != nullptr && m <= secular::kWide;
  int sweep = 0;
  if (use_wide) {
    TSG_CLK(4);
    {
      secular::ScratchWide S = secular::scratch_wide(wide);
      double* d_in = wide + secular::ScratchWide::doubles();
      double* z_in = d_in + secular::kWide;
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const double sg = i < r ? io.sigma[i] : 0.0;
        d_in[i] = sg * sg;
        z_in[i] = i < r ? io.p[i] : io.k;
      }
      __syncthreads();
      // block-wide: one thread per root / coordinate / column
      sweep = secular::eig_rank_one_wide(m, d_in, z_in, S, io.inner + L.lam, io.inner + L.W);
    }
    TSG_CLK(5);
  } else {
  double acc = 0.0;
  for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
    const int i = idx % m, j = idx / m;
    if (i > j) continue;
    double dot = 0.0;
    for (int l = 0; l < rows; ++l) dot += Sp(io, l, i) * Sp(io, l, j);
    G[i + j * m] = dot;
    G[j + i * m] = dot;
    acc += (i == j) ? dot * dot : 2.0 * dot * dot;
  }
  for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x)
    V[idx] = ((idx % m) == (idx / m)) ? 1.0 : 0.0;
  const double tol = kOffDiagTolFactor * sqrt(block_sum(acc, red));
  const int np = m + (m & 1), half = np / 2;
  for (; sweep < kMaxSweeps; ++sweep) {
    double o2 = 0.0;
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
      const int i = idx % m, j = idx / m;
      if (i != j) o2 += G[idx] * G[idx];
    }
    const double off = sqrt(block_sum(o2, red));
    if (off <= tol || m < 2) break;
    for (int rd = 0; rd < np - 1; ++rd) {
      for (int mm = threadIdx.x; mm < half; mm += blockDim.x) {
        int x, y;
        if (mm == 0) {
          x = rd % (np - 1);
          y = np - 1;
        } else {
          x = (rd + mm) % (np - 1);
          y = (rd + np - 1 - mm) % (np - 1);
        }
        RotL R;
        R.p = min(x, y);
        R.q = max(x, y);
        R.c = 1.0;
        R.s = 0.0;
        R.t = 0.0;
        if (R.q < m) {
          const double gpq = G[R.p + R.q * m];
          if (gpq != 0.0) {
            const double theta = (G[R.q + R.q * m] - G[R.p + R.p * m]) / (2.0 * gpq);
            const double t = (theta >= 0.0) ? 1.0 / (theta + sqrt(1.0 + theta * theta))
                                            : 1.0 / (theta - sqrt(1.0 + theta * theta));
            const double cc = 1.0 / sqrt(1.0 + t * t);
            R.c = cc;
            R.s = t * cc;
            R.t = t;
          }
        }
        rot[mm] = R;
      }
      __syncthreads();
      for (int bi = threadIdx.x; bi < half * half; bi += blockDim.x) {
        const int m1 = bi / half, m2 = bi % half;
        if (m1 > m2) continue;
        const RotL A = rot[m1], B = rot[m2];
        const bool idA = (A.s == 0.0 && A.t == 0.0), idB = (B.s == 0.0 && B.t == 0.0);
        if (idA && idB) continue;
        const int p1 = A.p, q1 = A.q, p2 = B.p, q2 = B.q;
        const bool q1v = q1 < m, q2v = q2 < m;
        if (m1 == m2) {
          const double gpq = G[p1 + q1 * m], gpp = G[p1 + p1 * m], gqq = G[q1 + q1 * m];
          G[p1 + p1 * m] = gpp - A.t * gpq;
          G[q1 + q1 * m] = gqq + A.t * gpq;
          G[p1 + q1 * m] = 0.0;
          G[q1 + p1 * m] = 0.0;
          continue;
        }
        const double b00 = G[p1 + p2 * m];
        const double b01 = q2v ? G[p1 + q2 * m] : 0.0;
        const double b10 = q1v ? G[q1 + p2 * m] : 0.0;
        const double b11 = (q1v && q2v) ? G[q1 + q2 * m] : 0.0;
        const double t00 = A.c * b00 - A.s * b10, t01 = A.c * b01 - A.s * b11;
        const double t10 = A.s * b00 + A.c * b10, t11 = A.s * b01 + A.c * b11;
        const double o00 = B.c * t00 - B.s * t01, o01 = B.s * t00 + B.c * t01;
        const double o10 = B.c * t10 - B.s * t11, o11 = B.s * t10 + B.c * t11;
        G[p1 + p2 * m] = o00;
        G[p2 + p1 * m] = o00;
        if (q2v) {
          G[p1 + q2 * m] = o01;
          G[q2 + p1 * m] = o01;
        }
        if (q1v) {
          G[q1 + p2 * m] = o10;
          G[p2 + q1 * m] = o10;
        }
        if (q1v && q2v) {
          G[q1 + q2 * m] = o11;
          G[q2 + q1 * m] = o11;
        }
      }
      for (int idx = threadIdx.x; idx < m * half; idx += blockDim.x) {
        const int i = idx % m, mm = idx / m;
        const RotL R = rot[mm];
        if (R.q >= m || (R.s == 0.0 && R.t == 0.0)) continue;
        const double vp = V[i + R.p * m], vq = V[i + R.q * m];
        V[i + R.p * m] = R.c * vp - R.s * vq;
        V[i + R.q * m] = R.s * vp + R.c * vq;
      }
      __syncthreads();
    }
  }
  __syncthreads();
  }  // !use_wide
  double* lam = io.inner + L.lam;
  double* W = io.inner + L.W;
  int* perm = reinterpret_cast<int*>(io.inner + L.perm);
  if (!use_wide) {
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double di = G[i + i * m];
    int rk = 0;
    for (int j = 0; j < m; ++j) {
      const double dj = G[j + j * m];
      if (dj > di || (dj == di && j < i)) ++rk;
    }
    perm[rk] = i;
  }
  __syncthreads();
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = wid; j < m; j += nw) {
      const int src = perm[j];
      double lambda = G[src + src * m];
      if (lambda < 0.0) lambda = 0.0;
      if (lane == 0) lam[j] = lambda;
      double best = -1.0;
      int arg = 0x7fffffff;
      for (int i = lane; i < m; i += 32) {
        const double av = fabs(V[i + src * m]);
        if (av > best) {
          best = av;
          arg = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(FULL, best, o);
        const int oa = __shfl_xor_sync(FULL, arg, o);
        if (ob > best || (ob == best && oa < arg)) {
          best = ob;
          arg = oa;
        }
      }
      const bool flip = V[arg + src * m] < 0.0;
      for (int i = lane; i < m; i += 32) {
        const double v = V[i + src * m];
        W[i + j * m] = flip ? -v : v;
      }
    }
  }
  __syncthreads();
  }  // !use_wide (the secular solver returns sorted, signed eigenpairs)
  if (threadIdx.x == 0) sh_rank = inner_truncate(io, lam, m, sweep);
  __syncthreads();
  if (use_wide) TSG_CLK(6);
  const int rank = sh_rank;
  double* U = io.inner + L.U;
  for (int j = threadIdx.x; j < rank; j += blockDim.x) io.sigma_new[j] = sqrt(lam[j]);
  if (use_wide) {
    // U = S' W / sigma and its MGS pass in shared memory (the secular
    // scratch is free now), a warp per column with lanes over the rows
    double* sU = wide;  // rows x rank, ld rows (<= 65 x 64)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int idx = threadIdx.x; idx < r * rank; idx += blockDim.x) {
      const int i = idx % r, j = idx / r;
      // rows i < r of S' are diag(s)
      sU[i + j * rows] = io.sigma[i] * W[i + j * m] * (1.0 / sqrt(lam[j]));
    }
    // last row [p^T k] W: a warp per column, lanes over the m terms (all loads
    // in flight), fixed tree
    for (int j = wid; j < rank; j += nw) {
      double s = 0.0;
      for (int l = lane; l < m; l += 32) s += Sp(io, r, l) * W[l + j * m];
      s = warp_sum(s);
      if (lane == 0) sU[r + j * rows] = s * (1.0 / sqrt(lam[j]));
    }
    __syncthreads();
    TSG_CLK(17);
    auto normalize = [&](double* u) {  // one warp
      double ss = 0.0;
      for (int l = lane; l < rows; l += 32) ss += u[l] * u[l];
      ss = warp_sum(ss);
      const double nrm = sqrt(ss);
      __syncwarp();
      if (nrm > 0.0)
        for (int l = lane; l < rows; l += 32) u[l] /= nrm;
      __syncwarp();
    };
    if (wid == 0 && rank > 0) normalize(sU);
    __syncthreads();
    // one barrier per column: the warp that updates column i + 1 normalises it
    // right away (the same operations in the same order as a separate pass)
    for (int i = 0; i < rank; ++i) {
      const double* ui = sU + i * rows;
      for (int j = i + 1 + wid; j < rank; j += nw) {
        double* uj = sU + j * rows;
        double dot = 0.0;
        for (int l = lane; l < rows; l += 32) dot += ui[l] * uj[l];
        dot = warp_sum(dot);
        for (int l = lane; l < rows; l += 32) uj[l] -= dot * ui[l];
        __syncwarp();
        if (j == i + 1) normalize(uj);
      }
      __syncthreads();
    }
    TSG_CLK(7);
    for (int idx = threadIdx.x; idx < rows * rank; idx += blockDim.x) U[idx] = sU[idx];
    double* M = io.inner + L.M;
    double* w = io.inner + L.w;
    for (int idx = threadIdx.x; idx < rank * r; idx += blockDim.x) {
      const int jn = idx % rank, j = idx / rank;
      double s = 0.0;
      for (int l = 0; l < r; ++l) s += sU[l + jn * rows] * io.pgram[l + j * r];
      M[jn + j * rank] = s;
    }
    for (int j = threadIdx.x; j < rank; j += blockDim.x) w[j] = sU[r + j * rows];
    __syncthreads();
    TSG_CLK(2);
    return;
  }
  for (int idx = threadIdx.x; idx < rows * rank; idx += blockDim.x) {
    const int i = idx % rows, j = idx / rows;
    double s = 0.0;
    for (int l = 0; l < m; ++l) {
      const double wl = W[l + j * m];
      if (wl == 0.0) continue;
      s += Sp(io, i, l) * wl;
    }
    U[i + j * rows] = s * (1.0 / sqrt(lam[j]));
  }
  __syncthreads();
  // MGS, right-looking, thread per column (the reference's sequential dot order)
  for (int i = 0; i < rank; ++i) {
    double* ui = U + i * rows;
    if (threadIdx.x == 0) {
      double ss = 0.0;
      for (int l = 0; l < rows; ++l) ss += ui[l] * ui[l];
      const double nrm = sqrt(ss);
      if (nrm > 0.0)
        for (int l = 0; l < rows; ++l) ui[l] /= nrm;
    }
    __syncthreads();
    for (int j = i + 1 + threadIdx.x; j < rank; j += blockDim.x) {
      double* uj = U + j * rows;
      double dot = 0.0;
      for (int l = 0; l < rows; ++l) dot += ui[l] * uj[l];
      for (int l = 0; l < rows; ++l) uj[l] -= dot * ui[l];
    }
    __syncthreads();
  }
  double* M = io.inner + L.M;
  double* w = io.inner + L.w;
  for (int idx = threadIdx.x; idx < rank * r; idx += blockDim.x) {
    const int jn = idx % rank, j = idx / rank;
    double s = 0.0;
    for (int l = 0; l < r; ++l) s += U[l + jn * rows] * io.pgram[l + j * r];
    M[jn + j * rank] = s;
  }
  for (int j = threadIdx.x; j < rank; j += blockDim.x) w[j] = U[r + j * rows];
  __syncthreads();
}

// ---------------------------------------------------------------- helpers
// p_gram = left^T left (isvd.cpp:86-100): per (l, j) sum over rows in
// order, zero multipliers skipped, mirrored.
__device__ void pgram_block(const double* __restrict__ left, long long n_d, int capr, int r,
                            double* pg) {
  for (int idx = threadIdx.x; idx < r * r; idx += blockDim.x) {
    const int l = idx % r, j = idx / r;
    if (l > j) continue;
    double s = 0.0;
    for (long long i = 0; i < n_d; ++i) {
      const double w = left[i * capr + j];
      if (w == 0.0) continue;
      s += left[i * capr + l] * w;
    }
    pg[l + j * r] = s;
    pg[j + l * r] = s;
  }
}

// Append a record to the device ring (metrics + control snapshot): fields,
// gpu-scope fence, then the count. The host sees it once a tail kernel
// (decide_finish) has copied it to the mapped ring, or by a copy at drain.
__device__ void publish(Ctrl* c, const Metrics& m, RecRing* ring) {
  const unsigned long long k = c->records;
  const int pos = (int)(k % kRecRing);
  ring->rec[pos] = m;
  c->records = k + 1;
  ring->ctrl[pos] = *c;
  __threadfence();
  *reinterpret_cast<volatile unsigned long long*>(&ring->done) = k + 1;
}

__device__ void finalize_record(Ctrl* c, const SliceCtl* sl, double d, double cs, RecRing* ring,
                                int order, const SpatialRanks& sr) {
  // one batch of independent loads, then stores (no load-after-store chains)
  const int r_new = c->r_new, status = c->status, sweeps = c->sweeps;
  const long long n_d = c->n_d, ins = c->insertions;
  const double slice_sq = sl->slice_sq, proj_sq = c->proj_sq, margin = c->trunc_margin;
  const double sq_err = c->squared_error, ns = c->nonstream_discarded_sq, tot = c->total_input_sq;
  double res[kMaxD];
#pragma unroll
  for (int k = 0; k < kMaxD; ++k) res[k] = sl->res_sq[k];
  c->coupling_diff_sq = d;
  c->core_sq = cs;
  if (sqrt(d) > kCouplingTol * sqrt(cs) + 1e-300 && status == 0) c->status = 2;  // streaming.cpp:55-63
  c->r = r_new;
  c->n_d = n_d + 1;
  c->insertions = ins + 1;
  Metrics m;
  m.slice_index = n_d;
#pragma unroll
  for (int k = 0; k < kMaxD; ++k) m.ranks[k] = (k + 1 < order) ? sr.v[k] : 0;
  m.ranks[order - 1] = r_new;
  m.slice_norm = sqrt(slice_sq);
  m.projected_norm = sqrt(proj_sq);
#pragma unroll
  for (int k = 0; k < kMaxD; ++k) m.mode_residuals[k] = (k + 1 < order) ? sqrt(res[k]) : 0.0;
  const double booked = sq_err + ns;
  m.error_estimate = tot <= 0.0 ? 0.0 : sqrt(fmax(booked, 0.0) / tot);
  m.expanded_mask = 0;
  m.trunc_margin = margin;
  m.sweeps = sweeps;
  publish(c, m, ring);
}

// Row update of Q and the core for rows [i0, i1): Qn = [Q q] W,
// Cn = C M^T + b w^T; returns the coupling partials (isvd.cpp:217-225,
// streaming.cpp:208-218).
template <int RMAX>
__device__ void update_rows(const Ctrl* ctrl, const double* __restrict__ q,
                            const double* __restrict__ cin, const double* __restrict__ e,
                            const double* __restrict__ b, const double* W, const double* M,
                            const double* w, const double* __restrict__ sig_new, long long n,
                            long long i0, long long i1, long long stride, double* qn, double* cn,
                            double& dacc, double& cacc) {
  const int r = ctrl->r, rn = ctrl->r_new, deg = ctrl->degenerate;
  const int m = deg ? r : r + 1;
  const double inv = deg ? 0.0 : 1.0 / sqrt(ctrl->e_sq);
  for (long long i = i0; i < i1; i += stride) {
    double qr[RMAX + 1], cr[RMAX];
#pragma unroll
    for (int l = 0; l < RMAX; ++l) {
      qr[l] = l < r ? q[i + (long long)l * n] : 0.0;
      cr[l] = l < r ? cin[i + (long long)l * n] : 0.0;
    }
    qr[RMAX] = 0.0;
    const double qi = deg ? 0.0 : e[i] * inv;
    const double bi = b[i];
    for (int jn = 0; jn < rn; ++jn) {
      double sq = 0.0, sc = 0.0;
      // zero multipliers are skipped in the reference (matrix.cpp:44-52);
      // adding 0 * x is exact for finite x, so they are not tested here
#pragma unroll
      for (int l = 0; l < RMAX; ++l) {
        if (l < r) {
          sq += qr[l] * W[l + jn * m];
          sc += cr[l] * M[jn + l * rn];
        }
      }
      if (!deg) sq += qi * W[r + jn * m];
      sc += w[jn] * bi;
      qn[i + (long long)jn * n] = sq;
      cn[i + (long long)jn * n] = sc;
      const double diff = sc - sq * sig_new[jn];
      dacc += diff * diff;
      cacc += sc * sc;
    }
  }
}

// Generic (any r) row update reading rows from global memory.
__device__ void update_rows_generic(const Ctrl* ctrl, const double* __restrict__ q,
                                    const double* __restrict__ cin, const double* __restrict__ e,
                                    const double* __restrict__ b, const double* W, const double* M,
                                    const double* w, const double* __restrict__ sig_new, long long n,
                                    long long i0, long long i1, long long stride, double* qn,
                                    double* cn, double& dacc, double& cacc) {
  const int r = ctrl->r, rn = ctrl->r_new, deg = ctrl->degenerate;
  const int m = deg ? r : r + 1;
  const double inv = deg ? 0.0 : 1.0 / sqrt(ctrl->e_sq);
  for (long long i = i0; i < i1; i += stride) {
    const double qi = deg ? 0.0 : e[i] * inv;
    const double bi = b[i];
    for (int jn = 0; jn < rn; ++jn) {
      double sq = 0.0, sc = 0.0;
      for (int l = 0; l < r; ++l) {
        const double wl = W[l + jn * m];
        if (wl != 0.0) sq += q[i + (long long)l * n] * wl;
        const double ml = M[jn + l * rn];
        if (ml != 0.0) sc += cin[i + (long long)l * n] * ml;
      }
      if (!deg) {
        const double wl = W[r + jn * m];
        if (wl != 0.0) sq += qi * wl;
      }
      const double wj = w[jn];
      if (wj != 0.0) sc += wj * bi;
      qn[i + (long long)jn * n] = sq;
      cn[i + (long long)jn * n] = sc;
      const double diff = sc - sq * sig_new[jn];
      dacc += diff * diff;
      cacc += sc * sc;
    }
  }
}

// left <- blkdiag(left, 1) P' (isvd.cpp:227-237; right_multiply :66-84)
__device__ void left_rows(const Ctrl* ctrl, const double* __restrict__ left, long long n_d,
                          int capr, const double* U, double* left_new, long long tid,
                          long long stride) {
  const int r = ctrl->r, rn = ctrl->r_new;
  const int rows = r + 1;
  const long long total = (n_d + 1) * capr;
  for (long long idx = tid; idx < total; idx += stride) {
    const long long i = idx / capr;
    const int j = (int)(idx % capr);
    double v = 0.0;
    if (j < rn) {
      if (i < n_d) {
        for (int l = 0; l < r; ++l) v += left[i * capr + l] * U[l + j * rows];
      } else {
        v = U[r + j * rows];
      }
    }
    left_new[idx] = v;
  }
}

// ============================================================ fused path
// One CTA (1024 threads); e and the projection coefficients stay on chip.
template <int RMAX>
__global__ void __launch_bounds__(512, 1) isvd_fused_kernel(IsvdBufs B) {
  extern __shared__ double fsm[];
  __shared__ double red[32];
  __shared__ double sp1[RMAX + 1], sp2[RMAX + 1], sp[RMAX + 1];
  __shared__ int sperm[33];
  __shared__ double sh_bsq, sh_esq;
  Ctrl* c = B.ctrl;
  const int r = c->r;
  const long long n = B.n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const InnerLayout L = inner_layout(B.capr);
  double* pg = B.inner + L.pg;
  double* se = fsm;                    // n doubles
  double* sG = se + n;                 // 32 x 33
  double* sV = sG + 32 * 33;
  double* sU = sV + 32 * 33;
  TSG_CLK(0);
  // p_gram (old left) for the core rotation
  const long long n_d = c->n_d;
  pgram_block(B.left, n_d, B.capr, r, pg);
  __syncthreads();
  TSG_CLK(8);
  // Two classical Gram-Schmidt passes (CGS2) split b = Q p + e
  // (isvd.cpp:172-191 uses two MGS passes: same projector, parallel form).
  // Row-parallel: each thread accumulates all r dot products of its rows.
  __shared__ double wpart[16][RMAX + 1];
  const double* __restrict__ q = B.q;
  const double* __restrict__ bv = B.b;
  auto reduce_to = [&](double (&acc)[RMAX + 1], double* dst, int cnt) {
#pragma unroll
    for (int j = 0; j <= RMAX; ++j) {
      const double v = warp_sum(acc[j]);
      if (lane == 0) wpart[wid][j] = v;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
      double s = 0.0;
      for (int w = 0; w < 16; ++w) s += wpart[w][j];
      dst[j] = s;
    }
    __syncthreads();
  };
  double acc[RMAX + 1];
#pragma unroll
  for (int j = 0; j <= RMAX; ++j) acc[j] = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const double bi = bv[i];
#pragma unroll
    for (int j = 0; j < RMAX; ++j)
      if (j < r) acc[j] += q[i + (long long)j * n] * bi;
    acc[RMAX] += bi * bi;
  }
  reduce_to(acc, sp1, RMAX + 1);
  const double bs = sp1[RMAX];
#pragma unroll
  for (int j = 0; j <= RMAX; ++j) acc[j] = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    double qr[RMAX];
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < RMAX; ++j) {
      qr[j] = j < r ? q[i + (long long)j * n] : 0.0;
      s += qr[j] * sp1[j];
    }
    const double e1 = bv[i] - s;
    se[i] = e1;
#pragma unroll
    for (int j = 0; j < RMAX; ++j) acc[j] += qr[j] * e1;
  }
  reduce_to(acc, sp2, RMAX);
  double es = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < RMAX; ++j)
      if (j < r) s += q[i + (long long)j * n] * sp2[j];
    const double v = se[i] - s;
    se[i] = v;
    es += v * v;
  }
  es = block_sum(es, red);
  TSG_CLK(1);
  for (int j = threadIdx.x; j < r; j += blockDim.x) sp[j] = sp1[j] + sp2[j];
  if (threadIdx.x == 0) {
    sh_bsq = bs;
    sh_esq = es;
    c->proj_sq = bs;
    c->e_sq = es;
  }
  __syncthreads();
  // inner SVD in warp 0
  if (wid == 0) {
    InnerIO io;
    io.ctrl = c;
    io.r = r;
    io.sigma = B.sigma;
    io.p = sp;
    io.k = sqrt(sh_esq);
    io.deg = (io.k <= kOrthEps * sqrt(sh_bsq)) ? 1 : 0;  // isvd.cpp:191
    io.delta = B.slot->delta;
    io.pgram = pg;
    io.inner = B.inner;
    io.sigma_new = B.sigma_new;
    io.capr = B.capr;
    inner_solve_warp<RMAX + 1>(io, sG, sU);
  }
  __syncthreads();
  TSG_CLK(2);
  // stage the small factors, then Q / core rows, coupling partials; left rows
  double* stW = sU + 32 * 33;
  double* stM = stW + 33 * 33;
  double* stw = stM + 33 * 33;
  double* sts = stw + 33;
  {
    const int rr = c->r, rn = c->r_new, mm = c->degenerate ? rr : rr + 1;
    for (int i = threadIdx.x; i < mm * rn; i += blockDim.x) stW[i] = B.inner[L.W + i];
    for (int i = threadIdx.x; i < rn * rr; i += blockDim.x) stM[i] = B.inner[L.M + i];
    for (int i = threadIdx.x; i < rn; i += blockDim.x) {
      stw[i] = B.inner[L.w + i];
      sts[i] = B.sigma_new[i];
    }
  }
  __syncthreads();
  double dacc = 0.0, cacc = 0.0;
  update_rows<RMAX>(c, B.q, B.c, se, B.b, stW, stM, stw, sts, n, threadIdx.x, n, blockDim.x,
                    B.qn, B.cn, dacc, cacc);
  left_rows(c, B.left, n_d, B.capr, B.inner + L.U, B.left_new, threadIdx.x, blockDim.x);
  dacc = block_sum(dacc, red);
  cacc = block_sum(cacc, red);
  TSG_CLK(3);
  if (threadIdx.x == 0) {
    SpatialRanks sr;
    for (int k = 0; k < kMaxD; ++k) sr.v[k] = B.spatial_ranks[k];
    finalize_record(c, B.slot, dacc, cacc, B.ring, B.order, sr);
    TSG_CLK(9);
  }
}

// ============================================================ split path
// p_gram for the split path: the same per-(l, j) row-ordered sums as
// pgram_block, but the rows are staged through shared memory in tiles
// (coalesced loads, double buffered) instead of every thread walking the
// row-major factor with one dependent L2 round trip per row (390 us at
// n_d = 400, r = 36; ~15 us tiled).
constexpr int kPgTile = 32;
constexpr int kPgThreads = 256;  // a light CTA: it must fit beside a persistent mode-0 CTA
constexpr int kPgPairs = 8;      // (l, j) pairs per thread: r^2 <= 2048 (r <= 45)
__global__ void __launch_bounds__(kPgThreads) pgram_kernel(const Ctrl* ctrl, const double* __restrict__ left,
                                                            int capr, double* pg) {
  extern __shared__ double tile[];  // 2 x kPgTile x r
  const long long n_d = ctrl->n_d;
  const int r = ctrl->r;
  const int tid = threadIdx.x;
  const int npair = r * r;
  int pl[kPgPairs], pj[kPgPairs];
  bool act[kPgPairs];
  double acc[kPgPairs];
#pragma unroll
  for (int q = 0; q < kPgPairs; ++q) {
    const int idx = tid + kPgThreads * q;
    pl[q] = idx < npair ? idx % r : 0;
    pj[q] = idx < npair ? idx / r : 0;
    act[q] = idx < npair && pl[q] <= pj[q];
    acc[q] = 0.0;
  }
  const long long ntiles = (n_d + kPgTile - 1) / kPgTile;
  auto load = [&](long long t, double* dst) {
    const long long i0 = t * kPgTile;
    for (int e = tid; e < kPgTile * r; e += kPgThreads) {
      const int ii = e / r, c = e % r;
      dst[e] = (i0 + ii < n_d) ? left[(i0 + ii) * capr + c] : 0.0;
    }
  };
  if (ntiles > 0) load(0, tile);
  __syncthreads();
  for (long long t = 0; t < ntiles; ++t) {
    const double* cur = tile + (t & 1) * kPgTile * r;
    if (t + 1 < ntiles) load(t + 1, tile + ((t + 1) & 1) * kPgTile * r);
#pragma unroll
    for (int q = 0; q < kPgPairs; ++q) {
      if (!act[q]) continue;
      double sacc = acc[q];
#pragma unroll 8
      for (int ii = 0; ii < kPgTile; ++ii) {
        const double w = cur[ii * r + pj[q]];
        if (w != 0.0) sacc += cur[ii * r + pl[q]] * w;
      }
      acc[q] = sacc;
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < kPgPairs; ++q)
    if (act[q]) {
      pg[pl[q] + pj[q] * r] = acc[q];
      pg[pj[q] + pl[q] * r] = acc[q];
    }
  // r > 45: the remaining pairs the slow way (not reached by the configs)
  for (int idx = tid + kPgThreads * kPgPairs; idx < npair; idx += kPgThreads) {
    const int l = idx % r, j = idx / r;
    if (l > j) continue;
    double sacc = 0.0;
    for (long long i = 0; i < n_d; ++i) {
      const double w = left[i * capr + j];
      if (w == 0.0) continue;
      sacc += left[i * capr + l] * w;
    }
    pg[l + j * r] = sacc;
    pg[j + l * r] = sacc;
  }
}

// out[j] = sum over the nblk per-block partials of column j (j < r): a warp per
// column, lanes stride the blocks so every load is in flight at once, fixed
// shuffle tree. Pass 2, pass 3 and the inner kernel all sum in this order, so
// they see the same bits. (One thread per column used to walk the ~180
// partials one dependent L2 round trip at a time.)
__device__ __forceinline__ void column_sums(const double* __restrict__ part, int nblk, int capr,
                                            int r, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = wid; j < r; j += nw) {
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s += part[(long long)b * (capr + 1) + j];
    s = warp_sum(s);
    if (lane == 0) out[j] = s;
  }
}

__global__ void __launch_bounds__(256) isvd_pass1_kernel(const Ctrl* ctrl, const double* __restrict__ q,
                                                         const double* __restrict__ b, long long n,
                                                         long long rows_per, int capr,
                                                         double* __restrict__ part) {
  const int r = ctrl->r;
  const long long i0 = blockIdx.x * rows_per, i1 = min(n, i0 + rows_per);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* out = part + (long long)blockIdx.x * (capr + 1);
  for (int j = wid; j < r; j += nw) {
    const double* qj = q + (long long)j * n;
    double s = 0.0;
#pragma unroll 4
    for (long long i = i0 + lane; i < i1; i += 32) s += qj[i] * b[i];
    s = warp_sum(s);
    if (lane == 0) out[j] = s;
  }
  if (wid == nw - 1) {
    double s = 0.0;
#pragma unroll 4
    for (long long i = i0 + lane; i < i1; i += 32) s += b[i] * b[i];
    s = warp_sum(s);
    if (lane == 0) out[capr] = s;
  }
}

__global__ void __launch_bounds__(256) isvd_pass2_kernel(const Ctrl* ctrl, const double* __restrict__ q,
                                                         const double* __restrict__ b, long long n,
                                                         long long rows_per, int capr, int nblk,
                                                         const double* __restrict__ part1,
                                                         double* __restrict__ e,
                                                         double* __restrict__ part2) {
  extern __shared__ double ps[];
  const int r = ctrl->r;
  column_sums(part1, nblk, capr, r, ps);
  __syncthreads();
  const long long i0 = blockIdx.x * rows_per, i1 = min(n, i0 + rows_per);
  for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    double s = 0.0;
#pragma unroll 4
    for (int j = 0; j < r; ++j) s += q[i + (long long)j * n] * ps[j];
    e[i] = b[i] - s;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* out = part2 + (long long)blockIdx.x * (capr + 1);
  for (int j = wid; j < r; j += nw) {
    const double* qj = q + (long long)j * n;
    double s = 0.0;
#pragma unroll 4
    for (long long i = i0 + lane; i < i1; i += 32) s += qj[i] * e[i];
    s = warp_sum(s);
    if (lane == 0) out[j] = s;
  }
}

__global__ void __launch_bounds__(256) isvd_pass3_kernel(const Ctrl* ctrl, const double* __restrict__ q,
                                                         long long n, long long rows_per, int capr,
                                                         int nblk, const double* __restrict__ part2,
                                                         double* __restrict__ e,
                                                         double* __restrict__ part3) {
  extern __shared__ double ps[];
  __shared__ double red[32];
  const int r = ctrl->r;
  column_sums(part2, nblk, capr, r, ps);
  __syncthreads();
  const long long i0 = blockIdx.x * rows_per, i1 = min(n, i0 + rows_per);
  double acc = 0.0;
  for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    double s = 0.0;
#pragma unroll 4
    for (int j = 0; j < r; ++j) s += q[i + (long long)j * n] * ps[j];
    const double v = e[i] - s;
    e[i] = v;
    acc += v * v;
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) part3[blockIdx.x] = acc;
}

struct InnerArgs {
  Ctrl* ctrl;
  const SliceCtl* slot;
  const double* sigma;
  double* sigma_new;
  const double* part1;
  const double* part2;
  const double* part3;
  int nblk;
  int capr;
  double* inner;
  int use_smem;
  int wide;  // secular solver for 32 < m <= 64 (scratch in dynamic shared memory)
};

__global__ void __launch_bounds__(512) isvd_inner_kernel(InnerArgs a) {
  extern __shared__ double ism[];
  __shared__ double red[32];
  __shared__ double sh_bsq, sh_esq;
  __shared__ int sperm[33];
  const InnerLayout L = inner_layout(a.capr);
  Ctrl* c = a.ctrl;
  const int r = c->r;
  double* p = a.inner + L.p;
  TSG_CLK(0);
  {
    // p_j = sum_b part1[b][j] + sum_b part2[b][j]: a warp per column, lanes
    // stride the blocks (all loads in flight), fixed shuffle tree. (One
    // thread per column walked the ~180 partials of each array one dependent
    // L2 round trip at a time: ~55 us of the 170 us inner kernel.)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = wid; j < r; j += nw) {
      double s1 = 0.0, s2 = 0.0;
      for (int b = lane; b < a.nblk; b += 32) {
        s1 += a.part1[(long long)b * (a.capr + 1) + j];
        s2 += a.part2[(long long)b * (a.capr + 1) + j];
      }
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      if (lane == 0) p[j] = s1 + s2;
    }
  }
  double bs = 0.0, es = 0.0;
  for (int b = threadIdx.x; b < a.nblk; b += blockDim.x) {
    bs += a.part1[(long long)b * (a.capr + 1) + a.capr];
    es += a.part3[b];
  }
  bs = block_sum(bs, red);
  es = block_sum(es, red);
  if (threadIdx.x == 0) {
    sh_bsq = bs;
    sh_esq = es;
    c->proj_sq = bs;
    c->e_sq = es;
  }
  __syncthreads();
  TSG_CLK(1);
  InnerIO io;
  io.ctrl = c;
  io.r = r;
  io.sigma = a.sigma;
  io.p = p;
  io.k = sqrt(sh_esq);
  io.deg = (io.k <= kOrthEps * sqrt(sh_bsq)) ? 1 : 0;
  io.delta = a.slot->delta;
  io.pgram = a.inner + L.pg;
  io.inner = a.inner;
  io.sigma_new = a.sigma_new;
  io.capr = a.capr;
  const int m = io.deg ? r : r + 1;
  if (m <= 32) {
    if (threadIdx.x < 32) {
      double* sG = ism;
      inner_solve_warp<33>(io, sG, sG + 64 * 33);
    }
  } else {
    double* G = a.use_smem ? ism : a.inner + L.G;
    double* V = a.use_smem ? ism + (long long)m * m : a.inner + L.V;
    inner_solve_block(io, G, V, a.wide ? ism : nullptr);
  }
}

template <int RMAX>
__global__ void __launch_bounds__(256) isvd_update_kernel(const Ctrl* ctrl, const double* __restrict__ q,
                                                          const double* __restrict__ cin,
                                                          const double* __restrict__ e,
                                                          const double* __restrict__ b,
                                                          const double* __restrict__ inner,
                                                          const double* __restrict__ sigma_new,
                                                          long long n, int capr,
                                                          double* __restrict__ qn,
                                                          double* __restrict__ cn,
                                                          double* __restrict__ part) {
  __shared__ double red[32];
  const InnerLayout L = inner_layout(capr);
  double dacc = 0.0, cacc = 0.0;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if constexpr (RMAX > 0)
    update_rows<RMAX>(ctrl, q, cin, e, b, inner + L.W, inner + L.M, inner + L.w, sigma_new, n, tid,
                      n, stride, qn, cn, dacc, cacc);
  else
    update_rows_generic(ctrl, q, cin, e, b, inner + L.W, inner + L.M, inner + L.w, sigma_new, n,
                        tid, n, stride, qn, cn, dacc, cacc);
  dacc = block_sum(dacc, red);
  cacc = block_sum(cacc, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = dacc;
    part[2 * blockIdx.x + 1] = cacc;
  }
}

// Split-path row update with the small factors in shared memory: a thread
// owns a row and keeps its 2 x RN outputs in registers while it streams the
// row's r entries of Q and of the core once (coalesced over the rows); W and
// M^T are read as warp-wide broadcasts (ld.shared.v2). Each output is the same
// l-ordered sum as update_rows (bit-identical), without its LDG per FMA and
// its 2 x RMAX register row copies: 128 -> ~20 us at n = 46656, r = 36.
// RN >= r_new (zero-padded columns).
template <int RN>
__global__ void __launch_bounds__(128) isvd_update_acc_kernel(
    const Ctrl* ctrl, const double* __restrict__ q, const double* __restrict__ cin,
    const double* __restrict__ e, const double* __restrict__ b, const double* __restrict__ inner,
    const double* __restrict__ sigma_new, long long n, int capr, double* __restrict__ qn,
    double* __restrict__ cn, double* __restrict__ part) {
  extern __shared__ double usm[];  // sW (r+1) x RN | sM r x RN | sw RN | ssig RN
  __shared__ double red[32];
  const InnerLayout L = inner_layout(capr);
  const int r = ctrl->r, rn = ctrl->r_new, deg = ctrl->degenerate;
  const int m = deg ? r : r + 1;
  const double* W = inner + L.W;
  const double* M = inner + L.M;
  const double* w = inner + L.w;
  double* sW = usm;
  double* sM = sW + (r + 1) * RN;
  double* sw = sM + r * RN;
  double* ssig = sw + RN;
  for (int idx = threadIdx.x; idx < (r + 1) * RN; idx += blockDim.x) {
    const int l = idx / RN, jn = idx % RN;
    sW[idx] = (jn < rn && l < m) ? W[l + jn * m] : 0.0;
  }
  for (int idx = threadIdx.x; idx < r * RN; idx += blockDim.x) {
    const int l = idx / RN, jn = idx % RN;
    sM[idx] = jn < rn ? M[jn + l * rn] : 0.0;
  }
  for (int jn = threadIdx.x; jn < RN; jn += blockDim.x) {
    sw[jn] = jn < rn ? w[jn] : 0.0;
    ssig[jn] = jn < rn ? sigma_new[jn] : 0.0;
  }
  __syncthreads();
  const double inv = deg ? 0.0 : 1.0 / sqrt(ctrl->e_sq);
  double dacc = 0.0, cacc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double sq[RN], sc[RN];
#pragma unroll
    for (int jn = 0; jn < RN; ++jn) sq[jn] = sc[jn] = 0.0;
    for (int l = 0; l < r; ++l) {
      const double qv = q[i + (long long)l * n];
      const double cv = cin[i + (long long)l * n];
      const double2* wr = reinterpret_cast<const double2*>(sW + l * RN);
      const double2* mr = reinterpret_cast<const double2*>(sM + l * RN);
#pragma unroll
      for (int jn = 0; jn < RN / 2; ++jn) {
        const double2 wv = wr[jn], mv = mr[jn];
        sq[2 * jn] += qv * wv.x;
        sq[2 * jn + 1] += qv * wv.y;
        sc[2 * jn] += cv * mv.x;
        sc[2 * jn + 1] += cv * mv.y;
      }
    }
    const double qi = deg ? 0.0 : e[i] * inv;
    const double bi = b[i];
#pragma unroll
    for (int jn = 0; jn < RN; ++jn) {
      if (!deg) sq[jn] += qi * sW[r * RN + jn];
      sc[jn] += sw[jn] * bi;
      if (jn < rn) {
        qn[i + (long long)jn * n] = sq[jn];
        cn[i + (long long)jn * n] = sc[jn];
        const double diff = sc[jn] - sq[jn] * ssig[jn];
        dacc += diff * diff;
        cacc += sc[jn] * sc[jn];
      }
    }
  }
  dacc = block_sum(dacc, red);
  cacc = block_sum(cacc, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = dacc;
    part[2 * blockIdx.x + 1] = cacc;
  }
}

__global__ void isvd_left_kernel(const Ctrl* ctrl, const double* __restrict__ left, int capr,
                                 const double* __restrict__ inner,
                                 double* __restrict__ left_new) {
  const InnerLayout L = inner_layout(capr);
  left_rows(ctrl, left, ctrl->n_d, capr, inner + L.U, left_new,
            blockIdx.x * (long long)blockDim.x + threadIdx.x, (long long)gridDim.x * blockDim.x);
}

__global__ void isvd_finalize_kernel(Ctrl* c, const SliceCtl* sl, const double* __restrict__ part,
                                     int nblk, RecRing* ring, int order, SpatialRanks sr) {
  __shared__ double red[32];
  double d = 0.0, cs = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
    d += part[2 * b];
    cs += part[2 * b + 1];
  }
  d = block_sum(d, red);
  cs = block_sum(cs, red);
  if (threadIdx.x == 0) finalize_record(c, sl, d, cs, ring, order, sr);
}

// ------------------------------------------------------- other entry points
__global__ void zero_slice_kernel(Ctrl* c, const SliceCtl* sl, double* left, int capr,
                                  RecRing* ring, int order, SpatialRanks sr) {
  const long long nd = c->n_d;
  for (int j = threadIdx.x; j < capr; j += blockDim.x) left[nd * capr + j] = 0.0;
  __syncthreads();
  if (threadIdx.x != 0) return;
  (void)sl;
  Metrics m;
  m.slice_index = nd;
  c->n_d = nd + 1;
  for (int k = 0; k < kMaxD; ++k) m.ranks[k] = (k + 1 < order) ? sr.v[k] : 0;
  m.ranks[order - 1] = c->r;
  m.slice_norm = 0.0;
  m.projected_norm = 0.0;
  for (int k = 0; k < kMaxD; ++k) m.mode_residuals[k] = 0.0;
  const double booked = c->squared_error + c->nonstream_discarded_sq;
  m.error_estimate = c->total_input_sq <= 0.0 ? 0.0 : sqrt(fmax(booked, 0.0) / c->total_input_sq);
  m.expanded_mask = 0;
  m.trunc_margin = 0.0;
  m.sweeps = 0;
  publish(c, m, ring);
}

__global__ void init_isvd_kernel(Ctrl* c, const double* __restrict__ core, long long n, int r,
                                 const double* __restrict__ lam, double* __restrict__ q,
                                 double* __restrict__ sigma, const double* __restrict__ left_cm,
                                 long long n_init, double* __restrict__ left_rm, int capr) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long idx = tid; idx < n * r; idx += stride) {
    const int j = (int)(idx / n);
    const double inv = 1.0 / sqrt(lam[j]);  // streaming.cpp:96-108
    q[idx] = core[idx] * inv;
  }
  for (long long idx = tid; idx < n_init * capr; idx += stride) {
    const long long i = idx / capr;
    const int j = (int)(idx % capr);
    left_rm[idx] = j < r ? left_cm[i + j * n_init] : 0.0;
  }
  if (tid < r) sigma[tid] = sqrt(lam[tid]);
  if (tid == 0) {
    c->r = r;
    c->n_d = n_init;
    c->insertions = 0;
  }
}

__global__ void coupling_kernel(Ctrl* c, const double* __restrict__ core,
                                const double* __restrict__ q, const double* __restrict__ sigma,
                                long long n, int r) {
  __shared__ double red[32];
  double d = 0.0, cs = 0.0;
  for (long long idx = threadIdx.x; idx < n * r; idx += blockDim.x) {
    const int j = (int)(idx / n);
    const double cv = core[idx];
    const double diff = cv - q[idx] * sigma[j];
    d += diff * diff;
    cs += cv * cv;
  }
  d = block_sum(d, red);
  cs = block_sum(cs, red);
  if (threadIdx.x == 0) {
    c->coupling_diff_sq = d;
    c->core_sq = cs;
    c->status = (sqrt(d) > kCouplingTol * sqrt(cs) + 1e-300) ? 2 : 0;
  }
}

inline int grid_for(long long total, int block = 256, int cap = 148 * 8) {
  long long g = (total + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// Dynamic shared memory beyond the default needs the attribute whenever
// static + dynamic exceeds 48 KB; set it for every requested size.
template <class K>
void ensure_smem(K kernel, size_t bytes) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

#include "isvd_small.cuh"
#include "isvd_grid.cuh"
#include "isvd_cta.cuh"
#include "isvd_clu.cuh"

namespace {
template <int RMAX, int RPT, bool QREG = true>
void launch_small(const IsvdBufs& B0, cudaStream_t st) {
  IsvdBufs B = B0;
  const size_t core_bytes = sizeof(double) * (size_t)B.n * (size_t)B.r_hint;
  B.stage_core = core_bytes <= 120 * 1024 ? 1 : 0;
  const size_t smem = sizeof(double) * kSmallFixed + (B.stage_core ? core_bytes + 16 : 16);
  ensure_smem(isvd_small_kernel<RMAX, RPT, QREG>, smem);
  isvd_small_kernel<RMAX, RPT, QREG><<<1, 512, smem, st>>>(B);
}
template <int RMAX>
void launch_grid(const IsvdBufs& B, cudaStream_t st) {
  const int G = (int)((B.n + kGridRows - 1) / kGridRows);
  const size_t smem =
      sizeof(double) * ((size_t)kSmallFixed + (size_t)B.n + 2 * RMAX * kGridRows + 2);
  ensure_smem(isvd_grid_kernel<RMAX>, smem);
  isvd_grid_kernel<RMAX><<<G, 256, smem, st>>>(B);
}
template <int RMAX, int RPT>
void launch_cta(const IsvdBufs& B, cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t)cta::smem_doubles(B.n, B.r_hint);
  ensure_smem(cta::isvd_cta_kernel<RMAX, RPT>, smem);
  cta::isvd_cta_kernel<RMAX, RPT><<<1, cta::kThreads, smem, st>>>(B);
}
template <int RMAX>
void launch_clu(const IsvdBufs& B, cudaStream_t st) {
  // rows per CTA: even (16-byte aligned bulk copies), at most 128 (one per thread)
  int G = (int)((B.n + clu::kT - 1) / clu::kT);
  if (G > clu::kMaxG) G = clu::kMaxG;
  if (G < 1) G = 1;
  int R0 = (int)((B.n + G - 1) / G);
  R0 = (R0 + 1) & ~1;
  G = (int)((B.n + R0 - 1) / R0);
  const size_t smem = sizeof(double) * (size_t)clu::smem_doubles(R0, B.r_hint);
  ensure_smem(clu::isvd_clu_kernel<RMAX, 1>, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G, 1, 1);
  cfg.blockDim = dim3(clu::kT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, clu::isvd_clu_kernel<RMAX, 1>, B, R0);
}
void launch_clu_r(const IsvdBufs& B, cudaStream_t st) {
  const int rh = B.r_hint;
  if (rh <= 8) launch_clu<8>(B, st);
  else if (rh <= 12) launch_clu<12>(B, st);
  else if (rh <= 14) launch_clu<14>(B, st);
  else if (rh <= 16) launch_clu<16>(B, st);
  else if (rh <= 20) launch_clu<20>(B, st);
  else launch_clu<24>(B, st);
}
void launch_cta_r(const IsvdBufs& B, cudaStream_t st) {
  const int rh = B.r_hint;
  if (rh <= 8) launch_cta<8, 4>(B, st);
  else if (rh <= 12) launch_cta<12, 4>(B, st);
  else if (rh <= 14) launch_cta<14, 4>(B, st);
  else if (rh <= 16) launch_cta<16, 4>(B, st);
  else if (rh <= 20) launch_cta<20, 4>(B, st);
  else launch_cta<24, 4>(B, st);
}
// n <= 512 * RPT, r_hint <= RMAX; false when not applicable
bool try_small(const IsvdBufs& B, cudaStream_t st) {
  static const bool off = std::getenv("TSG_OLD_ISVD") != nullptr;
  static const bool small_only = std::getenv("TSG_ISVD_SMALL") != nullptr;
  static const int use_cta = [] {
    const char* e = std::getenv("TSG_ISVD_CTA");
    return e ? std::atoi(e) : 1;
  }();
  if (off || B.r_hint < 1 || B.r_hint > 31) return false;
  const int rh = B.r_hint;
  // single CTA, branch-free inner solve (isvd_cta.cuh)
  // cluster of CTAs (isvd_clu.cuh): rows split, DSMEM reductions
  if (use_cta == 1 && !small_only && B.n <= clu::kMaxG * clu::kT && B.n >= 64 && rh <= 24 &&
      (B.n % 2) == 0) {
    launch_clu_r(B, st);
    return true;
  }
  // (Q columns and b bulk-copied to shared memory: even n, and they must fit)
  if (use_cta && !small_only && B.n <= 4 * cta::kThreads && rh <= 24 && (B.n % 2) == 0 &&
      sizeof(double) * cta::smem_doubles(B.n, rh) <= 227 * 1024) {
    launch_cta_r(B, st);
    return true;
  }
  if (!small_only && B.hand && B.gsync && B.n <= kGridMaxRows) {
    if (rh <= 4) launch_grid<4>(B, st);
    else if (rh <= 8) launch_grid<8>(B, st);
    else if (rh <= 12) launch_grid<12>(B, st);
    else if (rh <= 16) launch_grid<16>(B, st);
    else if (rh <= 24) launch_grid<24>(B, st);
    else launch_grid<32>(B, st);
    return true;
  }
  if (B.n <= 512) {
    if (rh <= 4) launch_small<4, 1>(B, st);
    else if (rh <= 8) launch_small<8, 1>(B, st);
    else if (rh <= 12) launch_small<12, 1>(B, st);
    else if (rh <= 16) launch_small<16, 1>(B, st);
    else if (rh <= 24) launch_small<24, 1>(B, st);
    else launch_small<32, 1>(B, st);
    return true;
  }
  if (B.n <= 1024) {
    if (rh <= 4) launch_small<4, 2>(B, st);
    else if (rh <= 8) launch_small<8, 2>(B, st);
    else if (rh <= 12) launch_small<12, 2>(B, st);
    else if (rh <= 16) launch_small<16, 2>(B, st);
    else if (rh <= 24) launch_small<24, 2, false>(B, st);
    else launch_small<32, 2, false>(B, st);
    return true;
  }
  return false;
}
}  // namespace

// Fused single-CTA chain when n <= kFusedRows and r + 1 <= 32. Beyond the
// grid kernel's 4096 rows one CTA is the slower choice (config 5 at
// n = 8000: 0.67 ms per insertion against ~0.1 ms for the split kernels).
constexpr long long kFusedRows = 4096;

void launch_isvd(const IsvdBufs& B0, cudaStream_t st) {
  if (try_small(B0, st)) {
    g_launches += 1;
    return;
  }
  if (B0.commit_modes > 0) {
    launch_commit_modes(B0.ctrl, B0.slot, 0, B0.commit_modes, 1, st);
  }
  const IsvdBufs& B = B0;
  const long long n = B.n;
  const int capr = B.capr;
  SpatialRanks sr;
  for (int k = 0; k < kMaxD; ++k) sr.v[k] = B.spatial_ranks[k];
  if (n <= kFusedRows && B.r_hint + 1 <= 32 && B.r_hint >= 1) {
    const size_t smem = sizeof(double) * (n + 3 * 32 * 33 + 2 * 33 * 33 + 66);
    switch ((B.r_hint + 3) / 4) {
#define TSG_FUSED(R)                                  \
  case R / 4:                                         \
    ensure_smem(isvd_fused_kernel<R>, smem);          \
    isvd_fused_kernel<R><<<1, 512, smem, st>>>(B);    \
    break;
      TSG_FUSED(4)
      TSG_FUSED(8)
      TSG_FUSED(12)
      TSG_FUSED(16)
      TSG_FUSED(20)
      TSG_FUSED(24)
      TSG_FUSED(28)
      TSG_FUSED(32)
#undef TSG_FUSED
    }
    g_launches += 1;
    return;
  }
  long long rows_per = 256;
  long long nblk = (n + rows_per - 1) / rows_per;
  if (nblk > 296) {
    nblk = 296;
    rows_per = (n + nblk - 1) / nblk;
  }
  const int nb = (int)nblk;
  double* part1 = B.partial;
  double* part2 = part1 + (long long)nb * (capr + 1);
  double* part3 = part2 + (long long)nb * (capr + 1);
  double* part4 = part3 + nb;
  const InnerLayout L = inner_layout(capr);
  // TSG_SPLIT_CLK=1 (with TSG_NO_GRAPH=1): CUDA events between the split
  // kernels, averages printed every 32 insertions (diagnostic only)
  static const bool clk = std::getenv("TSG_SPLIT_CLK") != nullptr;
  static cudaEvent_t cev[10];
  static double cacc[10];
  static int ccount = 0;
  static bool cinit = false, clive = false;
  auto mark = [&](int i) {
    if (!clk) return;
    cudaEventRecord(cev[i], st);
  };
  if (clk) {
    if (!cinit) {
      for (auto& e : cev) cudaEventCreate(&e);
      cinit = true;
    }
    if (clive) {
      cudaEventSynchronize(cev[9]);
      for (int i = 0; i < 9; ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, cev[i], cev[i + 1]);
        cacc[i] += ms;
      }
      if (++ccount % 32 == 0) {
        static const char* nm[9] = {"pgram", "pass1", "pass2", "pass3", "inner", "update", "left", "finalize", "-"};
        std::fprintf(stderr, "split insertion (n %lld, capr %d), avg us:", n, capr);
        for (int i = 0; i < 8; ++i) std::fprintf(stderr, " %s %.1f", nm[i], cacc[i] / ccount * 1e3);
        std::fprintf(stderr, "\n");
      }
    }
    clive = true;
  }
  mark(0);
  pgram_kernel<<<1, kPgThreads, sizeof(double) * 2 * kPgTile * capr, st>>>(B.ctrl, B.left, capr,
                                                                           B.inner + L.pg);
  mark(1);
  isvd_pass1_kernel<<<nb, 256, 0, st>>>(B.ctrl, B.q, B.b, n, rows_per, capr, part1);
  mark(2);
  isvd_pass2_kernel<<<nb, 256, sizeof(double) * capr, st>>>(B.ctrl, B.q, B.b, n, rows_per, capr,
                                                            nb, part1, B.e, part2);
  mark(3);
  isvd_pass3_kernel<<<nb, 256, sizeof(double) * capr, st>>>(B.ctrl, B.q, n, rows_per, capr, nb,
                                                            part2, B.e, part3);
  mark(4);
  InnerArgs ia;
  ia.ctrl = B.ctrl;
  ia.slot = B.slot;
  ia.sigma = B.sigma;
  ia.sigma_new = B.sigma_new;
  ia.part1 = part1;
  ia.part2 = part2;
  ia.part3 = part3;
  ia.nblk = nb;
  ia.capr = capr;
  ia.inner = B.inner;
  const long long m = capr + 1;
  size_t smem = 2 * m * m * sizeof(double);
  ia.use_smem = smem <= 160 * 1024 ? 1 : 0;
  if (!ia.use_smem) smem = 0;
  smem = std::max(smem, sizeof(double) * 3 * 32 * 33);
  static const bool no_wide = std::getenv("TSG_NO_WIDE_SECULAR") != nullptr;  // A/B: block Jacobi
  ia.wide = no_wide ? 0 : 1;
  if (ia.wide) smem = std::max(smem, sizeof(double) * (size_t)kWideScratch);
  ensure_smem(isvd_inner_kernel, smem);
  isvd_inner_kernel<<<1, 512, smem, st>>>(ia);
  mark(5);
  int gu = grid_for(n, 256, 148 * 4);
  static const bool old_update = std::getenv("TSG_OLD_UPDATE") != nullptr;  // A/B
  const int rn_max = B.r_hint + 1;  // r_new <= r + 1 <= r_hint + 1
  if (!old_update && rn_max <= 48 && B.r_hint >= 1) {
    gu = grid_for(n, 128, 148 * 4);
    const size_t usm = sizeof(double) * ((size_t)(2 * rn_max + 1) * 48 + 96);
#define TSG_UPD(RN)                                                                          \
  {                                                                                          \
    ensure_smem(isvd_update_acc_kernel<RN>, usm);                                            \
    isvd_update_acc_kernel<RN><<<gu, 128, usm, st>>>(B.ctrl, B.q, B.c, B.e, B.b, B.inner,    \
                                                     B.sigma_new, n, capr, B.qn, B.cn, part4); \
  }
    if (rn_max <= 16) TSG_UPD(16)
    else if (rn_max <= 24) TSG_UPD(24)
    else if (rn_max <= 32) TSG_UPD(32)
    else if (rn_max <= 40) TSG_UPD(40)
    else TSG_UPD(48)
#undef TSG_UPD
  } else if (capr <= 16)
    isvd_update_kernel<16><<<gu, 256, 0, st>>>(B.ctrl, B.q, B.c, B.e, B.b, B.inner, B.sigma_new, n,
                                               capr, B.qn, B.cn, part4);
  else if (capr <= 32)
    isvd_update_kernel<32><<<gu, 256, 0, st>>>(B.ctrl, B.q, B.c, B.e, B.b, B.inner, B.sigma_new, n,
                                               capr, B.qn, B.cn, part4);
  else if (capr <= 48)
    isvd_update_kernel<48><<<gu, 256, 0, st>>>(B.ctrl, B.q, B.c, B.e, B.b, B.inner, B.sigma_new, n,
                                               capr, B.qn, B.cn, part4);
  else
    isvd_update_kernel<0><<<gu, 256, 0, st>>>(B.ctrl, B.q, B.c, B.e, B.b, B.inner, B.sigma_new, n,
                                              capr, B.qn, B.cn, part4);
  mark(6);
  isvd_left_kernel<<<grid_for(B.cap_rows * capr), 256, 0, st>>>(B.ctrl, B.left, capr, B.inner,
                                                                 B.left_new);
  mark(7);
  isvd_finalize_kernel<<<1, 256, 0, st>>>(B.ctrl, B.slot, part4, gu, B.ring, B.order, sr);
  mark(8);
  mark(9);
  g_launches += 8;
}

// Periodic re-orthogonalization (ISVDOptions::reorthogonalize_every,
// isvd.cpp:243-248): modified Gram-Schmidt over the columns of the streaming
// factor (GrowableRowMatrix::reorthogonalize, isvd.cpp:102-124) and of the
// right factor (orthonormalize_columns, linalg.cpp:64-78), in that order.
// One CTA per matrix: for each column j, the dots with the earlier columns
// are taken one at a time against the partially updated column (the
// reference's order); reductions are fixed-order block sums. Element (i, j)
// lives at a[i * rs + j * cs]; rows = ctrl->n_d (left) or n (right), cols =
// ctrl->r (both as the insertion left them).
__global__ void __launch_bounds__(1024) reorth_kernel(const Ctrl* ctrl, double* a, long long rows_fixed,
                                                       long long rs, long long cs) {
  __shared__ double scratch[32];
  const long long rows = rows_fixed > 0 ? rows_fixed : ctrl->n_d;
  const int cols = ctrl->r;
  for (int j = 0; j < cols; ++j) {
    for (int i = 0; i < j; ++i) {
      double d = 0.0;
      for (long long r = threadIdx.x; r < rows; r += blockDim.x) d = fma(a[r * rs + i * cs], a[r * rs + j * cs], d);
      d = block_sum(d, scratch);
      for (long long r = threadIdx.x; r < rows; r += blockDim.x) a[r * rs + j * cs] -= d * a[r * rs + i * cs];
      __syncthreads();
    }
    double sq = 0.0;
    for (long long r = threadIdx.x; r < rows; r += blockDim.x) {
      const double v = a[r * rs + j * cs];
      sq = fma(v, v, sq);
    }
    sq = block_sum(sq, scratch);
    const double nrm = sqrt(sq);
    if (nrm > 0.0)
      for (long long r = threadIdx.x; r < rows; r += blockDim.x) a[r * rs + j * cs] /= nrm;
    __syncthreads();
  }
}

void launch_reorth(const Ctrl* ctrl, double* left, int capr, double* q, long long n, cudaStream_t st) {
  reorth_kernel<<<1, 1024, 0, st>>>(ctrl, left, 0, capr, 1);
  reorth_kernel<<<1, 1024, 0, st>>>(ctrl, q, n, 1, n);
  g_launches += 2;
}

void launch_zero_slice(Ctrl* ctrl, const SliceCtl* slot, double* left, int capr, RecRing* ring,
                       int order, const long long* spatial, cudaStream_t st) {
  SpatialRanks sr;
  for (int k = 0; k < kMaxD; ++k) sr.v[k] = spatial[k];
  zero_slice_kernel<<<1, 256, 0, st>>>(ctrl, slot, left, capr, ring, order, sr);
  ++g_launches;
}

void launch_init_isvd(Ctrl* ctrl, const double* core, long long n, int r, const double* evals_last,
                      double* q, double* sigma, const double* left_cm, long long n_init,
                      double* left_rm, int capr, cudaStream_t st) {
  const long long total = n * r > n_init * capr ? n * r : n_init * capr;
  init_isvd_kernel<<<grid_for(total), 256, 0, st>>>(ctrl, core, n, r, evals_last, q, sigma,
                                                    left_cm, n_init, left_rm, capr);
  ++g_launches;
}

void launch_coupling_check(Ctrl* ctrl, const double* core, const double* q, const double* sigma,
                           long long n, int r, double* partial, cudaStream_t st) {
  (void)partial;
  coupling_kernel<<<1, 1024, 0, st>>>(ctrl, core, q, sigma, n, r);
  ++g_launches;
}

}  // namespace tsg
