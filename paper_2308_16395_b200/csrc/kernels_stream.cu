// Per-slice streaming update kernels (reference proj/src/streaming.cpp and
// proj/src/isvd.cpp): mode-k projection with fused residual norm, the
// branch decision, ledgers, the incremental SVD row insertion and the core
// rotation with the coupling check fused into its epilogue.
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"
#include "proj_dmma.cuh"

namespace tsg {

namespace {

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// ------------------------------------------------------------ projection
// Generic fused projection (any mode): tile = BC mode-k fibres staged in
// shared memory together with U; P = U^T X_tile, then E = X - U P and the
// squared norms (streaming.cpp:128-133, tensor.cpp:106-162).
__global__ void __launch_bounds__(256) project_kernel(ProjArgs a, int BC, int u_smem) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  const long long left = a.v.left, N = a.v.n, right = a.v.right;
  const int R = a.R;
  const long long cols = left * right;
  const long long ntiles = (cols + BC - 1) / BC;
  double* Us = sm;
  double* Xs = Us + (u_smem ? N * R : 0);
  double* Ps = Xs + N * BC;
  if (u_smem)
    for (long long idx = threadIdx.x; idx < N * R; idx += blockDim.x) {
      const long long i = idx % N, j = idx / N;
      Us[i * R + j] = a.u[idx];
    }
  double racc = 0.0, xacc = 0.0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long c0 = tile * BC;
    __syncthreads();
    for (long long e = threadIdx.x; e < N * BC; e += blockDim.x) {
      long long i, j;
      if (left == 1) {
        j = e / N;
        i = e % N;
      } else {
        j = e % BC;
        i = e / BC;
      }
      const long long c = c0 + j;
      double val = 0.0;
      if (c < cols) {
        const long long l = c % left, r = c / left;
        val = a.x[r * left * N + i * left + l];
      }
      Xs[i * BC + j] = val;
    }
    __syncthreads();
    for (long long o = threadIdx.x; o < (long long)R * BC; o += blockDim.x) {
      const long long c = o % BC, j = o / BC;
      double s = 0.0;
      for (long long i = 0; i < N; ++i) {
        const double uij = u_smem ? Us[i * R + j] : __ldg(&a.u[i + j * N]);
        s += uij * Xs[i * BC + c];
      }
      Ps[j * BC + c] = s;
      const long long cc = c0 + c;
      if (a.p && cc < cols) {
        const long long l = cc % left, r = cc / left;
        a.p[r * left * R + j * left + l] = s;
      }
    }
    __syncthreads();
    if (a.residual) {
      for (long long e = threadIdx.x; e < N * BC; e += blockDim.x) {
        long long i, j;
        if (left == 1) {
          j = e / N;
          i = e % N;
        } else {
          j = e % BC;
          i = e / BC;
        }
        const long long c = c0 + j;
        if (c >= cols) continue;
        const double x = Xs[i * BC + j];
        double s = 0.0;
        for (int jj = 0; jj < R; ++jj) {
          const double uij = u_smem ? Us[i * R + jj] : __ldg(&a.u[i + (long long)jj * N]);
          s += uij * Ps[jj * BC + j];
        }
        const double ev = x - s;
        racc += ev * ev;
        xacc += x * x;
        if (a.e) {
          const long long l = c % left, r = c / left;
          a.e[r * left * N + i * left + l] = ev;
        }
      }
    }
  }
  racc = block_sum(racc, red);
  xacc = block_sum(xacc, red);
  if (threadIdx.x == 0 && a.partial) {
    a.partial[2 * blockIdx.x] = racc;
    a.partial[2 * blockIdx.x + 1] = xacc;
  }
}

// ----------------------------------------------------------- decisions
__global__ void decide_kernel(DecideArgs a) {
  __shared__ double red[32];
  __shared__ double res[kMaxD];
  __shared__ double xsq;
  for (int k = a.first_mode; k < a.nmodes; ++k) {
    double acc = 0.0, acx = 0.0;
    for (int b = threadIdx.x; b < a.cnt[k]; b += blockDim.x) {
      acc += a.partial[a.off[k] + 2 * b];
      acx += a.partial[a.off[k] + 2 * b + 1];
    }
    acc = block_sum(acc, red);
    acx = block_sum(acx, red);
    if (threadIdx.x == 0) {
      res[k] = acc;
      if (k == 0) xsq = acx;
    }
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  Ctrl* c = a.ctrl;
  if (a.first_mode == 0) {
    c->slice_sq = xsq;
    c->zero_slice = (xsq == 0.0);
    const double slice_norm = sqrt(xsq);
    c->delta = a.tau * slice_norm / sqrt((double)a.order);  // streaming.cpp:187-188
  }
  int em = -1;
  for (int k = a.first_mode; k < a.nmodes; ++k) {
    c->res_sq[k] = res[k];
    if (em < 0 && !(sqrt(res[k]) <= c->delta)) em = k;  // streaming.cpp:135
  }
  c->expand_mode = em;
}

__global__ void commit_modes_kernel(Ctrl* c, int m0, int m1, int with_total) {
  if (threadIdx.x != 0) return;
  if (with_total) {
    const double sn = sqrt(c->slice_sq);
    c->total_input_sq += sn * sn;  // streaming.cpp:169
  }
  for (int k = m0; k < m1; ++k) {
    const double rn = sqrt(c->res_sq[k]);
    c->nonstream_discarded_sq += rn * rn;  // streaming.cpp:137
  }
}

__global__ void ledger_add_kernel(Ctrl* c, const double* v) {
  if (threadIdx.x == 0) c->nonstream_discarded_sq += *v;  // streaming.cpp:150
}

// ------------------------------------------------------------------ ISVD
// p_gram = left^T left before the insertion (isvd.cpp:86-100,
// streaming.cpp:199): per-(l,j) sums in row order, zero entries skipped,
// lower triangle mirrored.
__global__ void pgram_kernel(const Ctrl* ctrl, const double* __restrict__ left, long long n_d,
                             int capr, double* __restrict__ pg) {
  const int r = ctrl->r;
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

// Two classical Gram-Schmidt passes (CGS2) split b = Q p + e
// (isvd.cpp:172-191 does two MGS passes; same projector, parallel form).
// Pass 1: partial p1 = Q^T b and ||b||^2 per CTA.
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
    for (long long i = i0 + lane; i < i1; i += 32) s += qj[i] * b[i];
    s = warp_sum(s);
    if (lane == 0) out[j] = s;
  }
  if (wid == nw - 1) {
    double s = 0.0;
    for (long long i = i0 + lane; i < i1; i += 32) s += b[i] * b[i];
    s = warp_sum(s);
    if (lane == 0) out[capr] = s;
  }
}

// Pass 2: e1 = b - Q p1 on the CTA's rows, then partial p2 = Q^T e1.
__global__ void __launch_bounds__(256) isvd_pass2_kernel(const Ctrl* ctrl, const double* __restrict__ q,
                                                         const double* __restrict__ b, long long n,
                                                         long long rows_per, int capr, int nblk,
                                                         const double* __restrict__ part1,
                                                         double* __restrict__ e,
                                                         double* __restrict__ part2) {
  extern __shared__ double ps[];
  const int r = ctrl->r;
  for (int j = threadIdx.x; j < r; j += blockDim.x) {
    double s = 0.0;
    for (int bb = 0; bb < nblk; ++bb) s += part1[(long long)bb * (capr + 1) + j];
    ps[j] = s;
  }
  __syncthreads();
  const long long i0 = blockIdx.x * rows_per, i1 = min(n, i0 + rows_per);
  for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < r; ++j) s += q[i + (long long)j * n] * ps[j];
    e[i] = b[i] - s;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* out = part2 + (long long)blockIdx.x * (capr + 1);
  for (int j = wid; j < r; j += nw) {
    const double* qj = q + (long long)j * n;
    double s = 0.0;
    for (long long i = i0 + lane; i < i1; i += 32) s += qj[i] * e[i];
    s = warp_sum(s);
    if (lane == 0) out[j] = s;
  }
}

// Pass 3: e = e1 - Q p2 and partial ||e||^2.
__global__ void __launch_bounds__(256) isvd_pass3_kernel(const Ctrl* ctrl, const double* __restrict__ q,
                                                         long long n, long long rows_per, int capr,
                                                         int nblk, const double* __restrict__ part2,
                                                         double* __restrict__ e,
                                                         double* __restrict__ part3) {
  extern __shared__ double ps[];
  __shared__ double red[32];
  const int r = ctrl->r;
  for (int j = threadIdx.x; j < r; j += blockDim.x) {
    double s = 0.0;
    for (int bb = 0; bb < nblk; ++bb) s += part2[(long long)bb * (capr + 1) + j];
    ps[j] = s;
  }
  __syncthreads();
  const long long i0 = blockIdx.x * rows_per, i1 = min(n, i0 + rows_per);
  double acc = 0.0;
  for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < r; ++j) s += q[i + (long long)j * n] * ps[j];
    const double v = e[i] - s;
    e[i] = v;
    acc += v * v;
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) part3[blockIdx.x] = acc;
}

}  // namespace

// Scratch layout of the inner SVD (all column-major):
struct InnerLayout {
  long long W, U, M, w, lam, G, V, p, perm;
  long long total;
};
__host__ __device__ static InnerLayout inner_layout(int capr) {
  const long long m = capr + 1;
  InnerLayout L;
  long long o = 0;
  L.W = o; o += m * m;     // eigenvectors of S'^T S' (kept columns = right factor)
  L.U = o; o += m * m;     // left factor P' of S'
  L.M = o; o += m * m;     // core rotation M = P'_top^T p_gram
  L.w = o; o += m;         // last row of P'
  L.lam = o; o += m;       // eigenvalues
  L.G = o; o += m * m;     // global fallback for large inner problems
  L.V = o; o += m * m;
  L.p = o; o += m;         // p = p1 + p2
  L.perm = o; o += m;      // int scratch (stored in doubles' space)
  L.total = o;
  return L;
}
int isvd_inner_scratch(int capr) { return (int)inner_layout(capr).total; }

namespace {

struct InnerArgs {
  Ctrl* ctrl;
  const double* sigma;
  double* sigma_new;
  const double* part1;
  const double* part2;
  const double* part3;
  int nblk;
  int capr;
  const double* pgram;
  double* inner;
  int use_smem;
};

// small_svd_truncated on the (r+1)-sized middle matrix (isvd.cpp:201-215,
// linalg.cpp:210-259) plus the core-rotation factors (streaming.cpp:203-208).
__global__ void __launch_bounds__(512) isvd_inner_kernel(InnerArgs a) {
  extern __shared__ unsigned char smraw[];
  __shared__ double red[32];
  __shared__ double sh_k, sh_bsq;
  __shared__ int sh_deg, sh_rank;
  __shared__ double sh_disc;
  const InnerLayout L = inner_layout(a.capr);
  Ctrl* c = a.ctrl;
  const int r = c->r;
  double* p = a.inner + L.p;
  // reduce the projection passes
  for (int j = threadIdx.x; j <= r; j += blockDim.x) {
    if (j < r) {
      double s1 = 0.0, s2 = 0.0;
      for (int b = 0; b < a.nblk; ++b) s1 += a.part1[(long long)b * (a.capr + 1) + j];
      for (int b = 0; b < a.nblk; ++b) s2 += a.part2[(long long)b * (a.capr + 1) + j];
      p[j] = s1 + s2;
    }
  }
  {
    double bs = 0.0, es = 0.0;
    for (int b = threadIdx.x; b < a.nblk; b += blockDim.x) {
      bs += a.part1[(long long)b * (a.capr + 1) + a.capr];
      es += a.part3[b];
    }
    bs = block_sum(bs, red);
    es = block_sum(es, red);
    if (threadIdx.x == 0) {
      sh_bsq = bs;
      sh_k = sqrt(es);
      sh_deg = (sh_k <= kOrthEps * sqrt(bs)) ? 1 : 0;  // isvd.cpp:191
      c->proj_sq = bs;
      c->e_sq = es;
    }
  }
  __syncthreads();
  const double k = sh_k;
  const int deg = sh_deg;
  const int m = deg ? r : r + 1;   // columns of S'
  const int rows = r + 1;          // rows of S'
  double* G;
  double* V;
  if (a.use_smem) {
    G = reinterpret_cast<double*>(smraw);
    V = G + (long long)m * m;
  } else {
    G = a.inner + L.G;
    V = a.inner + L.V;
  }
  // S'(i,j): diag(s) over [p^T k]; G = S'^T S' (gram_transposed, rows order)
  auto Sp = [&](int i, int j) -> double {
    if (i < r) return (i == j) ? a.sigma[j] : 0.0;
    return (j < r) ? p[j] : k;
  };
  double acc = 0.0;
  for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
    const int i = idx % m, j = idx / m;
    if (i > j) continue;
    double dot = 0.0;
    for (int l = 0; l < rows; ++l) dot += Sp(l, i) * Sp(l, j);
    G[i + j * m] = dot;
    G[j + i * m] = dot;
    acc += (i == j) ? dot * dot : 2.0 * dot * dot;
  }
  for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x)
    V[idx] = ((idx % m) == (idx / m)) ? 1.0 : 0.0;
  const double tol = kOffDiagTolFactor * sqrt(block_sum(acc, red));
  // Jacobi (shared with sym_eig_kernel)
  struct RotL {
    double c, s, t;
    int p, q;
  };
  __shared__ RotL rot[128];
  // reuse the eigen routine through a local copy of its logic
  const int np = m + (m & 1);
  const int half = np / 2;
  int sweep = 0;
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
  // sort (stable, descending), clamp, sign rule -> lam, W
  double* lam = a.inner + L.lam;
  double* W = a.inner + L.W;
  int* perm = reinterpret_cast<int*>(a.inner + L.perm);
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
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
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
  // floor + truncation (linalg.cpp:224-240)
  if (threadIdx.x == 0) {
    const double smax = sqrt(lam[0]);
    int rank = 0;
    double disc = 0.0, margin = 0.0;
    if (smax > 0.0) {
      const double fl = kSigmaZeroFactor * smax;
      for (int i = 0; i < m; ++i)
        if (sqrt(lam[i]) <= fl) lam[i] = 0.0;
      const double budget = c->delta * c->delta;
      double s = 0.0;
      int rr = m;
      double prev_excess = -1.0;
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
    }
    sh_rank = rank;
    sh_disc = disc;
    c->trunc_margin = margin;
    c->sweeps = sweep;
    double added = disc;
    if (deg) added += k * k;
    c->added_error_sq = added;
    c->squared_error += added;  // isvd.cpp:212-215
    c->r_new = rank;
    c->degenerate = deg;
  }
  __syncthreads();
  const int rank = sh_rank;
  // sigma_new, U = S' W / sigma then MGS (linalg.cpp:250-258)
  double* U = a.inner + L.U;
  for (int j = threadIdx.x; j < rank; j += blockDim.x) a.sigma_new[j] = sqrt(lam[j]);
  for (int idx = threadIdx.x; idx < rows * rank; idx += blockDim.x) {
    const int i = idx % rows, j = idx / rows;
    double s = 0.0;
    for (int l = 0; l < m; ++l) {
      const double wl = W[l + j * m];
      if (wl == 0.0) continue;
      s += Sp(i, l) * wl;
    }
    const double inv = 1.0 / sqrt(lam[j]);
    U[i + j * rows] = s * inv;
  }
  __syncthreads();
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = 0; i < rank; ++i) {
      double* ui = U + i * rows;
      double ss = 0.0;
      for (int l = threadIdx.x; l < rows; l += blockDim.x) ss += ui[l] * ui[l];
      const double nrm = sqrt(block_sum(ss, red));
      if (nrm > 0.0)
        for (int l = threadIdx.x; l < rows; l += blockDim.x) ui[l] /= nrm;
      __syncthreads();
      for (int j = i + 1 + wid; j < rank; j += nw) {
        double* uj = U + j * rows;
        double dot = 0.0;
        for (int l = lane; l < rows; l += 32) dot += ui[l] * uj[l];
        dot = warp_sum(dot);
        for (int l = lane; l < rows; l += 32) uj[l] -= dot * ui[l];
      }
      __syncthreads();
    }
  }
  // M = P'_top^T p_gram (rank x r), w = last row of P' (streaming.cpp:203-218)
  double* M = a.inner + L.M;
  double* w = a.inner + L.w;
  for (int idx = threadIdx.x; idx < rank * r; idx += blockDim.x) {
    const int jn = idx % rank, j = idx / rank;
    double s = 0.0;
    for (int l = 0; l < r; ++l) s += U[l + jn * rows] * a.pgram[l + j * r];
    M[jn + j * rank] = s;
  }
  for (int j = threadIdx.x; j < rank; j += blockDim.x) w[j] = U[r + j * rows];
}

// [Q q] W and C M^T + b w^T, row-parallel, plus coupling partials
// (isvd.cpp:217-225, streaming.cpp:208-224, streaming.cpp:39-64).
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
  const int r = ctrl->r, rn = ctrl->r_new, deg = ctrl->degenerate;
  const int m = deg ? r : r + 1;
  const double inv = deg ? 0.0 : 1.0 / sqrt(ctrl->e_sq);
  const double* W = inner + L.W;
  const double* M = inner + L.M;
  const double* w = inner + L.w;
  double dacc = 0.0, cacc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double qi = deg ? 0.0 : e[i] * inv;
    const double bi = b[i];
    for (int jn = 0; jn < rn; ++jn) {
      double sq = 0.0;
      for (int l = 0; l < r; ++l) {
        const double wl = W[l + jn * m];
        if (wl == 0.0) continue;
        sq += q[i + (long long)l * n] * wl;
      }
      if (!deg) {
        const double wl = W[r + jn * m];
        if (wl != 0.0) sq += qi * wl;
      }
      double sc = 0.0;
      for (int l = 0; l < r; ++l) {
        const double ml = M[jn + l * rn];
        if (ml == 0.0) continue;
        sc += cin[i + (long long)l * n] * ml;
      }
      const double wj = w[jn];
      if (wj != 0.0) sc += wj * bi;
      qn[i + (long long)jn * n] = sq;
      cn[i + (long long)jn * n] = sc;
      const double diff = sc - sq * sigma_new[jn];
      dacc += diff * diff;
      cacc += sc * sc;
    }
  }
  dacc = block_sum(dacc, red);
  cacc = block_sum(cacc, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = dacc;
    part[2 * blockIdx.x + 1] = cacc;
  }
}

// left <- blkdiag(left, 1) P' (isvd.cpp:227-237; right_multiply :66-84)
__global__ void isvd_left_kernel(const Ctrl* ctrl, const double* __restrict__ left,
                                 long long n_d, int capr, const double* __restrict__ inner,
                                 double* __restrict__ left_new) {
  const InnerLayout L = inner_layout(capr);
  const int r = ctrl->r, rn = ctrl->r_new;
  const int rows = r + 1;
  const double* U = inner + L.U;
  const long long total = (n_d + 1) * capr;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
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

__global__ void isvd_finalize_kernel(Ctrl* c, const double* __restrict__ part, int nblk,
                                     Metrics* rec, int order, SpatialRanks sr) {
  __shared__ double red[32];
  double d = 0.0, cs = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
    d += part[2 * b];
    cs += part[2 * b + 1];
  }
  d = block_sum(d, red);
  cs = block_sum(cs, red);
  if (threadIdx.x != 0) return;
  c->coupling_diff_sq = d;
  c->core_sq = cs;
  if (sqrt(d) > kCouplingTol * sqrt(cs) + 1e-300) c->status = 2;  // streaming.cpp:55-63
  c->r = c->r_new;
  rec->slice_index = c->n_d;
  c->n_d += 1;
  c->insertions += 1;
  for (int k = 0; k + 1 < order; ++k) rec->ranks[k] = sr.v[k];
  rec->ranks[order - 1] = c->r;
  rec->slice_norm = sqrt(c->slice_sq);
  rec->projected_norm = sqrt(c->proj_sq);
  for (int k = 0; k + 1 < order; ++k) rec->mode_residuals[k] = sqrt(c->res_sq[k]);
  const double booked = c->squared_error + c->nonstream_discarded_sq;
  rec->error_estimate = c->total_input_sq <= 0.0 ? 0.0 : sqrt(fmax(booked, 0.0) / c->total_input_sq);
  rec->trunc_margin = c->trunc_margin;
  rec->sweeps = c->sweeps;
}

__global__ void zero_slice_kernel(Ctrl* c, double* left, int capr, Metrics* rec, int order,
                                  SpatialRanks sr) {
  const long long nd = c->n_d;
  for (int j = threadIdx.x; j < capr; j += blockDim.x) left[nd * capr + j] = 0.0;
  __syncthreads();
  if (threadIdx.x != 0) return;
  rec->slice_index = nd;
  c->n_d = nd + 1;
  for (int k = 0; k + 1 < order; ++k) rec->ranks[k] = sr.v[k];
  rec->ranks[order - 1] = c->r;
  rec->slice_norm = 0.0;
  rec->projected_norm = 0.0;
  for (int k = 0; k + 1 < order; ++k) rec->mode_residuals[k] = 0.0;
  const double booked = c->squared_error + c->nonstream_discarded_sq;
  rec->error_estimate = c->total_input_sq <= 0.0 ? 0.0 : sqrt(fmax(booked, 0.0) / c->total_input_sq);
  rec->trunc_margin = 0.0;
  rec->sweeps = 0;
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

}  // namespace

int launch_project(const ProjArgs& a, cudaStream_t st) {
  static const bool force_generic = std::getenv("TSG_GENERIC_PROJ") != nullptr;
  static const bool debug = std::getenv("TSG_DEBUG_SYNC") != nullptr;
  if (!force_generic) {
    const int grid = dmma_proj::launch(a, a.stream_in, st);
    if (debug) {
      cudaError_t e = cudaStreamSynchronize(st);
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e != cudaSuccess)
        fprintf(stderr, "proj_dmma failed: %s (left %lld N %lld right %lld R %d grid %d)\n",
                cudaGetErrorString(e), a.v.left, a.v.n, a.v.right, a.R, grid);
    }
    if (grid > 0) {
      ++g_launches;
      return grid;
    }
  }
  const long long N = a.v.n;
  const long long cols = a.v.left * a.v.right;
  const long long budget = 200 * 1024 / 8;  // doubles of shared memory
  int u_smem = (N * a.R <= budget / 2) ? 1 : 0;
  long long rem = budget - (u_smem ? N * a.R : 0);
  long long bc = rem / (N + a.R);
  if (bc > 64) bc = 64;
  if (bc >= 8) bc = bc / 8 * 8;
  if (bc < 1) bc = 1;
  const size_t smem = 8 * ((u_smem ? N * a.R : 0) + N * bc + a.R * bc);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(project_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 205 * 1024);
    attr = true;
  }
  const long long ntiles = (cols + bc - 1) / bc;
  long long grid = ntiles < 148 ? ntiles : 148;
  if (grid < 1) grid = 1;
  project_kernel<<<(int)grid, 256, smem, st>>>(a, (int)bc, u_smem);
  ++g_launches;
  return (int)grid;
}

void launch_decide(const DecideArgs& a, cudaStream_t st) {
  decide_kernel<<<1, 256, 0, st>>>(a);
  ++g_launches;
}

void launch_commit_modes(Ctrl* ctrl, int m0, int m1, int with_total, cudaStream_t st) {
  commit_modes_kernel<<<1, 32, 0, st>>>(ctrl, m0, m1, with_total);
  ++g_launches;
}

void launch_ledger_add_nonstream(Ctrl* ctrl, const double* value, cudaStream_t st) {
  ledger_add_kernel<<<1, 32, 0, st>>>(ctrl, value);
  ++g_launches;
}

void launch_isvd(const IsvdBufs& B, cudaStream_t st) {
  const long long n = B.n;
  const int capr = B.capr;
  // row blocks for the projection passes
  long long rows_per = 1024;
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
  pgram_kernel<<<1, 256, 0, st>>>(B.ctrl, B.left, B.n_d, capr, B.pgram);
  isvd_pass1_kernel<<<nb, 256, 0, st>>>(B.ctrl, B.q, B.b, n, rows_per, capr, part1);
  isvd_pass2_kernel<<<nb, 256, sizeof(double) * capr, st>>>(B.ctrl, B.q, B.b, n, rows_per, capr,
                                                            nb, part1, B.e, part2);
  isvd_pass3_kernel<<<nb, 256, sizeof(double) * capr, st>>>(B.ctrl, B.q, n, rows_per, capr, nb,
                                                            part2, B.e, part3);
  InnerArgs ia;
  ia.ctrl = B.ctrl;
  ia.sigma = B.sigma;
  ia.sigma_new = B.sigma_new;
  ia.part1 = part1;
  ia.part2 = part2;
  ia.part3 = part3;
  ia.nblk = nb;
  ia.capr = capr;
  ia.pgram = B.pgram;
  ia.inner = B.inner;
  const long long m = capr + 1;
  const size_t smem = 2 * m * m * sizeof(double);
  ia.use_smem = smem <= 160 * 1024 ? 1 : 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(isvd_inner_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 164 * 1024);
    attr = true;
  }
  isvd_inner_kernel<<<1, 512, ia.use_smem ? smem : 0, st>>>(ia);
  const int gu = grid_for(n, 256, 148 * 4);
  isvd_update_kernel<<<gu, 256, 0, st>>>(B.ctrl, B.q, B.c, B.e, B.b, B.inner, B.sigma_new, n, capr,
                                         B.qn, B.cn, part4);
  isvd_left_kernel<<<grid_for((B.n_d + 1) * capr), 256, 0, st>>>(B.ctrl, B.left, B.n_d, capr,
                                                                  B.inner, B.left_new);
  SpatialRanks sr;
  for (int k = 0; k < kMaxD; ++k) sr.v[k] = B.spatial_ranks[k];
  isvd_finalize_kernel<<<1, 256, 0, st>>>(B.ctrl, part4, gu, B.metrics, B.order, sr);
  g_launches += 8;
}

void launch_zero_slice(Ctrl* ctrl, double* left, int capr, Metrics* rec, int order,
                       const long long* spatial, cudaStream_t st) {
  SpatialRanks sr;
  for (int k = 0; k < kMaxD; ++k) sr.v[k] = spatial[k];
  zero_slice_kernel<<<1, 256, 0, st>>>(ctrl, left, capr, rec, order, sr);
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
