// Eigendecomposition of D + z z^T in one warp (secular equation), for the
// ISVD inner problem: S'^T S' = diag(s_1^2, ..., s_r^2, 0) + z z^T with
// z = [p; k] (isvd.cpp:201-209). The reference obtains the same spectrum by
// cyclic Jacobi on the explicitly formed Gram matrix (linalg.cpp:120-181);
// here each lane solves one root of f(l) = 1 + sum_i z_i^2 / (d_i - l) with a
// bracketed one-pole rational iteration, eigenvectors come from Loewner's
// formula (numerically orthogonal), and tiny z_i / close poles are deflated.
// Output: eigenvalues descending (clamped >= 0) and eigenvectors with the
// reference's sign rule, ready for the truncation rule.
#pragma once
#include <cfloat>

#ifndef SEC_CLK
#define SEC_CLK(i)
#endif
namespace tsg {
namespace secular {

constexpr unsigned FULL = 0xffffffffu;
constexpr int P = 33;  // shared-memory pitch

// 1/x to full double precision: hardware approximation + two Newton steps.
__device__ __forceinline__ double rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

// 1/sqrt(x) for x > 0: hardware approximation + two Newton steps (~1 ulp);
// a fraction of the cost of the IEEE sqrt / division sequences.
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  return y * fma(-h * y, y, 1.5);
}
__device__ __forceinline__ double sqrt_nr(double x) { return x > 0.0 ? x * rsqrt_nr(x) : 0.0; }

// f(tau) pieces around origin pole o: returns f, accumulates phi' (without o)
// and erretm (sum of |terms|).
__device__ __forceinline__ void eval(const double* dK, const double* wK, int K, int o,
                                     double sigma, double tau, double& f, double& phi_out,
                                     double& dphi, double& err) {
  double phi = 0.0, dp = 0.0, ea = 0.0;
  for (int i = 0; i < K; ++i) {
    if (i == o) continue;
    const double ri = rcp((dK[i] - sigma) - tau);
    const double q = wK[i] * ri;
    phi += q;
    dp += q * ri;
    ea += fabs(q);
  }
  const double qo = -wK[o] * rcp(tau);
  f = 1.0 + phi + qo;
  phi_out = phi;
  dphi = dp;
  err = 1.0 + ea + fabs(qo);
}

// Solve root j (0 = largest) of the non-deflated problem (poles dK
// descending, weights wK = z^2 > 0). Returns origin index and offset tau.
__device__ int solve_root(const double* dK, const double* wK, int K, double wsum, int j,
                          int& o_out, double& tau_out) {
  int o;
  double lo, hi;  // bracket in tau: f(lo) < 0 < f(hi)
  if (j == 0) {
    o = 0;
    lo = 0.0;
    hi = wsum;
  } else {
    const double mid = 0.5 * (dK[j] + dK[j - 1]);
    // f at the midpoint, origin-free
    double fm = 1.0;
    for (int i = 0; i < K; ++i) fm += wK[i] * rcp(dK[i] - mid);
    if (fm >= 0.0) {  // root in (d_j, mid]: origin = lower pole d_j
      o = j;
      lo = 0.0;
      hi = mid - dK[j];
    } else {          // root in (mid, d_{j-1}): origin = upper pole
      o = j - 1;
      lo = mid - dK[j - 1];
      hi = 0.0;
    }
  }
  const double sigma = dK[o];
  const bool pos = (o == j);  // tau > 0 when the origin is the lower pole
  double tau = 0.5 * (lo + hi);
  if (tau == 0.0) tau = pos ? hi : lo;
  int it = 0;
  for (; it < 60; ++it) {
    double f, phi, dphi, err;
    eval(dK, wK, K, o, sigma, tau, f, phi, dphi, err);
    if (f < 0.0)
      lo = tau;
    else
      hi = tau;
    if (fabs(f) <= 8.0 * DBL_EPSILON * err) break;
    // one-pole + linear model: 1 + phi + phi'(t - tau) - w_o / t = 0
    const double A = 1.0 + phi - dphi * tau;
    const double Dd = A * A + 4.0 * dphi * wK[o];
    const double sq = sqrt(Dd);
    double t;
    if (dphi > 0.0) {
      if (pos)
        t = (A > 0.0) ? 2.0 * wK[o] / (A + sq) : (-A + sq) / (2.0 * dphi);
      else
        t = (A < 0.0) ? 2.0 * wK[o] / (A - sq) : (-A - sq) / (2.0 * dphi);
    } else {
      t = wK[o] / A;  // single pole: (1 + phi) t = w_o
    }
    if (!(t > lo && t < hi)) t = 0.5 * (lo + hi);
    if (fabs(t - tau) <= 2.0 * DBL_EPSILON * fabs(tau)) {
      tau = t;
      break;
    }
    tau = t;
    if (hi - lo <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi))) break;
  }
  o_out = o;
  tau_out = tau;
  return it;
}

// Full solve in warp 0. d (m, descending, >= 0) and z (m) in shared memory.
// Outputs lam (m, descending) and W (m x m column-major, ld m), plus the
// same sorted eigenvectors in sW (pitch P) for the caller.
// Scratch (shared): sQ (m x P, rotations), dK, wK, sig, tau (each 32),
// idx, perm (int 32), defl flags.
struct Scratch {
  double* sQ;      // 32 x P
  double* dK;      // 32
  double* wK;      // 32
  double* zK;      // 32
  double* ls;      // 32 (sigma of root)
  double* lt;      // 32 (tau of root)
  double* zh;      // 32 (Loewner z-hat)
  double* lamall;  // 32
  int* idx;        // 32 non-deflated coordinates
  int* perm;       // 32
  int* flag;       // 32 deflated marks
};

__device__ int eig_rank_one(int m, const double* d_in, const double* z_in, Scratch S,
                            double* lam, double* W, double* sW) {
  const int lane = threadIdx.x & 31;
  __shared__ int sh_K, sh_rot;
  __shared__ double sh_wsum;
  __shared__ double dwork[32];
  // rotations basis
  for (int i = lane; i < m * m; i += 32) {
    const int a = i % m, b = i / m;
    S.sQ[a * P + b] = (a == b) ? 1.0 : 0.0;
  }
  if (lane < m) {
    dwork[lane] = d_in[lane];
    S.zK[lane] = z_in[lane];
  }
  __syncwarp();
  if (lane == 0) {
    double zn2 = 0.0;
    for (int i = 0; i < m; ++i) zn2 += S.zK[i] * S.zK[i];
    const double zn = sqrt(zn2);
    const double tol = 8.0 * DBL_EPSILON * (dwork[0] + zn2);
    for (int i = 0; i < m; ++i) S.flag[i] = (fabs(S.zK[i]) * zn <= tol) ? 1 : 0;
    // close poles: rotate the later coordinate's weight into the earlier one
    int prev = -1, rotated = 0;
    for (int i = 0; i < m; ++i) {
      if (S.flag[i]) continue;
      // |(d_p - d_i) c s| <= tol with c s = z_p z_i / (z_p^2 + z_i^2), tested
      // without the square root first
      if (prev >= 0 && fabs(dwork[prev] - dwork[i]) * fabs(S.zK[prev] * S.zK[i]) <=
                           tol * (S.zK[prev] * S.zK[prev] + S.zK[i] * S.zK[i])) {
        const double zp = S.zK[prev], zi = S.zK[i];
        const double rr = hypot(zp, zi);
        const double c = zp / rr, s = zi / rr;
        {
          rotated = 1;
          // G = [c s; -s c] on (prev, i): z_prev <- r, z_i <- 0
          const double dp = dwork[prev], di = dwork[i];
          dwork[prev] = c * c * dp + s * s * di;
          dwork[i] = s * s * dp + c * c * di;
          S.zK[prev] = rr;
          S.zK[i] = 0.0;
          for (int a = 0; a < m; ++a) {
            const double qp = S.sQ[a * P + prev], qi = S.sQ[a * P + i];
            S.sQ[a * P + prev] = c * qp + s * qi;
            S.sQ[a * P + i] = -s * qp + c * qi;
          }
          S.flag[i] = 1;
          continue;
        }
      }
      prev = i;
    }
    int K = 0;
    double wsum = 0.0;
    for (int i = 0; i < m; ++i)
      if (!S.flag[i]) {
        S.idx[K] = i;
        S.dK[K] = dwork[i];
        S.wK[K] = S.zK[i] * S.zK[i];
        wsum += S.wK[K];
        ++K;
      }
    sh_K = K;
    sh_wsum = wsum;
    sh_rot = rotated;
  }
  __syncwarp();
  const int K = sh_K;
  // roots
  int iters = 0;
  if (lane < K) {
    int o;
    double tau;
    iters = solve_root(S.dK, S.wK, K, sh_wsum, lane, o, tau);
    S.ls[lane] = S.dK[o];
    S.lt[lane] = tau;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) iters = max(iters, __shfl_xor_sync(FULL, iters, off));
  __syncwarp();
  // Loewner z-hat: zh_i^2 = (l_i - d_i) prod_{j != i} (l_j - d_i) / (d_j - d_i)
  if (lane < K) {
    const int i = lane;
    const double di = S.dK[i];
    double prod = (S.ls[i] - di) + S.lt[i];
    for (int j = 0; j < K; ++j) {
      if (j == i) continue;
      const double num = (S.ls[j] - di) + S.lt[j];
      prod *= num * rcp(S.dK[j] - di);
    }
    const double zi = S.zK[S.idx[i]];
    const double mag = sqrt(fabs(prod));
    S.zh[i] = (zi < 0.0) ? -mag : mag;
  }
  __syncwarp();
  // all eigenvalues (non-deflated roots then deflated poles) + sort
  __shared__ int src_kind[32];
  if (lane < m) {
    // position lane: lanes < K are roots, the rest map to deflated coordinates
    double lv;
    if (lane < K) {
      lv = S.ls[lane] + S.lt[lane];
      src_kind[lane] = lane;  // root id
    } else {
      int cnt = 0, coord = 0;
      for (int a = 0; a < m; ++a)
        if (S.flag[a]) {
          if (cnt == lane - K) {
            coord = a;
            break;
          }
          ++cnt;
        }
      lv = dwork[coord];
      src_kind[lane] = 32 + coord;  // deflated coordinate
    }
    S.lamall[lane] = lv;
  }
  __syncwarp();
  if (lane < m) {
    const double li = S.lamall[lane];
    int rk = 0;
    for (int j = 0; j < m; ++j) {
      const double lj = S.lamall[j];
      if (lj > li || (lj == li && j < lane)) ++rk;
    }
    S.perm[rk] = lane;
  }
  __syncwarp();
  // eigenvector columns (lane = output column), sign rule, clamp
  if (lane < m) {
    const int src = S.perm[lane];
    const int kind = src_kind[src];
    for (int a = 0; a < m; ++a) sW[a * P + lane] = 0.0;
    if (kind < 32) {
      const int j = kind;
      double nrm2 = 0.0;
      for (int i = 0; i < K; ++i) {
        const double t = S.zh[i] * rcp((S.dK[i] - S.ls[j]) - S.lt[j]);
        nrm2 += t * t;
      }
      const double inv = 1.0 / sqrt(nrm2);
      if (!sh_rot) {
        for (int i = 0; i < K; ++i)
          sW[S.idx[i] * P + lane] = S.zh[i] * rcp((S.dK[i] - S.ls[j]) - S.lt[j]) * inv;
      } else {
        for (int i = 0; i < K; ++i) {
          const double c = S.zh[i] * rcp((S.dK[i] - S.ls[j]) - S.lt[j]) * inv;
          const int coord = S.idx[i];
          for (int a = 0; a < m; ++a) sW[a * P + lane] += S.sQ[a * P + coord] * c;
        }
      }
    } else {
      const int coord = kind - 32;
      for (int a = 0; a < m; ++a) sW[a * P + lane] = S.sQ[a * P + coord];
    }
    int arg = 0;
    double best = fabs(sW[lane]);
    for (int a = 1; a < m; ++a) {
      const double av = fabs(sW[a * P + lane]);
      if (av > best) {
        best = av;
        arg = a;
      }
    }
    const bool flip = sW[arg * P + lane] < 0.0;
    for (int a = 0; a < m; ++a) {
      const double v = flip ? -sW[a * P + lane] : sW[a * P + lane];
      sW[a * P + lane] = v;
      W[a + lane * m] = v;
    }
    const double lv = S.lamall[src];
    lam[lane] = lv < 0.0 ? 0.0 : lv;
  }
  __syncwarp();
  return iters;
}


// Wide variant: the same algorithm as eig_rank_one for 32 < m <= kWide (the
// inner problem of streams whose rank passes 31: configs 3 and 5), one warp,
// each lane taking coordinates / roots lane, lane + 32. Scratch comes from
// the caller (shared memory): sQ and sW are m x PW (PW = kWide + 1), the
// double arrays kWide entries each, the int arrays kWide entries each.
constexpr int kWide = 64;
constexpr int PW = kWide + 1;
struct ScratchWide {
  double *sQ, *sW;
  double *dwork, *dK, *wK, *zK, *ls, *lt, *zh, *lamall;
  int *idx, *perm, *flag, *kind;
  __host__ __device__ static constexpr int doubles() { return 2 * kWide * PW + 8 * kWide + 2 * kWide; }
};
__device__ inline ScratchWide scratch_wide(double* base) {
  ScratchWide S;
  S.sQ = base;
  S.sW = S.sQ + kWide * PW;
  S.dwork = S.sW + kWide * PW;
  S.dK = S.dwork + kWide;
  S.wK = S.dK + kWide;
  S.zK = S.wK + kWide;
  S.ls = S.zK + kWide;
  S.lt = S.ls + kWide;
  S.zh = S.lt + kWide;
  S.lamall = S.zh + kWide;
  int* ib = reinterpret_cast<int*>(S.lamall + kWide);
  S.idx = ib;
  S.perm = ib + kWide;
  S.flag = ib + 2 * kWide;
  S.kind = ib + 3 * kWide;
  return S;
}

// d_in (m, descending, >= 0), z_in (m): eigenvalues of diag(d) + z z^T into
// lam (descending, clamped >= 0), eigenvectors into W (m x m column-major,
// ld m) with the reference's sign rule. Called by EVERY thread of the CTA
// (block barriers inside): one thread per root / coordinate / column, so the
// 33..64-column problem takes about as long as one root instead of two per
// lane of a single warp; the sequential Givens deflation of close poles runs
// only when a close pair exists (rare), after a parallel scan.
__device__ __noinline__ int eig_rank_one_wide(int m, const double* d_in, const double* z_in, ScratchWide S,
                                 double* lam, double* W) {
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ int sh_K, sh_rot, sh_close, sh_iters;
  __shared__ double sh_wsum, sh_zn2;
  for (int i = tid; i < m * PW; i += nt) {
    const int a_ = i / PW, b_ = i - a_ * PW;
    S.sQ[i] = (a_ == b_) ? 1.0 : 0.0;
  }
  for (int i = tid; i < m; i += nt) {
    S.dwork[i] = d_in[i];
    S.zK[i] = z_in[i];
  }
  if (tid == 0) {
    sh_close = 0;
    sh_iters = 0;
  }
  __syncthreads();
  if (tid < 32) {  // ||z||^2 in coordinate order per lane, fixed tree
    double zn2 = 0.0;
    for (int i = tid; i < m; i += 32) zn2 += S.zK[i] * S.zK[i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) zn2 += __shfl_xor_sync(FULL, zn2, off);
    if (tid == 0) sh_zn2 = zn2;
  }
  __syncthreads();
  const double zn2 = sh_zn2;
  const double tol = 8.0 * DBL_EPSILON * (S.dwork[0] + zn2);
  const double zn = sqrt(zn2);
  for (int i = tid; i < m; i += nt) S.flag[i] = (fabs(S.zK[i]) * zn <= tol) ? 1 : 0;
  __syncthreads();
  // any close pair among consecutive kept coordinates?
  for (int i = tid; i < m; i += nt) {
    if (S.flag[i]) continue;
    int prev = i - 1;
    while (prev >= 0 && S.flag[prev]) --prev;
    if (prev >= 0 && fabs(S.dwork[prev] - S.dwork[i]) * fabs(S.zK[prev] * S.zK[i]) <=
                         tol * (S.zK[prev] * S.zK[prev] + S.zK[i] * S.zK[i]))
      sh_close = 1;
  }
  __syncthreads();
  if (tid == 0) {
    int rotated = 0;
    if (sh_close) {
      // close poles: rotate the later coordinate's weight into the earlier one
      int prev = -1;
      for (int i = 0; i < m; ++i) {
        if (S.flag[i]) continue;
        if (prev >= 0 && fabs(S.dwork[prev] - S.dwork[i]) * fabs(S.zK[prev] * S.zK[i]) <=
                             tol * (S.zK[prev] * S.zK[prev] + S.zK[i] * S.zK[i])) {
          const double zp = S.zK[prev], zi = S.zK[i];
          const double rr = hypot(zp, zi);
          const double c = zp / rr, sn = zi / rr;
          rotated = 1;
          const double dp = S.dwork[prev], di = S.dwork[i];
          S.dwork[prev] = c * c * dp + sn * sn * di;
          S.dwork[i] = sn * sn * dp + c * c * di;
          S.zK[prev] = rr;
          S.zK[i] = 0.0;
          for (int a_ = 0; a_ < m; ++a_) {
            const double qp = S.sQ[a_ * PW + prev], qi = S.sQ[a_ * PW + i];
            S.sQ[a_ * PW + prev] = c * qp + sn * qi;
            S.sQ[a_ * PW + i] = -sn * qp + c * qi;
          }
          S.flag[i] = 1;
          continue;
        }
        prev = i;
      }
    }
    int K = 0;
    double wsum = 0.0;
    for (int i = 0; i < m; ++i)
      if (!S.flag[i]) {
        S.idx[K] = i;
        S.dK[K] = S.dwork[i];
        S.wK[K] = S.zK[i] * S.zK[i];
        wsum += S.wK[K];
        ++K;
      }
    sh_K = K;
    sh_wsum = wsum;
    sh_rot = rotated;
  }
  __syncthreads();
  SEC_CLK(10);
  const int K = sh_K;
  for (int j = tid; j < K; j += nt) {
    int o;
    double tau;
    const int it = solve_root(S.dK, S.wK, K, sh_wsum, j, o, tau);
    S.ls[j] = S.dK[o];
    S.lt[j] = tau;
    atomicMax(&sh_iters, it);
  }
  __syncthreads();
  SEC_CLK(11);
  // Loewner z-hat
  for (int i = tid; i < K; i += nt) {
    const double di = S.dK[i];
    double prod = (S.ls[i] - di) + S.lt[i];
    for (int j = 0; j < K; ++j) {
      if (j == i) continue;
      const double num = (S.ls[j] - di) + S.lt[j];
      prod *= num * rcp(S.dK[j] - di);
    }
    const double zi = S.zK[S.idx[i]];
    const double mag = sqrt(fabs(prod));
    S.zh[i] = (zi < 0.0) ? -mag : mag;
  }
  // all eigenvalues: non-deflated roots, then deflated poles in coordinate order
  for (int q = tid; q < m; q += nt) {
    double lv;
    if (q < K) {
      lv = S.ls[q] + S.lt[q];
      S.kind[q] = q;
    } else {
      int cnt = 0, coord = 0;
      for (int a_ = 0; a_ < m; ++a_)
        if (S.flag[a_]) {
          if (cnt == q - K) {
            coord = a_;
            break;
          }
          ++cnt;
        }
      lv = S.dwork[coord];
      S.kind[q] = kWide + coord;
    }
    S.lamall[q] = lv;
  }
  __syncthreads();
  for (int q = tid; q < m; q += nt) {
    const double li = S.lamall[q];
    int rk = 0;
    for (int j = 0; j < m; ++j) {
      const double lj = S.lamall[j];
      if (lj > li || (lj == li && j < q)) ++rk;
    }
    S.perm[rk] = q;
  }
  __syncthreads();
  SEC_CLK(12);
  // eigenvector columns, sign rule, clamp
  for (int col = tid; col < m; col += nt) {
    const int src = S.perm[col];
    const int kind = S.kind[src];
    for (int a_ = 0; a_ < m; ++a_) S.sW[a_ * PW + col] = 0.0;
    if (kind < kWide) {
      const int j = kind;
      double nrm2 = 0.0;
      for (int i = 0; i < K; ++i) {
        const double t = S.zh[i] * rcp((S.dK[i] - S.ls[j]) - S.lt[j]);
        nrm2 += t * t;
      }
      const double inv = 1.0 / sqrt(nrm2);
      if (!sh_rot) {
        for (int i = 0; i < K; ++i)
          S.sW[S.idx[i] * PW + col] = S.zh[i] * rcp((S.dK[i] - S.ls[j]) - S.lt[j]) * inv;
      } else {
        for (int i = 0; i < K; ++i) {
          const double c = S.zh[i] * rcp((S.dK[i] - S.ls[j]) - S.lt[j]) * inv;
          const int coord = S.idx[i];
          for (int a_ = 0; a_ < m; ++a_) S.sW[a_ * PW + col] += S.sQ[a_ * PW + coord] * c;
        }
      }
    } else {
      const int coord = kind - kWide;
      for (int a_ = 0; a_ < m; ++a_) S.sW[a_ * PW + col] = S.sQ[a_ * PW + coord];
    }
    int arg = 0;
    double best = fabs(S.sW[col]);
    for (int a_ = 1; a_ < m; ++a_) {
      const double av = fabs(S.sW[a_ * PW + col]);
      if (av > best) {
        best = av;
        arg = a_;
      }
    }
    const bool flip = S.sW[arg * PW + col] < 0.0;
    for (int a_ = 0; a_ < m; ++a_) {
      const double v = flip ? -S.sW[a_ * PW + col] : S.sW[a_ * PW + col];
      W[a_ + col * m] = v;
    }
    const double lv = S.lamall[src];
    lam[col] = lv < 0.0 ? 0.0 : lv;
  }
  __syncthreads();
  return sh_iters;
}

// Register-resident variant for m <= KM: the deflation scan, root solve,
// Loewner z-hat and eigenvectors run lane-parallel over unrolled register
// arrays (no shared-memory loops on the critical path). Close poles (which
// need the sequential Givens deflation) fall back to eig_rank_one. Same
// outputs and conventions as eig_rank_one.
template <int N>
__device__ __forceinline__ double tsum(double (&t)[N]) {  // binary tree, in place
#pragma unroll
  for (int w = 1; w < N; w <<= 1) {
#pragma unroll
    for (int i = 0; i + w < N; i += 2 * w) t[i] = __dadd_rn(t[i], t[i + w]);
  }
  return t[0];
}
template <int N>
__device__ __forceinline__ double tprod(double (&t)[N]) {
#pragma unroll
  for (int w = 1; w < N; w <<= 1) {
#pragma unroll
    for (int i = 0; i + w < N; i += 2 * w) t[i] = __dmul_rn(t[i], t[i + w]);
  }
  return t[0];
}

// dd[i] = d_i - sigma (origin-shifted poles, padded entries huge with w = 0)
template <int KM>
__device__ __forceinline__ double eval_reg(const double (&dd)[KM], const double (&wK)[KM], int o,
                                           double wo, double tau, double& phi_out, double& dphi,
                                           double& err) {
  double q[KM], qr[KM], aq[KM];
#pragma unroll
  for (int i = 0; i < KM; ++i) {
    const double ri = rcp(dd[i] - tau);
    const double qi = (i == o) ? 0.0 : wK[i] * ri;
    q[i] = qi;
    qr[i] = qi * ri;
    aq[i] = fabs(qi);
  }
  const double qo = -wo * rcp(tau);
  const double phi = tsum<KM>(q);
  phi_out = phi;
  dphi = tsum<KM>(qr);
  err = 1.0 + tsum<KM>(aq) + fabs(qo);
  return 1.0 + phi + qo;
}

template <int KM>
__device__ int solve_root_reg(const double (&dK)[KM], const double (&wK)[KM], const double* sdK,
                              const double* swK, int K, double wsum, int j, int& o_out,
                              double& tau_out) {
  int o;
  double lo, hi;
  if (j == 0) {
    o = 0;
    lo = 0.0;
    hi = wsum;
  } else {
    const double dj = sdK[j], dj1 = sdK[j - 1];
    const double mid = 0.5 * (dj + dj1);
    double t[KM];
#pragma unroll
    for (int i = 0; i < KM; ++i) t[i] = (i < K) ? wK[i] * rcp(dK[i] - mid) : 0.0;
    const double fm = 1.0 + tsum<KM>(t);
    if (fm >= 0.0) {
      o = j;
      lo = 0.0;
      hi = mid - dj;
    } else {
      o = j - 1;
      lo = mid - dj1;
      hi = 0.0;
    }
  }
  const double sigma = sdK[o], wo = swK[o];
  double dd[KM];
#pragma unroll
  for (int i = 0; i < KM; ++i) dd[i] = dK[i] - sigma;
  const bool pos = (o == j);
  double tau = 0.5 * (lo + hi);
  if (tau == 0.0) tau = pos ? hi : lo;
  int it = 0;
  for (; it < 60; ++it) {
    double phi, dphi, err;
    const double f = eval_reg<KM>(dd, wK, o, wo, tau, phi, dphi, err);
    if (f < 0.0)
      lo = tau;
    else
      hi = tau;
    if (fabs(f) <= 8.0 * DBL_EPSILON * err) break;
    const double A = 1.0 + phi - dphi * tau;
    const double Dd = A * A + 4.0 * dphi * wo;
    const double sq = sqrt_nr(Dd);
    // one reciprocal for every branch of the quadratic's stable root
    double num, den;
    if (dphi > 0.0) {
      const bool first = pos ? (A > 0.0) : (A < 0.0);
      const double as = pos ? A + sq : A - sq;
      num = first ? 2.0 * wo : (pos ? -A + sq : -A - sq);
      den = first ? as : 2.0 * dphi;
    } else {
      num = wo;
      den = A;
    }
    double t = num * rcp(den);
    if (!(t > lo && t < hi)) t = 0.5 * (lo + hi);
    if (fabs(t - tau) <= 2.0 * DBL_EPSILON * fabs(tau)) {
      tau = t;
      break;
    }
    tau = t;
    if (hi - lo <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi))) break;
  }
  o_out = o;
  tau_out = tau;
  return it;
}

template <int KM>
__device__ int eig_rank_one_fast(int m, const double* d_in, const double* z_in, Scratch S,
                                 double* lam, double* W, double* sW) {
  const int lane = threadIdx.x & 31;
  const double di = lane < m ? d_in[lane] : 0.0;
  const double zi = lane < m ? z_in[lane] : 0.0;
  double zn2 = zi * zi;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) zn2 += __shfl_xor_sync(FULL, zn2, o);
  const double d0 = __shfl_sync(FULL, di, 0);
  const double zn = sqrt_nr(zn2);
  const double tol = 8.0 * DBL_EPSILON * (d0 + zn2);
  const bool flag = (lane >= m) || (fabs(zi) * zn <= tol);
  const unsigned keep = __ballot_sync(FULL, !flag);
  // close poles between consecutive kept coordinates need sequential Givens
  // deflation (rare): hand the whole problem to the scalar-lane solver
  const unsigned below = keep & ((1u << lane) - 1u);
  const int prev = below ? 31 - __clz(below) : lane;
  const double dp = __shfl_sync(FULL, di, prev), zp = __shfl_sync(FULL, zi, prev);
  const bool close = !flag && below &&
                     fabs(dp - di) * fabs(zp * zi) <= tol * (zp * zp + zi * zi);
  if (__any_sync(FULL, close) || m > KM) return eig_rank_one(m, d_in, z_in, S, lam, W, sW);
  SEC_CLK(10);
  const int K = __popc(keep);
  const int pos = __popc(below);
  if (!flag) {
    S.dK[pos] = di;
    S.wK[pos] = zi * zi;
    S.idx[pos] = lane;
  }
  double wsum = flag ? 0.0 : zi * zi;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(FULL, wsum, o);
  __syncwarp();
  // padded register copies: absent poles sit at +huge with zero weight
  double dK[KM], wK[KM];
#pragma unroll
  for (int i = 0; i < KM; ++i) {
    dK[i] = i < K ? S.dK[i] : 1e300;
    wK[i] = i < K ? S.wK[i] : 0.0;
  }
  int iters = 0;
  double my_ls = 0.0, my_lt = 0.0;
  if (lane < K) {
    int o;
    double tau;
    iters = solve_root_reg<KM>(dK, wK, S.dK, S.wK, K, wsum, lane, o, tau);
    my_ls = S.dK[o];
    my_lt = tau;
    S.ls[lane] = my_ls;
    S.lt[lane] = tau;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) iters = max(iters, __shfl_xor_sync(FULL, iters, off));
  __syncwarp();
  SEC_CLK(11);
  // Loewner z-hat (lane i < K)
  double zh_me = 0.0;
  if (lane < K) {
    const double dki = S.dK[lane];
    // own factor first: every factor's tree position is independent of KM
    double fac[KM + 1];
    fac[0] = (my_ls - dki) + my_lt;
#pragma unroll
    for (int j = 0; j < KM; ++j)
      fac[j + 1] = (j < K && j != lane) ? ((S.ls[j] - dki) + S.lt[j]) * rcp(dK[j] - dki) : 1.0;
    const double prod = tprod<KM + 1>(fac);
    const double mag = sqrt_nr(fabs(prod));
    zh_me = (z_in[S.idx[lane]] < 0.0) ? -mag : mag;
    S.zh[lane] = zh_me;
  }
  // all eigenvalues: roots (lanes < K) then deflated poles in coordinate order
  const unsigned defl = (~keep) & ((m >= 32) ? FULL : ((1u << m) - 1u));
  double lv = 0.0;
  int kind = -1;
  if (lane < K) {
    lv = my_ls + my_lt;
    kind = lane;
  } else if (lane < m) {
    // (lane - K)-th deflated coordinate
    unsigned mm = defl;
    for (int c = 0; c < lane - K; ++c) mm &= mm - 1u;
    const int coord = __ffs(mm) - 1;
    lv = d_in[coord];  // no rotation: the deflated eigenvalue is the pole
    kind = 32 + coord;
  }
  S.lamall[lane] = lv;
  __syncwarp();
  SEC_CLK(12);
  __shared__ int src_kind[32];
  src_kind[lane] = kind;
  if (lane < m) {
    int rk = 0;
    for (int j = 0; j < m; ++j) {
      const double lj = S.lamall[j];
      if (lj > lv || (lj == lv && j < lane)) ++rk;
    }
    S.perm[rk] = lane;
  }
  __syncwarp();
  SEC_CLK(13);
  if (lane < m) {
    const int src = S.perm[lane];
    const int kd = src_kind[src];
    for (int a = 0; a < m; ++a) sW[a * P + lane] = 0.0;
    if (kd < 32) {
      const double lsj = S.ls[kd], ltj = S.lt[kd];
      double t[KM], t2[KM];
#pragma unroll
      for (int i = 0; i < KM; ++i) {
        t[i] = (i < K) ? S.zh[i] * rcp((dK[i] - lsj) - ltj) : 0.0;
        t2[i] = t[i] * t[i];
      }
      const double inv = rsqrt_nr(tsum<KM>(t2));
      // sign rule: first coordinate of largest magnitude made positive
      // (coordinates of the kept poles are increasing in i)
      double best = -1.0, bv = 0.0;
#pragma unroll
      for (int i = 0; i < KM; ++i) {
        const double v = t[i] * inv;
        t[i] = v;
        if (i < K && fabs(v) > best) {
          best = fabs(v);
          bv = v;
        }
      }
      const double sgn = bv < 0.0 ? -1.0 : 1.0;
#pragma unroll
      for (int i = 0; i < KM; ++i)
        if (i < K) sW[S.idx[i] * P + lane] = sgn * t[i];
    } else {
      sW[(kd - 32) * P + lane] = 1.0;
    }
    for (int a = 0; a < m; ++a) W[a + lane * m] = sW[a * P + lane];
    const double l = S.lamall[src];
    lam[lane] = l < 0.0 ? 0.0 : l;
  }
  __syncwarp();
  return iters;
}

}  // namespace secular
}  // namespace tsg
