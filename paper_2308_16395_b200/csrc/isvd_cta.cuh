// Single-CTA insertion with a branch-free inner solve (n <= 1024 rows).
//
// Why: on the B200 a taken branch costs a warp tens of cycles (measured:
// a loop body with two uniform branches runs at ~130 cycles per iteration
// against 9 cycles for its one dependent DFMA, tools/micro/mufu_lat.cu),
// and the insertion is one latency chain executed by one warp: the
// data-dependent control flow of the general secular solver (iteration
// loops with early exits, per-pole deflation branches, a sort) made the
// inner solve ~17k cycles. Here the common case is straight-line code over
// compile-time sized register arrays:
//   * roots: NIT unrolled iterations of the same bracketed one-pole +
//     linear model as secular::solve_root_reg, frozen by selects once
//     converged (a lane that has not converged after NIT, or a problem that
//     needs deflation -- tiny z_i or close poles -- takes the general solver,
//     a rare branch);
//   * the roots of D + z z^T come out descending (root j lies in
//     (d_j, d_{j-1})), so no sort is needed;
//   * Loewner z-hat, eigenvectors and the sign rule as in the general solver;
//   * truncation (linalg.cpp:183-208) replicated lane-uniformly;
//   * P' = S' W / sigma re-orthonormalised by one classical Gram-Schmidt
//     pass (its columns are orthonormal to O(eps kappa^2); CGS and the
//     reference's MGS agree to the square of that defect).
// The rest of the chain matches isvd_small_kernel / isvd_grid_kernel:
// ledger commit, two-pass CGS2 split (||e||^2 = ||e1||^2 - ||p2||^2), p_gram
// of the left factor by the other warps during the inner solve, Q / core /
// left row updates, coupling check, record. One CTA, no inter-CTA handoff.
// Reference: isvd.cpp:163-250 (add_row), linalg.cpp:210-259
// (small_svd_truncated), streaming.cpp:196-224.
#pragma once

namespace {
namespace cta {

using secular::rcp;
using secular::rsqrt_nr;
using secular::sqrt_nr;
using secular::tprod;
using secular::tsum;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// Returns the rank (>= 1), or -1 when the general solver must run. c may be
// null (a redundant solve that must not write the ledgers).
// Inputs (shared): ssig[r], sp[r]; k = ||e||. Outputs (shared): sW (pitch
// 33, rows < m, cols < rank: W = eigenvectors of S'^T S'), sU (pitch 33,
// rows <= r, cols < rank: P'), ssn[rank]; ctrl ledgers / diagnostics.
template <int RM, int NIT>
__device__ int inner_fast(Ctrl* c, int r, int deg, const double* ssig, const double* sp, double k,
                          double delta, double sq_err, double* sW, double* sU, double* ssn) {
  constexpr int P = 33;
  constexpr double EPS = DBL_EPSILON;
  const int lane = threadIdx.x & 31;
  const int m = deg ? r : r + 1;
  const bool valid = lane < m;
  // my pole / weight; padding poles sit far below with zero weight
  const int li = lane < r ? lane : (r > 0 ? r - 1 : 0);
  const double sg = ssig[li], pz = sp[li];
  double dj = lane < r ? sg * sg : 0.0;
  double zj = lane < r ? pz : (lane == r ? k : 0.0);
  if (!valid) {
    dj = -1e300;
    zj = 0.0;
  }
  const double wj = zj * zj;
  double dv[RM], wv[RM];
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    dv[i] = __shfl_sync(FULL, dj, i);
    wv[i] = __shfl_sync(FULL, wj, i);
  }
  double zn2 = wj;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) zn2 += __shfl_xor_sync(FULL, zn2, o);
  const double zn = sqrt_nr(zn2);
  const double tol = 8.0 * EPS * (dv[0] + zn2);
  // deflation (tiny weight, or close consecutive poles): general solver
  const double dprev = __shfl_up_sync(FULL, dj, 1), zprev = __shfl_up_sync(FULL, zj, 1);
  const bool tiny = valid && fabs(zj) * zn <= tol;
  const bool close = valid && lane > 0 && fabs(dprev - dj) * fabs(zprev * zj) <= tol * (zprev * zprev + zj * zj);
  if (__any_sync(FULL, tiny || close)) return -1;
  const double wsum = zn2;
  TSG_CLK(10);

  // ---- root of this lane (lanes >= m solve a copy of the last root)
  const int jj = valid ? lane : m - 1;
  const double dJ = __shfl_sync(FULL, dj, jj);
  const double dJm1 = __shfl_sync(FULL, dj, jj > 0 ? jj - 1 : 0);
  const double mid = 0.5 * (dJ + dJm1);
  double fm;
  {
    double t[RM];
#pragma unroll
    for (int i = 0; i < RM; ++i) t[i] = wv[i] * rcp(dv[i] - mid);
    fm = 1.0 + tsum<RM>(t);
  }
  const bool lower = (jj == 0) || (fm >= 0.0);
  const int o = lower ? jj : jj - 1;
  double lo = lower ? 0.0 : mid - dJm1;
  double hi = lower ? (jj == 0 ? wsum : mid - dJ) : 0.0;
  const double sigma = lower ? dJ : dJm1;
  const double wo = __shfl_sync(FULL, wj, o);
  const bool pos = lower;
  double tau = 0.5 * (lo + hi);
  if (tau == 0.0) tau = pos ? hi : lo;
  double dd[RM];
#pragma unroll
  for (int i = 0; i < RM; ++i) dd[i] = dv[i] - sigma;
  bool done = false;
  int iters = 0;
  // rolled: one loop branch per iteration, against a register footprint that
  // would spill if NIT iterations were scheduled together
#pragma unroll 1
  for (int it = 0; it < NIT; ++it) {
    double q[RM], qr[RM], aq[RM];
#pragma unroll
    for (int i = 0; i < RM; ++i) {
      const double ri = rcp(dd[i] - tau);
      const double qi = (i == o) ? 0.0 : wv[i] * ri;
      q[i] = qi;
      qr[i] = qi * ri;
      aq[i] = fabs(qi);
    }
    const double qo = -wo * rcp(tau);
    const double phi = tsum<RM>(q);
    const double dphi = tsum<RM>(qr);
    const double err = 1.0 + tsum<RM>(aq) + fabs(qo);
    const double f = 1.0 + phi + qo;
    const double nlo = f < 0.0 ? tau : lo;
    const double nhi = f < 0.0 ? hi : tau;
    const bool conv = fabs(f) <= 8.0 * EPS * err;
    const double A = 1.0 + phi - dphi * tau;
    const double Dd = A * A + 4.0 * dphi * wo;
    const double sq = sqrt_nr(Dd);
    const bool first = pos ? (A > 0.0) : (A < 0.0);
    const double as = pos ? A + sq : A - sq;
    const double num = dphi > 0.0 ? (first ? 2.0 * wo : (pos ? -A + sq : -A - sq)) : wo;
    const double den = dphi > 0.0 ? (first ? as : 2.0 * dphi) : A;
    double t = num * rcp(den);
    if (!(t > nlo && t < nhi)) t = 0.5 * (nlo + nhi);
    const bool stall = fabs(t - tau) <= 2.0 * EPS * fabs(tau);
    const bool tiny_br = nhi - nlo <= 2.0 * EPS * fmax(fabs(nlo), fabs(nhi));
    if (!done) {
      lo = nlo;
      hi = nhi;
      if (!conv) {
        tau = t;
        ++iters;
      }
      done = conv || stall || tiny_br;
    }
  }
  if (__any_sync(FULL, valid && !done)) return -1;
  TSG_CLK(11);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) iters = max(iters, __shfl_xor_sync(FULL, iters, off));

  // ---- Loewner z-hat of coordinate `lane`
  double ls[RM], lt[RM];
#pragma unroll
  for (int j = 0; j < RM; ++j) {
    ls[j] = __shfl_sync(FULL, sigma, j);
    lt[j] = __shfl_sync(FULL, tau, j);
  }
  double zh;
  {
    double fac[RM + 1];
    fac[0] = (sigma - dj) + tau;
#pragma unroll
    for (int j = 0; j < RM; ++j)
      fac[j + 1] = (j < m && j != lane) ? ((ls[j] - dj) + lt[j]) * rcp(dv[j] - dj) : 1.0;
    const double prod = tprod<RM + 1>(fac);
    const double mag = sqrt_nr(fabs(prod));
    zh = zj < 0.0 ? -mag : mag;
  }
  double zhv[RM];
#pragma unroll
  for (int i = 0; i < RM; ++i) zhv[i] = __shfl_sync(FULL, zh, i);
  TSG_CLK(12);
  // ---- eigenvector `lane` (descending eigenvalue order = lane order)
  double v[RM];
  {
    double t2[RM];
#pragma unroll
    for (int i = 0; i < RM; ++i) {
      v[i] = i < m ? zhv[i] * rcp((dv[i] - sigma) - tau) : 0.0;
      t2[i] = v[i] * v[i];
    }
    const double inv = rsqrt_nr(tsum<RM>(t2));
    double best = -1.0, bv = 0.0;
#pragma unroll
    for (int i = 0; i < RM; ++i) {
      v[i] *= inv;
      const bool better = i < m && fabs(v[i]) > best;  // first coordinate of largest magnitude
      best = better ? fabs(v[i]) : best;
      bv = better ? v[i] : bv;
    }
    const double sgn = bv < 0.0 ? -1.0 : 1.0;
#pragma unroll
    for (int i = 0; i < RM; ++i) v[i] *= sgn;
  }
  TSG_CLK(13);
  double lj = sigma + tau;
  if (lj < 0.0) lj = 0.0;
  if (!valid) lj = 0.0;

  // ---- truncation (linalg.cpp:224-240, isvd.cpp:210-215), lane-uniform
  const double smax = sqrt_nr(__shfl_sync(FULL, lj, 0));
  const double fl = kSigmaZeroFactor * smax;
  if (valid && sqrt_nr(lj) <= fl) lj = 0.0;
  double lv[RM];
#pragma unroll
  for (int i = 0; i < RM; ++i) lv[i] = __shfl_sync(FULL, lj, i);
  const double budget = delta * delta;
  double s = 0.0, prev_excess = -1.0;
  int rr = m;
#pragma unroll
  for (int i = RM - 1; i >= 0; --i) {
    const bool act = i < m && prev_excess < 0.0;
    const double nx = s + lv[i];
    const bool keep = act && nx <= budget;
    s = keep ? nx : s;
    rr = keep ? i : rr;
    prev_excess = (act && !keep) ? nx : prev_excess;
  }
  const int rank = rr < 1 ? 1 : rr;
  double disc = 0.0;
#pragma unroll
  for (int j = RM - 1; j >= 0; --j) disc += (j < m && j >= rank) ? lv[j] : 0.0;
  double margin = 0.0;
  if (budget > 0.0) {
    double mg = fabs(budget - s) / budget;
    if (prev_excess >= 0.0) mg = fmin(mg, fabs(prev_excess - budget) / budget);
    margin = mg;
  }
  if (lane == 0 && c) {
    const double added = disc + (deg ? k * k : 0.0);
    c->trunc_margin = margin;
    c->sweeps = iters;
    c->added_error_sq = added;
    c->squared_error = sq_err + added;  // isvd.cpp:212-215
    c->r_new = rank;
    c->degenerate = deg;
  }
  TSG_CLK(5);
  // W = eigenvectors (rows < m), columns < rank
  if (lane < rank) {
#pragma unroll
    for (int i = 0; i < RM; ++i)
      if (i < m) sW[i * P + lane] = v[i];
  }
  // ---- P' = S' W / sigma (rows l < r: s_l w_l; row r: z^T w), one CGS pass
  double u[RM];
  {
    const double inv = rsqrt_nr(lj > 0.0 ? lj : 1.0);
    if (lane < rank) ssn[lane] = lj * inv;
    double prt[RM];
#pragma unroll
    for (int l = 0; l < RM; ++l) prt[l] = l < m ? __shfl_sync(FULL, zj, l) * v[l] : 0.0;
    const double sz = tsum<RM>(prt);
#pragma unroll
    for (int l = 0; l < RM; ++l) {
      const double sl = __shfl_sync(FULL, sg, l);
      u[l] = l < r ? sl * v[l] * inv : (l == r ? sz * inv : 0.0);
      if (lane >= rank) u[l] = 0.0;
    }
  }
  TSG_CLK(6);
#pragma unroll
  for (int l = 0; l < RM; ++l) sU[l * P + lane] = u[l];
  __syncwarp();
  // G_ij = u_i . u_j (i < j) into sG (shared), then u_j -= sum_i G_ij u_i
  // (classical, from the unmodified columns)
  double* sG = sW + 32 * 33 * 3;  // sWcm: the general solver's W copy (unused on this path)
#pragma unroll 4
  for (int i = 0; i < RM; ++i) {
    double pr[RM];
#pragma unroll
    for (int l = 0; l < RM; ++l) pr[l] = sU[l * P + i] * u[l];
    const double gi = tsum<RM>(pr);
    sG[i * 32 + lane] = (i < lane) ? gi : 0.0;
  }
#pragma unroll 4
  for (int i = 0; i < RM; ++i) {
    const double gi = sG[i * 32 + lane];
#pragma unroll
    for (int l = 0; l < RM; ++l) u[l] = fma(-gi, sU[l * P + i], u[l]);
  }
  {
    double sq2[RM];
#pragma unroll
    for (int l = 0; l < RM; ++l) sq2[l] = u[l] * u[l];
    const double ss = tsum<RM>(sq2);
    const double inv = ss > 0.0 ? rsqrt_nr(ss) : 0.0;
#pragma unroll
    for (int l = 0; l < RM; ++l) u[l] *= inv;
  }
  __syncwarp();
  if (lane < rank) {
#pragma unroll
    for (int l = 0; l < RM; ++l)
      if (l <= r) sU[l * P + lane] = u[l];
  }
  __syncwarp();
  return rank;
}

// Rows per thread RPT (n <= 256 RPT). Q (columns < r_hint) and b reach
// shared memory by bulk copies (TMA engine, one per Q column) at entry, so no
// thread holds rows in registers across the inner solve; the old core is read
// in the update (L2-resident: written by the previous insertion).
__host__ __device__ constexpr long long smem_doubles(long long n, int rhint) {
  return kSmallFixed + n * (rhint + 1) + 4;
}

template <int RMAX, int RPT>
__global__ void __launch_bounds__(kThreads, 1) isvd_cta_kernel(IsvdBufs B) {
  constexpr int RM = RMAX + 1;
  constexpr int P = 33;
  extern __shared__ __align__(16) double dsm[];
  double* sW = dsm;
  double* sU = sW + 32 * 33;
  double* sQ = sU + 32 * 33;
  double* sWcm = sQ + 32 * 33;
  double* spg = sWcm + 33 * 33;
  double* sM = spg + 32 * 32;
  const long long n = B.n;
  const int rhint = B.r_hint;
  // Q columns < r_hint, ld n, at a 16-byte aligned shared address (bulk copies)
  double* qs = dsm + kSmallFixed;
  if ((unsigned)__cvta_generic_to_shared(qs) & 15u) ++qs;
  double* bs = qs + n * rhint;         // b
  __shared__ __align__(8) unsigned long long qbar;
  __shared__ double wp[kWarps][33];
  __shared__ double red[32];
  __shared__ double sp1[33], sp2[33], sp[33];
  __shared__ double sx[8 * 32];
  __shared__ int si[3 * 32];
  __shared__ double sd[32], sz[33], ssig[33], ssn[33], sw[33], slam[33];
  __shared__ double sh_bsq, sh_esq, sh_delta, sh_sqerr;
  __shared__ int sh_rank, sh_deg;
  Ctrl* c = B.ctrl;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  TSG_CLK(0);
  if (tid == 0) {
    const unsigned bytes = (unsigned)(n * 8);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&qbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&qbar)),
                 "r"(bytes * (unsigned)(rhint + 1))
                 : "memory");
    for (int l = 0; l < rhint; ++l)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              (unsigned)__cvta_generic_to_shared(qs + l * n)),
          "l"(B.q + l * n), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(&qbar))
          : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(bs)),
        "l"(B.b), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(&qbar))
        : "memory");
  }
  // every thread reads r / n_d (one broadcast round trip)
  const int r = __ldcg(&c->r);
  const long long n_d = __ldcg(&c->n_d);
  // the small factors' padding is read (times zero) by the unrolled row
  // updates: keep it finite
  for (int i = tid; i < 3 * 32 * 33 + 33 * 33 + 32 * 32 + 33 * 32; i += kThreads) dsm[i] = 0.0;
  if (tid == 0) {
    const SliceCtl* sl = B.slot;
    if (B.commit_modes > 0) {
      const double sn = sqrt(sl->slice_sq);
      double tot = c->total_input_sq, ns = c->nonstream_discarded_sq;
      tot += sn * sn;  // streaming.cpp:169
      for (int kk = 0; kk < B.commit_modes; ++kk) {
        const double rn = sqrt(sl->res_sq[kk]);
        ns += rn * rn;  // streaming.cpp:137
      }
      c->total_input_sq = tot;
      c->nonstream_discarded_sq = ns;
    }
    sh_delta = sl->delta;
    sh_sqerr = c->squared_error;
  }
  if (tid < 32) ssig[tid] = tid < r ? B.sigma[tid] : 0.0;
  __syncthreads();  // mbarrier initialised
  {
    const unsigned a = (unsigned)__cvta_generic_to_shared(&qbar);
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(a)
        : "memory");
  }
  TSG_CLK(8);
  auto qrow = [&](long long row, double (&q)[RMAX]) {
    const long long rc = row < n ? row : 0;
#pragma unroll
    for (int l = 0; l < RMAX; ++l) {
      const double v = qs[(l < rhint ? l : 0) * n + rc];
      q[l] = (l < r && row < n) ? v : 0.0;
    }
  };
  // ---- CGS2 split b = Q p + e (isvd.cpp:172-191), two classical passes;
  // ||e||^2 = ||e1||^2 - ||p2||^2 (see isvd_grid.cuh)
  double bsq_part = 0.0;
  {
    double acc[RMAX];
#pragma unroll
    for (int l = 0; l < RMAX; ++l) acc[l] = 0.0;
#pragma unroll
    for (int p = 0; p < RPT; ++p) {
      const long long row = tid + (long long)kThreads * p;
      double q[RMAX];
      qrow(row, q);
      const double bb = row < n ? bs[row] : 0.0;
#pragma unroll
      for (int l = 0; l < RMAX; ++l) acc[l] = fma(q[l], bb, acc[l]);
      bsq_part = fma(bb, bb, bsq_part);
    }
    block_reduce_vec<RMAX, true, kWarps>(acc, wp, sp1);
  }
  double e1[RPT];
  double e1sq = 0.0;
  {
    double acc[RMAX], c1[RMAX];
#pragma unroll
    for (int l = 0; l < RMAX; ++l) {
      acc[l] = 0.0;
      c1[l] = sp1[l];
    }
#pragma unroll
    for (int p = 0; p < RPT; ++p) {
      const long long row = tid + (long long)kThreads * p;
      double q[RMAX];
      qrow(row, q);
      const double bb = row < n ? bs[row] : 0.0;
      double pr[RMAX];
#pragma unroll
      for (int l = 0; l < RMAX; ++l) pr[l] = q[l] * c1[l];
      e1[p] = bb - tree_sum<RMAX>(pr);
      e1sq = fma(e1[p], e1[p], e1sq);
#pragma unroll
      for (int l = 0; l < RMAX; ++l) acc[l] = fma(q[l], e1[p], acc[l]);
    }
    block_reduce_vec<RMAX, true, kWarps>(acc, wp, sp2);
  }
  {
    double ev[2] = {e1sq, bsq_part};
    block_reduce_vec<2, false, kWarps>(ev, wp, red);
  }
  TSG_CLK(1);
  if (tid < 33) sp[tid] = sp1[tid] + sp2[tid];
  if (tid == 0) {
    double p2sq = 0.0;
    for (int l = 0; l < r; ++l) p2sq = fma(sp2[l], sp2[l], p2sq);
    const double esq = fmax(red[0] - p2sq, 0.0);
    sh_bsq = red[1];
    sh_esq = esq;
    c->proj_sq = red[1];
    c->e_sq = esq;
    sh_deg = (sqrt(esq) <= kOrthEps * sqrt(red[1])) ? 1 : 0;  // isvd.cpp:191
  }
  __syncthreads();
  // ---- inner problem (warp 0) || p_gram of the old left factor (warps 1..)
  if (wid == 0) {
    TSG_CLK(4);
    const double kk = sqrt(sh_esq);
    int rank = (r + 1 <= RM && r >= 1) ? inner_fast<RM, 6>(c, r, sh_deg, ssig, sp, kk, sh_delta, sh_sqerr,
                                                            sW, sU, ssn)
                                       : -1;
    if (rank < 0) {
      if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&g_isvd_clk[26]), 1ull);
      // deflation / slow convergence: the general solver
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
      rank = inner_warp_small<RM>(c, r, ssig, sp, kk, sh_deg, sh_delta, sh_sqerr, ssn, sW, sU, sd, sz,
                                  S, slam, sWcm);
    }
    TSG_CLK(7);
    if (lane == 0) sh_rank = rank;
  } else {
    const int npair = r * (r + 1) / 2;
    for (int pidx = wid - 1; pidx < npair; pidx += kWarps - 1) {
      int j = 0, rem = pidx;
      while (rem > j) {
        rem -= j + 1;
        ++j;
      }
      const int l = rem;
      double s = 0.0;
      for (long long i = lane; i < n_d; i += 32) s = fma(B.left[i * B.capr + l], B.left[i * B.capr + j], s);
      s = warp_sum(s);
      if (lane == 0) {
        spg[l + j * r] = s;
        spg[j + l * r] = s;
      }
    }
  }
  __syncthreads();
  TSG_CLK(2);
  const int rank = sh_rank;
  const int deg = sh_deg;
  // M = P'_top^T p_gram (rank x r), w = last row of P' (streaming.cpp:199-218)
  for (int idx = tid; idx < rank * r; idx += kThreads) {
    const int jn = idx % rank, j = idx / rank;
    double s = 0.0;
    for (int l = 0; l < r; ++l) s = fma(sU[l * P + jn], spg[l + j * r], s);
    sM[jn + j * rank] = s;
  }
  if (tid < rank) {
    sw[tid] = sU[r * P + tid];
    B.sigma_new[tid] = ssn[tid];
  }
  __syncthreads();
  TSG_CLK(16);
  // ---- own rows: e = e1 - Q p2; Qn = [Q q] W, Cn = C M^T + b w^T; coupling
  double dacc = 0.0, cacc = 0.0;
  {
    const double inv = deg ? 0.0 : 1.0 / sqrt(sh_esq);
    double c2[RMAX];
#pragma unroll
    for (int l = 0; l < RMAX; ++l) c2[l] = sp2[l];
#pragma unroll 1
    for (int p = 0; p < RPT; ++p) {
      const long long i = tid + (long long)kThreads * p;
      if (i >= n) break;
      double q[RMAX], cr[RMAX];
      qrow(i, q);
#pragma unroll
      for (int l = 0; l < RMAX; ++l) cr[l] = B.c[i + (long long)(l < r ? l : 0) * n];
#pragma unroll
      for (int l = 0; l < RMAX; ++l) cr[l] = l < r ? cr[l] : 0.0;
      const double bb = bs[i];
      double ep = e1[0];
#pragma unroll
      for (int pp = 1; pp < RPT; ++pp) ep = p == pp ? e1[pp] : ep;
      double pr[RMAX];
#pragma unroll
      for (int l = 0; l < RMAX; ++l) pr[l] = q[l] * c2[l];
      const double e = ep - tree_sum<RMAX>(pr);
      const double qi = deg ? 0.0 : e * inv;
      constexpr int JB = 8;
#pragma unroll
      for (int j0 = 0; j0 < RM; j0 += JB) {
        if (j0 < rank) {
          double sq[JB], sc[JB];
#pragma unroll
          for (int jj = 0; jj < JB; ++jj) {
            sq[jj] = 0.0;
            sc[jj] = 0.0;
          }
#pragma unroll
          for (int l = 0; l < RMAX; ++l) {
#pragma unroll
            for (int jj = 0; jj < JB; ++jj) {
              sq[jj] = fma(q[l], sW[l * P + j0 + jj], sq[jj]);
              sc[jj] = fma(cr[l], sM[j0 + jj + l * rank], sc[jj]);
            }
          }
#pragma unroll
          for (int jj = 0; jj < JB; ++jj) {
            const int jn = j0 + jj;
            if (jn < rank) {
              double q2 = sq[jj];
              if (!deg) q2 = fma(qi, sW[r * P + jn], q2);
              const double c2v = fma(sw[jn], bb, sc[jj]);
              B.qn[i + (long long)jn * n] = q2;
              B.cn[i + (long long)jn * n] = c2v;
              const double diff = fma(-q2, ssn[jn], c2v);
              dacc = fma(diff, diff, dacc);
              cacc = fma(c2v, c2v, cacc);
            }
          }
        }
      }
    }
  }
  TSG_CLK(14);
  // ---- left <- blkdiag(left, 1) P' (isvd.cpp:227-237)
  {
    const long long total = (n_d + 1) * B.capr;
    for (long long idx = tid; idx < total; idx += kThreads) {
      const long long i = idx / B.capr;
      const int j = (int)(idx % B.capr);
      double v = 0.0;
      if (j < rank) {
        if (i < n_d) {
          for (int l = 0; l < r; ++l) v = fma(B.left[i * B.capr + l], sU[l * P + j], v);
        } else {
          v = sU[r * P + j];
        }
      }
      B.left_new[idx] = v;
    }
  }
  TSG_CLK(15);
  {
    double dv[2] = {dacc, cacc};
    block_reduce_vec<2, false, kWarps>(dv, wp, red);
  }
  TSG_CLK(3);
  // ---- ledgers, record, publication (warp 0)
  if (wid == 0) {
    __shared__ Metrics sm_rec;
    __shared__ Ctrl sm_ctl;
    if (lane == 0) {
      const double dd = red[0], cs = red[1];
      Ctrl cc = *c;
      const SliceCtl* sl = B.slot;
      cc.degenerate = deg;
      cc.coupling_diff_sq = dd;
      cc.core_sq = cs;
      if (sqrt(dd) > kCouplingTol * sqrt(cs) + 1e-300 && cc.status == 0) cc.status = 2;  // streaming.cpp:55-63
      cc.r = rank;
      cc.r_new = rank;
      cc.n_d = n_d + 1;
      cc.insertions = cc.insertions + 1;
      Metrics mm;
      mm.slice_index = n_d;
      for (int kk = 0; kk < kMaxD; ++kk) mm.ranks[kk] = (kk + 1 < B.order) ? B.spatial_ranks[kk] : 0;
      mm.ranks[B.order - 1] = rank;
      mm.slice_norm = sqrt(sl->slice_sq);
      mm.projected_norm = sqrt(sh_bsq);
      for (int kk = 0; kk < kMaxD; ++kk) mm.mode_residuals[kk] = (kk + 1 < B.order) ? sqrt(sl->res_sq[kk]) : 0.0;
      const double booked = cc.squared_error + cc.nonstream_discarded_sq;
      mm.error_estimate = cc.total_input_sq <= 0.0 ? 0.0 : sqrt(fmax(booked, 0.0) / cc.total_input_sq);
      mm.expanded_mask = 0;
      mm.trunc_margin = cc.trunc_margin;
      mm.sweeps = cc.sweeps;
      const unsigned long long kr = cc.records;
      cc.records = kr + 1;
      *c = cc;
      sm_rec = mm;
      sm_ctl = cc;
    }
    __syncwarp();
    const unsigned long long kr = sm_ctl.records - 1;
    const int pos = (int)(kr % kRecRing);
    {
      const unsigned long long* srcm = reinterpret_cast<const unsigned long long*>(&sm_rec);
      unsigned long long* dstm = reinterpret_cast<unsigned long long*>(&B.ring->rec[pos]);
      for (int w = lane; w < (int)(sizeof(Metrics) / 8); w += 32) dstm[w] = srcm[w];
      const unsigned long long* srcc = reinterpret_cast<const unsigned long long*>(&sm_ctl);
      unsigned long long* dstc = reinterpret_cast<unsigned long long*>(&B.ring->ctrl[pos]);
      for (int w = lane; w < (int)(sizeof(Ctrl) / 8); w += 32) dstc[w] = srcc[w];
    }
    // device ring (gpu scope): the tail kernel publishes it to the host
    __threadfence();
    __syncwarp();
    if (lane == 0) *reinterpret_cast<volatile unsigned long long*>(&B.ring->done) = kr + 1;
  }
  TSG_CLK(9);
}

}  // namespace cta
}  // namespace
