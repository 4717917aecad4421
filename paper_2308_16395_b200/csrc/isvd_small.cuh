// Latency-optimised single-CTA insertion for n <= 512 * RPT rows (the
// configurations whose insertion would otherwise bound the stream rate).
// Included by isvd.cu (shares its helpers). Same arithmetic contract as
// isvd_fused_kernel (isvd.cpp:163-250 add_row, streaming.cpp:196-224), with
// the latency chain restructured:
//   * the slice's ledger commit (streaming.cpp:137,169) runs here, not in a
//     separate kernel;
//   * Q and b rows stay in registers across the CGS2 passes and the update;
//     the old core is staged into shared memory by cp.async at entry;
//   * warp 0 solves the inner problem (register secular solver, MGS) while
//     warps 1..15 form p_gram = left^T left (isvd.cpp:86-100);
//   * small factors never round-trip through global memory;
//   * the record is published by a warp-parallel copy.
#pragma once

namespace {

// Sum of an unrolled register array (tree order, deterministic).
template <int N>
__device__ __forceinline__ double tree_sum(const double (&a)[N]) {
  double t[N];
#pragma unroll
  for (int i = 0; i < N; ++i) t[i] = a[i];
  // __dadd_rn: no contraction with the producers of a[], so the result does not
  // depend on how a given instantiation was scheduled
#pragma unroll
  for (int w = 1; w < N; w <<= 1) {
#pragma unroll
    for (int i = 0; i + w < N; i += 2 * w) t[i] = __dadd_rn(t[i], t[i + w]);
  }
  return t[0];
}

// Block-wide reduction of NV per-thread values into dst[0..NV) (512 threads).
// Warp stage: transposed butterfly (NV padded to a power of two <= 32);
// block stage: NV threads sum the 16 warp partials in warp order.
// FIXED selects the 32-wide layout regardless of NV, so that the summation
// order of coefficient j does not depend on the register bound RMAX.
template <int NV, bool FIXED = false, int NWP = 16>
__device__ __forceinline__ void block_reduce_vec(double (&v)[NV], double (*wp)[33], double* dst) {
  constexpr int P2 = FIXED ? 32 : NV <= 1 ? 1 : NV <= 2 ? 2 : NV <= 4 ? 4 : NV <= 8 ? 8 : NV <= 16 ? 16 : 32;
  constexpr int L2 = P2 == 1 ? 0 : P2 == 2 ? 1 : P2 == 4 ? 2 : P2 == 8 ? 3 : P2 == 16 ? 4 : 5;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double a[P2];
#pragma unroll
  for (int i = 0; i < P2; ++i) a[i] = i < NV ? v[i] : 0.0;
#pragma unroll
  for (int st = 0; st < L2; ++st) {
    const int o = 16 >> st;
    const int half = P2 >> (st + 1);
    const bool hi = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = hi ? a[i] : a[i + half];
      const double keep = hi ? a[i + half] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
#pragma unroll
  for (int o = 16 >> L2; o > 0; o >>= 1) a[0] += __shfl_xor_sync(0xffffffffu, a[0], o);
  const int j = lane >> (5 - L2);
  if ((lane & ((32 >> L2) - 1)) == 0 && j < NV) wp[wid][j] = a[0];
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NWP; ++w) s += wp[w][threadIdx.x];
    dst[threadIdx.x] = s;
  }
  __syncthreads();
}

// Inner problem in warp 0, outputs in shared memory:
//   sW (pitch 33): eigenvectors of S'^T S' (columns = right factor W, sorted)
//   sUo (pitch 33): left factor P' = S' W / sigma after one MGS pass
//   ssn: sigma_new (rank entries); returns rank (lane-uniform).
template <int RM>
__device__ int inner_warp_small(Ctrl* c, int r, const double* ssig, const double* sp, double k,
                                int deg, double delta, double sq_err, double* ssn, double* sW,
                                double* sUo, double* sd, double* sz, secular::Scratch S,
                                double* lam_g, double* W_g) {
  const int lane = threadIdx.x & 31;
  const int m = deg ? r : r + 1;
  constexpr int P = 33;
  if (lane < m) {
    const double sg = lane < r ? ssig[lane] : 0.0;
    sd[lane] = sg * sg;
    sz[lane] = lane < r ? sp[lane] : k;
  }
  __syncwarp();
  const int iters = secular::eig_rank_one_fast<RM>(m, sd, sz, S, lam_g, W_g, sW);
  TSG_CLK(5);
  // eigenvalue `lane` (descending, clamped) in a register
  double lj = lane < m ? lam_g[lane] : 0.0;
  // truncation (linalg.cpp:224-240, isvd.cpp:210-215): sigma floor lane-parallel
  const double smax = secular::sqrt_nr(__shfl_sync(FULL, lj, 0));
  int rank = 0;
  if (smax > 0.0) {
    const double fl = kSigmaZeroFactor * smax;
    if (lane < m && secular::sqrt_nr(lj) <= fl) lj = 0.0;
    double lv[RM];
#pragma unroll
    for (int i = 0; i < RM; ++i) lv[i] = __shfl_sync(FULL, lj, i);
    if (lane == 0) {
      const double budget = delta * delta;
      double s = 0.0, prev_excess = -1.0;
      int rr = m;
#pragma unroll
      for (int i = RM - 1; i >= 0; --i) {
        if (i < m && prev_excess < 0.0) {
          const double nx = s + lv[i];
          if (nx <= budget) {
            s = nx;
            rr = i;
          } else {
            prev_excess = nx;
          }
        }
      }
      rank = rr < 1 ? 1 : rr;
      double disc = 0.0;
#pragma unroll
      for (int j = RM - 1; j >= 0; --j)
        if (j < m && j >= rank) disc += lv[j];
      double margin = 0.0;
      if (budget > 0.0) {
        double mg = fabs(budget - s) / budget;
        if (prev_excess >= 0.0) mg = fmin(mg, fabs(prev_excess - budget) / budget);
        margin = mg;
      }
      double added = disc;
      if (deg) added += k * k;
      c->trunc_margin = margin;
      c->sweeps = iters;
      c->added_error_sq = added;
      c->squared_error = sq_err + added;  // isvd.cpp:212-215
      c->r_new = rank;
      c->degenerate = deg;
    }
  } else if (lane == 0) {
    c->status = 3;  // S' == 0 cannot happen with r >= 1 and sigma > 0
    c->r_new = 0;
    c->degenerate = deg;
  }
  rank = __shfl_sync(FULL, rank, 0);
  TSG_CLK(6);
  // U = S' W / sigma (column `lane` in registers; rows i < r of S' are diag(s))
  double u[RM];
#pragma unroll
  for (int l = 0; l < RM; ++l) u[l] = 0.0;
  if (lane < rank) {
    const double inv = secular::rsqrt_nr(lj);
    const double sn = lj * inv;
    ssn[lane] = sn;
    double prt[RM];
#pragma unroll
    for (int l = 0; l < RM; ++l) prt[l] = l < m ? sz[l] * sW[l * P + lane] : 0.0;
    const double s = tree_sum<RM>(prt);
#pragma unroll
    for (int l = 0; l < RM; ++l) {
      if (l < r) u[l] = ssig[l] * sW[l * P + lane] * inv;
      else if (l == r) u[l] = s * inv;
    }
  }
  // one MGS pass, right-looking (linalg.cpp:64-78)
  for (int i = 0; i < rank; ++i) {
    if (lane == i) {
      double sq[RM];
#pragma unroll
      for (int l = 0; l < RM; ++l) sq[l] = u[l] * u[l];
      const double ss = tree_sum<RM>(sq);
      if (ss > 0.0) {
        const double inv = secular::rsqrt_nr(ss);
#pragma unroll
        for (int l = 0; l < RM; ++l) u[l] *= inv;
      }
    }
    double ui[RM], pr[RM];
#pragma unroll
    for (int l = 0; l < RM; ++l) {
      ui[l] = __shfl_sync(FULL, u[l], i);
      pr[l] = ui[l] * u[l];
    }
    const double dot = tree_sum<RM>(pr);
    if (lane > i && lane < rank) {
#pragma unroll
      for (int l = 0; l < RM; ++l) u[l] = fma(-dot, ui[l], u[l]);
    }
  }
  if (lane < rank) {
#pragma unroll
    for (int l = 0; l < RM; ++l)
      if (l <= r) sUo[l * P + lane] = u[l];
  }
  __syncwarp();
  return rank;
}

// doubles of fixed dynamic shared memory ahead of the staged core (even)
constexpr int kSmallFixed = 3 * 32 * 33 + 33 * 33 + 32 * 32 + 33 * 32 + 1;

template <int RMAX, int RPT, bool QREG>
__global__ void __launch_bounds__(512, 1) isvd_small_kernel(IsvdBufs B) {
  constexpr int RM = RMAX + 1;
  constexpr int QR = QREG ? RMAX : 1;  // Q rows held in registers, else re-read (same arithmetic)
  constexpr int P = 33;
  extern __shared__ double dsm[];  // small factors, then the staged old core (n x r_hint)
  double* sW = dsm;                 // 32 x 33
  double* sU = sW + 32 * 33;        // 32 x 33
  double* sQ = sU + 32 * 33;        // 32 x 33 (rotation scratch of the fallback solver)
  double* sWcm = sQ + 32 * 33;      // 33 x 33
  double* spg = sWcm + 33 * 33;     // 32 x 32
  double* sM = spg + 32 * 32;       // 33 x 32
  double* fsm = dsm + kSmallFixed;  // staged core (16-byte aligned)
  __shared__ double wp[16][33];
  __shared__ double red[32];
  __shared__ double sp1[RM + 1], sp2[RM + 1], sp[RM + 1];
  __shared__ double sx[8 * 32];
  __shared__ int si[3 * 32];
  __shared__ double sd[32], sz[33], ssig[33], ssn[33], sw[33];
  __shared__ double slam[33];
  __shared__ double sh_bsq, sh_esq, sh_delta, sh_sqerr;
  __shared__ int sh_r, sh_rank, sh_deg;
  __shared__ long long sh_nd;
  Ctrl* c = B.ctrl;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const long long n = B.n;
  TSG_CLK(0);
  // ---- entry: ledger commit + control scalars (thread 0), core staging
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
    sh_r = c->r;
    sh_nd = c->n_d;
    sh_delta = sl->delta;
    sh_sqerr = c->squared_error;
  }
  const bool stage_core = B.stage_core != 0;
  if (stage_core) {
    const long long cnt = n * (long long)B.r_hint;  // columns >= r are never read
    const long long chunks = cnt >> 1;
    for (long long i = tid; i < chunks; i += 512) {
      const unsigned dst = (unsigned)__cvta_generic_to_shared(fsm + 2 * i);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(B.c + 2 * i));
    }
    if ((cnt & 1) && tid == 0) fsm[cnt - 1] = B.c[cnt - 1];
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  __syncthreads();
  const int r = sh_r;
  const long long n_d = sh_nd;
  // ---- Q and b rows in registers
  double qr[RPT][QR], bv[RPT];
#pragma unroll
  for (int p = 0; p < RPT; ++p) {
    const long long i = tid + 512LL * p;
    const bool ok = i < n;
    bv[p] = ok ? B.b[i] : 0.0;
#pragma unroll
    for (int l = 0; l < QR; ++l) qr[p][l] = (QREG && ok && l < r) ? B.q[i + (long long)l * n] : 0.0;
  }
  auto Qv = [&](int p, int l) -> double {
    if (QREG) return qr[p][QREG ? l : 0];
    const long long i = tid + 512LL * p;
    return (i < n && l < r) ? B.q[i + (long long)l * n] : 0.0;
  };
  TSG_CLK(8);
  // ---- CGS2 split b = Q p + e (isvd.cpp:172-191; two classical passes)
  double bsq_part = 0.0;
  {
    double acc[RMAX];
#pragma unroll
    for (int l = 0; l < RMAX; ++l) acc[l] = 0.0;
#pragma unroll
    for (int p = 0; p < RPT; ++p) {
#pragma unroll
      for (int l = 0; l < RMAX; ++l) acc[l] = fma(Qv(p, l), bv[p], acc[l]);
      bsq_part = fma(bv[p], bv[p], bsq_part);
    }
    block_reduce_vec<RMAX, true>(acc, wp, sp1);
  }
  double e[RPT];
  {
    double acc[RMAX];
#pragma unroll
    for (int l = 0; l < RMAX; ++l) acc[l] = 0.0;
    double c1[RMAX];
#pragma unroll
    for (int l = 0; l < RMAX; ++l) c1[l] = sp1[l];
#pragma unroll
    for (int p = 0; p < RPT; ++p) {
      double pr[RMAX];
#pragma unroll
      for (int l = 0; l < RMAX; ++l) pr[l] = Qv(p, l) * c1[l];
      e[p] = bv[p] - tree_sum<RMAX>(pr);
#pragma unroll
      for (int l = 0; l < RMAX; ++l) acc[l] = fma(Qv(p, l), e[p], acc[l]);
    }
    block_reduce_vec<RMAX, true>(acc, wp, sp2);
  }
  {
    double c2[RMAX];
#pragma unroll
    for (int l = 0; l < RMAX; ++l) c2[l] = sp2[l];
    double es = 0.0;
#pragma unroll
    for (int p = 0; p < RPT; ++p) {
      double pr[RMAX];
#pragma unroll
      for (int l = 0; l < RMAX; ++l) pr[l] = Qv(p, l) * c2[l];
      e[p] = e[p] - tree_sum<RMAX>(pr);
      if (tid + 512LL * p < n) es = fma(e[p], e[p], es);
    }
    double ev[2] = {es, bsq_part};
    block_reduce_vec<2>(ev, wp, red);
  }
  TSG_CLK(1);
  if (tid < RMAX) sp[tid] = sp1[tid] + sp2[tid];
  if (tid == 0) {
    sh_bsq = red[1];
    sh_esq = red[0];
    c->proj_sq = red[1];
    c->e_sq = red[0];
    sh_deg = (sqrt(red[0]) <= kOrthEps * sqrt(red[1])) ? 1 : 0;  // isvd.cpp:191
  }
  if (tid < 32) ssig[tid] = tid < r ? B.sigma[tid] : 0.0;
  __syncthreads();
  // ---- inner problem (warp 0) || p_gram of the old left factor (warps 1..15)
  if (wid == 0) {
    const double kk = sqrt(sh_esq);
    const int deg = sh_deg;
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
    TSG_CLK(4);
    const int rank = inner_warp_small<RM>(c, r, ssig, sp, kk, deg, sh_delta, sh_sqerr, ssn, sW, sU,
                                          sd, sz, S, slam, sWcm);
    TSG_CLK(7);
    if (lane == 0) {
      sh_rank = rank;
      c->r_new = rank;
    }
  } else {
    // p_gram[l][j] = sum_i left[i][l] left[i][j] (pairs l <= j), warp per pair
    const int npair = r * (r + 1) / 2;
    for (int pidx = wid - 1; pidx < npair; pidx += 15) {
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
  // M = P'_top^T p_gram (rank x r), w = last row of P'
  for (int idx = tid; idx < rank * r; idx += 512) {
    const int jn = idx % rank, j = idx / rank;
    double s = 0.0;
    for (int l = 0; l < r; ++l) s = fma(sU[l * P + jn], spg[l + j * r], s);
    sM[jn + j * rank] = s;
  }
  if (tid < rank) {
    sw[tid] = sU[r * P + tid];
    B.sigma_new[tid] = ssn[tid];
  }
  TSG_CLK(16);
  if (stage_core) asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  TSG_CLK(17);
  // ---- Q / core rows: Qn = [Q q] W, Cn = C M^T + b w^T, coupling partials
  double dacc = 0.0, cacc = 0.0;
  {
    const double inv = deg ? 0.0 : 1.0 / sqrt(sh_esq);
#pragma unroll
    for (int p = 0; p < RPT; ++p) {
      const long long i = tid + 512LL * p;
      if (i >= n) continue;
      double cr[RMAX];
#pragma unroll
      for (int l = 0; l < RMAX; ++l)
        cr[l] = l < r ? (stage_core ? fsm[i + (long long)l * n] : B.c[i + (long long)l * n]) : 0.0;
      const double qi = deg ? 0.0 : e[p] * inv;
      // output columns in blocks of JB advance together (independent chains)
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
            if (l < r) {
              const double ql = Qv(p, l), cl = cr[l];
#pragma unroll
              for (int jj = 0; jj < JB; ++jj) {
                sq[jj] = fma(ql, sW[l * P + j0 + jj], sq[jj]);
                sc[jj] = fma(cl, sM[j0 + jj + l * rank], sc[jj]);
              }
            }
          }
#pragma unroll
          for (int jj = 0; jj < JB; ++jj) {
            const int jn = j0 + jj;
            if (jn < rank) {
              double q2 = sq[jj];
              if (!deg) q2 = fma(qi, sW[r * P + jn], q2);
              const double c2 = fma(sw[jn], bv[p], sc[jj]);
              B.qn[i + (long long)jn * n] = q2;
              B.cn[i + (long long)jn * n] = c2;
              const double diff = fma(-q2, ssn[jn], c2);
              dacc = fma(diff, diff, dacc);
              cacc = fma(c2, c2, cacc);
            }
          }
        }
      }
      if (p == 0) TSG_CLK(18);
    }
  }
  TSG_CLK(14);
  // left <- blkdiag(left, 1) P' (isvd.cpp:227-237)
  {
    const int rows = r + 1;
    (void)rows;
    const long long total = (n_d + 1) * B.capr;
    for (long long idx = tid; idx < total; idx += 512) {
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
    block_reduce_vec<2>(dv, wp, red);
  }
  TSG_CLK(3);
  // ---- ledgers, record, publication (warp 0)
  if (wid == 0) {
    __shared__ Metrics sm_rec;
    __shared__ Ctrl sm_ctl;
    if (lane == 0) {
      const double dd = red[0], cs = red[1];
      Ctrl cc = *c;  // one batch of loads
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

}  // namespace
