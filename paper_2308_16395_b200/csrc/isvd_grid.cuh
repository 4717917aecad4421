// Multi-CTA insertion for n <= kGridMaxRows: the serial part (ledger commit,
// CGS2 split, inner problem, p_gram) runs in CTA 0 ("leader") exactly as in
// isvd_small_kernel; the row-parallel part (Q / core row updates, left
// rows, coupling partials) is spread over ceil(n / 128) CTAs, which prefetch
// their rows and wait on the leader's handoff flag. The last CTA to finish
// reduces the coupling partials in CTA order and publishes the record.
// Included by isvd.cu after isvd_small.cuh (shares its helpers).
// Reference: isvd.cpp:163-250 (add_row), streaming.cpp:196-224.
#pragma once

namespace {

constexpr int kGridRows = 128;          // update rows per CTA
constexpr long long kGridMaxRows = 4096;

// handoff layout (doubles)
constexpr int kHW = 0;                   // W, pitch 33 (rows l < m, cols < rank)
constexpr int kHU = 33 * 33;             // P', pitch 33 (rows <= r)
constexpr int kHM = 2 * 33 * 33;         // M (jn + l * rank)
constexpr int kHw = 3 * 33 * 33;         // w
constexpr int kHsn = kHw + 33;           // sigma_new
constexpr int kHs1 = kHsn + 33;          // sp1
constexpr int kHs2 = kHs1 + 33;          // sp2
constexpr int kHsc = kHs2 + 33;          // scalars: inv_e, rank, deg

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int RMAX>
__global__ void __launch_bounds__(256, 2) isvd_grid_kernel(IsvdBufs B) {
  constexpr int RM = RMAX + 1;
  constexpr int P = 33;
  constexpr int NW = 8;
  extern __shared__ double dsm[];
  double* sW = dsm;
  double* sU = sW + 32 * 33;
  double* sQ = sU + 32 * 33;
  double* sWcm = sQ + 32 * 33;
  double* spg = sWcm + 33 * 33;
  double* sM = spg + 32 * 32;
  double* se1 = dsm + kSmallFixed;  // leader: e1 per row (n)
  __shared__ double wp[NW][33];
  __shared__ double red[32];
  __shared__ double sp1[RM + 1], sp2[RM + 1], sp[RM + 1];
  __shared__ double sx[8 * 32];
  __shared__ int si[3 * 32];
  __shared__ double sd[32], sz[33], ssig[33], ssn[33], sw[33], slam[33];
  __shared__ double sh_bsq, sh_esq, sh_delta, sh_sqerr, sh_inv;
  __shared__ int sh_r, sh_rank, sh_deg, sh_last;
  __shared__ long long sh_nd;
  __shared__ unsigned sh_epoch;
  Ctrl* c = B.ctrl;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const long long n = B.n;
  const bool leader = blockIdx.x == 0;
  unsigned* gs = B.gsync;
  double* hand = B.hand;
  if (leader) TSG_CLK(0);
  if (leader && tid == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    g_isvd_clk[24] = (long long)g;
  }
  if (tid == 0) {
    sh_epoch = __ldcg(gs);  // written by the previous launch (kernel boundary)
    sh_r = c->r;    // c->r and c->n_d change only in the final record (this kernel's end)
    sh_nd = c->n_d;
    if (leader) {
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
  }
  if (leader) TSG_CLK(21);
  __syncthreads();
  if (leader) TSG_CLK(22);
  const int r = sh_r;
  const long long n_d = sh_nd;
  const unsigned epoch = sh_epoch;
  // this CTA's rows, prefetched before any waiting
  const long long row = (long long)blockIdx.x * kGridRows + tid;
  const bool has_row = tid < kGridRows && row < n;
  // all loads unconditional from clamped (valid, written) addresses so they
  // issue back to back; out-of-range entries are zeroed by a 0/1 factor
  // (a predicated load followed by a zeroing move serialises on the register)
  double qv[RMAX], cv[RMAX], bvr;
  {
    const long long rowc = has_row ? row : 0;
    double mk[RMAX];
#pragma unroll
    for (int l = 0; l < RMAX; ++l) {
      const long long idx = rowc + (long long)(l < r ? l : 0) * n;
      qv[l] = B.q[idx];
      cv[l] = B.c[idx];
      mk[l] = (has_row && l < r) ? 1.0 : 0.0;
    }
    bvr = B.b[rowc];
#pragma unroll
    for (int l = 0; l < RMAX; ++l) {
      qv[l] *= mk[l];
      cv[l] *= mk[l];
    }
    if (!has_row) bvr = 0.0;
  }
  if (leader) {
    TSG_CLK(8);
    // ---- CGS2 over all rows (isvd.cpp:172-191), same arithmetic per row as
    // the followers' recomputation below
    double bsq_part = 0.0;
    // Q columns l >= r are read from column 0 and zeroed by a 0/1 factor:
    // unconditional loads issue back to back (see the row prefetch above)
    double mk[RMAX];
    long long coff[RMAX];
#pragma unroll
    for (int l = 0; l < RMAX; ++l) {
      mk[l] = l < r ? 1.0 : 0.0;
      coff[l] = (long long)(l < r ? l : 0) * n;
    }
    {
      double acc[RMAX];
#pragma unroll
      for (int l = 0; l < RMAX; ++l) acc[l] = 0.0;
      for (long long i = tid; i < n; i += 256) {
        const double bi = B.b[i];
        double qq[RMAX];
#pragma unroll
        for (int l = 0; l < RMAX; ++l) qq[l] = B.q[i + coff[l]];
#pragma unroll
        for (int l = 0; l < RMAX; ++l) acc[l] = fma(qq[l] * mk[l], bi, acc[l]);
        bsq_part = fma(bi, bi, bsq_part);
      }
      block_reduce_vec<RMAX, true, NW>(acc, wp, sp1);
    }
    double e1sq = 0.0;
    {
      double acc[RMAX];
#pragma unroll
      for (int l = 0; l < RMAX; ++l) acc[l] = 0.0;
      for (long long i = tid; i < n; i += 256) {
        double qq[RMAX], pr[RMAX];
#pragma unroll
        for (int l = 0; l < RMAX; ++l) qq[l] = B.q[i + coff[l]];
#pragma unroll
        for (int l = 0; l < RMAX; ++l) {
          qq[l] *= mk[l];
          pr[l] = qq[l] * sp1[l];
        }
        const double e1 = B.b[i] - tree_sum<RMAX>(pr);
        e1sq = fma(e1, e1, e1sq);
#pragma unroll
        for (int l = 0; l < RMAX; ++l) acc[l] = fma(qq[l], e1, acc[l]);
      }
      block_reduce_vec<RMAX, true, NW>(acc, wp, sp2);
    }
    {
      // ||e||^2 for e = e1 - Q p2 without a third pass over the rows:
      // ||e1||^2 - 2 p2^T Q^T e1 + ||Q p2||^2 = ||e1||^2 - ||p2||^2 up to
      // terms of order ||p2||^2 (Q^T Q - I), i.e. ~1e-24 ||b||^2: p2 is the
      // reorthogonalisation correction, ~eps ||b||
      double ev[2] = {e1sq, bsq_part};
      block_reduce_vec<2, false, NW>(ev, wp, red);
    }
    TSG_CLK(1);
    if (tid < RMAX) sp[tid] = sp1[tid] + sp2[tid];
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
    if (tid < 32) ssig[tid] = tid < r ? B.sigma[tid] : 0.0;
    __syncthreads();
    // ---- inner problem (warp 0) || p_gram of the old left factor (warps 1..7)
    if (wid == 0) {
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
      const int rank = inner_warp_small<RM>(c, r, ssig, sp, sqrt(sh_esq), sh_deg, sh_delta, sh_sqerr,
                                            ssn, sW, sU, sd, sz, S, slam, sWcm);
      TSG_CLK(7);
      if (lane == 0) sh_rank = rank;
    } else {
      const int npair = r * (r + 1) / 2;
      for (int pidx = wid - 1; pidx < npair; pidx += NW - 1) {
        int j = 0, rem = pidx;
        while (rem > j) {
          rem -= j + 1;
          ++j;
        }
        const int l = rem;
        double s = 0.0;
        for (long long i = lane; i < n_d; i += 32)
          s = fma(B.left[i * B.capr + l], B.left[i * B.capr + j], s);
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
    for (int idx = tid; idx < rank * r; idx += 256) {
      const int jn = idx % rank, j = idx / rank;
      double s = 0.0;
      for (int l = 0; l < r; ++l) s = fma(sU[l * P + jn], spg[l + j * r], s);
      sM[jn + j * rank] = s;
    }
    if (tid < rank) {
      sw[tid] = sU[r * P + tid];
      B.sigma_new[tid] = ssn[tid];
    }
    if (tid == 0) sh_inv = sh_deg ? 0.0 : 1.0 / sqrt(sh_esq);
    __syncthreads();
    TSG_CLK(16);
    if (gridDim.x > 1) {
      // ---- handoff to the followers
      const int m = sh_deg ? r : r + 1;
      for (int idx = tid; idx < 33 * 33; idx += 256) {
        const int l = idx / P, j = idx % P;
        if (l < m && j < rank) __stcg(hand + kHW + idx, sW[idx]);
        if (l <= r && j < rank) __stcg(hand + kHU + idx, sU[idx]);
      }
      for (int idx = tid; idx < rank * r; idx += 256) __stcg(hand + kHM + idx, sM[idx]);
      if (tid < rank) {
        __stcg(hand + kHw + tid, sw[tid]);
        __stcg(hand + kHsn + tid, ssn[tid]);
      }
      if (tid < RMAX) {
        __stcg(hand + kHs1 + tid, sp1[tid]);
        __stcg(hand + kHs2 + tid, sp2[tid]);
      }
      if (tid == 0) {
        __stcg(hand + kHsc + 0, sh_inv);
        __stcg(hand + kHsc + 1, (double)rank);
        __stcg(hand + kHsc + 2, (double)sh_deg);
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) st_release(gs + 1, epoch + 1);
    }
    TSG_CLK(17);
  } else {
    if (tid == 0) {
      while (ld_acquire(gs + 1) != epoch + 1) {
      }
    }
    __syncthreads();
    const int rank = (int)__ldcg(hand + kHsc + 1);
    const int deg = (int)__ldcg(hand + kHsc + 2);
    const int m = deg ? r : r + 1;
    for (int idx = tid; idx < 33 * 33; idx += 256) {
      const int l = idx / P, j = idx % P;
      if (l < m && j < rank) sW[idx] = __ldcg(hand + kHW + idx);
      if (l <= r && j < rank) sU[idx] = __ldcg(hand + kHU + idx);
    }
    for (int idx = tid; idx < rank * r; idx += 256) sM[idx] = __ldcg(hand + kHM + idx);
    if (tid < rank) {
      sw[tid] = __ldcg(hand + kHw + tid);
      ssn[tid] = __ldcg(hand + kHsn + tid);
    }
    if (tid < RMAX) {
      sp1[tid] = __ldcg(hand + kHs1 + tid);
      sp2[tid] = __ldcg(hand + kHs2 + tid);
    }
    if (tid == 0) {
      sh_inv = __ldcg(hand + kHsc + 0);
      sh_deg = deg;
      sh_rank = rank;
    }
    __syncthreads();
  }
  const int rank = sh_rank;
  const int deg = sh_deg;
  // ---- own rows: e (same arithmetic as the leader's CGS2), Qn, Cn, coupling
  double dacc = 0.0, cacc = 0.0;
  // row values addressed by a runtime index in the rolled loop below
  double* rowq = se1 + (leader ? n : 0);                 // [l * 128 + tid]
  double* rowc = rowq + RMAX * kGridRows;
  if (has_row) {
#pragma unroll
    for (int l = 0; l < RMAX; ++l) {
      rowq[l * kGridRows + tid] = qv[l];
      rowc[l * kGridRows + tid] = cv[l];
    }
  }
  auto qv_at = [&](int l) { return rowq[l * kGridRows + tid]; };
  auto cv_at = [&](int l) { return rowc[l * kGridRows + tid]; };
  if (has_row) {
    double pr[RMAX];
#pragma unroll
    for (int l = 0; l < RMAX; ++l) pr[l] = qv[l] * sp1[l];
    const double e1 = bvr - tree_sum<RMAX>(pr);
#pragma unroll
    for (int l = 0; l < RMAX; ++l) pr[l] = qv[l] * sp2[l];
    const double e = e1 - tree_sum<RMAX>(pr);
    const double qi = deg ? 0.0 : e * sh_inv;
    if (leader) TSG_CLK(19);
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
        // rolled over l (short hot loop: straight-line code executed once per
        // launch is instruction-fetch bound)
#pragma unroll 1
        for (int l = 0; l < r; ++l) {
          const double ql = qv_at(l), cl = cv_at(l);
#pragma unroll
          for (int jj = 0; jj < JB; ++jj) {
            sq[jj] = fma(ql, sW[l * P + j0 + jj], sq[jj]);
            sc[jj] = fma(cl, sM[j0 + jj + l * rank], sc[jj]);
          }
        }
#pragma unroll
        for (int jj = 0; jj < JB; ++jj) {
          const int jn = j0 + jj;
          if (jn < rank) {
            double q2 = sq[jj];
            if (!deg) q2 = fma(qi, sW[r * P + jn], q2);
            const double c2 = fma(sw[jn], bvr, sc[jj]);
            B.qn[row + (long long)jn * n] = q2;
            B.cn[row + (long long)jn * n] = c2;
            const double diff = fma(-q2, ssn[jn], c2);
            dacc = fma(diff, diff, dacc);
            cacc = fma(c2, c2, cacc);
          }
        }
      }
      if (leader && j0 == 0) TSG_CLK(20);
    }
  }
  if (leader) TSG_CLK(18);
  // ---- left <- blkdiag(left, 1) P' (isvd.cpp:227-237): this CTA's slab of
  // rows, threads 128..255 (all threads when the CTA has no update rows)
  {
    const long long total_rows = n_d + 1;
    const long long per = (total_rows + gridDim.x - 1) / gridDim.x;
    const long long r0 = (long long)blockIdx.x * per;
    const long long r1 = r0 + per < total_rows ? r0 + per : total_rows;
    const int t0 = tid - kGridRows;
    const int nt = 256 - kGridRows;
    if (tid >= kGridRows) {
      for (long long idx = r0 * B.capr + t0; idx < r1 * B.capr; idx += nt) {
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
  }
  if (leader) TSG_CLK(14);
  {
    double dv[2] = {dacc, cacc};
    block_reduce_vec<2, false, NW>(dv, wp, red);
  }
  // ---- arrival; the last CTA reduces in CTA order and publishes
  double* part = B.partial;
  if (tid == 0) {
    __stcg(part + 2 * blockIdx.x, red[0]);
    __stcg(part + 2 * blockIdx.x + 1, red[1]);
    __threadfence();
    const unsigned prev = atomicAdd(gs + 2, 1u);
    sh_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!sh_last) return;
  __threadfence();
  if (wid == 0) {
    double dd = 0.0, cs = 0.0;
    if (lane == 0) {
      for (unsigned b = 0; b < gridDim.x; ++b) {
        dd += __ldcg(part + 2 * b);
        cs += __ldcg(part + 2 * b + 1);
      }
    }
    __shared__ Metrics sm_rec;
    __shared__ Ctrl sm_ctl;
    if (lane == 0) {
      Ctrl cc;
      {
        const volatile Ctrl* vc = c;  // leader's ledger writes precede its arrival
        cc.squared_error = vc->squared_error;
        cc.total_input_sq = vc->total_input_sq;
        cc.nonstream_discarded_sq = vc->nonstream_discarded_sq;
        cc.proj_sq = vc->proj_sq;
        cc.e_sq = vc->e_sq;
        cc.added_error_sq = vc->added_error_sq;
        cc.trunc_margin = vc->trunc_margin;
        cc.n_d = vc->n_d;
        cc.insertions = vc->insertions;
        cc.r = vc->r;
        cc.r_new = vc->r_new;
        cc.degenerate = vc->degenerate;
        cc.status = vc->status;
        cc.sweeps = vc->sweeps;
        cc.records = vc->records;
      }
      const SliceCtl* sl = B.slot;
      cc.coupling_diff_sq = dd;
      cc.core_sq = cs;
      if (sqrt(dd) > kCouplingTol * sqrt(cs) + 1e-300 && cc.status == 0) cc.status = 2;  // streaming.cpp:55-63
      const int rn = cc.r_new;
      cc.r = rn;
      cc.n_d = n_d + 1;
      cc.insertions = cc.insertions + 1;
      Metrics mm;
      mm.slice_index = n_d;
      for (int kk = 0; kk < kMaxD; ++kk) mm.ranks[kk] = (kk + 1 < B.order) ? B.spatial_ranks[kk] : 0;
      mm.ranks[B.order - 1] = rn;
      mm.slice_norm = sqrt(sl->slice_sq);
      mm.projected_norm = sqrt(cc.proj_sq);
      for (int kk = 0; kk < kMaxD; ++kk)
        mm.mode_residuals[kk] = (kk + 1 < B.order) ? sqrt(sl->res_sq[kk]) : 0.0;
      const double booked = cc.squared_error + cc.nonstream_discarded_sq;
      mm.error_estimate = cc.total_input_sq <= 0.0 ? 0.0 : sqrt(fmax(booked, 0.0) / cc.total_input_sq);
      mm.expanded_mask = 0;
      mm.trunc_margin = cc.trunc_margin;
      mm.sweeps = cc.sweeps;
      cc.records = cc.records + 1;
      *c = cc;
      sm_rec = mm;
      sm_ctl = cc;
      // re-arm the grid handshake for the next insertion
      gs[2] = 0u;
      gs[0] = epoch + 1;
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
    if (lane == 0) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      g_isvd_clk[25] = (long long)g;
    }
  }
  if (leader) TSG_CLK(9);
}

}  // namespace
