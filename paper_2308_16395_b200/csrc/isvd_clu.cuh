// Insertion on one thread-block cluster (n <= 8 * 128 * RPT rows).
//
// The row work of add_row (CGS2 passes over Q, the Q / core updates) is
// FP64-throughput bound on one SM (C2: 1000 rows x ~200 FMAs ~ 3k cycles of
// one SM's FP64 pipe, plus shared-memory operand traffic), so it is split
// over the G <= 8 CTAs of a cluster, each owning a contiguous block of rows
// that reaches its shared memory by bulk copies (Q columns < r_hint, b). The
// two CGS reductions are exchanged through distributed shared memory: every
// CTA pushes its partial vector into slot [rank] of every CTA, one cluster
// barrier, then each CTA sums the G slots in rank order -- all CTAs hold
// bitwise identical sums. The small inner problem is then solved
// redundantly by warp 0 of every CTA (identical inputs, deterministic
// arithmetic: identical W, P', sigma, rank), so no factor is handed off
// through global memory; the coupling partials are pushed to CTA 0, which
// commits the ledgers and publishes the record after a last cluster barrier.
// Reference: isvd.cpp:163-250 (add_row), streaming.cpp:196-224.
#pragma once


namespace {
namespace clu {

namespace cg = cooperative_groups;
constexpr int kT = 128;
constexpr int kW = kT / 32;
constexpr int kMaxG = 8;

__host__ __device__ constexpr long long smem_doubles(long long r0, int rhint) {
  return kSmallFixed + r0 * (rhint + 1) + 4;
}

template <int RMAX, int RPT>
__global__ void __launch_bounds__(kT, 1) isvd_clu_kernel(IsvdBufs B, int R0) {
  constexpr int RM = RMAX + 1;
  constexpr int P = 33;
  constexpr int NV = RMAX + 1;  // pass-1 vector: Q^T b and ||b||^2
  cg::cluster_group cl = cg::this_cluster();
  const int crk = (int)cl.block_rank();
  const int G = (int)cl.num_blocks();
  extern __shared__ __align__(16) double dsm[];
  double* sW = dsm;
  double* sU = sW + 32 * 33;
  double* sQ = sU + 32 * 33;
  double* sWcm = sQ + 32 * 33;
  double* spg = sWcm + 33 * 33;
  double* sM = spg + 32 * 32;
  const long long n = B.n;
  const int rhint = B.r_hint;
  const long long row0 = (long long)crk * R0;
  const long long nloc = (n - row0) < R0 ? (n - row0) : R0;
  double* qs = dsm + kSmallFixed;
  if ((unsigned)__cvta_generic_to_shared(qs) & 15u) ++qs;
  double* bs = qs + (long long)R0 * rhint;
  __shared__ __align__(8) unsigned long long qbar;
  __shared__ double wp[kW][33];
  __shared__ double red[32];
  __shared__ double slot1[kMaxG][33], slot2[kMaxG][33], slotc[kMaxG][2];
  __shared__ double sp1[33], sp2[33], sp[33];
  __shared__ double sx[8 * 32];
  __shared__ int si[3 * 32];
  __shared__ double sd[32], sz[33], ssig[33], ssn[33], sw[33], slam[33];
  __shared__ double sh_bsq, sh_esq, sh_delta, sh_sqerr;
  __shared__ int sh_rank, sh_deg;
  __shared__ Ctrl dummy_ctrl;
  Ctrl* c = B.ctrl;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (crk == 0) TSG_CLK(0);
  if (tid == 0) {
    const unsigned bytes = (unsigned)(nloc * 8);
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&qbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
                 "r"(bytes * (unsigned)(rhint + 1))
                 : "memory");
    for (int l = 0; l < rhint; ++l)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              (unsigned)__cvta_generic_to_shared(qs + (long long)l * R0)),
          "l"(B.q + l * n + row0), "r"(bytes), "r"(bar)
          : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(bs)),
        "l"(B.b + row0), "r"(bytes), "r"(bar)
        : "memory");
  }
  const int r = __ldcg(&c->r);
  const long long n_d = __ldcg(&c->n_d);
  for (int i = tid; i < 3 * 32 * 33 + 33 * 33 + 32 * 32 + 33 * 32; i += kT) dsm[i] = 0.0;
  if (tid == 0) {
    const SliceCtl* sl = B.slot;
    // every CTA reads the ledger before CTA 0 rewrites it (after two cluster
    // barriers)
    sh_delta = sl->delta;
    sh_sqerr = c->squared_error;
    if (crk == 0 && B.commit_modes > 0) {
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
  }
  if (tid < 32) ssig[tid] = tid < r ? B.sigma[tid] : 0.0;
  __syncthreads();
  {
    const unsigned a = (unsigned)__cvta_generic_to_shared(&qbar);
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(a)
        : "memory");
  }
  if (crk == 0) TSG_CLK(8);
  auto qrow = [&](long long lr, double (&q)[RMAX]) {
    const long long rc = lr < nloc ? lr : 0;
#pragma unroll
    for (int l = 0; l < RMAX; ++l) {
      const double v = qs[(long long)(l < rhint ? l : 0) * R0 + rc];
      q[l] = (l < r && lr < nloc) ? v : 0.0;
    }
  };
  // push this CTA's NV-vector into slot [crk] of every CTA of the cluster
  auto push = [&](double (*slots)[33], const double* v, int nv) {
    if (tid < nv) {
      const double x = v[tid];
      for (int g = 0; g < G; ++g) *cl.map_shared_rank(&slots[crk][tid], g) = x;
    }
  };
  // ---- CGS2 pass 1: p1 = Q^T b, ||b||^2
  {
    double acc[NV];
#pragma unroll
    for (int l = 0; l < NV; ++l) acc[l] = 0.0;
#pragma unroll
    for (int p = 0; p < RPT; ++p) {
      const long long lr = tid + (long long)kT * p;
      double q[RMAX];
      qrow(lr, q);
      const double bb = lr < nloc ? bs[lr] : 0.0;
#pragma unroll
      for (int l = 0; l < RMAX; ++l) acc[l] = fma(q[l], bb, acc[l]);
      acc[RMAX] = fma(bb, bb, acc[RMAX]);
    }
    block_reduce_vec<NV, true, kW>(acc, wp, red);
    push(slot1, red, NV);
  }
  cl.sync();
  if (tid < NV) {
    double s = 0.0;
    for (int g = 0; g < G; ++g) s += slot1[g][tid];
    sp1[tid] = s;
  }
  __syncthreads();
  // ---- pass 2: e1 = b - Q p1, p2 = Q^T e1, ||e1||^2
  double e1[RPT];
  {
    double acc[NV], c1[RMAX];
#pragma unroll
    for (int l = 0; l < NV; ++l) acc[l] = 0.0;
#pragma unroll
    for (int l = 0; l < RMAX; ++l) c1[l] = sp1[l];
#pragma unroll
    for (int p = 0; p < RPT; ++p) {
      const long long lr = tid + (long long)kT * p;
      double q[RMAX];
      qrow(lr, q);
      const double bb = lr < nloc ? bs[lr] : 0.0;
      double pr[RMAX];
#pragma unroll
      for (int l = 0; l < RMAX; ++l) pr[l] = q[l] * c1[l];
      e1[p] = bb - tree_sum<RMAX>(pr);
      acc[RMAX] = fma(e1[p], e1[p], acc[RMAX]);
#pragma unroll
      for (int l = 0; l < RMAX; ++l) acc[l] = fma(q[l], e1[p], acc[l]);
    }
    block_reduce_vec<NV, true, kW>(acc, wp, red);
    push(slot2, red, NV);
  }
  cl.sync();
  if (tid < NV) {
    double s = 0.0;
    for (int g = 0; g < G; ++g) s += slot2[g][tid];
    sp2[tid] = s;
  }
  __syncthreads();
  if (crk == 0) TSG_CLK(1);
  if (tid < 33) sp[tid] = sp1[tid] + sp2[tid];
  if (tid == 0) {
    double p2sq = 0.0;
    for (int l = 0; l < r; ++l) p2sq = fma(sp2[l], sp2[l], p2sq);
    const double bsq = sp1[RMAX], e1sq = sp2[RMAX];
    const double esq = fmax(e1sq - p2sq, 0.0);
    sh_bsq = bsq;
    sh_esq = esq;
    if (crk == 0) {
      c->proj_sq = bsq;
      c->e_sq = esq;
    }
    sh_deg = (sqrt(esq) <= kOrthEps * sqrt(bsq)) ? 1 : 0;  // isvd.cpp:191
  }
  __syncthreads();
  // ---- inner problem (warp 0, redundantly in every CTA) || p_gram (warps 1..)
  if (wid == 0) {
    if (crk == 0) TSG_CLK(4);
    const double kk = sqrt(sh_esq);
    Ctrl* cw = crk == 0 ? c : &dummy_ctrl;
    int rank = (r + 1 <= RM && r >= 1)
                   ? cta::inner_fast<RM, 6>(crk == 0 ? c : nullptr, r, sh_deg, ssig, sp, kk, sh_delta,
                                            sh_sqerr, sW, sU, ssn)
                   : -1;
    if (rank < 0) {
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
      rank = inner_warp_small<RM>(cw, r, ssig, sp, kk, sh_deg, sh_delta, sh_sqerr, ssn, sW, sU, sd, sz, S,
                                  slam, sWcm);
    }
    if (crk == 0) TSG_CLK(7);
    if (lane == 0) sh_rank = rank;
  } else {
    const int npair = r * (r + 1) / 2;
    for (int pidx = wid - 1; pidx < npair; pidx += kW - 1) {
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
  if (crk == 0) TSG_CLK(2);
  const int rank = sh_rank;
  const int deg = sh_deg;
  for (int idx = tid; idx < rank * r; idx += kT) {
    const int jn = idx % rank, j = idx / rank;
    double s = 0.0;
    for (int l = 0; l < r; ++l) s = fma(sU[l * P + jn], spg[l + j * r], s);
    sM[jn + j * rank] = s;
  }
  if (tid < rank) {
    sw[tid] = sU[r * P + tid];
    if (crk == 0) B.sigma_new[tid] = ssn[tid];
  }
  __syncthreads();
  if (crk == 0) TSG_CLK(16);
  // ---- own rows
  double dacc = 0.0, cacc = 0.0;
  {
    const double inv = deg ? 0.0 : 1.0 / sqrt(sh_esq);
    double c2[RMAX];
#pragma unroll
    for (int l = 0; l < RMAX; ++l) c2[l] = sp2[l];
#pragma unroll
    for (int p = 0; p < RPT; ++p) {
      const long long lr = tid + (long long)kT * p;
      if (lr >= nloc) break;
      const long long i = row0 + lr;
      double q[RMAX], cr[RMAX];
      qrow(lr, q);
#pragma unroll
      for (int l = 0; l < RMAX; ++l) cr[l] = B.c[i + (long long)(l < r ? l : 0) * n];
#pragma unroll
      for (int l = 0; l < RMAX; ++l) cr[l] = l < r ? cr[l] : 0.0;
      const double bb = bs[lr];
      double pr[RMAX];
#pragma unroll
      for (int l = 0; l < RMAX; ++l) pr[l] = q[l] * c2[l];
      const double e = e1[p] - tree_sum<RMAX>(pr);
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
          // padded to RMAX: q[l] = cr[l] = 0 and the small factors' padding
          // is zero for l >= r (no per-l branch)
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
  if (crk == 0) TSG_CLK(14);
  // ---- left <- blkdiag(left, 1) P' (isvd.cpp:227-237), rows split over CTAs
  {
    const long long total_rows = n_d + 1;
    const long long per = (total_rows + G - 1) / G;
    const long long r0 = (long long)crk * per;
    const long long r1 = r0 + per < total_rows ? r0 + per : total_rows;
    for (long long idx = r0 * B.capr + tid; idx < r1 * B.capr; idx += kT) {
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
  if (crk == 0) TSG_CLK(15);
  {
    double dv[2] = {dacc, cacc};
    block_reduce_vec<2, false, kW>(dv, wp, red);
    if (tid < 2) *cl.map_shared_rank(&slotc[crk][tid], 0) = red[tid];
  }
  cl.sync();
  if (crk != 0) return;
  TSG_CLK(3);
  if (wid == 0) {
    __shared__ Metrics sm_rec;
    __shared__ Ctrl sm_ctl;
    if (lane == 0) {
      double dd = 0.0, cs = 0.0;
      for (int g = 0; g < G; ++g) {
        dd += slotc[g][0];
        cs += slotc[g][1];
      }
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
  if (threadIdx.x == 0) {  // diagnostics: per-phase sums over all insertions
    for (int i = 1; i < 24; ++i)
      if (g_isvd_clk[i] >= g_isvd_clk[0]) g_isvd_acc[i] += g_isvd_clk[i] - g_isvd_clk[0];
    g_isvd_acc[31] += 1;
  }
}

}  // namespace clu
}  // namespace
