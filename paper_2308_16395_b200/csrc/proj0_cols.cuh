// Mode-0 fused projection + residual on FP64 DMMA with column-owning warps.
//
// The row-split DMMA kernel (proj0_tma_kernel) spreads a fibre's rows over
// the 8 warps of a CTA, so every 8-column tile pays a shared-memory
// cross-warp reduction and two CTA barriers, and with two CTAs per SM only
// two tiles are in flight: its math adds to the slice stream instead of
// hiding under it. The FP64 FMA-pipe variant (proj0_fma.cuh) avoids the
// reduction but is shared-memory bound: every DFMA needs its U operand from
// shared memory (a 128-bit load costs 4 wavefronts whatever the broadcast),
// ~1 wavefront per warp-DFMA against one port per SM.
//
// Here a warp owns whole fibres (columns): an 8*MC-column tile, all N rows,
// both GEMMs, no cross-warp traffic and no CTA barrier in the main loop.
//   phase 1  P^T (8 x 8RT per mc) = X^T U     K = N rows, 2 K-steps per 8-row
//            group with the k-permutation lane t -> rows 8grp+2t+i, so one
//            16-byte load feeds both steps; U image 1 stores rank
//            8nt+4i+t in column 8nt+2t+i (pitch 8RT+2: conflict-free)
//   phase 2  Rec^T (8 x 8 per row group) = P^T U^T   K = ranks, and the
//            phase-1 accumulators ARE the A fragments (lane (g,t) holds
//            ranks 8rt+4i+t); a K-step of ranks >= R is skipped (HALF);
//            U image 2 is row-major by natural rank (pitch 8RT+4)
//   epilogue e = x - rec, ||e||^2 (x reloaded from the tile), ||x||^2 from
//            phase 1's loads.
// Per 8 columns: 50*RT (phase 1) + 25*(2RT-HALF) (phase 2) DMMAs for N = 200;
// shared-memory wavefronts ~0.55 per DMMA-cycle, so the FP64 pipe, not the
// port, is the bound. Tiles arrive by per-column bulk copies (TMA engine)
// into an NB-deep per-warp ring with one mbarrier per buffer; tiles are
// assigned statically, so per-CTA partial sums are deterministic.
// Reference: streaming.cpp:126-155, tensor.cpp:106-162 (ttm mode-0 path).
#pragma once

#include "kernels.cuh"
#include "proj0_fma.cuh"

namespace tsg {
namespace cols0 {

using fma0::bulk_col;
using fma0::fibre_pitch;
using fma0::s32;
using fma0::wait_parity;

// not volatile: the compiler may interleave independent accumulator chains
// (a volatile asm keeps the written order, which put dependent DMMAs back to
// back and capped a warp at one DMMA per DMMA latency)
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__host__ __device__ inline long long upad_cols_offset_dev(long long N, int R) {
  return (N + 7) / 8 * 8 * (8 * ((R + 7) / 8) + 4);  // = upad_cols_offset (kernels_stream.cu)
}

// Ranks past the last full 8-rank DMMA tile that the register-resident kernel
// computes on the FP64 FMA pipe instead of padding a whole rank tile with
// zeros (R = 9..11 with N = 200 / 256: C2's R = 10 executes 75 + FMA work
// instead of 175 DMMAs per 8 columns). DMMA and DFMA share one FP64 datapath
// (profiles/r02/coissue_dmma_dfma.txt), so this only removes padded work.
// The prebuilt U images (cols_u_kernel) follow the same rule.
// MEASURED AND REJECTED as the default (TSG_COLS0_LO=1 enables it for A/B):
// C2 mode 0 alone 30.4 us against 26.8 us with the padded second rank tile,
// 37-39 us against 32 us inside the pipeline. Parity-clean either way. The
// kernel is not FP64-datapath bound at 57 % DMMA-pipe utilisation: the extra
// shared-memory operand loads and the issue slots of the 200 FMAs per tile
// cost more than the 75 DMMAs they replace.
inline int cols_lo(long long N, int R) {
  static const bool on = [] {
    const char* e = std::getenv("TSG_COLS0_LO");
    return e ? std::atoi(e) != 0 : false;
  }();
  return (on && (N == 200 || N == 256) && R >= 9 && R <= 11) ? R - 8 : 0;
}
inline int cols_rt(long long N, int R) { return cols_lo(N, R) ? R / 8 : (R + 7) / 8; }

template <int RT>
__host__ __device__ constexpr int p1_pitch() { return 8 * RT + 2; }
template <int RT>
__host__ __device__ constexpr int p2_pitch() { return 8 * RT + 4; }

template <int RT, int MC, int NW, int NB>
__host__ __device__ constexpr long long smem_doubles(long long N) {
  return N * (p1_pitch<RT>() + p2_pitch<RT>()) + (long long)NW * NB * 8 * MC * fibre_pitch(N) +
         NW * NB /*bars*/ + 2 * NW;
}

template <int RT, int MC, int NW, int NB, bool HALF>
__global__ void __launch_bounds__(32 * NW, 1) proj0_cols_kernel(ProjArgs a) {
  extern __shared__ __align__(128) double csm[];
  constexpr int P1 = p1_pitch<RT>(), P2 = p2_pitch<RT>();
  constexpr int TC = 8 * MC;
  const int N = (int)a.v.n;
  const int ngroups = N >> 3;
  const long long cols = a.v.right;
  const int R = a.R;
  const long long NP = fibre_pitch(N);
  double* U1 = csm;
  double* U2 = U1 + (long long)N * P1;
  double* bufs = U2 + (long long)N * P2;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(bufs + (long long)NW * NB * TC * NP);
  double* wred = reinterpret_cast<double*>(bars + NW * NB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const long long ntiles = (cols + TC - 1) / TC;
  const long long W = (long long)gridDim.x * NW;
  const long long w0 = (long long)blockIdx.x * NW + warp;
  double* mybuf = bufs + (long long)warp * NB * TC * NP;
  unsigned long long* mybar = bars + NB * warp;
  const bool ef = a.stream_in == 2;
  unsigned long long pol = 0ull;
  if (ef) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  if (lane == 0) {
    for (int b = 0; b < NB; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s32(&mybar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](long long tl, int b) {
    const long long c0 = tl * TC;
    const long long nc = (cols - c0) < TC ? (cols - c0) : TC;
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s32(&mybar[b])),
                   "r"((unsigned)(nc * N * 8))
                   : "memory");
    __syncwarp();
    if (lane < nc)
      bulk_col(mybuf + (long long)b * TC * NP + lane * NP, a.x + (c0 + lane) * N, (unsigned)(N * 8),
               &mybar[b], pol, ef);
  };
  // prologue: the first NB-1 tiles of this warp
  for (int k = 0; k < NB - 1; ++k)
    if (w0 + k * W < ntiles) issue(w0 + k * W, k);
  // U images (ranks >= R zero); consecutive threads read consecutive rows
  for (int idx = threadIdx.x; idx < N * 8 * RT; idx += 32 * NW) {
    const int rk = idx / N, i = idx - rk * N;
    const double v = rk < R ? a.u[(long long)rk * N + i] : 0.0;
    // image 1: rank 8nt + 4ii + tt at column 8nt + 2tt + ii
    const int nt = rk >> 3, ii = (rk >> 2) & 1, tt = rk & 3;
    U1[i * P1 + 8 * nt + 2 * tt + ii] = v;
    U2[i * P2 + rk] = v;
  }
  __syncthreads();

  double racc = 0.0, xacc = 0.0;
  int j = 0;
#pragma unroll 1
  for (long long tl = w0; tl < ntiles; tl += W, ++j) {
    const int b = j % NB;
    {
      const long long nx = tl + (long long)(NB - 1) * W;
      if (nx < ntiles) {
        // buffer (j + NB - 1) % NB was last read by this warp's tile j - 1
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue(nx, (j + NB - 1) % NB);
      }
    }
    wait_parity(&mybar[b], (unsigned)((j / NB) & 1));
    if (a.karg1 == 7) continue;  // profiling only: stream, no math
    const double* xt = mybuf + (long long)b * TC * NP;
    bool cv[MC];
    const double* xc[MC];
#pragma unroll
    for (int mc = 0; mc < MC; ++mc) {
      cv[mc] = tl * TC + 8 * mc + g < cols;
      xc[mc] = xt + (cv[mc] ? 8 * mc + g : 0) * NP + 2 * t;
    }
    // ---- phase 1 (two K halves: even / odd row groups, summed at the end)
    double acc[2][MC][RT][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int mc = 0; mc < MC; ++mc)
#pragma unroll
        for (int rt = 0; rt < RT; ++rt) acc[h][mc][rt][0] = acc[h][mc][rt][1] = 0.0;
    double xs[MC];
#pragma unroll
    for (int mc = 0; mc < MC; ++mc) xs[mc] = 0.0;
    const double* u1 = U1 + 2 * t * P1 + g;
    auto p1 = [&](int grp, double (&ac)[MC][RT][2]) {
      double2 xv[MC];
#pragma unroll
      for (int mc = 0; mc < MC; ++mc) xv[mc] = *reinterpret_cast<const double2*>(xc[mc] + 8 * grp);
      double bb[2][RT];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int rt = 0; rt < RT; ++rt) bb[i][rt] = u1[(8 * grp + i) * P1 + 8 * rt];
#pragma unroll
      for (int mc = 0; mc < MC; ++mc) {
#pragma unroll
        for (int rt = 0; rt < RT; ++rt) {
          dmma(ac[mc][rt][0], ac[mc][rt][1], xv[mc].x, bb[0][rt]);
          dmma(ac[mc][rt][0], ac[mc][rt][1], xv[mc].y, bb[1][rt]);
        }
        xs[mc] = fma(xv[mc].x, xv[mc].x, xs[mc]);
        xs[mc] = fma(xv[mc].y, xv[mc].y, xs[mc]);
      }
    };
    int grp = 0;
#pragma unroll 1
    for (; grp + 1 < ngroups; grp += 2) {
      p1(grp, acc[0]);
      p1(grp + 1, acc[1]);
    }
    if (grp < ngroups) p1(grp, acc[0]);
    double pa[MC][RT][2];
#pragma unroll
    for (int mc = 0; mc < MC; ++mc)
#pragma unroll
      for (int rt = 0; rt < RT; ++rt)
#pragma unroll
        for (int i = 0; i < 2; ++i) pa[mc][rt][i] = acc[0][mc][rt][i] + acc[1][mc][rt][i];
    // ---- P (rank fastest); lane (g, t) holds ranks 8rt + 4i + t of column g
    if (a.p) {
#pragma unroll
      for (int mc = 0; mc < MC; ++mc)
        if (cv[mc]) {
          double* dst = a.p + (tl * TC + 8 * mc + g) * R;
#pragma unroll
          for (int rt = 0; rt < RT; ++rt)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int rk = 8 * rt + 4 * i + t;
              if (rk < R) dst[rk] = pa[mc][rt][i];
            }
        }
    }
    // ---- phase 2 + epilogue, two row groups per step (independent chains)
    double rs[MC];
#pragma unroll
    for (int mc = 0; mc < MC; ++mc) rs[mc] = 0.0;
    if (a.residual) {
      const double* u2 = U2 + g * P2 + t;
#pragma unroll 2
      for (int grp = 0; grp < ngroups; ++grp) {
        double c2[MC][2];
#pragma unroll
        for (int mc = 0; mc < MC; ++mc) c2[mc][0] = c2[mc][1] = 0.0;
#pragma unroll
        for (int rt = 0; rt < RT; ++rt)
#pragma unroll
          for (int i = 0; i < 2; ++i)
            if (!(HALF && rt == RT - 1 && i == 1)) {
              const double bv = u2[8 * grp * P2 + 8 * rt + 4 * i];
#pragma unroll
              for (int mc = 0; mc < MC; ++mc) dmma(c2[mc][0], c2[mc][1], pa[mc][rt][i], bv);
            }
#pragma unroll
        for (int mc = 0; mc < MC; ++mc) {
          const double2 xv = *reinterpret_cast<const double2*>(xc[mc] + 8 * grp);
          const double e0 = xv.x - c2[mc][0], e1 = xv.y - c2[mc][1];
          rs[mc] = fma(e0, e0, rs[mc]);
          rs[mc] = fma(e1, e1, rs[mc]);
        }
      }
    }
#pragma unroll
    for (int mc = 0; mc < MC; ++mc)
      if (cv[mc]) {
        racc += rs[mc];
        xacc += xs[mc];
      }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    racc += __shfl_xor_sync(0xffffffffu, racc, o);
    xacc += __shfl_xor_sync(0xffffffffu, xacc, o);
  }
  if (lane == 0) {
    wred[2 * warp] = racc;
    wred[2 * warp + 1] = xacc;
  }
  __syncthreads();
  if (threadIdx.x == 0 && a.partial) {
    double r_ = 0.0, x_ = 0.0;
    for (int w = 0; w < NW; ++w) {
      r_ += wred[2 * w];
      x_ += wred[2 * w + 1];
    }
    a.partial[2 * blockIdx.x] = r_;
    a.partial[2 * blockIdx.x + 1] = x_;
  }
}

// Register-resident variant (N = 8*NG known at compile time, 8-column
// tiles): a lane's 2*NG slice values are loaded into registers as soon as
// its tile lands, the warp's single shared buffer is handed straight back to
// the TMA engine for the warp's next tile, and both GEMMs and the epilogue run
// from registers. One buffer per warp double-buffers in effect, so 12 warps
// (3 per SM sub-partition, which the DMMA issue pattern needs) fit next to
// the U images.
template <int RT, int NW, int NG, bool HALF, int LO = 0>
__global__ void __launch_bounds__(32 * NW, 1) proj0_colsr_kernel(ProjArgs a) {
  extern __shared__ __align__(128) double csm[];
  constexpr int P1 = p1_pitch<RT>(), P2 = p2_pitch<RT>();
  constexpr int N = 8 * NG;
  constexpr long long NP = fibre_pitch(N);
  const long long cols = a.v.right;
  const int R = a.R;
  double* U1 = csm;
  double* U2 = U1 + N * P1;
  double* bufs = U2 + N * P2;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(bufs + (long long)NW * 8 * NP);
  double* wred = reinterpret_cast<double*>(bars + NW + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const long long ntiles = (cols + 7) / 8;
  const long long W = (long long)gridDim.x * NW;
  const long long w0 = (long long)blockIdx.x * NW + warp;
  double* mybuf = bufs + (long long)warp * 8 * NP;
  unsigned long long* mybar = bars + warp;
  const bool ef = a.stream_in == 2;
  unsigned long long pol = 0ull;
  if (ef) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s32(mybar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](long long tl) {
    const long long c0 = tl * 8;
    const long long nc = (cols - c0) < 8 ? (cols - c0) : 8;
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s32(mybar)),
                   "r"((unsigned)(nc * N * 8))
                   : "memory");
    __syncwarp();
    if (lane < nc)
      bulk_col(mybuf + lane * NP, a.x + (c0 + lane) * N, (unsigned)(N * 8), mybar, pol, ef);
  };
  const bool noload = a.karg1 & 64;  // profiling only: compute on stale shared memory, no loads
  if (w0 < ntiles && !noload) issue(w0);
  if (a.upad) {
    // both images in one bulk copy from the engine's prebuilt buffer
    unsigned long long& ubar = bars[NW];
    if (threadIdx.x == 0) {
      const unsigned bytes = (unsigned)(N * (P1 + P2) * 8);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s32(&ubar)));
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s32(&ubar)), "r"(bytes)
                   : "memory");
      bulk_col(U1, a.upad + upad_cols_offset_dev(N, R), bytes, &ubar, 0ull, false);
    }
    __syncthreads();
    wait_parity(&ubar, 0u);
  } else {
    for (int idx = threadIdx.x; idx < N * 8 * RT; idx += 32 * NW) {
      const int rk = idx / N, i = idx - rk * N;
      const double v = rk < R ? a.u[(long long)rk * N + i] : 0.0;
      const int nt = rk >> 3, ii = (rk >> 2) & 1, tt = rk & 3;
      U1[i * P1 + 8 * nt + 2 * tt + ii] = v;
      U2[i * P2 + rk] = v;
    }
    for (int idx = threadIdx.x; idx < N * LO; idx += 32 * NW) {  // left-over ranks: image 2 only
      const int l = idx / N, i = idx - l * N;
      U2[i * P2 + 8 * RT + l] = a.u[(long long)(8 * RT + l) * N + i];
    }
    __syncthreads();
  }
  const double* u1 = U1 + 2 * t * P1 + g;
  const double* u2 = U2 + g * P2 + t;
  // left-over ranks 8RT .. 8RT+LO-1 of rows 8grp + 2t, 8grp + 2t + 1 (the rows
  // of this lane's slice values): image 2, natural rank order
  const double* ulo = U2 + 2 * t * P2 + 8 * RT;

  double racc = 0.0, xacc = 0.0;
  int j = 0;
#pragma unroll 1
  for (long long tl = w0; tl < ntiles; tl += W, ++j) {
    if (!noload) wait_parity(mybar, (unsigned)(j & 1));
    const bool cv = tl * 8 + g < cols;
    const double* xc = mybuf + (cv ? g : 0) * NP + 2 * t;
    double2 xr[NG];
#pragma unroll
    for (int grp = 0; grp < NG; ++grp) xr[grp] = *reinterpret_cast<const double2*>(xc + 8 * grp);
    // the buffer is free once every lane holds its values
    if (tl + W < ntiles && !noload) {
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      issue(tl + W);
    }
    if (a.karg1 == 7) continue;  // profiling only
    // ---- phase 1: four accumulator chains (two K halves x RT tiles)
    double acc[2][RT][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int rt = 0; rt < RT; ++rt) acc[h][rt][0] = acc[h][rt][1] = 0.0;
    double xs = 0.0;
    double lp[2][LO > 0 ? LO : 1];
#pragma unroll
    for (int l = 0; l < (LO > 0 ? LO : 1); ++l) lp[0][l] = lp[1][l] = 0.0;
    const int dbg = a.karg1;  // profiling only: 16 skip phase 2, 32 skip phase 1
    // two row groups per step, written so consecutive DMMAs belong to
    // different accumulator chains: (grp, rt, x) for both groups, then
    // (grp, rt, y)
    if (!(dbg & 32)) {
#pragma unroll
      for (int grp = 0; grp < NG; grp += 2) {
        const bool two = grp + 1 < NG;
        double b0[2][RT], b1[2][RT];
#pragma unroll
        for (int rt = 0; rt < RT; ++rt) {
          b0[0][rt] = u1[(8 * grp) * P1 + 8 * rt];
          b0[1][rt] = u1[(8 * grp + 1) * P1 + 8 * rt];
          b1[0][rt] = two ? u1[(8 * grp + 8) * P1 + 8 * rt] : 0.0;
          b1[1][rt] = two ? u1[(8 * grp + 9) * P1 + 8 * rt] : 0.0;
        }
        const double2 x0 = xr[grp];
        const double2 x1 = two ? xr[grp + 1] : make_double2(0.0, 0.0);
#pragma unroll
        for (int rt = 0; rt < RT; ++rt) dmma(acc[0][rt][0], acc[0][rt][1], x0.x, b0[0][rt]);
#pragma unroll
        for (int rt = 0; rt < RT; ++rt) dmma(acc[1][rt][0], acc[1][rt][1], x1.x, b1[0][rt]);
#pragma unroll
        for (int rt = 0; rt < RT; ++rt) dmma(acc[0][rt][0], acc[0][rt][1], x0.y, b0[1][rt]);
#pragma unroll
        for (int rt = 0; rt < RT; ++rt) dmma(acc[1][rt][0], acc[1][rt][1], x1.y, b1[1][rt]);
        xs = fma(x0.x, x0.x, xs);
        xs = fma(x0.y, x0.y, xs);
        xs = fma(x1.x, x1.x, xs);
        xs = fma(x1.y, x1.y, xs);
        if constexpr (LO > 0) {
          // left-over ranks on the FMA pipe: this lane's rows of column g
          if constexpr (LO == 2) {  // ranks 8RT, 8RT+1 are one 16-byte load per row
            const double2 a0 = *reinterpret_cast<const double2*>(ulo + (8 * grp) * P2);
            const double2 a1 = *reinterpret_cast<const double2*>(ulo + (8 * grp + 1) * P2);
            lp[0][0] = fma(x0.x, a0.x, lp[0][0]);
            lp[0][1] = fma(x0.x, a0.y, lp[0][1]);
            lp[0][0] = fma(x0.y, a1.x, lp[0][0]);
            lp[0][1] = fma(x0.y, a1.y, lp[0][1]);
            if (two) {
              const double2 b0_ = *reinterpret_cast<const double2*>(ulo + (8 * grp + 8) * P2);
              const double2 b1_ = *reinterpret_cast<const double2*>(ulo + (8 * grp + 9) * P2);
              lp[1][0] = fma(x1.x, b0_.x, lp[1][0]);
              lp[1][1] = fma(x1.x, b0_.y, lp[1][1]);
              lp[1][0] = fma(x1.y, b1_.x, lp[1][0]);
              lp[1][1] = fma(x1.y, b1_.y, lp[1][1]);
            }
          } else {
#pragma unroll
            for (int l = 0; l < LO; ++l) {
              lp[0][l] = fma(x0.x, ulo[(8 * grp) * P2 + l], lp[0][l]);
              lp[0][l] = fma(x0.y, ulo[(8 * grp + 1) * P2 + l], lp[0][l]);
              if (two) {
                lp[1][l] = fma(x1.x, ulo[(8 * grp + 8) * P2 + l], lp[1][l]);
                lp[1][l] = fma(x1.y, ulo[(8 * grp + 9) * P2 + l], lp[1][l]);
              }
            }
          }
        }
      }
    }
    double pl[LO > 0 ? LO : 1];
    if constexpr (LO > 0) {
      // sum over the four lanes (t) that share column g: every lane ends with
      // the same bits (commutative pairings)
#pragma unroll
      for (int l = 0; l < LO; ++l) {
        double v = lp[0][l] + lp[1][l];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        pl[l] = v;
      }
    }
    double pa[RT][2];
#pragma unroll
    for (int rt = 0; rt < RT; ++rt)
#pragma unroll
      for (int i = 0; i < 2; ++i) pa[rt][i] = acc[0][rt][i] + acc[1][rt][i];
    if (a.p && cv) {
      double* dst = a.p + (tl * 8 + g) * R;
#pragma unroll
      for (int rt = 0; rt < RT; ++rt)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int rk = 8 * rt + 4 * i + t;
          if (rk < R) dst[rk] = pa[rt][i];
        }
      if constexpr (LO > 0) {
#pragma unroll
        for (int l = 0; l < LO; ++l)
          if (t == l) dst[8 * RT + l] = pl[l];
      }
    }
    // ---- phase 2 + epilogue from registers
    double rs = 0.0;
    if (a.residual && !(dbg & 16)) {
      // K-steps of phase 2 (the skipped all-padding step excluded)
      constexpr int KS = 2 * RT - (HALF ? 1 : 0);
      // two row groups per step with all B fragments loaded first, so the
      // two 3-DMMA chains interleave instead of waiting on each other
      auto kofs = [](int k) { return 8 * (k >> 1) + 4 * (k & 1); };
#pragma unroll
      for (int grp = 0; grp < NG; grp += 2) {
        const bool two = grp + 1 < NG;
        double bv0[KS], bv1[KS];
#pragma unroll
        for (int k = 0; k < KS; ++k) {
          bv0[k] = u2[8 * grp * P2 + kofs(k)];
          bv1[k] = two ? u2[8 * (grp + 1) * P2 + kofs(k)] : 0.0;
        }
        double c0 = -xr[grp].x, c1 = -xr[grp].y;
        double d0 = two ? -xr[grp + 1].x : 0.0, d1 = two ? -xr[grp + 1].y : 0.0;
#pragma unroll
        for (int k = 0; k < KS; ++k) {
          dmma(c0, c1, pa[k >> 1][k & 1], bv0[k]);
          if (two) dmma(d0, d1, pa[k >> 1][k & 1], bv1[k]);
        }
        if constexpr (LO > 0) {
          if constexpr (LO == 2) {
            const double2 a0 = *reinterpret_cast<const double2*>(ulo + (8 * grp) * P2);
            const double2 a1 = *reinterpret_cast<const double2*>(ulo + (8 * grp + 1) * P2);
            c0 = fma(a0.x, pl[0], c0);
            c0 = fma(a0.y, pl[1], c0);
            c1 = fma(a1.x, pl[0], c1);
            c1 = fma(a1.y, pl[1], c1);
            if (two) {
              const double2 b0_ = *reinterpret_cast<const double2*>(ulo + (8 * grp + 8) * P2);
              const double2 b1_ = *reinterpret_cast<const double2*>(ulo + (8 * grp + 9) * P2);
              d0 = fma(b0_.x, pl[0], d0);
              d0 = fma(b0_.y, pl[1], d0);
              d1 = fma(b1_.x, pl[0], d1);
              d1 = fma(b1_.y, pl[1], d1);
            }
          } else {
#pragma unroll
            for (int l = 0; l < LO; ++l) {
              c0 = fma(ulo[(8 * grp) * P2 + l], pl[l], c0);
              c1 = fma(ulo[(8 * grp + 1) * P2 + l], pl[l], c1);
              if (two) {
                d0 = fma(ulo[(8 * grp + 8) * P2 + l], pl[l], d0);
                d1 = fma(ulo[(8 * grp + 9) * P2 + l], pl[l], d1);
              }
            }
          }
        }
        rs = fma(c0, c0, rs);
        rs = fma(c1, c1, rs);
        if (two) {
          rs = fma(d0, d0, rs);
          rs = fma(d1, d1, rs);
        }
      }
    }
    if (cv) {
      racc += rs;
      xacc += xs;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    racc += __shfl_xor_sync(0xffffffffu, racc, o);
    xacc += __shfl_xor_sync(0xffffffffu, xacc, o);
  }
  if (lane == 0) {
    wred[2 * warp] = racc;
    wred[2 * warp + 1] = xacc;
  }
  __syncthreads();
  if (threadIdx.x == 0 && a.partial) {
    double r_ = 0.0, x_ = 0.0;
    for (int w = 0; w < NW; ++w) {
      r_ += wred[2 * w];
      x_ += wred[2 * w + 1];
    }
    a.partial[2 * blockIdx.x] = r_;
    a.partial[2 * blockIdx.x + 1] = x_;
  }
}

template <int RT, int NW, int NG, bool HALF, int LO = 0>
inline int launch_r(const ProjArgs& a, cudaStream_t st, int free_sms) {
  constexpr long long N = 8 * NG;
  const size_t smem =
      sizeof(double) * (N * (p1_pitch<RT>() + p2_pitch<RT>()) + NW * 8 * fibre_pitch(N) + NW + 1 + 2 * NW);
  if (smem > 227 * 1024) return -1;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(proj0_colsr_kernel<RT, NW, NG, HALF, LO>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
      return -1;
    attr = true;
  }
  const long long ntiles = (a.v.right + 7) / 8;
  const long long slots = (long long)(kNumSMs - free_sms) * NW;
  const long long per = (ntiles + slots - 1) / slots;
  const long long warps = (ntiles + per - 1) / per;
  int grid = (int)((warps + NW - 1) / NW);
  if (grid < 1) grid = 1;
  proj0_colsr_kernel<RT, NW, NG, HALF, LO><<<grid, 32 * NW, smem, st>>>(a);
  return grid;
}

// one full DMMA rank tile + LO left-over ranks on the FMA pipe (R = 9..11)
template <int NW, int NG>
inline int launch_lo(const ProjArgs& a, cudaStream_t st, int free_sms, int lo) {
  switch (lo) {
    case 1: return launch_r<1, NW, NG, false, 1>(a, st, free_sms);
    case 2: return launch_r<1, NW, NG, false, 2>(a, st, free_sms);
    case 3: return launch_r<1, NW, NG, false, 3>(a, st, free_sms);
  }
  return -1;
}

template <int RT, int NW, int NG>
inline int launch_rh(const ProjArgs& a, cudaStream_t st, int free_sms) {
  return (a.R <= 8 * (RT - 1) + 4) ? launch_r<RT, NW, NG, true>(a, st, free_sms)
                                    : launch_r<RT, NW, NG, false>(a, st, free_sms);
}

template <int RT, int MC, int NW, int NB, bool HALF>
inline int launch_t(const ProjArgs& a, cudaStream_t st, int free_sms) {
  const size_t smem = sizeof(double) * smem_doubles<RT, MC, NW, NB>(a.v.n);
  if (smem > 227 * 1024) return -1;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(proj0_cols_kernel<RT, MC, NW, NB, HALF>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
      return -1;
    attr = true;
  }
  const long long tc = 8 * MC;
  const long long ntiles = (a.v.right + tc - 1) / tc;
  const long long slots = (long long)(kNumSMs - free_sms) * NW;
  const long long per = (ntiles + slots - 1) / slots;
  const long long warps = (ntiles + per - 1) / per;
  int grid = (int)((warps + NW - 1) / NW);
  if (grid < 1) grid = 1;
  proj0_cols_kernel<RT, MC, NW, NB, HALF><<<grid, 32 * NW, smem, st>>>(a);
  return grid;
}

template <int RT, int MC, int NW, int NB>
inline int launch_h(const ProjArgs& a, cudaStream_t st, int free_sms) {
  return (a.R <= 8 * (RT - 1) + 4) ? launch_t<RT, MC, NW, NB, true>(a, st, free_sms)
                                    : launch_t<RT, MC, NW, NB, false>(a, st, free_sms);
}

// Envelope: mode 0, N a multiple of 8 up to 512, R <= 32, residual norm only.
inline int launch(const ProjArgs& a, cudaStream_t st) {
  static const int mode = [] {
    const char* e = std::getenv("TSG_PROJ0_COLS");
    return e ? std::atoi(e) : 1;
  }();
  if (!mode || a.e || a.v.left != 1 || (a.v.n & 7) || a.v.n > 512 || a.R < 1 || a.R > 32) return -1;
  static const int free_sms = [] {
    const char* e = std::getenv("TSG_COLS0_FREE_SMS");
    return e ? std::atoi(e) : 8;
  }();
  const int RT = (a.R + 7) / 8;
  int g = -1;
  if (const int lo = cols_lo(a.v.n, a.R)) {
    if (a.v.n == 200) g = launch_lo<12, 25>(a, st, free_sms, lo);
    if (a.v.n == 256) g = launch_lo<8, 32>(a, st, free_sms, lo);
    return g;  // the prebuilt images follow cols_rt: no other kernel reads them
  }
  // A/B variants (TSG_PROJ0_COLS): 1 = 6 warps x 2 buffers, 2 = 8 warps x 1,
  // 3 = 12 warps x 1, 4 = 4 warps x 3; each falls back to the 4 x 2 shape
  // when its shared memory does not fit
  if (mode == 1 || mode == 6) {  // register-resident tiles for the configs' mode-0 sizes
    const int nw = mode == 6 ? 16 : 12;
    if (a.v.n == 200 && RT == 2) g = nw == 12 ? launch_rh<2, 12, 25>(a, st, free_sms) : launch_rh<2, 16, 25>(a, st, free_sms);
    if (a.v.n == 200 && RT == 1) g = launch_rh<1, 12, 25>(a, st, free_sms);
    if (a.v.n == 64 && RT == 1) g = launch_rh<1, 12, 8>(a, st, free_sms);
    if (a.v.n == 256 && RT == 1) g = launch_rh<1, 8, 32>(a, st, free_sms);
    if (a.v.n == 256 && RT == 2) g = launch_rh<2, 8, 32>(a, st, free_sms);
    if (g > 0) return g;
  }
  switch (mode) {
    case 5:
      if (RT == 1) g = launch_h<1, 1, 6, 2>(a, st, free_sms);
      if (RT == 2) g = launch_h<2, 1, 6, 2>(a, st, free_sms);
      break;
    case 2:
      if (RT == 1) g = launch_h<1, 1, 8, 1>(a, st, free_sms);
      if (RT == 2) g = launch_h<2, 1, 8, 1>(a, st, free_sms);
      break;
    case 3:
      if (RT == 1) g = launch_h<1, 1, 12, 1>(a, st, free_sms);
      if (RT == 2) g = launch_h<2, 1, 12, 1>(a, st, free_sms);
      break;
    case 4:
      if (RT == 1) g = launch_h<1, 1, 4, 3>(a, st, free_sms);
      if (RT == 2) g = launch_h<2, 1, 4, 3>(a, st, free_sms);
      break;
  }
  if (g > 0) return g;
  // fallback within the envelope: 8-column tiles, 4 warps, double buffer
  switch (RT) {
    case 1: return launch_h<1, 1, 4, 2>(a, st, free_sms);
    case 2: return launch_h<2, 1, 4, 2>(a, st, free_sms);
    case 3: return launch_h<3, 1, 4, 2>(a, st, free_sms);
    case 4: return launch_h<4, 1, 4, 2>(a, st, free_sms);
  }
  return -1;
}

}  // namespace cols0
}  // namespace tsg
