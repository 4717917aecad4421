// Mode-0 fused projection + residual on the FP64 FMA pipe, for small ranks.
//
// Why FMA and not DMMA here: on sm_100a the FP64 tensor path (DMMA.8x8x4)
// and the FP64 FMA pipe share one FP64 throughput (tools/micro/coissue.cu:
// DMMA alone 36.9 TF/s, DFMA alone 32.4, any mix 32-35 — no co-issue), and
// with R = 10 the DMMA shapes pad the ranks to 16 in U^T X and to 12 in U P
// (1.4x the algorithmic flops) and split the fibre rows across warps, which
// costs a cross-warp reduction and two CTA barriers per tile. Here every
// flop is algorithmic and no warp ever waits on another:
//
//   * a warp owns a tile of 8*MCOL consecutive mode-0 fibres (columns); lane
//     (c, q) = (lane >> 2, lane & 3) owns columns c + 8m and the row pairs
//     {8s + 2q, 8s + 2q + 1} of them, so the 4 q-lanes of a column split its
//     N rows and sum their partial p = U^T x with two xor-shuffles (the sums
//     are identical on the 4 lanes: a + b == b + a);
//   * phase 1: p[m][l] += U[i][l] x[i] over the lane's rows (sequential FMA
//     chains, fixed order), ||x||^2 on the side; phase 2: rec = U p,
//     e = x - rec, ||e||^2 (streaming.cpp:129-133, tensor.cpp:120-143);
//   * the tile reaches shared memory by bulk copies (TMA engine,
//     cp.async.bulk, one per column into a padded pitch NP = N rounded up to
//     8 mod 16 doubles, so the lanes' 16-byte loads are bank-conflict free),
//     double buffered per warp and completed on a per-buffer mbarrier: the
//     copy of the warp's next tile overlaps the math of the current one;
//   * U is staged once per CTA row-major with an odd 16-byte pitch (the four
//     rows a load instruction touches fall in distinct banks);
//   * tiles are assigned statically (warp w of the grid takes tiles w, w+W,
//     ...): each CTA's partial sums are a deterministic function of the
//     input, so sync/async runs and sharded ranks agree bitwise.
//
// Reference: streaming.cpp:126-155 (process_nonstreaming_mode, mode 0),
// tensor.cpp:106-162 (ttm mode-0 fast path).
#pragma once

#include "kernels.cuh"

namespace tsg {
namespace fma0 {

__device__ __forceinline__ unsigned s32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bulk_col(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar, unsigned long long pol, bool ef) {
  if (ef)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
            s32(dst)),
        "l"(src), "r"(bytes), "r"(s32(bar)), "l"(pol)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            s32(dst)),
        "l"(src), "r"(bytes), "r"(s32(bar))
        : "memory");
}

__device__ __forceinline__ void wait_parity(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n"
      "}\n" ::"r"(s32(bar)),
      "r"(parity)
      : "memory");
}

// padded fibre pitch: N rounded up to 8 (mod 16) doubles
__host__ __device__ constexpr long long fibre_pitch(long long N) { return ((N + 7) / 16) * 16 + 8; }
// U row pitch in doubles: even and 2 (mod 4) (odd in 16-byte units)
__host__ __device__ constexpr int u_pitch(int RP) { return (RP % 4 == 2) ? RP : RP + 2; }

template <int RP, int MCOL, int NW, int NB>
__host__ __device__ constexpr long long smem_doubles(long long N) {
  return N * u_pitch(RP) + (long long)NW * NB * 8 * MCOL * fibre_pitch(N) + NW * 2 /*bars*/ + 2 * NW;
}

template <int RP, int MCOL, int NW, int NB>
__global__ void __launch_bounds__(32 * NW, 1) proj0_fma_kernel(ProjArgs a) {
  extern __shared__ __align__(128) double fsm[];
  constexpr int UP = u_pitch(RP);
  constexpr int TC = 8 * MCOL;  // columns per warp tile
  const int N = (int)a.v.n;
  const long long cols = a.v.right;
  const int R = a.R;
  const long long NP = fibre_pitch(N);
  double* Us = fsm;
  double* bufs = Us + (long long)N * UP;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(bufs + (long long)NW * NB * TC * NP);
  double* wred = reinterpret_cast<double*>(bars + 2 * NW);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = lane >> 2, q = lane & 3;
  const long long ntiles = (cols + TC - 1) / TC;
  const long long W = (long long)gridDim.x * NW;
  const long long w0 = (long long)blockIdx.x * NW + warp;
  double* mybuf = bufs + (long long)warp * NB * TC * NP;
  unsigned long long* mybar = bars + 2 * warp;
  const bool ef = a.stream_in == 2;
  unsigned long long pol = 0ull;
  if (ef) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));

  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s32(&mybar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s32(&mybar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  // tile tl -> buffer b: lane 0 posts the byte count, lanes copy one column each
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
  if (w0 < ntiles) issue(w0, 0);
  // U, row-major with pitch UP (ranks >= R zero), once per CTA
  for (int idx = threadIdx.x; idx < N * UP; idx += 32 * NW) {
    const int l = idx / N, i = idx - l * N;  // consecutive threads: consecutive rows (coalesced)
    Us[i * UP + l] = l < R ? a.u[(long long)l * N + i] : 0.0;
  }
  __syncthreads();

  double racc = 0.0, xacc = 0.0;
  const int npair = N / 8;  // row pairs per lane
  int j = 0;
#pragma unroll 1
  for (long long tl = w0; tl < ntiles; tl += W, ++j) {
    const int b = NB == 2 ? (j & 1) : 0;
    if (NB == 2 && tl + W < ntiles) {
      // the other buffer was last read by this warp's previous tile
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      issue(tl + W, b ^ 1);
    }
    if (NB == 1 && j > 0) {
      // single buffer: the next tile's copy starts once this warp is done
      // with the previous one (the other warps of the SM compute meanwhile)
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      issue(tl, 0);
    }
    wait_parity(&mybar[b], (unsigned)((NB == 2 ? (j >> 1) : j) & 1));
    if (a.karg1 == 7) continue;  // profiling only (tools/proj0_one.py flag 64): stream, no math
    const double* xt = mybuf + (long long)b * TC * NP;
    // columns past the end (last tile only) read column 0's fibre and their
    // sums are dropped once per tile (no per-element masking)
    bool cv[MCOL];
    int cc[MCOL];
#pragma unroll
    for (int m = 0; m < MCOL; ++m) {
      cv[m] = tl * TC + c + 8 * m < cols;
      cc[m] = cv[m] ? c + 8 * m : 0;
    }
    double xt_acc[MCOL], rt_acc[MCOL];
#pragma unroll
    for (int m = 0; m < MCOL; ++m) xt_acc[m] = rt_acc[m] = 0.0;
    // ---- phase 1: p = U^T x over the lane's rows, ||x||^2
    double p[MCOL][RP];
#pragma unroll
    for (int m = 0; m < MCOL; ++m)
#pragma unroll
      for (int l = 0; l < RP; ++l) p[m][l] = 0.0;
#pragma unroll 2
    for (int s = 0; s < npair; ++s) {
      const int row = 8 * s + 2 * q;
      double2 xv[MCOL];
#pragma unroll
      for (int m = 0; m < MCOL; ++m) xv[m] = *reinterpret_cast<const double2*>(xt + cc[m] * NP + row);
      double u0[RP], u1[RP];
#pragma unroll
      for (int l = 0; l < RP; l += 2) {
        const double2 a0 = *reinterpret_cast<const double2*>(Us + row * UP + l);
        const double2 a1 = *reinterpret_cast<const double2*>(Us + (row + 1) * UP + l);
        u0[l] = a0.x;
        u0[l + 1] = a0.y;
        u1[l] = a1.x;
        u1[l + 1] = a1.y;
      }
#pragma unroll
      for (int m = 0; m < MCOL; ++m) {
#pragma unroll
        for (int l = 0; l < RP; ++l) p[m][l] = fma(u0[l], xv[m].x, p[m][l]);
#pragma unroll
        for (int l = 0; l < RP; ++l) p[m][l] = fma(u1[l], xv[m].y, p[m][l]);
        xt_acc[m] = fma(xv[m].x, xv[m].x, xt_acc[m]);
        xt_acc[m] = fma(xv[m].y, xv[m].y, xt_acc[m]);
      }
    }
#pragma unroll
    for (int m = 0; m < MCOL; ++m)
      if (cv[m]) xacc += xt_acc[m];
    // the four row quarters of each column (identical sums on all four lanes)
#pragma unroll
    for (int m = 0; m < MCOL; ++m)
#pragma unroll
      for (int l = 0; l < RP; ++l) {
        p[m][l] += __shfl_xor_sync(0xffffffffu, p[m][l], 1);
        p[m][l] += __shfl_xor_sync(0xffffffffu, p[m][l], 2);
      }
    // ---- P (rank fastest: P[c * R + l]); lane q stores ranks l = q (mod 4)
    if (a.p) {
#pragma unroll
      for (int m = 0; m < MCOL; ++m)
        if (cv[m]) {
          double* dst = a.p + (tl * TC + c + 8 * m) * R;
#pragma unroll
          for (int l = 0; l < RP; ++l)
            if ((l & 3) == q && l < R) dst[l] = p[m][l];
        }
    }
    // ---- phase 2: e = x - U p, ||e||^2
    if (a.residual) {
#pragma unroll 2
      for (int s = 0; s < npair; ++s) {
        const int row = 8 * s + 2 * q;
        double2 xv[MCOL];
#pragma unroll
        for (int m = 0; m < MCOL; ++m) xv[m] = *reinterpret_cast<const double2*>(xt + cc[m] * NP + row);
        double u0[RP], u1[RP];
#pragma unroll
        for (int l = 0; l < RP; l += 2) {
          const double2 a0 = *reinterpret_cast<const double2*>(Us + row * UP + l);
          const double2 a1 = *reinterpret_cast<const double2*>(Us + (row + 1) * UP + l);
          u0[l] = a0.x;
          u0[l + 1] = a0.y;
          u1[l] = a1.x;
          u1[l + 1] = a1.y;
        }
        // 4*MCOL independent chains (even / odd ranks split), interleaved
        double ra[MCOL][2], rb[MCOL][2];
#pragma unroll
        for (int m = 0; m < MCOL; ++m) ra[m][0] = ra[m][1] = rb[m][0] = rb[m][1] = 0.0;
#pragma unroll
        for (int l = 0; l < RP; l += 2)
#pragma unroll
          for (int m = 0; m < MCOL; ++m) {
            ra[m][0] = fma(u0[l], p[m][l], ra[m][0]);
            ra[m][1] = fma(u1[l], p[m][l], ra[m][1]);
            rb[m][0] = fma(u0[l + 1], p[m][l + 1], rb[m][0]);
            rb[m][1] = fma(u1[l + 1], p[m][l + 1], rb[m][1]);
          }
#pragma unroll
        for (int m = 0; m < MCOL; ++m) {
          const double e0 = xv[m].x - (ra[m][0] + rb[m][0]);
          const double e1 = xv[m].y - (ra[m][1] + rb[m][1]);
          rt_acc[m] = fma(e0, e0, rt_acc[m]);
          rt_acc[m] = fma(e1, e1, rt_acc[m]);
        }
      }
#pragma unroll
      for (int m = 0; m < MCOL; ++m)
        if (cv[m]) racc += rt_acc[m];
    }
  }
  // ---- per-CTA partials (fixed order: lanes by butterfly, warps in order)
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
    double rs = 0.0, xs = 0.0;
    for (int w = 0; w < NW; ++w) {
      rs += wred[2 * w];
      xs += wred[2 * w + 1];
    }
    a.partial[2 * blockIdx.x] = rs;
    a.partial[2 * blockIdx.x + 1] = xs;
  }
}

template <int RP, int MCOL, int NW, int NB = 2>
inline int launch_t(const ProjArgs& a, cudaStream_t st, int free_sms) {
  const size_t smem = sizeof(double) * smem_doubles<RP, MCOL, NW, NB>(a.v.n);
  if (smem > 227 * 1024) return -1;
  static size_t attr = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(proj0_fma_kernel<RP, MCOL, NW, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024) != cudaSuccess)
      return -1;
    attr = 227 * 1024;
  }
  const long long tc = 8 * MCOL;
  const long long ntiles = (a.v.right + tc - 1) / tc;
  // balance: every warp gets the same number of tiles (the makespan is the
  // per-warp maximum), on at most kNumSMs - free_sms CTAs
  const long long slots = (long long)(kNumSMs - free_sms) * NW;
  const long long per = (ntiles + slots - 1) / slots;
  const long long warps = (ntiles + per - 1) / per;
  const int grid = (int)((warps + NW - 1) / NW);
  proj0_fma_kernel<RP, MCOL, NW, NB><<<grid < 1 ? 1 : grid, 32 * NW, smem, st>>>(a);
  return grid < 1 ? 1 : grid;
}

// Envelope: mode 0 (contiguous fibres), N a multiple of 8 up to 256, R <= 16,
// residual norm only (no residual tensor). Returns -1 outside it.
inline int launch(const ProjArgs& a, cudaStream_t st) {
  static const int mode = [] {
    const char* e = std::getenv("TSG_PROJ0_FMA");
    return e ? std::atoi(e) : 1;
  }();
  if (!mode || a.e || a.v.left != 1 || (a.v.n & 7) || a.v.n > 256 || a.R < 1 || a.R > 16) return -1;
  if (a.v.right >= (1LL << 40)) return -1;
  static const int free_sms = [] {
    const char* e = std::getenv("TSG_FMA0_FREE_SMS");
    return e ? std::atoi(e) : 8;
  }();
  const int RP = (a.R + 1) & ~1;
  if (mode == 1) {
    int g = -1;
    switch (RP) {
      case 2: g = launch_t<2, 2, 4>(a, st, free_sms); break;
      case 4: g = launch_t<4, 2, 4>(a, st, free_sms); break;
      case 6: g = launch_t<6, 2, 4>(a, st, free_sms); break;
      case 8: g = launch_t<8, 2, 4>(a, st, free_sms); break;
      case 10: g = launch_t<10, 2, 4>(a, st, free_sms); break;
      case 12: g = launch_t<12, 2, 4>(a, st, free_sms); break;
      case 14: g = launch_t<14, 2, 4>(a, st, free_sms); break;
      case 16: g = launch_t<16, 2, 4>(a, st, free_sms); break;
    }
    if (g > 0) return g;
  }
  if (mode == 3) {  // A/B: 16-column tiles, 8 warps, one buffer per warp
    switch (RP) {
      case 8: return launch_t<8, 2, 8, 1>(a, st, free_sms);
      case 10: return launch_t<10, 2, 8, 1>(a, st, free_sms);
      case 12: return launch_t<12, 2, 8, 1>(a, st, free_sms);
      default: return -1;
    }
  }
  if (mode == 4) {  // A/B: 8-column tiles, 12 warps, one buffer per warp
    switch (RP) {
      case 8: return launch_t<8, 1, 12, 1>(a, st, free_sms);
      case 10: return launch_t<10, 1, 12, 1>(a, st, free_sms);
      case 12: return launch_t<12, 1, 12, 1>(a, st, free_sms);
      default: return -1;
    }
  }
  // 8-column tiles (wide fibres, or the mode-2 A/B variant with 8 warps)
  if (mode == 2) {  // A/B variant: 8-column tiles, 8 warps
    switch (RP) {
      case 2: return launch_t<2, 1, 8>(a, st, free_sms);
      case 4: return launch_t<4, 1, 8>(a, st, free_sms);
      case 6: return launch_t<6, 1, 8>(a, st, free_sms);
      case 8: return launch_t<8, 1, 8>(a, st, free_sms);
      case 10: return launch_t<10, 1, 8>(a, st, free_sms);
      case 12: return launch_t<12, 1, 8>(a, st, free_sms);
      default: return -1;
    }
  }
  switch (RP) {
    case 2: return launch_t<2, 1, 4>(a, st, free_sms);
    case 4: return launch_t<4, 1, 4>(a, st, free_sms);
    case 6: return launch_t<6, 1, 4>(a, st, free_sms);
    case 8: return launch_t<8, 1, 4>(a, st, free_sms);
    case 10: return launch_t<10, 1, 4>(a, st, free_sms);
    case 12: return launch_t<12, 1, 4>(a, st, free_sms);
    case 14: return launch_t<14, 1, 4>(a, st, free_sms);
    case 16: return launch_t<16, 1, 4>(a, st, free_sms);
    default: return -1;
  }
}

}  // namespace fma0
}  // namespace tsg
