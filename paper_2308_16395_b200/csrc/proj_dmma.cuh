// FP64 tensor-core (DMMA) fused mode-k projection + residual kernel.
//
// For a mode-k view (left, N, right) of the tensor, every column
// c = (l, r) is one mode-k fibre x_c (N values, stride `left`). A CTA tile is
// BN = 8*MC consecutive columns; the 8 warps split the fibre rows in groups
// of 8 (warp w owns groups w, w+8, ...). Per tile:
//   phase 1  P^T (BN x R) = X^T U    (mma.sync m8n8k4 f64, K = the warp's rows)
//            cross-warp sum of the partial P^T through shared memory
//   phase 2  Rec^T (BN x N) = P^T U^T (K = R), E = X - Rec, ||E||^2, ||X||^2
// The K index inside phase 1 is permuted (k-step (grp, i), lane t -> row
// 8 grp + 2t + i) so that the A fragments a thread feeds phase 1 are exactly
// the X elements its phase-2 accumulators cover, and phase 2's K index is
// permuted (k-step (rt, i), lane t -> rank 8 rt + 2t + i) so its A fragments
// are exactly the thread's reduced phase-1 accumulators. X therefore lives in
// registers only (read once from HBM, prefetched one tile ahead), U is staged
// once per CTA in shared memory with a conflict-minimal row pitch (8 RT + 4).
// Reference: streaming.cpp:128-133 (ttm pair + residual), tensor.cpp:106-162.
#pragma once
#include "kernels.cuh"

namespace tsg {
namespace dmma_proj {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int RT, int MC>
constexpr int red_doubles() {
  return 9 * MC * RT * 2 * 32;  // 8 warp partials + the reduced copy
}

// CTAs per SM for a tile shape: two when the register footprint allows, so
// one CTA's reduction barriers overlap the other's DMMA work.
constexpr int pick_minb(int RT, int MC, int GM) { return (MC * GM <= 8 && RT * MC <= 8) ? 2 : 1; }

template <int RT, int MC, int GM>
__global__ void __launch_bounds__(256, pick_minb(RT, MC, GM)) proj_dmma_kernel(ProjArgs a, int streaming_in) {
  extern __shared__ double sm[];
  __shared__ double sred[32];
  constexpr int RPAD = 8 * RT + 4;
  constexpr int PER = MC * RT * 2;  // accumulator doubles per lane
  const long long left = a.v.left, N = a.v.n, right = a.v.right;
  const long long cols = left * right;
  const int R = a.R;
  const int ngroups = (int)((N + 7) / 8);
  double* Us = sm;
  double* red = Us + (long long)ngroups * 8 * RPAD;
  if (a.upad) {
    // straight 16-byte copy of the pre-padded image (RPAD is even)
    const int total2 = ngroups * 8 * RPAD / 2;
    const double2* src = reinterpret_cast<const double2*>(a.upad);
    double2* dst = reinterpret_cast<double2*>(Us);
#pragma unroll 8
    for (int idx = threadIdx.x; idx < total2; idx += blockDim.x) dst[idx] = __ldg(src + idx);
  } else {
    // coalesced read of the column-major U, transposed into the padded rows
    const int rows8 = ngroups * 8;
    const int total = rows8 * RPAD;
#pragma unroll 4
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
      const int col = idx / rows8, row = idx - col * rows8;
      Us[row * RPAD + col] = (row < N && col < R) ? __ldg(a.u + row + (long long)col * N) : 0.0;
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const long long ntiles = (cols + 8 * MC - 1) / (8 * MC);
  const double* __restrict__ x = a.x;

  double X[MC][GM][2], Xn[MC][GM][2];
  // column c = l + r*left starts at r*left*N + l = c*N - l*(N-1); 32-bit
  // division only (cols < 2^31 is checked at launch), none when left == 1
  const unsigned uleft = (unsigned)left;
  auto col_base = [&](long long c) -> long long {
    if (uleft == 1u) return c * N;
    const unsigned l = (unsigned)c % uleft;
    return c * N - (long long)l * (N - 1);
  };
  auto load_tile = [&](long long tile, double (&dst)[MC][GM][2]) {
#pragma unroll
    for (int mc = 0; mc < MC; ++mc) {
      const long long c = tile * 8 * MC + 8 * mc + g;
      const bool cv = c < cols;
      const long long base = cv ? col_base(c) : 0;
#pragma unroll
      for (int gi = 0; gi < GM; ++gi) {
        const int grp = warp + 8 * gi;
        const long long row = 8LL * grp + 2 * t;
        double v0 = 0.0, v1 = 0.0;
        if (cv && grp < ngroups) {
          if (left == 1 && row + 1 < N && ((base + row) & 1) == 0) {
            const double2 v = streaming_in ? __ldcs(reinterpret_cast<const double2*>(x + base + row))
                                           : *reinterpret_cast<const double2*>(x + base + row);
            v0 = v.x;
            v1 = v.y;
          } else {
            if (row < N) v0 = streaming_in ? __ldcs(x + base + row * left) : x[base + row * left];
            if (row + 1 < N)
              v1 = streaming_in ? __ldcs(x + base + (row + 1) * left) : x[base + (row + 1) * left];
          }
        }
        dst[mc][gi][0] = v0;
        dst[mc][gi][1] = v1;
      }
    }
  };

  // With one CTA per SM the next tile is prefetched into registers; with two,
  // the co-resident CTA hides the load latency and registers stay <= 128.
  constexpr bool kPrefetch = pick_minb(RT, MC, GM) == 1;
  // Tiles are handed out by an atomic counter when one is given, so CTAs that
  // start late (an SM busy with the previous slice's insertion) take fewer.
  // The index two tiles ahead is fetched by thread 0 at the start of a tile
  // and published at the reduction barrier, so the atomic's latency hides
  // behind phase 1.
  __shared__ long long s_next;
  const bool dyn = a.tile_counter != nullptr;
  double racc = 0.0, xacc = 0.0;
  long long tile = blockIdx.x;
  long long next;
  if (dyn) {
    if (threadIdx.x == 0) s_next = (long long)gridDim.x + atomicAdd(a.tile_counter, 1u);
    __syncthreads();
    next = s_next;
  } else {
    next = tile + gridDim.x;
  }
  if (kPrefetch && tile < ntiles) load_tile(tile, X);
#pragma unroll 1
  for (; tile < ntiles;) {
    if (kPrefetch) {
      if (next < ntiles) load_tile(next, Xn);
    } else {
      load_tile(tile, X);
    }
    long long after = 0;
    if (dyn && threadIdx.x == 0) after = (long long)gridDim.x + atomicAdd(a.tile_counter, 1u);
    // ---- phase 1: partial P^T over the warp's rows
    double acc[MC][RT][2];
#pragma unroll
    for (int mc = 0; mc < MC; ++mc)
#pragma unroll
      for (int rt = 0; rt < RT; ++rt) acc[mc][rt][0] = acc[mc][rt][1] = 0.0;
#pragma unroll
    for (int gi = 0; gi < GM; ++gi) {
      const int grp = warp + 8 * gi;
      if (grp < ngroups) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const double* urow = Us + (8 * grp + 2 * t + i) * RPAD + g;
          double b[RT];
#pragma unroll
          for (int rt = 0; rt < RT; ++rt) b[rt] = urow[8 * rt];
#pragma unroll
          for (int mc = 0; mc < MC; ++mc)
#pragma unroll
            for (int rt = 0; rt < RT; ++rt) dmma(acc[mc][rt][0], acc[mc][rt][1], X[mc][gi][i], b[rt]);
        }
      }
    }
    // ---- cross-warp reduction (reduce-scatter then gather; fixed order)
    double* myred = red + warp * (PER * 32);
#pragma unroll
    for (int mc = 0; mc < MC; ++mc)
#pragma unroll
      for (int rt = 0; rt < RT; ++rt)
#pragma unroll
        for (int i = 0; i < 2; ++i) myred[((mc * RT + rt) * 2 + i) * 32 + lane] = acc[mc][rt][i];
    if (dyn && threadIdx.x == 0) s_next = after;
    __syncthreads();
    double* fin = red + 8 * (PER * 32);
    for (int slot = warp; slot < PER; slot += 8) {
      double sacc = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) sacc += red[w * (PER * 32) + slot * 32 + lane];
      fin[slot * 32 + lane] = sacc;
    }
    __syncthreads();
#pragma unroll
    for (int mc = 0; mc < MC; ++mc)
#pragma unroll
      for (int rt = 0; rt < RT; ++rt)
#pragma unroll
        for (int i = 0; i < 2; ++i) acc[mc][rt][i] = fin[((mc * RT + rt) * 2 + i) * 32 + lane];
    // ---- store P (each (mc, rt) block written by one warp)
    if (a.p) {
#pragma unroll
      for (int mc = 0; mc < MC; ++mc) {
        const long long c = tile * 8 * MC + 8 * mc + g;
        if (c < cols) {
          // (l, r) -> r*left*R + l = c*R - l*(R-1)
          const long long l = (uleft == 1u) ? 0 : (long long)((unsigned)c % uleft);
          double* pout = a.p + c * R - l * (R - 1);
#pragma unroll
          for (int rt = 0; rt < RT; ++rt) {
            if (((mc * RT + rt) & 7) != warp) continue;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int j = 8 * rt + 2 * t + i;
              if (j < R) pout[(long long)j * left] = acc[mc][rt][i];
            }
          }
        }
      }
    }
    // ---- phase 2: reconstruction, residual and norms
    if (a.residual) {
#pragma unroll
      for (int gi = 0; gi < GM; ++gi) {
        const int grp = warp + 8 * gi;
        if (grp < ngroups) {
          double c2[MC][2];
#pragma unroll
          for (int mc = 0; mc < MC; ++mc) c2[mc][0] = c2[mc][1] = 0.0;
          const double* urow = Us + (8 * grp + g) * RPAD + 2 * t;
#pragma unroll
          for (int rt = 0; rt < RT; ++rt)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const double b = urow[8 * rt + i];
#pragma unroll
              for (int mc = 0; mc < MC; ++mc) dmma(c2[mc][0], c2[mc][1], acc[mc][rt][i], b);
            }
#pragma unroll
          for (int mc = 0; mc < MC; ++mc)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const double xv = X[mc][gi][i];
              const double ev = xv - c2[mc][i];
              racc += ev * ev;
              xacc += xv * xv;
            }
          if (a.e) {
#pragma unroll
            for (int mc = 0; mc < MC; ++mc) {
              const long long c = tile * 8 * MC + 8 * mc + g;
              if (c < cols) {
                const long long cb = col_base(c);
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                  const long long row = 8LL * grp + 2 * t + i;
                  if (row < N) a.e[cb + row * left] = X[mc][gi][i] - c2[mc][i];
                }
              }
            }
          }
        }
      }
    }
    if (kPrefetch) {
#pragma unroll
      for (int mc = 0; mc < MC; ++mc)
#pragma unroll
        for (int gi = 0; gi < GM; ++gi) {
          X[mc][gi][0] = Xn[mc][gi][0];
          X[mc][gi][1] = Xn[mc][gi][1];
        }
    }
    tile = next;
    next = dyn ? s_next : tile + gridDim.x;
  }
  racc = block_sum(racc, sred);
  xacc = block_sum(xacc, sred);
  if (threadIdx.x == 0 && a.partial) {
    a.partial[2 * blockIdx.x] = racc;
    a.partial[2 * blockIdx.x + 1] = xacc;
  }
}

template <int RT, int MC, int GM>
inline size_t smem_bytes(long long N) {
  const long long ngroups = (N + 7) / 8;
  return sizeof(double) * (ngroups * 8 * (8 * RT + 4) + red_doubles<RT, MC>());
}

template <int RT, int MC, int GM>
inline int launch_t(const ProjArgs& a, int streaming_in, cudaStream_t st) {
  const size_t smem = smem_bytes<RT, MC, GM>(a.v.n);
  static size_t attr = 48 * 1024;
  if (smem > attr) {
    if (cudaFuncSetAttribute(proj_dmma_kernel<RT, MC, GM>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return -1;
    attr = smem;
  }
  const long long cols = a.v.left * a.v.right;
  const long long ntiles = (cols + 8 * MC - 1) / (8 * MC);
  // one SM is left to the concurrently running insertion kernel
  const long long slots = (long long)(kNumSMs - 1) * pick_minb(RT, MC, GM);
  const int grid = (int)(ntiles < slots ? (ntiles < 1 ? 1 : ntiles) : slots);
  proj_dmma_kernel<RT, MC, GM><<<grid, 256, smem, st>>>(a, streaming_in);
  return grid;
}

// Column tiles per CTA tile: wide tiles for small R (B-fragment reuse), while
// keeping the register-resident X (2 MC GM doubles, double-buffered) bounded.
constexpr int pick_mc(int RT, int GM) { return RT <= 2 ? (GM <= 2 ? 4 : 2) : (RT <= 6 ? 2 : 1); }

template <int RT, int GM>
inline int launch_rt(const ProjArgs& a, int streaming_in, cudaStream_t st) {
  return launch_t<RT, pick_mc(RT, GM), GM>(a, streaming_in, st);
}

// Picks (RT, MC, GM); returns -1 when the shape is outside the DMMA kernel's
// envelope (N > 512, R > 64 or shared memory too large).
template <int GM>
inline int dispatch_rt(const ProjArgs& a, int streaming_in, cudaStream_t st) {
  switch ((a.R + 7) / 8) {
    case 1: return launch_rt<1, GM>(a, streaming_in, st);
    case 2: return launch_rt<2, GM>(a, streaming_in, st);
    case 3: return launch_rt<3, GM>(a, streaming_in, st);
    case 4: return launch_rt<4, GM>(a, streaming_in, st);
    case 5: return launch_rt<5, GM>(a, streaming_in, st);
    case 6: return launch_rt<6, GM>(a, streaming_in, st);
    case 7: return launch_rt<7, GM>(a, streaming_in, st);
    case 8: return launch_rt<8, GM>(a, streaming_in, st);
    default: return -1;
  }
}

inline int launch(const ProjArgs& a, int streaming_in, cudaStream_t st) {
  const long long N = a.v.n;
  if (N > 512 || a.R > 64 || a.R < 1) return -1;
  if (a.v.left * a.v.right >= (1LL << 31) || a.v.left >= (1LL << 31)) return -1;
  const int RT = (a.R + 7) / 8;
  const long long ngroups = (N + 7) / 8;
  const long long smem = 8 * (ngroups * 8 * (8 * RT + 4)) + 8LL * 9 * 4 * RT * 2 * 32;
  if (smem > 220 * 1024) return -1;
  const int GM = (int)((ngroups + 7) / 8);
  if (GM <= 1) return dispatch_rt<1>(a, streaming_in, st);
  if (GM <= 2) return dispatch_rt<2>(a, streaming_in, st);
  if (GM <= 4) return dispatch_rt<4>(a, streaming_in, st);
  return dispatch_rt<8>(a, streaming_in, st);
}

}  // namespace dmma_proj
}  // namespace tsg
