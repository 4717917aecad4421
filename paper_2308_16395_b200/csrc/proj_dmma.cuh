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
// permuted (k-step (rt, i), lane t -> rank 8 rt + 4i + t; the U image holds
// rank 8rt + 4i + t in column 8rt + 2t + i) so its A fragments are exactly
// the thread's reduced phase-1 accumulators and a K-step of ranks >= R
// (R - 8(RT-1) <= 4: the last tile's i = 1 step) is skipped. X therefore lives in
// registers only (read once from HBM, prefetched one tile ahead), U is staged
// once per CTA in shared memory with a conflict-minimal row pitch (8 RT + 4).
// Reference: streaming.cpp:128-133 (ttm pair + residual), tensor.cpp:106-162.
#pragma once
#include <cstdlib>

#include "kernels.cuh"

namespace tsg {
namespace dmma_proj {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {

  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int RT, int MC, int NW = 8>
constexpr int red_doubles() {
  return (NW + 1) * MC * RT * 2 * 32;  // NW warp partials + the reduced copy
}

// CTAs per SM for a tile shape: two when the register footprint allows, so
// one CTA's reduction barriers overlap the other's DMMA work.
constexpr int pick_minb(int RT, int MC, int GM) { return (MC * GM <= 8 && RT * MC <= 8) ? 2 : 1; }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// mbarrier + bulk-copy (TMA) helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Same copy with an L2 evict-first policy: a slice streamed once should not
// push the small hot state the insertion kernel reads (Q, core, the streaming
// factor) out of L2.
__device__ __forceinline__ unsigned long long l2_evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_ef(void* dst, const void* src, unsigned bytes,
                                            unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// STAGES > 0: contiguous mode-0 fibres staged through a per-thread-private
// cp.async ring in shared memory (each thread copies exactly the 16-byte
// pairs it later reads, so no barrier guards the ring).
template <int RT, int MC, int GM, int STAGES, int NW = 8>
__global__ void __launch_bounds__(32 * NW, STAGES > 0 ? 1 : (NW == 8 ? pick_minb(RT, MC, GM) : 2))
    proj_dmma_kernel(ProjArgs a) {
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
  double2* ring = reinterpret_cast<double2*>(red + (NW + 1) * PER * 32);  // [STAGES][MC][GM][32 NW]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const long long ntiles = (cols + 8 * MC - 1) / (8 * MC);
  const int streaming_in = a.karg0;
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
        const int grp = warp + NW * gi;
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
  constexpr bool kPrefetch = STAGES == 0 && pick_minb(RT, MC, GM) == 1;
  auto ring_issue = [&](long long tl, int stage) {
#pragma unroll
    for (int mc = 0; mc < MC; ++mc) {
      const long long c = tl * 8 * MC + 8 * mc + g;
      const bool cv = c < cols;
#pragma unroll
      for (int gi = 0; gi < GM; ++gi) {
        const int grp = warp + NW * gi;
        const long long row = 8LL * grp + 2 * t;
        const bool ok = cv && grp < ngroups && row < N;
        const int bytes = ok ? (row + 1 < N ? 16 : 8) : 0;
        const double* src = ok ? x + c * N + row : x;
        cp_async16(ring + (((stage * MC + mc) * GM + gi) * (32 * NW) + threadIdx.x), src, bytes);
      }
    }
  };
  // Tiles are handed out by an atomic counter when one is given, so CTAs that
  // start late (an SM busy with the previous slice's insertion) take fewer.
  // The index two tiles ahead is fetched by thread 0 at the start of a tile
  // and published at the reduction barrier, so the atomic's latency hides
  // behind phase 1.
  __shared__ long long s_next;
  const bool dyn = STAGES == 0 && a.tile_counter != nullptr;
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
  if constexpr (STAGES > 0) {
#pragma unroll
    for (int st_ = 0; st_ < STAGES - 1; ++st_) {
      const long long tl = tile + (long long)st_ * gridDim.x;
      if (tl < ntiles) ring_issue(tl, st_);
      cp_async_commit();
    }
  }
  // stage U while the first tile's loads are in flight
  if (a.upad) {
    // straight 16-byte copy of the pre-padded image (RPAD is even); the
    // first tile's X loads are already in flight
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
      const int rk = (col & ~7) + 4 * (col & 1) + ((col & 7) >> 1);
      Us[row * RPAD + col] = (row < N && col < 8 * RT && rk < R) ? __ldg(a.u + row + (long long)rk * N) : 0.0;
    }
  }
  __syncthreads();
  int it = 0;
#pragma unroll 1
  for (; tile < ntiles; ++it) {
    if constexpr (STAGES > 0) {
      const long long tl = tile + (long long)(STAGES - 1) * gridDim.x;
      if (tl < ntiles) ring_issue(tl, (it + STAGES - 1) % STAGES);
      cp_async_commit();
      cp_async_wait<STAGES - 1>();
      const int stage = it % STAGES;
#pragma unroll
      for (int mc = 0; mc < MC; ++mc)
#pragma unroll
        for (int gi = 0; gi < GM; ++gi) {
          const double2 v = ring[((stage * MC + mc) * GM + gi) * (32 * NW) + threadIdx.x];
          X[mc][gi][0] = v.x;
          X[mc][gi][1] = v.y;
        }
    } else if (kPrefetch) {
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
      const int grp = warp + NW * gi;
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
    // the next tile index is read right after the barrier that publishes it:
    // thread 0 rewrites s_next in the next iteration before that iteration's
    // first barrier, so reading it at the end of this one would race
    long long next_pub = 0;
    if (a.debug_skip & 2) {  // profiling only
      if (dyn && threadIdx.x == 0) s_next = after;
      __syncthreads();
      next_pub = s_next;
    } else {
    double* myred = red + warp * (PER * 32);
#pragma unroll
    for (int mc = 0; mc < MC; ++mc)
#pragma unroll
      for (int rt = 0; rt < RT; ++rt)
#pragma unroll
        for (int i = 0; i < 2; ++i) myred[((mc * RT + rt) * 2 + i) * 32 + lane] = acc[mc][rt][i];
    if (dyn && threadIdx.x == 0) s_next = after;
    __syncthreads();
    next_pub = s_next;
    double* fin = red + NW * (PER * 32);
    for (int slot = warp; slot < PER; slot += NW) {
      double sacc = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) sacc += red[w * (PER * 32) + slot * 32 + lane];
      fin[slot * 32 + lane] = sacc;
    }
    __syncthreads();
#pragma unroll
    for (int mc = 0; mc < MC; ++mc)
#pragma unroll
      for (int rt = 0; rt < RT; ++rt)
#pragma unroll
        for (int i = 0; i < 2; ++i) acc[mc][rt][i] = fin[((mc * RT + rt) * 2 + i) * 32 + lane];
    }
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
            if (((mc * RT + rt) % NW) != warp) continue;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int j = 8 * rt + 4 * i + t;
              if (j < R) pout[(long long)j * left] = acc[mc][rt][i];
            }
          }
        }
      }
    }
    // ---- phase 2: reconstruction, residual and norms. All groups' DMMA
    // chains are issued before any epilogue so their latencies overlap.
    if (a.residual) {
      double c2[GM][MC][2];
#pragma unroll
      for (int gi = 0; gi < GM; ++gi)
#pragma unroll
        for (int mc = 0; mc < MC; ++mc) c2[gi][mc][0] = c2[gi][mc][1] = 0.0;
#pragma unroll
      for (int rt = 0; rt < RT; ++rt)
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int gi = 0; gi < GM; ++gi) {
            const int grp = warp + NW * gi;
            if (grp < ngroups) {
              const double b = Us[(8 * grp + g) * RPAD + 2 * t + 8 * rt + i];
#pragma unroll
              for (int mc = 0; mc < MC; ++mc) dmma(c2[gi][mc][0], c2[gi][mc][1], acc[mc][rt][i], b);
            }
          }
#pragma unroll
      for (int gi = 0; gi < GM; ++gi) {
        const int grp = warp + NW * gi;
        if (grp < ngroups) {
#pragma unroll
          for (int mc = 0; mc < MC; ++mc)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const double xv = X[mc][gi][i];
              const double ev = xv - c2[gi][mc][i];
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
                  if (row < N) a.e[cb + row * left] = X[mc][gi][i] - c2[gi][mc][i];
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
    if constexpr (STAGES > 0) {
      tile += gridDim.x;  // static schedule: the ring prefetches by stride
    } else {
      tile = next;
      next = dyn ? next_pub : tile + gridDim.x;
    }
  }
  racc = block_sum(racc, sred);
  xacc = block_sum(xacc, sred);
  if (threadIdx.x == 0 && a.partial) {
    a.partial[2 * blockIdx.x] = racc;
    a.partial[2 * blockIdx.x + 1] = xacc;
  }
}

template <int RT, int MC, int GM, int STAGES, int NW = 8>
inline size_t smem_bytes(long long N) {
  const long long ngroups = (N + 7) / 8;
  return sizeof(double) * (ngroups * 8 * (8 * RT + 4) + red_doubles<RT, MC, NW>()) +
         (size_t)STAGES * MC * GM * 32 * NW * 16;
}

template <int RT, int MC, int GM, int STAGES, int NW = 8>
inline int launch_t(const ProjArgs& a, int streaming_in, cudaStream_t st) {
  const size_t smem = smem_bytes<RT, MC, GM, STAGES, NW>(a.v.n);
  if (smem > 220 * 1024) return -1;
  // (the attribute bounds the dynamic part only; 48 KB of dynamic shared
  // memory plus the static reduction scratch exceeds the default opt-in)
  static size_t attr = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(proj_dmma_kernel<RT, MC, GM, STAGES, NW>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return -1;
    attr = smem;
  }
  const long long cols = a.v.left * a.v.right;
  const long long ntiles = (cols + 8 * MC - 1) / (8 * MC);
  // SMs left to the concurrently running insertion kernels (TSG_PROJ_FREE_SMS)
  static const int free_sms = [] {
    const char* e = std::getenv("TSG_PROJ_FREE_SMS");
    return e ? std::atoi(e) : 1;
  }();
  const long long slots = (long long)(kNumSMs - free_sms) *
                          (STAGES > 0 ? 1 : (NW == 8 ? pick_minb(RT, MC, GM) : 2));
  const int grid = (int)(ntiles < slots ? (ntiles < 1 ? 1 : ntiles) : slots);
  ProjArgs b = a;
  b.karg0 = streaming_in;
  proj_dmma_kernel<RT, MC, GM, STAGES, NW><<<grid, 32 * NW, smem, st>>>(b);
  return grid;
}


// ---------------------------------------------------------------------------
// Mode-0 fast path: contiguous BN-column tiles (BN * N doubles) stream into a
// dense NS-stage shared-memory ring with one bulk copy (TMA, cp.async.bulk)
// per tile and an mbarrier per stage, keeping ~(NS-1) tiles in flight per SM
// (load latency, not bandwidth, limited the register-prefetch path). The
// math is the same two-phase DMMA scheme as proj_dmma_kernel.
template <int RT, int MC, int GM, bool WE, int MINB = 1, bool HALF = false>
__global__ void __launch_bounds__(256, MINB) proj0_tma_kernel(ProjArgs a) {
  const int NS = a.karg0;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ double sred[32];
  constexpr int RPAD = 8 * RT + 4;
  constexpr int PER = MC * RT * 2;
  constexpr int BN = 8 * MC;
  const long long N = a.v.n, cols = a.v.right;  // left == 1
  const int R = a.R;
  const int ngroups = (int)((N + 7) / 8);
  double* ring = reinterpret_cast<double*>(smraw);
  double* Us = ring + (long long)NS * BN * N;
  double* red = Us + (long long)ngroups * 8 * RPAD;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(red + 9 * PER * 32);
  unsigned long long* ubar = bar + NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool last_ok = warp + 8 * (GM - 1) < ngroups;  // warp-uniform
  const int g = lane >> 2, t = lane & 3;
  const long long ntiles = (cols + BN - 1) / BN;
  const double* xsrc = a.x;
  const bool ef = a.stream_in == 2;  // slice read exactly once: evict-first in L2
  const unsigned long long pol = ef ? l2_evict_first_policy() : 0ull;
  auto issue = [&](long long tl, int stage) {
    const long long c0 = tl * BN;
    const long long nc = (cols - c0) < BN ? (cols - c0) : BN;
    const unsigned bytes = (unsigned)(nc * N * 8);
    mbar_expect_tx(&bar[stage], bytes);
    if (ef)
      bulk_g2s_ef(ring + (long long)stage * BN * N, xsrc + c0 * N, bytes, &bar[stage], pol);
    else
      bulk_g2s(ring + (long long)stage * BN * N, xsrc + c0 * N, bytes, &bar[stage]);
  };
  if (threadIdx.x == 0) {
    for (int s_ = 0; s_ < NS; ++s_) mbar_init(&bar[s_], 1);
    mbar_init(ubar, 1);
    mbar_fence_init();
    // U first (one bulk copy of the pre-padded image), then the first tiles
    const unsigned ubytes = (unsigned)(ngroups * 8 * RPAD * sizeof(double));
    mbar_expect_tx(ubar, ubytes);
    bulk_g2s(Us, a.upad, ubytes, ubar);
    for (int s_ = 0; s_ < NS - 1; ++s_) {
      const long long tl = blockIdx.x + (long long)s_ * gridDim.x;
      if (tl < ntiles) issue(tl, s_);
    }
  }
  __syncthreads();
  mbar_wait(ubar, 0);
  double racc = 0.0, xacc = 0.0;
  int it = 0;
#pragma unroll 1
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int stage = it % NS;
    // refill the stage consumed in the previous iteration (every thread has
    // passed that iteration's reduction barriers)
    if (threadIdx.x == 0) {
      const long long tl = tile + (long long)(NS - 1) * gridDim.x;
      if (tl < ntiles) issue(tl, (it + NS - 1) % NS);
    }
    mbar_wait(&bar[stage], (unsigned)((it / NS) & 1));
    if (a.karg1 == 7) {  // profiling only (tools/proj0_one.py): stream the slice, no math
      __syncthreads();
      continue;
    }
    const double* xt = ring + (long long)stage * BN * N;
    double X[MC][GM][2];
#pragma unroll
    for (int mc = 0; mc < MC; ++mc) {
      const int cl = 8 * mc + g;
      const bool cv = tile * BN + cl < cols;
#pragma unroll
      for (int gi = 0; gi < GM; ++gi) {
        const int grp = warp + 8 * gi;
        const int row = 8 * grp + 2 * t;
        double2 v = make_double2(0.0, 0.0);
        if (cv && grp < ngroups && row < N) v = *reinterpret_cast<const double2*>(xt + cl * N + row);
        X[mc][gi][0] = v.x;
        X[mc][gi][1] = v.y;
      }
    }
    // ---- phase 1: partial P^T over the warp's rows
    double acc[MC][RT][2];
#pragma unroll
    for (int mc = 0; mc < MC; ++mc)
#pragma unroll
      for (int rt = 0; rt < RT; ++rt) acc[mc][rt][0] = acc[mc][rt][1] = 0.0;
    // slots gi < GM-1 always hold a row group; the last one only for some
    // warps (a real branch, so no predicated-off DMMA occupies the pipe)
    auto p1 = [&](int gi) {
      const int grp = warp + 8 * gi;
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
    };
    const int dbg = a.karg1;  // profiling only: 8 skip reduction, 16 skip phase 2, 32 skip phase 1
    if (!(dbg & 32)) {
#pragma unroll
      for (int gi = 0; gi + 1 < GM; ++gi) p1(gi);
      if (last_ok) p1(GM - 1);
    }
    // ---- cross-warp reduction (reduce-scatter then gather; fixed order)
    if (!(dbg & 8)) {
    double* myred = red + warp * (PER * 32);
#pragma unroll
    for (int mc = 0; mc < MC; ++mc)
#pragma unroll
      for (int rt = 0; rt < RT; ++rt)
#pragma unroll
        for (int i = 0; i < 2; ++i) myred[((mc * RT + rt) * 2 + i) * 32 + lane] = acc[mc][rt][i];
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
    } else {
      __syncthreads();  // the ring refill relies on one barrier per tile
    }
    // ---- store P (P[c*R + j]); each (mc, rt) block by one warp
    if (a.p) {
#pragma unroll
      for (int mc = 0; mc < MC; ++mc) {
        const long long c = tile * BN + 8 * mc + g;
        if (c < cols) {
#pragma unroll
          for (int rt = 0; rt < RT; ++rt) {
            if (((mc * RT + rt) & 7) != warp) continue;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int j = 8 * rt + 4 * i + t;
              if (j < R) a.p[c * R + j] = acc[mc][rt][i];
            }
          }
        }
      }
    }
    // ---- phase 2 (all groups' DMMA chains first, then the epilogue)
    if (a.residual && !(dbg & 16)) {
      double c2[GM][MC][2];
#pragma unroll
      for (int gi = 0; gi < GM; ++gi)
#pragma unroll
        for (int mc = 0; mc < MC; ++mc) c2[gi][mc][0] = c2[gi][mc][1] = 0.0;
      auto p2 = [&](int gi, int rt, int i) {
        const int grp = warp + 8 * gi;
        const double b = Us[(8 * grp + g) * RPAD + 2 * t + 8 * rt + i];
#pragma unroll
        for (int mc = 0; mc < MC; ++mc) dmma(c2[gi][mc][0], c2[gi][mc][1], acc[mc][rt][i], b);
      };
      // K-step (rt, i) = ranks 8rt + 4i .. +3: the last tile's second step is
      // all padding when HALF
#pragma unroll
      for (int rt = 0; rt < RT; ++rt)
#pragma unroll
        for (int i = 0; i < 2; ++i)
          if (!(HALF && rt == RT - 1 && i == 1)) {
#pragma unroll
            for (int gi = 0; gi + 1 < GM; ++gi) p2(gi, rt, i);
          }
      if (last_ok) {
#pragma unroll
        for (int rt = 0; rt < RT; ++rt)
#pragma unroll
          for (int i = 0; i < 2; ++i)
            if (!(HALF && rt == RT - 1 && i == 1)) p2(GM - 1, rt, i);
      }
#pragma unroll
      for (int gi = 0; gi < GM; ++gi) {
        const int grp = warp + 8 * gi;
        if (grp < ngroups) {
#pragma unroll
          for (int mc = 0; mc < MC; ++mc)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const double xv = X[mc][gi][i];
              const double ev = xv - c2[gi][mc][i];
              racc += ev * ev;
              xacc += xv * xv;
            }
          if constexpr (WE) {
#pragma unroll
            for (int mc = 0; mc < MC; ++mc) {
              const long long c = tile * BN + 8 * mc + g;
              if (c < cols) {
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                  const long long row = 8LL * grp + 2 * t + i;
                  if (row < N) a.e[c * N + row] = X[mc][gi][i] - c2[gi][mc][i];
                }
              }
            }
          }
        }
      }
    }
  }
  racc = block_sum(racc, sred);
  xacc = block_sum(xacc, sred);
  if (threadIdx.x == 0 && a.partial) {
    a.partial[2 * blockIdx.x] = racc;
    a.partial[2 * blockIdx.x + 1] = xacc;
  }
}

inline size_t smem0_bytes(int RT, int MC, long long N, int NS) {
  const long long ngroups = (N + 7) / 8;
  return sizeof(double) * ((long long)NS * 8 * MC * N + ngroups * 8 * (8 * RT + 4) +
                           9 * MC * RT * 2 * 32) +
         (NS + 1) * sizeof(unsigned long long);
}

template <int RT, int MC, int GM, bool WE, int MINB, bool HALF>
inline int launch0_th(const ProjArgs& a, cudaStream_t st) {
  const size_t cap = MINB == 1 ? 225 * 1024 : 111 * 1024;
  int NS = 8;
  while (NS >= 3 && smem0_bytes(RT, MC, a.v.n, NS) > cap) --NS;
  if (NS < 3) return -1;
  const size_t smem = smem0_bytes(RT, MC, a.v.n, NS);
  static size_t attr = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(proj0_tma_kernel<RT, MC, GM, WE, MINB, HALF>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap) != cudaSuccess)
      return -1;
    attr = cap;
  }
  const long long ntiles = (a.v.right + 8 * MC - 1) / (8 * MC);
  // leave room for the concurrent tail / insertion kernels
  static const long long cap_ctas = [] {
    const char* e = std::getenv("TSG_M0_CTAS");
    return e ? std::atoll(e) : 0LL;
  }();
  // default: 8 SMs' worth of slots stay free for the overlapping kernels
  long long slots = (long long)(kNumSMs - 8) * MINB;
  if (cap_ctas > 0) slots = cap_ctas;
  const int grid = (int)(ntiles < slots ? (ntiles < 1 ? 1 : ntiles) : slots);
  ProjArgs b = a;
  b.karg0 = NS;
  proj0_tma_kernel<RT, MC, GM, WE, MINB, HALF><<<grid, 256, smem, st>>>(b);
  return grid;
}

template <int RT, int MC, int GM, bool WE, int MINB>
inline int launch0_t(const ProjArgs& a, cudaStream_t st) {
  return (a.R - 8 * (RT - 1) <= 4) ? launch0_th<RT, MC, GM, WE, MINB, true>(a, st)
                                   : launch0_th<RT, MC, GM, WE, MINB, false>(a, st);
}

template <int RT, int MC, int GM>
inline int launch0_rt(const ProjArgs& a, cudaStream_t st) {
  static const int variant = [] {
    const char* e = std::getenv("TSG_PROJ0_VARIANT");
    return e ? std::atoi(e) : 1;
  }();
  if (variant == 1 && RT <= 2) {  // 8-column tiles, two CTAs per SM
    const int g = a.e ? launch0_t<RT, 1, GM, true, 2>(a, st) : launch0_t<RT, 1, GM, false, 2>(a, st);
    if (g > 0) return g;
  }
  return a.e ? launch0_t<RT, MC, GM, true, 1>(a, st) : launch0_t<RT, MC, GM, false, 1>(a, st);
}

inline int launch0(const ProjArgs& a, cudaStream_t st) {
  const long long N = a.v.n;
  if (a.v.left != 1 || (N & 1) || N > 256 || a.R > 32 || a.R < 1 || !a.upad) return -1;
  if (a.v.right >= (1LL << 31)) return -1;
  const int ngroups = (int)((N + 7) / 8);
  const int RT = (a.R + 7) / 8;
  if (ngroups <= 8) {
    switch (RT) {
      case 1: return launch0_rt<1, 4, 1>(a, st);
      case 2: return launch0_rt<2, 4, 1>(a, st);
      case 3: return launch0_rt<3, 2, 1>(a, st);
      case 4: return launch0_rt<4, 2, 1>(a, st);
    }
  } else if (ngroups <= 16) {
    switch (RT) {
      case 1: return launch0_rt<1, 2, 2>(a, st);
      case 2: return launch0_rt<2, 2, 2>(a, st);
      case 3: return launch0_rt<3, 2, 2>(a, st);
      case 4: return launch0_rt<4, 2, 2>(a, st);
    }
  } else {
    switch (RT) {
      case 1: return launch0_rt<1, 2, 4>(a, st);
      case 2: return launch0_rt<2, 2, 4>(a, st);
      case 3: return launch0_rt<3, 2, 4>(a, st);
      case 4: return launch0_rt<4, 2, 4>(a, st);
    }
  }
  return -1;
}

// Column tiles per CTA tile: wide tiles for small R (B-fragment reuse), while
// keeping the register-resident X (2 MC GM doubles, double-buffered) bounded.
// (RT >= 3 with GM >= 4: one 8-column tile per CTA step keeps the register
// footprint at two CTAs per SM — measured 10 % faster on C3's 512 x 32 and
// 5 % on 256 x 36 than two tiles per step at one CTA per SM)
constexpr int pick_mc(int RT, int GM) {
  return RT <= 2 ? (GM <= 2 ? 4 : 2) : ((RT <= 6 && GM < 4) ? 2 : 1);
}

template <int RT, int GM>
inline int launch_rt(const ProjArgs& a, int streaming_in, cudaStream_t st) {
  // contiguous fibres (mode 0, even N): cp.async ring when it fits
  static const int ring_mode = [] {
    const char* e = std::getenv("TSG_PROJ_RING");
    return e ? std::atoi(e) : 1;
  }();
  if constexpr (GM <= 4 && RT <= 4) {
    if (ring_mode && a.v.left == 1 && (a.v.n & 1) == 0) {
      const int g = ring_mode == 2 ? launch_t<RT, 4, GM, 2>(a, streaming_in, st)
                                   : launch_t<RT, 2, GM, 3>(a, streaming_in, st);
      if (g > 0) return g;
    }
  }
  static const int mc1 = [] {
    const char* e = std::getenv("TSG_PROJ_MC1");
    return e ? std::atoi(e) : 0;
  }();
  if constexpr (pick_mc(RT, GM) > 1) {
    if (mc1) return launch_t<RT, 1, GM, 0>(a, streaming_in, st);
  }
  const int g = launch_t<RT, pick_mc(RT, GM), GM, 0>(a, streaming_in, st);
  if constexpr (pick_mc(RT, GM) > 1) {
    if (g < 0) return launch_t<RT, 1, GM, 0>(a, streaming_in, st);  // smaller reduction area
  }
  return g;
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

// 21..25 row groups (161 <= N <= 200): 5 warps x 5 groups balance the K split
template <int RT>
inline int launch_nw5(const ProjArgs& a, int streaming_in, cudaStream_t st) {
  return launch_t<RT, 2, 5, 0, 5>(a, streaming_in, st);
}

inline int launch(const ProjArgs& a, int streaming_in, cudaStream_t st) {
  const long long N = a.v.n;
  static const int tma0 = [] {
    const char* e = std::getenv("TSG_PROJ_TMA");
    return e ? std::atoi(e) : 1;
  }();
  if (tma0 && a.debug_skip == 0) {
    const int g0 = launch0(a, st);
    if (g0 > 0) return g0;
  }
  static const int nw5 = [] {
    const char* e = std::getenv("TSG_PROJ_NW5");
    return e ? std::atoi(e) : 1;
  }();
  if (nw5 && N > 160 && N <= 200 && a.R <= 32 && a.v.left * a.v.right < (1LL << 31)) {
    int g = -1;
    switch ((a.R + 7) / 8) {
      case 1: g = launch_nw5<1>(a, streaming_in, st); break;
      case 2: g = launch_nw5<2>(a, streaming_in, st); break;
      case 3: g = launch_nw5<3>(a, streaming_in, st); break;
      case 4: g = launch_nw5<4>(a, streaming_in, st); break;
    }
    if (g > 0) return g;
  }
  if (N > 512 || a.R > 64 || a.R < 1) return -1;
  if (a.v.left * a.v.right >= (1LL << 31) || a.v.left >= (1LL << 31)) return -1;
  const int RT = (a.R + 7) / 8;
  const long long ngroups = (N + 7) / 8;
  // the U image alone must fit; launch_t checks the exact footprint of the
  // (MC, stages) variant it picks (the reduction area depends on MC)
  if (8 * (ngroups * 8 * (8 * RT + 4)) > 200 * 1024) return -1;
  const int GM = (int)((ngroups + 7) / 8);
  if (GM <= 1) return dispatch_rt<1>(a, streaming_in, st);
  if (GM <= 2) return dispatch_rt<2>(a, streaming_in, st);
  if (GM <= 4) return dispatch_rt<4>(a, streaming_in, st);
  return dispatch_rt<8>(a, streaming_in, st);
}

}  // namespace dmma_proj
}  // namespace tsg
