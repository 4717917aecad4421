// Fused tail of one slice's projection chain: the small trailing modes
// k = m0..d-2 (their inputs are already projected along the large leading
// mode(s), so they sit in L2) and the branch decision, in ONE cooperative
// kernel with a grid barrier between modes (streaming.cpp:126-137, 187-188;
// tensor.cpp:106-162 for the mode products).
//
// Mode k: every mode-k fibre x (length N_k, stride `left`) is handled by one
// warp: lanes own fibre elements, p = U_k^T x is an all-reduce over the warp
// (fixed butterfly order -> deterministic), then e = x - U_k p and ||e||^2
// accumulate per lane. U_k is staged once per CTA in shared memory. Per-CTA
// partial sums are reduced in a fixed order by CTA 0, which then decides.
#include <cooperative_groups.h>

#include <cstdlib>

#include "decide.cuh"
#include "kernels.cuh"

namespace tsg {

namespace cg = cooperative_groups;

namespace {

template <int RMAX, int NT>
__global__ void __launch_bounds__(256) tail_kernel(TailArgs t) {
  constexpr int P2 = RMAX <= 4 ? 4 : RMAX <= 8 ? 8 : RMAX <= 16 ? 16 : 32;
  constexpr int LOG2P = P2 == 4 ? 2 : P2 == 8 ? 3 : P2 == 16 ? 4 : 5;
  constexpr int NP = 32 * NT;  // padded fibre length (rows of the U image)
  extern __shared__ double Us[];  // per tail mode: NP x RMAX, zero padded
  __shared__ double sp[8][P2];
  __shared__ double red[32];
  __shared__ double res[kMaxD];
  __shared__ double xsq;
  __shared__ int last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long nwarps = (long long)gridDim.x * 8;
  const long long gw = (long long)blockIdx.x * 8 + wid;
  auto stamp = [&](int i) {
    if (t.clk && threadIdx.x == 0) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      t.clk[blockIdx.x * 16 + i] = g;
    }
  };
  auto cstamp = [&](int i) {
    if (t.clk && threadIdx.x == 0) t.clk[16 * kMaxGrid + i] = clock64();
  };
  stamp(0);
  // first fibre of the first mode in flight before anything else
  double xv[NT];
  auto load_fibre = [&](const double* x, long long f, long long left, int n) {
    const long long l = f % left, r = f / left;
    const double* __restrict__ xf = x + l + r * left * n;
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      const int i = lane + 32 * q;
      xv[q] = xf[(long long)(i < n ? i : 0) * left];  // unconditional: loads issue together
    }
#pragma unroll
    for (int q = 0; q < NT; ++q) xv[q] *= (lane + 32 * q < n) ? 1.0 : 0.0;
  };
  bool have = false;
  if (t.m0 < t.m1 && gw < t.left[t.m0] * t.right[t.m0]) {
    load_fibre(t.x, gw, t.left[t.m0], (int)t.N[t.m0]);
    have = true;
  }
  // zero-padded U images of every tail mode (branch-free inner loops)
  for (int k = t.m0; k < t.m1; ++k) {
    const int n = (int)t.N[k], R = t.R[k];
    const double* __restrict__ u = t.u[k];
    double* dst = Us + (k - t.m0) * NP * RMAX;
    constexpr int TOT = NP * RMAX;
    constexpr int PER = (TOT + 255) / 256;
    double tmp[PER];
#pragma unroll
    for (int s2 = 0; s2 < PER; ++s2) {
      const int idx = threadIdx.x + 256 * s2;
      const int i = idx % NP, j = idx / NP;
      const bool ok = idx < TOT && i < n && j < R;
      tmp[s2] = u[ok ? i + (long long)j * n : 0] * (ok ? 1.0 : 0.0);
    }
#pragma unroll
    for (int s2 = 0; s2 < PER; ++s2) {
      const int idx = threadIdx.x + 256 * s2;
      if (idx < TOT) dst[idx] = tmp[s2];
    }
  }
  // CTA 0 reduces the stand-alone kernels' partial pairs meanwhile
  const DecideArgs& a = t.da;
  if (blockIdx.x == 0) {
    for (int k = a.first_mode; k < t.m0; ++k) {
      double acc = 0.0, acx = 0.0;
      for (int b = threadIdx.x; b < a.cnt[k]; b += blockDim.x) {
        acc += a.partial[a.off[k] + 2 * b];
        acx += a.partial[a.off[k] + 2 * b + 1];
      }
      acc = block_sum(acc, red);
      acx = block_sum(acx, red);
      if (threadIdx.x == 0) {
        t.part[(long long)kMaxD * gridDim.x + k] = acc;
        if (k == 0) t.part[(long long)kMaxD * gridDim.x + kMaxD] = acx;
      }
    }
  }
  __syncthreads();
  stamp(1);
  const double* x = t.x;
  for (int k = t.m0; k < t.m1; ++k) {
    const int n = (int)t.N[k], R = t.R[k];
    const long long left = t.left[k], right = t.right[k];
    const double* __restrict__ Uk = Us + (k - t.m0) * NP * RMAX;
    double* __restrict__ out = t.out[k];
    double acc = 0.0;
    const long long F = left * right;
    for (long long f = gw; f < F; f += nwarps) {
      const long long l = f % left, r = f / left;
      if (!have) load_fibre(x, f, left, n);
      have = false;
      // p = U^T x: per-lane partials (all RMAX chains advance together)
      double v[P2];
#pragma unroll
      for (int j = 0; j < P2; ++j) v[j] = 0.0;
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        const int i = lane + 32 * q;
#pragma unroll
        for (int j = 0; j < RMAX; ++j) v[j] = fma(Uk[i + j * NP], xv[q], v[j]);
      }
      // transposed (reduce-scatter) butterfly: log2(P2) halving exchanges
      // leave lane group j with the sum of coefficient j; the remaining
      // offsets finish it (fixed order -> deterministic)
#pragma unroll
      for (int st = 0; st < LOG2P; ++st) {
        const int o = 16 >> st;
        const int half = P2 >> (st + 1);
        const bool hi = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
          const double send = hi ? v[i] : v[i + half];
          const double keep = hi ? v[i + half] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
#pragma unroll
      for (int o = 16 >> LOG2P; o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
      const int jme = lane >> (5 - LOG2P);
      if ((lane & ((32 >> LOG2P) - 1)) == 0) {
        sp[wid][jme] = v[0];
        if (jme < R) out[l + left * (jme + (long long)R * r)] = v[0];
      }
      __syncwarp();
      double pj[RMAX];
#pragma unroll
      for (int j = 0; j < RMAX; ++j) pj[j] = sp[wid][j];
      __syncwarp();
      // e = x - U p, ||e||^2
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        const int i = lane + 32 * q;
        double rec = 0.0;
#pragma unroll
        for (int j = 0; j < RMAX; ++j) rec = fma(Uk[i + j * NP], pj[j], rec);
        const double e = xv[q] - rec;
        acc = fma(e, e, acc);
      }
    }
    stamp(2 + 2 * (k - t.m0));
    acc = block_sum(acc, red);
    if (threadIdx.x == 0) t.part[(long long)k * gridDim.x + blockIdx.x] = acc;
    if (k + 1 < t.m1) {
      cg::this_grid().sync();
      stamp(3 + 2 * (k - t.m0));
    }
    x = out;
  }
  // the last CTA to finish reduces the partials and decides
  cstamp(0);
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(t.done, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  cstamp(1);
  __threadfence();
  // one warp per tail mode reduces that mode's per-CTA partials (all loads in
  // flight at once, fixed lane order); the last warp fetches the leading
  // modes' sums. No block-wide barrier before the decision.
  {
    const int nm = t.m1 - t.m0;
    const unsigned g = gridDim.x;
    if (wid < nm) {
      const int k = t.m0 + wid;
      const double* pk = t.part + (long long)k * g;
      double acc = 0.0;
      for (unsigned b = lane; b < g; b += 32) acc += __ldcg(pk + b);
      acc = warp_sum(acc);
      if (lane == 0) res[k] = acc;
    } else if (wid == nm && lane == 0) {
      for (int k = a.first_mode; k < t.m0; ++k) res[k] = __ldcg(t.part + (long long)kMaxD * g + k);
      if (a.first_mode == 0 && t.m0 > 0) xsq = __ldcg(t.part + (long long)kMaxD * g + kMaxD);
    }
  }
  __syncthreads();
  cstamp(2);
  if (threadIdx.x == 0) {
    *t.done = 0u;  // re-arm for the next launch
    decide_finish(a, xsq, res);
  }
  cstamp(3);
  stamp(15);
}

template <int RMAX, int NT>
int launch_t(const TailArgs& t, cudaStream_t st) {
  long long fmax = 1;
  size_t smem = 16;
  for (int k = t.m0; k < t.m1; ++k) {
    fmax = fmax > t.left[k] * t.right[k] ? fmax : t.left[k] * t.right[k];
    smem += sizeof(double) * 32 * NT * RMAX;
  }
  if (smem > 200 * 1024) return -1;
  auto fn = tail_kernel<RMAX, NT>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return -1;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem) != cudaSuccess ||
      per_sm < 1)
    return -1;
  long long grid = (fmax + 7) / 8;
  // one CTA per SM: short launch ramp, cheap grid barrier (TSG_TAIL_CTAS:
  // a smaller grid that fits next to a capped mode-0 grid)
  static const long long cap_env = [] {
    const char* e = std::getenv("TSG_TAIL_CTAS");
    return e ? std::atoll(e) : 0LL;
  }();
  const long long cap = cap_env > 0 ? cap_env : kNumSMs;
  if (grid > cap) grid = cap;
  if (grid > kMaxGrid) grid = kMaxGrid;
  if (grid < 1) grid = 1;
  TailArgs a = t;
  void* args[] = {&a};
  if (cudaLaunchCooperativeKernel((void*)fn, dim3((unsigned)grid), dim3(256), args, smem, st) !=
      cudaSuccess)
    return -1;
  ++g_launches;
  return (int)grid;
}

}  // namespace

bool tail_eligible(long long n, long long r) { return n >= 1 && n <= 512 && r >= 1 && r <= 32; }

int launch_tail(const TailArgs& t, cudaStream_t st) {
  int rmax = 1, nmax = 1;
  for (int k = t.m0; k < t.m1; ++k) {
    if (!tail_eligible(t.N[k], t.R[k])) return -1;
    rmax = rmax > t.R[k] ? rmax : t.R[k];
    nmax = nmax > (int)t.N[k] ? nmax : (int)t.N[k];
  }
  const int nt = nmax <= 128 ? 4 : nmax <= 256 ? 8 : 16;
#define TSG_TAIL(RM)                                      \
  if (rmax <= RM) {                                       \
    if (nt == 4) return launch_t<RM, 4>(t, st);           \
    if (nt == 8) return launch_t<RM, 8>(t, st);           \
    return launch_t<RM, 16>(t, st);                       \
  }
  TSG_TAIL(4)
  TSG_TAIL(8)
  TSG_TAIL(12)
  TSG_TAIL(16)
  TSG_TAIL(24)
  TSG_TAIL(32)
#undef TSG_TAIL
  return -1;
}

}  // namespace tsg
