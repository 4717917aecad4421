#include <cstdlib>
// Dense linear algebra kernels of the B200 streaming ST-HOSVD engine:
// Jacobi eigensolver, truncation rule, Gram (SYRK) kernels, MGS and the
// tensor relayouts used by basis expansion and stream_init.
//
// Reference behaviour followed (paths relative to /root/reference/proj):
//   sym_eig_desc          src/linalg.cpp:120-181 (rotation :27-60)
//   truncation_rank       src/linalg.cpp:183-208
//   gram_from_cols        src/linalg.cpp:80-94
//   gram_transposed       src/linalg.cpp:100-114
//   orthonormalize_columns src/linalg.cpp:64-78
//   orthonormality_defect src/matrix.cpp:118-131
//   unfold / pad / concat src/tensor.cpp:67-84, 168-209
#include <algorithm>
#include <cfloat>

#include "kernels.cuh"

namespace tsg {

long long g_launches = 0;

namespace {

struct Rot {
  double c, s, t;
  int p, q;
};

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// One CTA runs the whole eigensolve: sweeps of (np-1) rounds, each round
// rotating np/2 disjoint pairs at once (round-robin "circle" ordering) so
// every off-diagonal pair is annihilated once per sweep, as in the
// reference's cyclic sweep. Stopping rule, rotation formulas, stable sort,
// clamp and sign rule are the reference's (linalg.cpp:27-60,136-178).
__device__ __forceinline__ int jacobi_sweeps(double* G, double* V, int n,
                                             double tol, Rot* rot,
                                             double* red) {
  const int np = n + (n & 1);
  const int half = np / 2;
  const int rounds = np - 1;
  int sweep = 0;
  for (; sweep < kMaxSweeps; ++sweep) {
    double acc = 0.0;
    for (long long idx = threadIdx.x; idx < (long long)n * n; idx += blockDim.x) {
      const int i = (int)(idx % n), j = (int)(idx / n);
      if (i != j) {
        const double g = G[idx];
        acc += g * g;
      }
    }
    const double off = sqrt(block_sum(acc, red));
    if (off <= tol || n < 2) break;
    for (int rd = 0; rd < rounds; ++rd) {
      for (int m = threadIdx.x; m < half; m += blockDim.x) {
        int a, b;
        if (m == 0) {
          a = rd % (np - 1);
          b = np - 1;
        } else {
          a = (rd + m) % (np - 1);
          b = (rd + np - 1 - m) % (np - 1);
        }
        Rot R;
        R.p = min(a, b);
        R.q = max(a, b);
        R.c = 1.0;
        R.s = 0.0;
        R.t = 0.0;
        if (R.q < n) {
          const double gpq = G[R.p + (long long)R.q * n];
          if (gpq != 0.0) {
            const double gpp = G[R.p + (long long)R.p * n];
            const double gqq = G[R.q + (long long)R.q * n];
            const double theta = (gqq - gpp) / (2.0 * gpq);
            const double t = (theta >= 0.0)
                                 ? 1.0 / (theta + sqrt(1.0 + theta * theta))
                                 : 1.0 / (theta - sqrt(1.0 + theta * theta));
            const double c = 1.0 / sqrt(1.0 + t * t);
            R.c = c;
            R.s = t * c;
            R.t = t;
          }
        }
        rot[m] = R;
      }
      __syncthreads();
      const long long nblk = (long long)half * half;
      for (long long bi = threadIdx.x; bi < nblk; bi += blockDim.x) {
        const int m1 = (int)(bi / half), m2 = (int)(bi % half);
        if (m1 > m2) continue;
        const Rot A = rot[m1];
        const Rot B = rot[m2];
        const bool idA = (A.s == 0.0 && A.t == 0.0);
        const bool idB = (B.s == 0.0 && B.t == 0.0);
        if (idA && idB) continue;
        const int p1 = A.p, q1 = A.q, p2 = B.p, q2 = B.q;
        const bool q1v = q1 < n, q2v = q2 < n;
        if (m1 == m2) {
          // the rotated pair itself (linalg.cpp:50-53)
          const double gpq = G[p1 + (long long)q1 * n];
          const double gpp = G[p1 + (long long)p1 * n];
          const double gqq = G[q1 + (long long)q1 * n];
          G[p1 + (long long)p1 * n] = gpp - A.t * gpq;
          G[q1 + (long long)q1 * n] = gqq + A.t * gpq;
          G[p1 + (long long)q1 * n] = 0.0;
          G[q1 + (long long)p1 * n] = 0.0;
          continue;
        }
        // 2x2 block rows {p1,q1} x cols {p2,q2}: B' = J1^T B J2 (linalg.cpp:40-49)
        const double b00 = G[p1 + (long long)p2 * n];
        const double b01 = q2v ? G[p1 + (long long)q2 * n] : 0.0;
        const double b10 = q1v ? G[q1 + (long long)p2 * n] : 0.0;
        const double b11 = (q1v && q2v) ? G[q1 + (long long)q2 * n] : 0.0;
        const double t00 = A.c * b00 - A.s * b10;
        const double t01 = A.c * b01 - A.s * b11;
        const double t10 = A.s * b00 + A.c * b10;
        const double t11 = A.s * b01 + A.c * b11;
        const double o00 = B.c * t00 - B.s * t01;
        const double o01 = B.s * t00 + B.c * t01;
        const double o10 = B.c * t10 - B.s * t11;
        const double o11 = B.s * t10 + B.c * t11;
        G[p1 + (long long)p2 * n] = o00;
        G[p2 + (long long)p1 * n] = o00;
        if (q2v) {
          G[p1 + (long long)q2 * n] = o01;
          G[q2 + (long long)p1 * n] = o01;
        }
        if (q1v) {
          G[q1 + (long long)p2 * n] = o10;
          G[p2 + (long long)q1 * n] = o10;
        }
        if (q1v && q2v) {
          G[q1 + (long long)q2 * n] = o11;
          G[q2 + (long long)q1 * n] = o11;
        }
      }
      for (long long idx = threadIdx.x; idx < (long long)n * half; idx += blockDim.x) {
        const int i = (int)(idx % n), m = (int)(idx / n);
        const Rot R = rot[m];
        if (R.q >= n || (R.s == 0.0 && R.t == 0.0)) continue;
        const double vp = V[i + (long long)R.p * n], vq = V[i + (long long)R.q * n];
        V[i + (long long)R.p * n] = R.c * vp - R.s * vq;
        V[i + (long long)R.q * n] = R.s * vp + R.c * vq;
      }
      __syncthreads();
    }
  }
  return sweep;
}

// Stable descending sort of diag(G), clamp, copy columns with the sign rule.
__device__ __forceinline__ void jacobi_finish(const double* G, const double* V,
                                              int n, double* evals,
                                              double* evecs, int* perm) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double di = G[i + (long long)i * n];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double dj = G[j + (long long)j * n];
      if (dj > di || (dj == di && j < i)) ++rank;
    }
    perm[rank] = i;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = wid; j < n; j += nw) {
    const int src = perm[j];
    double lambda = G[src + (long long)src * n];
    if (lambda < 0.0) lambda = 0.0;
    if (lane == 0) evals[j] = lambda;
    // argmax |v| with first index on ties
    double best = -1.0;
    int arg = 0x7fffffff;
    for (int i = lane; i < n; i += 32) {
      const double a = fabs(V[i + (long long)src * n]);
      if (a > best) {
        best = a;
        arg = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
      if (ob > best || (ob == best && oa < arg)) {
        best = ob;
        arg = oa;
      }
    }
    const double pivot = V[arg + (long long)src * n];
    const bool flip = pivot < 0.0;
    for (int i = lane; i < n; i += 32) {
      const double v = V[i + (long long)src * n];
      evecs[i + (long long)j * n] = flip ? -v : v;
    }
  }
}

__global__ void __launch_bounds__(1024) sym_eig_kernel(const double* __restrict__ gin, int n,
                                                       double* evals, double* evecs,
                                                       double* work, int* sweeps_out) {
  extern __shared__ unsigned char smem_raw[];
  Rot* rot = reinterpret_cast<Rot*>(smem_raw);
  int* perm = reinterpret_cast<int*>(rot + (n + 2) / 2);
  __shared__ double red[32];
  double* G = work;
  double* V = work + (long long)n * n;
  double acc = 0.0;
  for (long long idx = threadIdx.x; idx < (long long)n * n; idx += blockDim.x) {
    const double g = gin[idx];
    G[idx] = g;
    V[idx] = ((idx % n) == (idx / n)) ? 1.0 : 0.0;
    acc += g * g;
  }
  const double tol = kOffDiagTolFactor * sqrt(block_sum(acc, red));
  const int sw = jacobi_sweeps(G, V, n, tol, rot, red);
  __syncthreads();
  jacobi_finish(G, V, n, evals, evecs, perm);
  if (threadIdx.x == 0 && sweeps_out) *sweeps_out = sw;
}

__global__ void truncate_kernel(double* ev, int n, double delta, int zero_floor,
                                long long* out_rank, double* out_disc) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (n == 0) {
    *out_rank = 0;
    *out_disc = 0.0;
    return;
  }
  if (zero_floor) {  // sthosvd.cpp:68-71, linalg.cpp:230-234
    const double smax = sqrt(ev[0]);
    const double fl = kSigmaZeroFactor * smax;
    for (int i = 0; i < n; ++i)
      if (sqrt(ev[i]) <= fl) ev[i] = 0.0;
  }
  const double budget = delta * delta;
  // trailing[r] = trailing[r+1] + ev[r], accumulated from the tail; the
  // admissible r form a suffix, so walk down while the budget holds.
  double s = 0.0;
  int r = n;

  for (int i = n - 1; i >= 0; --i) {
    const double next = s + ev[i];
    if (next <= budget) {
      s = next;
      r = i;

    } else {
      break;
    }
  }
  const int rank = r < 1 ? 1 : r;
  double disc = 0.0;
  for (int j = n - 1; j >= rank; --j) disc += ev[j];

  *out_rank = rank;
  *out_disc = disc;
}

// ---- Gram (SYRK) over a column-major rows x cols matrix, split over cols.
constexpr int GT = 64;  // tile
constexpr int GK = 16;  // k chunk

__global__ void __launch_bounds__(256) gram_partial_kernel(const double* __restrict__ a, int rows,
                                                           long long cols, long long chunk,
                                                           double* __restrict__ partial) {
  const int nt = (rows + GT - 1) / GT;
  // upper-triangular tile index -> (ti, tj), ti <= tj
  int t = blockIdx.x, ti = 0;
  while (t >= nt - ti) {
    t -= nt - ti;
    ++ti;
  }
  const int tj = ti + t;
  const long long c0 = (long long)blockIdx.y * chunk;
  const long long c1 = min(cols, c0 + chunk);
  __shared__ double As[GK][GT + 1];
  __shared__ double Bs[GK][GT + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int i0 = ti * GT, j0 = tj * GT;
  double acc[4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
  for (long long cc = c0; cc < c1; cc += GK) {
    for (int e = threadIdx.x; e < GT * GK; e += 256) {
      const int ii = e % GT, kk = e / GT;
      const long long c = cc + kk;
      const int i = i0 + ii, j = j0 + ii;
      As[kk][ii] = (i < rows && c < c1) ? a[i + c * rows] : 0.0;
      Bs[kk][ii] = (j < rows && c < c1) ? a[j + c * rows] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GK; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) av[x] = As[kk][ty + 16 * x];
#pragma unroll
      for (int y = 0; y < 4; ++y) bv[y] = Bs[kk][tx + 16 * y];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] += av[x] * bv[y];
    }
    __syncthreads();
  }
  double* out = partial + (long long)blockIdx.y * rows * rows;
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int i = i0 + ty + 16 * x, j = j0 + tx + 16 * y;
      if (i < rows && j < rows) out[i + (long long)j * rows] = acc[x][y];
    }
}

// Same partial Gram on the FP64 tensor cores: mma.sync m8n8k4 f64, a 64x64
// tile per CTA of four warps, warp (wr, wc) owns the 32x32 quarter
// (4 x 4 accumulator tiles: 16 DMMA per 8 fragment loads). K chunks of DK
// columns are staged in shared memory (pitch 72 doubles: the fragment reads
// of one warp hit every bank pair twice, the minimum for 32 x 8 bytes) and the
// next chunk is held in registers while the current one is consumed. Rows /
// columns past the end are zero.
constexpr int DK = 32;
constexpr int DPITCH = GT + 8;
constexpr int DTHREADS = 128;

__device__ __forceinline__ void gram_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(DTHREADS) gram_partial_dmma_kernel(const double* __restrict__ a,
                                                                     int rows, long long cols,
                                                                     long long chunk,
                                                                     double* __restrict__ partial) {
  const int nt = (rows + GT - 1) / GT;
  int t = blockIdx.x, ti = 0;
  while (t >= nt - ti) {
    t -= nt - ti;
    ++ti;
  }
  const int tj = ti + t;
  const long long c0 = (long long)blockIdx.y * chunk;
  const long long c1 = min(cols, c0 + chunk);
  __shared__ __align__(16) double As[DK][DPITCH];
  __shared__ __align__(16) double Bs[DK][DPITCH];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int wr = warp & 1, wc = warp >> 1;
  const int i0 = ti * GT, j0 = tj * GT;
  // staging: thread -> row ii = tid % 64, columns kk = kb + 2 e (e < DK / 2)
  constexpr int KS = DTHREADS / GT, NE = DK / KS;
  const int ii = threadIdx.x % GT, kb = threadIdx.x / GT;
  const bool iv = i0 + ii < rows, jv = j0 + ii < rows;
  const int ic = iv ? i0 + ii : rows - 1, jc = jv ? j0 + ii : rows - 1;
  double ra[NE], rb[NE];
  auto fetch = [&](long long cc) {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const long long c = cc + kb + KS * e;
      const bool cv = c < c1;
      const long long cl = cv ? c : c1 - 1;
      const double va = __ldg(a + ic + cl * rows);
      const double vb = __ldg(a + jc + cl * rows);
      ra[e] = (cv && iv) ? va : 0.0;
      rb[e] = (cv && jv) ? vb : 0.0;
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  if (c0 < c1) fetch(c0);
  for (long long cc = c0; cc < c1; cc += DK) {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      As[kb + KS * e][ii] = ra[e];
      Bs[kb + KS * e][ii] = rb[e];
    }
    __syncthreads();
    if (cc + DK < c1) fetch(cc + DK);
#pragma unroll
    for (int ks = 0; ks < DK / 4; ++ks) {
      const int k = 4 * ks + tq;
      double af[4], bf[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) af[x] = As[k][32 * wr + 8 * x + g];
#pragma unroll
      for (int y = 0; y < 4; ++y) bf[y] = Bs[k][32 * wc + 8 * y + g];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) gram_dmma(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
    }
    __syncthreads();
  }
  double* out = partial + (long long)blockIdx.y * rows * rows;
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = i0 + 32 * wr + 8 * x + g, j = j0 + 32 * wc + 8 * y + 2 * tq + h;
        if (i < rows && j < rows) out[i + (long long)j * rows] = acc[x][y][h];
      }
}

// Narrow modes (rows <= 8 TX <= 32): one diagonal tile of 8 TX rows holds the
// whole Gram, so each of the four warps computes all TX x TX MMA tiles over
// its share of the K steps (warp w: steps w, w + 4, ...; no per-MMA guards,
// rows past the end are zero in shared memory) and the four partial tiles
// are summed in warp order at the end.
constexpr int NK = 64;       // columns per staged chunk
constexpr int NPITCH = 40;   // 40 mod 16 = 8: conflict-free fragment reads
template <int TX>
__global__ void __launch_bounds__(128) gram_partial_narrow_kernel(const double* __restrict__ a,
                                                                  int rows, long long cols,
                                                                  long long chunk,
                                                                  double* __restrict__ partial) {
  constexpr int RT = 8 * TX;
  const long long c0 = (long long)blockIdx.y * chunk;
  const long long c1 = min(cols, c0 + chunk);
  constexpr int SMD = (NK * NPITCH > 3 * 32 * TX * TX * 2) ? NK * NPITCH : 3 * 32 * TX * TX * 2;
  __shared__ __align__(16) double sm[SMD];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  // staging: thread -> row ii = tid % RT, columns kb + (128 / RT) e
  constexpr int KS = 128 / RT, NE = NK / KS;
  const int ii = threadIdx.x % RT, kb = threadIdx.x / RT;
  const bool iv = ii < rows;
  const int ic = iv ? ii : rows - 1;
  double ra[NE];
  auto fetch = [&](long long cc) {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const long long c = cc + kb + KS * e;
      const bool cv = c < c1;
      const long long cl = cv ? c : c1 - 1;
      const double v = __ldg(a + ic + cl * rows);
      ra[e] = (cv && iv) ? v : 0.0;
    }
  };
  double acc[TX][TX][2];
#pragma unroll
  for (int x = 0; x < TX; ++x)
#pragma unroll
    for (int y = 0; y < TX; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  if (c0 < c1) fetch(c0);
  for (long long cc = c0; cc < c1; cc += NK) {
#pragma unroll
    for (int e = 0; e < NE; ++e) sm[(kb + KS * e) * NPITCH + ii] = ra[e];
    __syncthreads();
    if (cc + NK < c1) fetch(cc + NK);
#pragma unroll
    for (int s4 = 0; s4 < NK / 16; ++s4) {
      const int k = 4 * (4 * s4 + warp) + tq;
      double f[TX];
#pragma unroll
      for (int x = 0; x < TX; ++x) f[x] = sm[k * NPITCH + 8 * x + g];
#pragma unroll
      for (int x = 0; x < TX; ++x)
#pragma unroll
        for (int y = 0; y < TX; ++y) gram_dmma(acc[x][y][0], acc[x][y][1], f[x], f[y]);
    }
    __syncthreads();
  }
  constexpr int PER = TX * TX * 2;
  if (warp > 0) {
#pragma unroll
    for (int x = 0; x < TX; ++x)
#pragma unroll
      for (int y = 0; y < TX; ++y)
#pragma unroll
        for (int h = 0; h < 2; ++h) sm[((warp - 1) * PER + (x * TX + y) * 2 + h) * 32 + lane] = acc[x][y][h];
  }
  __syncthreads();
  if (warp != 0) return;
#pragma unroll
  for (int w = 0; w < 3; ++w)
#pragma unroll
    for (int x = 0; x < TX; ++x)
#pragma unroll
      for (int y = 0; y < TX; ++y)
#pragma unroll
        for (int h = 0; h < 2; ++h) acc[x][y][h] += sm[(w * PER + (x * TX + y) * 2 + h) * 32 + lane];
  double* out = partial + (long long)blockIdx.y * rows * rows;
#pragma unroll
  for (int x = 0; x < TX; ++x)
#pragma unroll
    for (int y = 0; y < TX; ++y)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = 8 * x + g, j = 8 * y + 2 * tq + h;
        if (i < rows && j < rows) out[i + (long long)j * rows] = acc[x][y][h];
      }
}

__global__ void gram_reduce_kernel(const double* __restrict__ partial, int rows, int splits,
                                   double* __restrict__ g) {
  const long long total = (long long)rows * rows;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int i = (int)(idx % rows), j = (int)(idx / rows);
    if (i > j) {
      const int t = i;
      i = j;
      j = t;
    }
    double s = 0.0;
    for (int sp = 0; sp < splits; ++sp) s += partial[(long long)sp * total + i + (long long)j * rows];
    g[idx] = s;
  }
}

// Small Grams with many K splits: one warp per element of the full square
// (each sums its upper-triangle mirror, so G is symmetric bit for bit), lanes
// take the splits strided by 32, then a fixed butterfly (deterministic order).
__global__ void gram_reduce_warp_kernel(const double* __restrict__ partial, int rows, int splits,
                                        double* __restrict__ g) {
  const long long total = (long long)rows * rows;
  const int lane = threadIdx.x & 31;
  for (long long idx = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; idx < total;
       idx += ((long long)gridDim.x * blockDim.x) >> 5) {
    int i = (int)(idx % rows), j = (int)(idx / rows);
    if (i > j) {
      const int t = i;
      i = j;
      j = t;
    }
    double s = 0.0;
    for (int sp = lane; sp < splits; sp += 32) s += partial[(long long)sp * total + i + (long long)j * rows];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) g[idx] = s;
  }
}

__global__ void gram_t_kernel(const double* __restrict__ a, long long rows, int cols,
                              double* __restrict__ g) {
  const long long total = (long long)cols * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx % cols), j = (int)(idx / cols);
    if (i > j) continue;
    const double* ai = a + (long long)i * rows;
    const double* aj = a + (long long)j * rows;
    double dot = 0.0;
    for (long long l = 0; l < rows; ++l) dot += ai[l] * aj[l];
    g[i + (long long)j * cols] = dot;
    g[j + (long long)i * cols] = dot;
  }
}

__global__ void gemm_nn_kernel(const double* __restrict__ a, long long lda,
                               const double* __restrict__ b, long long ldb, double* __restrict__ c,
                               long long ldc, long long m, int n, int k) {
  const long long total = m * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx % m;
    const int j = (int)(idx / m);
    double s = 0.0;
    for (int l = 0; l < k; ++l) {
      const double blj = b[l + j * ldb];
      if (blj == 0.0) continue;  // matrix.cpp:44-52 skips zero multipliers
      s += a[i + l * lda] * blj;
    }
    c[i + j * ldc] = s;
  }
}

__global__ void scale_cols_invsqrt_kernel(double* a, long long lda, long long m, int n,
                                          const double* __restrict__ ev) {
  const long long total = m * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx % m;
    const int j = (int)(idx / m);
    const double inv = 1.0 / sqrt(ev[j]);
    a[i + j * lda] *= inv;
  }
}

__global__ void __launch_bounds__(1024) mgs_kernel(double* a, long long lda, long long m, int n) {
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = 0; i < n; ++i) {
    double* ai = a + (long long)i * lda;
    double acc = 0.0;
    for (long long l = threadIdx.x; l < m; l += blockDim.x) acc += ai[l] * ai[l];
    const double norm = sqrt(block_sum(acc, red));
    if (norm > 0.0)
      for (long long l = threadIdx.x; l < m; l += blockDim.x) ai[l] /= norm;
    __syncthreads();
    for (int j = i + 1 + wid; j < n; j += nw) {
      double* aj = a + (long long)j * lda;
      double dot = 0.0;
      for (long long l = lane; l < m; l += 32) dot += ai[l] * aj[l];
      dot = warp_sum(dot);
      for (long long l = lane; l < m; l += 32) aj[l] -= dot * ai[l];
    }
    __syncthreads();
  }
}

__global__ void orth_defect_kernel(const double* __restrict__ a, long long lda, long long m,
                                   int n, double* out) {
  __shared__ double red[32];
  double worst = 0.0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int pidx = wid; pidx < n * n; pidx += nw) {
    const int i = pidx % n, j = pidx / n;
    if (i > j) continue;
    double dot = 0.0;
    for (long long l = lane; l < m; l += 32) dot += a[l + i * lda] * a[l + j * lda];
    dot = warp_sum(dot);
    const double d = fabs(dot - (i == j ? 1.0 : 0.0));
    if (d > worst) worst = d;
  }
  // block max
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
  if (lane == 0) red[wid] = worst;
  __syncthreads();
  if (threadIdx.x == 0) {
    double w = 0.0;
    for (int i = 0; i < nw; ++i) w = fmax(w, red[i]);
    *out = w;
  }
}

__global__ void unfold_kernel(const double* __restrict__ t, ModeView v, double* __restrict__ a) {
  const long long total = v.left * v.n * v.right;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    // source-order traversal: idx = l + i left + r left n
    const long long l = idx % v.left;
    const long long i = (idx / v.left) % v.n;
    const long long r = idx / (v.left * v.n);
    a[i + (l + r * v.left) * v.n] = t[idx];
  }
}

__global__ void pad_kernel(const double* __restrict__ t, ModeView v, long long extra,
                           double* __restrict__ out) {
  const long long nn = v.n + extra;
  const long long total = v.left * nn * v.right;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long l = idx % v.left;
    const long long i = (idx / v.left) % nn;
    const long long r = idx / (v.left * nn);
    out[idx] = (i < v.n) ? t[l + i * v.left + r * v.left * v.n] : 0.0;
  }
}

__global__ void concat_kernel(const double* __restrict__ a, const double* __restrict__ b,
                              long long left, long long na, long long nb, long long right,
                              double* __restrict__ out) {
  const long long nn = na + nb;
  const long long total = left * nn * right;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long l = idx % left;
    const long long i = (idx / left) % nn;
    const long long r = idx / (left * nn);
    out[idx] = (i < na) ? a[l + i * left + r * left * na] : b[l + (i - na) * left + r * left * nb];
  }
}

__global__ void sumsq_partial_kernel(const double* __restrict__ x, long long n,
                                     double* __restrict__ partial) {
  __shared__ double red[32];
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    acc += x[i] * x[i];
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

__global__ void sum_kernel(const double* __restrict__ partial, int n, double* out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partial[i];
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) *out = acc;
}

inline int grid_for(long long total, int block = 256, int cap = 148 * 16) {
  long long g = (total + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace

bool launch_sym_eig_coop(const double* g, int n, double* evals, double* evecs, double* work,
                         double* part, int* sweeps_out, cudaStream_t st);

void launch_sym_eig(const double* g, int n, double* evals, double* evecs, double* work,
                    int* sweeps_out, cudaStream_t st) {
  if (n <= 0) return;
  // work holds 3 n^2 doubles plus room for per-CTA partials (see engine)
  if (launch_sym_eig_coop(g, n, evals, evecs, work, work + 3LL * n * n, sweeps_out, st)) return;
  const size_t smem = sizeof(Rot) * ((n + 2) / 2) + sizeof(int) * (n + 1);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sym_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    attr = true;
  }
  sym_eig_kernel<<<1, 1024, smem, st>>>(g, n, evals, evecs, work, sweeps_out);
  ++g_launches;
}

void launch_truncate(double* evals, int n, double delta, int zero_floor, long long* out_rank,
                     double* out_disc, cudaStream_t st) {
  truncate_kernel<<<1, 32, 0, st>>>(evals, n, delta, zero_floor, out_rank, out_disc);
  ++g_launches;
}

int gram_splits(int rows, long long cols) {
  const int nt = (rows + GT - 1) / GT;
  const int tiles = nt * (nt + 1) / 2;
  static const long long waves = [] {  // TSG_GRAM_WAVES: CTAs per SM targeted
    const char* e = std::getenv("TSG_GRAM_WAVES");
    const long long w = e ? std::atoll(e) : 8LL;
    return w < 1 ? 1LL : (w > 64 ? 64LL : w);
  }();
  long long s = (waves * kNumSMs + tiles - 1) / tiles;
  const long long max_by_cols = (cols + 4 * GK - 1) / (4 * GK);
  if (s > max_by_cols) s = max_by_cols;
  // narrow modes need many CTAs to keep enough bytes in flight; the partial
  // buffer (splits x rows^2) stays <= 32 Mi doubles
  long long cap = (1LL << 25) / ((long long)rows * rows);
  if (cap < 1) cap = 1;
  if (cap > 4096) cap = 4096;
  if (s > cap) s = cap;
  if (s < 1) s = 1;
  return (int)s;
}

void launch_gram(const double* a, int rows, long long cols, double* g, double* partial,
                 cudaStream_t st) {
  const int nt = (rows + GT - 1) / GT;
  const int tiles = nt * (nt + 1) / 2;
  const int splits = gram_splits(rows, cols);
  long long chunk = (cols + splits - 1) / splits;
  chunk = (chunk + GK - 1) / GK * GK;
  static const bool ffma = [] {  // TSG_GRAM_FFMA=1: the CUDA-core SYRK (A/B)
    const char* e = std::getenv("TSG_GRAM_FFMA");
    return e && std::atoi(e) != 0;
  }();
  if (ffma)
    gram_partial_kernel<<<dim3(tiles, splits), 256, 0, st>>>(a, rows, cols, chunk, partial);
  else if (rows <= 16)
    gram_partial_narrow_kernel<2><<<dim3(1, splits), 128, 0, st>>>(a, rows, cols, chunk, partial);
  else if (rows <= 32)
    gram_partial_narrow_kernel<4><<<dim3(1, splits), 128, 0, st>>>(a, rows, cols, chunk, partial);
  else
    gram_partial_dmma_kernel<<<dim3(tiles, splits), DTHREADS, 0, st>>>(a, rows, cols, chunk, partial);
  if ((long long)rows * rows <= 64LL * 64 && splits >= 64)
    gram_reduce_warp_kernel<<<(int)std::min<long long>(((long long)rows * rows + 7) / 8, 8LL * kNumSMs),
                              256, 0, st>>>(partial, rows, splits, g);
  else
    gram_reduce_kernel<<<grid_for((long long)rows * rows), 256, 0, st>>>(partial, rows, splits, g);
  g_launches += 2;
}

void launch_gram_t(const double* a, long long rows, int cols, double* g, cudaStream_t st) {
  gram_t_kernel<<<grid_for((long long)cols * cols), 256, 0, st>>>(a, rows, cols, g);
  ++g_launches;
}

void launch_gemm_nn(const double* a, long long lda, const double* b, long long ldb, double* c,
                    long long ldc, long long m, int n, int k, cudaStream_t st) {
  if (m * n == 0) return;
  gemm_nn_kernel<<<grid_for(m * n), 256, 0, st>>>(a, lda, b, ldb, c, ldc, m, n, k);
  ++g_launches;
}

void launch_scale_cols_invsqrt(double* a, long long lda, long long m, int n, const double* evals,
                               cudaStream_t st) {
  if (m * n == 0) return;
  scale_cols_invsqrt_kernel<<<grid_for(m * n), 256, 0, st>>>(a, lda, m, n, evals);
  ++g_launches;
}

void launch_mgs(double* a, long long lda, long long m, int n, cudaStream_t st) {
  if (n == 0) return;
  mgs_kernel<<<1, 1024, 0, st>>>(a, lda, m, n);
  ++g_launches;
}

void launch_orth_defect(const double* a, long long lda, long long m, int n, double* out,
                        cudaStream_t st) {
  orth_defect_kernel<<<1, 1024, 0, st>>>(a, lda, m, n, out);
  ++g_launches;
}

void launch_unfold(const double* t, ModeView v, double* a, cudaStream_t st) {
  unfold_kernel<<<grid_for(v.left * v.n * v.right), 256, 0, st>>>(t, v, a);
  ++g_launches;
}

void launch_pad(const double* t, ModeView v, long long extra, double* out, cudaStream_t st) {
  pad_kernel<<<grid_for(v.left * (v.n + extra) * v.right), 256, 0, st>>>(t, v, extra, out);
  ++g_launches;
}

void launch_concat(const double* a, const double* b, long long left, long long na, long long nb,
                   long long right, double* out, cudaStream_t st) {
  concat_kernel<<<grid_for(left * (na + nb) * right), 256, 0, st>>>(a, b, left, na, nb, right,
                                                                    out);
  ++g_launches;
}

void launch_sumsq(const double* x, long long n, double* out, double* scratch, cudaStream_t st) {
  const int g = grid_for(n, 256, 1024);
  sumsq_partial_kernel<<<g, 256, 0, st>>>(x, n, scratch);
  sum_kernel<<<1, 1024, 0, st>>>(scratch, g, out);
  g_launches += 2;
}

}  // namespace tsg

// ---------------------------------------------------------------------------
// Cooperative multi-CTA Jacobi for large symmetric matrices (basis growth and
// stream_init Gram matrices, n up to a few hundred). Same ordering, formulas,
// stopping rule and finishing steps as the single-CTA solver; every CTA
// recomputes the round's rotations from the (grid-synchronised) matrix and
// applies its share of the 2x2 block and V updates, with one grid barrier
// per round.
#include <cooperative_groups.h>

namespace tsg {
namespace {

namespace cg = cooperative_groups;

struct RotC {
  double c, s, t;
  int p, q;
};

__global__ void __launch_bounds__(256) sym_eig_coop_kernel(const double* __restrict__ gin, int n,
                                                           double* evals, double* evecs,
                                                           double* work, double* part,
                                                           int* sweeps_out) {
  // G is double-buffered (work holds G0, V, G1): a round reads G_cur and
  // writes every entry of G_nxt, so one grid barrier per round suffices
  cg::grid_group grid = cg::this_grid();
  extern __shared__ unsigned char smem_raw[];
  RotC* rot = reinterpret_cast<RotC*>(smem_raw);
  __shared__ double red[32];
  double* G = work;
  double* V = work + (long long)n * n;
  double* Gn = work + 2LL * n * n;
  const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long gstride = (long long)gridDim.x * blockDim.x;
  const long long nn = (long long)n * n;
  double acc = 0.0;
  for (long long idx = gtid; idx < nn; idx += gstride) {
    const double g = gin[idx];
    G[idx] = g;
    V[idx] = ((idx % n) == (idx / n)) ? 1.0 : 0.0;
    acc += g * g;
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
  grid.sync();
  double tot = 0.0;
  for (int b = 0; b < (int)gridDim.x; ++b) tot += part[b];
  const double tol = kOffDiagTolFactor * sqrt(tot);
  const int np = n + (n & 1), half = np / 2;
  int sweep = 0;
  for (; sweep < kMaxSweeps; ++sweep) {
    double o2 = 0.0;
    for (long long idx = gtid; idx < nn; idx += gstride) {
      const int i = (int)(idx % n), j = (int)(idx / n);
      if (i != j) o2 += G[idx] * G[idx];
    }
    o2 = block_sum(o2, red);
    grid.sync();  // everyone has read the previous sweep's partials
    if (threadIdx.x == 0) part[blockIdx.x] = o2;
    grid.sync();
    double off = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) off += part[b];
    off = sqrt(off);
    if (off <= tol || n < 2) break;
    for (int rd = 0; rd < np - 1; ++rd) {
      for (int m = threadIdx.x; m < half; m += blockDim.x) {
        int a, b;
        if (m == 0) {
          a = rd % (np - 1);
          b = np - 1;
        } else {
          a = (rd + m) % (np - 1);
          b = (rd + np - 1 - m) % (np - 1);
        }
        RotC R;
        R.p = min(a, b);
        R.q = max(a, b);
        R.c = 1.0;
        R.s = 0.0;
        R.t = 0.0;
        if (R.q < n) {
          const double gpq = G[R.p + (long long)R.q * n];
          if (gpq != 0.0) {
            const double gpp = G[R.p + (long long)R.p * n];
            const double gqq = G[R.q + (long long)R.q * n];
            const double theta = (gqq - gpp) / (2.0 * gpq);
            const double t = (theta >= 0.0) ? 1.0 / (theta + sqrt(1.0 + theta * theta))
                                            : 1.0 / (theta - sqrt(1.0 + theta * theta));
            const double c = 1.0 / sqrt(1.0 + t * t);
            R.c = c;
            R.s = t * c;
            R.t = t;
          }
        }
        rot[m] = R;
      }
      __syncthreads();  // this CTA's copy of the round's rotations
      const long long nblk = (long long)half * half;
      for (long long bi = gtid; bi < nblk; bi += gstride) {
        const int m1 = (int)(bi / half), m2 = (int)(bi % half);
        if (m1 > m2) continue;
        const RotC A = rot[m1], B = rot[m2];
        const int p1 = A.p, q1 = A.q, p2 = B.p, q2 = B.q;
        const bool q1v = q1 < n, q2v = q2 < n;
        if (m1 == m2) {
          const double gpq = q1v ? G[p1 + (long long)q1 * n] : 0.0;
          const double gpp = G[p1 + (long long)p1 * n];
          const double gqq = q1v ? G[q1 + (long long)q1 * n] : 0.0;
          const bool idA = (A.s == 0.0 && A.t == 0.0);
          Gn[p1 + (long long)p1 * n] = idA ? gpp : gpp - A.t * gpq;
          if (q1v) {
            Gn[q1 + (long long)q1 * n] = idA ? gqq : gqq + A.t * gpq;
            Gn[p1 + (long long)q1 * n] = idA ? gpq : 0.0;
            Gn[q1 + (long long)p1 * n] = idA ? gpq : 0.0;
          }
          continue;
        }
        const double b00 = G[p1 + (long long)p2 * n];
        const double b01 = q2v ? G[p1 + (long long)q2 * n] : 0.0;
        const double b10 = q1v ? G[q1 + (long long)p2 * n] : 0.0;
        const double b11 = (q1v && q2v) ? G[q1 + (long long)q2 * n] : 0.0;
        // identity rotations (gpq == 0) have c = 1, s = 0: the same formulas
        // copy the block through
        const double t00 = A.c * b00 - A.s * b10, t01 = A.c * b01 - A.s * b11;
        const double t10 = A.s * b00 + A.c * b10, t11 = A.s * b01 + A.c * b11;
        const double o00 = B.c * t00 - B.s * t01, o01 = B.s * t00 + B.c * t01;
        const double o10 = B.c * t10 - B.s * t11, o11 = B.s * t10 + B.c * t11;
        Gn[p1 + (long long)p2 * n] = o00;
        Gn[p2 + (long long)p1 * n] = o00;
        if (q2v) {
          Gn[p1 + (long long)q2 * n] = o01;
          Gn[q2 + (long long)p1 * n] = o01;
        }
        if (q1v) {
          Gn[q1 + (long long)p2 * n] = o10;
          Gn[p2 + (long long)q1 * n] = o10;
        }
        if (q1v && q2v) {
          Gn[q1 + (long long)q2 * n] = o11;
          Gn[q2 + (long long)q1 * n] = o11;
        }
      }
      for (long long idx = gtid; idx < (long long)n * half; idx += gstride) {
        const int i = (int)(idx % n), m = (int)(idx / n);
        const RotC R = rot[m];
        if (R.q >= n || (R.s == 0.0 && R.t == 0.0)) continue;
        const double vp = V[i + (long long)R.p * n], vq = V[i + (long long)R.q * n];
        V[i + (long long)R.p * n] = R.c * vp - R.s * vq;
        V[i + (long long)R.q * n] = R.s * vp + R.c * vq;
      }
      grid.sync();
      double* tmp = G;
      G = Gn;
      Gn = tmp;
      __syncthreads();  // rot[] is rewritten next round
    }
  }
  if (blockIdx.x != 0) return;
  // finish (stable sort, clamp, sign rule) in CTA 0
  int* perm = reinterpret_cast<int*>(rot);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double di = G[i + (long long)i * n];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double dj = G[j + (long long)j * n];
      if (dj > di || (dj == di && j < i)) ++rank;
    }
    perm[rank] = i;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = wid; j < n; j += nw) {
    const int src = perm[j];
    double lambda = G[src + (long long)src * n];
    if (lambda < 0.0) lambda = 0.0;
    if (lane == 0) evals[j] = lambda;
    double best = -1.0;
    int arg = 0x7fffffff;
    for (int i = lane; i < n; i += 32) {
      const double a = fabs(V[i + (long long)src * n]);
      if (a > best) {
        best = a;
        arg = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
      if (ob > best || (ob == best && oa < arg)) {
        best = ob;
        arg = oa;
      }
    }
    const bool flip = V[arg + (long long)src * n] < 0.0;
    for (int i = lane; i < n; i += 32) {
      const double v = V[i + (long long)src * n];
      evecs[i + (long long)j * n] = flip ? -v : v;
    }
  }
  if (threadIdx.x == 0 && sweeps_out) *sweeps_out = sweep;
}

}  // namespace

// Large n: cooperative grid (one CTA per SM at most); small n: one CTA.
bool launch_sym_eig_coop(const double* g, int n, double* evals, double* evecs, double* work,
                         double* part, int* sweeps_out, cudaStream_t st) {
  static const int min_n = [] {  // below: the single-CTA solver (TSG_COOP_EIG_MIN)
    const char* e = std::getenv("TSG_COOP_EIG_MIN");
    return e ? std::atoi(e) : 96;
  }();
  if (n < min_n) return false;
  int dev = 0, coop = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return false;
  const size_t smem = std::max(sizeof(RotC) * ((n + 2) / 2), sizeof(int) * (n + 1));
  cudaFuncSetAttribute(sym_eig_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sym_eig_coop_kernel, 256, smem);
  int sms = kNumSMs;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long want = ((long long)n * n / 4 + 255) / 256;
  int grid = (int)std::min<long long>(std::max<long long>(want, 1), (long long)sms * std::max(per_sm, 1));
  grid = std::min(grid, 256);
  void* args[] = {(void*)&g, (void*)&n, (void*)&evals, (void*)&evecs, (void*)&work, (void*)&part,
                  (void*)&sweeps_out};
  if (cudaLaunchCooperativeKernel((void*)sym_eig_coop_kernel, grid, 256, args, smem, st) !=
      cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  ++g_launches;
  return true;
}

}  // namespace tsg
