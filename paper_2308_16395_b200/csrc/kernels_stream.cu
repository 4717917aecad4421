// Per-slice streaming update kernels (reference proj/src/streaming.cpp and
// proj/src/isvd.cpp): mode-k projection with fused residual norm, the
// branch decision, ledgers, the incremental SVD row insertion and the core
// rotation with the coupling check fused into its epilogue.
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"
#include "proj_dmma.cuh"
#include "proj0_fma.cuh"
#include "proj0_cols.cuh"
#include "decide.cuh"

namespace tsg {

namespace {

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// ------------------------------------------------------------ projection
// Generic fused projection (any mode): tile = BC mode-k fibres staged in
// shared memory together with U; P = U^T X_tile, then E = X - U P and the
// squared norms (streaming.cpp:128-133, tensor.cpp:106-162).
__global__ void __launch_bounds__(256) project_kernel(ProjArgs a) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  const int BC = a.karg0, u_smem = a.karg1;
  const long long left = a.v.left, N = a.v.n, right = a.v.right;
  const int R = a.R;
  const long long cols = left * right;
  const long long ntiles = (cols + BC - 1) / BC;
  double* Us = sm;
  double* Xs = Us + (u_smem ? N * R : 0);
  double* Ps = Xs + N * BC;
  if (u_smem)
    for (long long idx = threadIdx.x; idx < N * R; idx += blockDim.x) {
      const long long i = idx % N, j = idx / N;
      Us[i * R + j] = a.u[idx];
    }
  double racc = 0.0, xacc = 0.0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long c0 = tile * BC;
    __syncthreads();
    for (long long e = threadIdx.x; e < N * BC; e += blockDim.x) {
      long long i, j;
      if (left == 1) {
        j = e / N;
        i = e % N;
      } else {
        j = e % BC;
        i = e / BC;
      }
      const long long c = c0 + j;
      double val = 0.0;
      if (c < cols) {
        const long long l = c % left, r = c / left;
        val = a.x[r * left * N + i * left + l];
      }
      Xs[i * BC + j] = val;
    }
    __syncthreads();
    for (long long o = threadIdx.x; o < (long long)R * BC; o += blockDim.x) {
      const long long c = o % BC, j = o / BC;
      double s = 0.0;
      for (long long i = 0; i < N; ++i) {
        const double uij = u_smem ? Us[i * R + j] : __ldg(&a.u[i + j * N]);
        s += uij * Xs[i * BC + c];
      }
      Ps[j * BC + c] = s;
      const long long cc = c0 + c;
      if (a.p && cc < cols) {
        const long long l = cc % left, r = cc / left;
        a.p[r * left * R + j * left + l] = s;
      }
    }
    __syncthreads();
    if (a.residual) {
      for (long long e = threadIdx.x; e < N * BC; e += blockDim.x) {
        long long i, j;
        if (left == 1) {
          j = e / N;
          i = e % N;
        } else {
          j = e % BC;
          i = e / BC;
        }
        const long long c = c0 + j;
        if (c >= cols) continue;
        const double x = Xs[i * BC + j];
        double s = 0.0;
        for (int jj = 0; jj < R; ++jj) {
          const double uij = u_smem ? Us[i * R + jj] : __ldg(&a.u[i + (long long)jj * N]);
          s += uij * Ps[jj * BC + j];
        }
        const double ev = x - s;
        racc += ev * ev;
        xacc += x * x;
        if (a.e) {
          const long long l = c % left, r = c / left;
          a.e[r * left * N + i * left + l] = ev;
        }
      }
    }
  }
  racc = block_sum(racc, red);
  xacc = block_sum(xacc, red);
  if (threadIdx.x == 0 && a.partial) {
    a.partial[2 * blockIdx.x] = racc;
    a.partial[2 * blockIdx.x + 1] = xacc;
  }
}

// ----------------------------------------------------------- decisions
__global__ void decide_kernel(DecideArgs a) {
  __shared__ double red[32];
  __shared__ double res[kMaxD];
  __shared__ double xsq;
  for (int k = a.first_mode; k < a.nmodes; ++k) {
    double acc = 0.0, acx = 0.0;
    for (int b = threadIdx.x; b < a.cnt[k]; b += blockDim.x) {
      acc += a.partial[a.off[k] + 2 * b];
      acx += a.partial[a.off[k] + 2 * b + 1];
    }
    acc = block_sum(acc, red);
    acx = block_sum(acx, red);
    if (threadIdx.x == 0) {
      res[k] = acc;
      if (k == 0) xsq = acx;
    }
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  decide_finish(a, xsq, res);
}

__global__ void commit_modes_kernel(Ctrl* c, const SliceCtl* s, int m0, int m1, int with_total) {
  if (threadIdx.x != 0) return;
  if (with_total) {
    const double sn = sqrt(s->slice_sq);
    c->total_input_sq += sn * sn;  // streaming.cpp:169
  }
  for (int k = m0; k < m1; ++k) {
    const double rn = sqrt(s->res_sq[k]);
    c->nonstream_discarded_sq += rn * rn;  // streaming.cpp:137
  }
}

__global__ void ledger_add_kernel(Ctrl* c, const double* v) {
  if (threadIdx.x == 0) c->nonstream_discarded_sq += *v;  // streaming.cpp:150
}

__global__ void pad_u_kernel(const double* __restrict__ u, long long N, int R, int rpad,
                             long long rows8, double* __restrict__ out) {
  const long long total = rows8 * rpad;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long row = idx / rpad;
    const int col = (int)(idx % rpad);
    // image column 8rt + 2t + i holds rank 8rt + 4i + t (see proj_dmma.cuh)
    const int rk = (col & ~7) + 4 * (col & 1) + ((col & 7) >> 1);
    out[idx] = (row < N && col < (rpad & ~7) && rk < R) ? u[row + rk * N] : 0.0;
  }
}

// The column-owning mode-0 kernel's two U images (proj0_cols.cuh), stored
// right after the row-split image: image 1 (pitch 8RT+2) holds rank
// 8nt+4i+t in column 8nt+2t+i, image 2 (pitch 8RT+4) natural rank order.
__global__ void cols_u_kernel(const double* __restrict__ u, long long N, int R, int RT, int lo,
                              double* __restrict__ out) {
  const int p1 = 8 * RT + 2, p2 = 8 * RT + 4;
  const long long total = N * (p1 + p2);
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int rk;
    long long row;
    if (idx < N * p1) {
      row = idx / p1;
      const int col = (int)(idx % p1);
      rk = col < 8 * RT ? (col & ~7) + 4 * (col & 1) + ((col & 7) >> 1) : R;
    } else {
      const long long j2 = idx - N * p1;
      row = j2 / p2;
      rk = (int)(j2 % p2);
      if (rk >= 8 * RT + lo) rk = R;  // lo left-over ranks follow the DMMA tiles (cols_lo)
    }
    out[idx] = rk < R ? u[row + rk * N] : 0.0;
  }
}

}  // namespace

long long upad_size(long long N, int R) {
  const long long rows8 = (N + 7) / 8 * 8;
  const int rpad = 8 * ((R + 7) / 8) + 4;
  return rows8 * rpad + rows8 * (16 * ((R + 7) / 8) + 6);
}

long long upad_cols_offset(long long N, int R) {
  return (N + 7) / 8 * 8 * (8 * ((R + 7) / 8) + 4);
}

void launch_pad_u(const double* u, long long N, int R, double* out, cudaStream_t st) {
  const long long rows8 = (N + 7) / 8 * 8;
  const int rpad = 8 * ((R + 7) / 8) + 4;
  pad_u_kernel<<<(int)((rows8 * rpad + 255) / 256), 256, 0, st>>>(u, N, R, rpad, rows8, out);
  ++g_launches;
  if (N % 8 == 0) {
    const int RT = cols0::cols_rt(N, R), lo = cols0::cols_lo(N, R);
    cols_u_kernel<<<(int)((N * (16 * RT + 6) + 255) / 256), 256, 0, st>>>(u, N, R, RT, lo,
                                                                           out + rows8 * rpad);
    ++g_launches;
  }
}

namespace {

inline int grid_for(long long total, int block = 256, int cap = 148 * 8) {
  long long g = (total + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace

int launch_project(const ProjArgs& a, cudaStream_t st) {
  static const bool force_generic = std::getenv("TSG_GENERIC_PROJ") != nullptr;
  static const bool debug = std::getenv("TSG_DEBUG_SYNC") != nullptr;
  if (!force_generic) {
    int grid = a.debug_skip == 0 ? cols0::launch(a, st) : -1;
    if (grid <= 0 && a.debug_skip == 0) grid = fma0::launch(a, st);
    if (grid <= 0) grid = dmma_proj::launch(a, a.stream_in, st);
    if (debug) {
      cudaError_t e = cudaStreamSynchronize(st);
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e != cudaSuccess)
        fprintf(stderr, "proj_dmma failed: %s (left %lld N %lld right %lld R %d grid %d)\n",
                cudaGetErrorString(e), a.v.left, a.v.n, a.v.right, a.R, grid);
    }
    if (grid > 0) {
      ++g_launches;
      return grid;
    }
  }
  const long long N = a.v.n;
  const long long cols = a.v.left * a.v.right;
  const long long budget = 200 * 1024 / 8;  // doubles of shared memory
  int u_smem = (N * a.R <= budget / 2) ? 1 : 0;
  long long rem = budget - (u_smem ? N * a.R : 0);
  long long bc = rem / (N + a.R);
  if (bc > 64) bc = 64;
  if (bc >= 8) bc = bc / 8 * 8;
  if (bc < 1) bc = 1;
  const size_t smem = 8 * ((u_smem ? N * a.R : 0) + N * bc + a.R * bc);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(project_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 205 * 1024);
    attr = true;
  }
  const long long ntiles = (cols + bc - 1) / bc;
  long long grid = ntiles < 148 ? ntiles : 148;
  if (grid < 1) grid = 1;
  ProjArgs b = a;
  b.karg0 = (int)bc;
  b.karg1 = u_smem;
  project_kernel<<<(int)grid, 256, smem, st>>>(b);
  ++g_launches;
  return (int)grid;
}

void launch_decide(const DecideArgs& a, cudaStream_t st) {
  decide_kernel<<<1, 256, 0, st>>>(a);
  ++g_launches;
}

void launch_commit_modes(Ctrl* ctrl, const SliceCtl* slot, int m0, int m1, int with_total,
                         cudaStream_t st) {
  commit_modes_kernel<<<1, 32, 0, st>>>(ctrl, slot, m0, m1, with_total);
  ++g_launches;
}

void launch_ledger_add_nonstream(Ctrl* ctrl, const double* value, cudaStream_t st) {
  ledger_add_kernel<<<1, 32, 0, st>>>(ctrl, value);
  ++g_launches;
}

}  // namespace tsg
