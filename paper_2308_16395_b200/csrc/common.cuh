// Shared device-side definitions for the B200 streaming ST-HOSVD engine.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tsg {

constexpr int kMaxD = 8;
constexpr int kNumSMs = 148;
// Upper bound on the CTAs of any partial-sum-producing kernel (2 per SM).
constexpr int kMaxGrid = 2 * kNumSMs;

// Numeric constants that parity depends on (SURVEY §5 "Config / flags").
constexpr double kCouplingTol = 1e-8;       // streaming.cpp:15
constexpr double kOrthEps = 1e-12;          // isvd.cpp:12
constexpr double kOffDiagTolFactor = 1e-14; // linalg.cpp:13
constexpr int kMaxSweeps = 30;              // linalg.cpp:14
constexpr double kSigmaZeroFactor = 1e-14;  // linalg.cpp:16, sthosvd.cpp:13

// Device-resident control block: ledgers, per-slice scalars and the ISVD
// rank live on the device so the update chain never waits on the host.
struct Ctrl {
  // ledgers (streaming.hpp:42-43, isvd.hpp:78)
  double squared_error;
  double total_input_sq;
  double nonstream_discarded_sq;
  // per-insertion scalars (ISVD stream)
  double proj_sq;       // ||b||^2, b = vec(projected slice)
  double e_sq;          // ||e||^2 after the two projection passes
  double added_error_sq;
  double coupling_diff_sq, core_sq;
  double trunc_margin;
  long long n_d, insertions;
  int r, r_new, degenerate;
  int status;           // 0 ok, 2 coupling drift, 3 numerical
  int sweeps;
  unsigned long long records;  // per-insertion records published so far
};

struct Metrics {  // mirrors tsg_slice_metrics' device-filled part
  long long slice_index;
  long long ranks[kMaxD];
  double slice_norm, projected_norm, error_estimate;
  double mode_residuals[kMaxD];
  int expanded_mask;
  double trunc_margin;
  int sweeps;
};

// Per-slice decision record, written by the projection stream and read by
// the ISVD stream, so consecutive slices can be in flight at once.
struct SliceCtl {
  double slice_sq;      // ||y||^2
  double delta;         // tau ||y|| / sqrt(d)  (streaming.cpp:187-188)
  double res_sq[kMaxD]; // ||E_k||^2 per non-streaming mode
  int expand_mode;      // first mode whose residual exceeds delta, -1 none
  int zero_slice;
  unsigned long long seq;  // host mirror: decisions published for this parity
};

// Host-mapped ring of per-insertion records (metrics + control snapshot),
// filled by the device without a copy call; `done` publishes the count.
constexpr int kRecRing = 64;
struct RecRing {
  Metrics rec[kRecRing];
  Ctrl ctrl[kRecRing];
  unsigned long long done;
};



__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block-wide sum (fixed tree). `scratch` holds >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? scratch[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) scratch[0] = t;
  }
  __syncthreads();
  t = scratch[0];
  __syncthreads();
  return t;
}

}  // namespace tsg
