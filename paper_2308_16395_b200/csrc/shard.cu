// Kernels of the sharded streaming update.
//
// Rank g of G holds rows [lo_g, hi_g) of one spatial mode s of every slice
// (a dense sub-tensor; a contiguous chunk of the colexicographic slice when
// s is the last spatial mode). Modes 0..s-1 are projected locally; the one per-slice exchange is
// an allgather of [partial norm pairs | compressed local tensor] (the input
// of mode s restricted to the rank's rows). Every rank then assembles the
// identical full compressed tensor and partial pairs from the identical
// gathered bytes, so every decision and every state update is bitwise the
// same on all ranks (reductions run in rank order, never in arrival order).
#include "kernels.cuh"

namespace tsg {

namespace {

// pairs[k] = sum over the partial pairs of mode k (fixed order, one CTA).
__global__ void shard_pack_pairs_kernel(ShardPairs p, double* out) {
  __shared__ double red[32];
  for (int k = 0; k < p.nmodes; ++k) {
    double acc = 0.0, acx = 0.0;
    for (int b = threadIdx.x; b < p.cnt[k]; b += blockDim.x) {
      acc += p.partial[p.off[k] + 2 * b];
      acx += p.partial[p.off[k] + 2 * b + 1];
    }
    acc = block_sum(acc, red);
    acx = block_sum(acx, red);
    if (threadIdx.x == 0) {
      out[2 * k] = acc;
      out[2 * k + 1] = acx;
    }
  }
}

// Concatenate the ranks' parts along the shard mode and regroup the partial
// pairs per mode: pairs_out[k * 2G + 2g + j] = recv[g * count + 2k + j].
__global__ void shard_unpack_kernel(ShardLayout L, const double* __restrict__ recv,
                                    double* __restrict__ z, double* __restrict__ pairs_out) {
  const int g = blockIdx.y;
  const double* src = recv + (long long)g * L.count;
  if (pairs_out && blockIdx.x == 0)
    for (int i = threadIdx.x; i < L.header; i += blockDim.x) {
      const int k = i >> 1, j = i & 1;
      pairs_out[(long long)k * 2 * L.world + 2 * g + j] = src[i];
    }
  const long long chunk = L.inner * L.nloc[g];  // contiguous run per outer index
  const long long n = chunk * L.outer;
  double* dst = z + L.inner * L.lo[g];
  const long long pitch = L.inner * L.ns;
  src += L.header;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long o = i / chunk;
    dst[(i - o * chunk) + o * pitch] = src[i];
  }
}

}  // namespace

void launch_shard_pack_pairs(const ShardPairs& p, double* out, cudaStream_t st) {
  shard_pack_pairs_kernel<<<1, 256, 0, st>>>(p, out);
  ++g_launches;
}

void launch_shard_unpack(const ShardLayout& L, const double* recv, double* z, double* pairs_out,
                         cudaStream_t st) {
  long long mx = 1;
  for (int g = 0; g < L.world; ++g) {
    const long long e = L.inner * L.nloc[g] * L.outer;
    mx = e > mx ? e : mx;
  }
  long long bx = (mx + 255) / 256;
  if (bx > 2 * kNumSMs) bx = 2 * kNumSMs;
  if (bx < 1) bx = 1;
  shard_unpack_kernel<<<dim3((unsigned)bx, (unsigned)L.world), 256, 0, st>>>(L, recv, z, pairs_out);
  ++g_launches;
}

}  // namespace tsg
