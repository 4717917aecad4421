// Branch decision of one slice (streaming.cpp:126-137, 187-188), shared by
// the stand-alone decide kernel and the fused tail kernel. Thread 0 only.
#pragma once
#include "kernels.cuh"

namespace tsg {

// xsq: ||y||^2 (used when a.first_mode == 0); res[k]: ||E_k||^2 for the
// modes [a.first_mode, a.nmodes).
__device__ __forceinline__ void decide_finish(const DecideArgs& a, double xsq, const double* res) {
  // every field is computed in registers and stored to the device slot and the
  // host mirror from there (no load-after-store round trips)
  SliceCtl* c = a.slot;
  double delta, slice_sq = 0.0;
  int zero = 0;
  if (a.first_mode == 0 && !a.keep_delta) {
    slice_sq = xsq;
    zero = (xsq == 0.0);
    const double slice_norm = sqrt(xsq);
    delta = a.tau * slice_norm / sqrt((double)a.order);  // streaming.cpp:187-188
    c->slice_sq = slice_sq;
    c->zero_slice = zero;
    c->delta = delta;
  } else {
    delta = c->delta;
  }
  double rv[kMaxD];
  int em = -1;
#pragma unroll
  for (int k = 0; k < kMaxD; ++k) {
    rv[k] = 0.0;
    if (k >= a.first_mode && k < a.nmodes) {
      rv[k] = res[k];
      c->res_sq[k] = rv[k];
      if (em < 0 && !(sqrt(rv[k]) <= delta)) em = k;  // streaming.cpp:135
    }
  }
  c->expand_mode = em;
  if (a.host_slot && a.first_mode == 0) {
    // publish to the host without a copy call: fields, fence, then the count
    SliceCtl* h = a.host_slot;
    h->slice_sq = slice_sq;
    h->delta = delta;
#pragma unroll
    for (int k = 0; k < kMaxD; ++k) h->res_sq[k] = rv[k];
    h->expand_mode = em;
    h->zero_slice = zero;
    const unsigned long long q = *a.seq_counter + 1;
    *a.seq_counter = q;
    unsigned long long D = 0;
    if (a.ring_dev) {
      // insertion records completed so far (gpu-scope acquire), copied to the
      // host ring before the one system fence below
      D = *reinterpret_cast<const volatile unsigned long long*>(&a.ring_dev->done);
      __threadfence();
      unsigned long long P = *a.ring_pub;
      if (D > P + kRecRing - 1) P = D - (kRecRing - 1);
      for (unsigned long long k = P; k < D; ++k) {
        const int pos = (int)(k % kRecRing);
        const unsigned long long* sm = reinterpret_cast<const unsigned long long*>(&a.ring_dev->rec[pos]);
        unsigned long long* dm = reinterpret_cast<unsigned long long*>(&a.ring_host->rec[pos]);
        for (int w = 0; w < (int)(sizeof(Metrics) / 8); ++w) dm[w] = __ldcg(sm + w);
        const unsigned long long* sc = reinterpret_cast<const unsigned long long*>(&a.ring_dev->ctrl[pos]);
        unsigned long long* dc = reinterpret_cast<unsigned long long*>(&a.ring_host->ctrl[pos]);
        for (int w = 0; w < (int)(sizeof(Ctrl) / 8); ++w) dc[w] = __ldcg(sc + w);
      }
      *a.ring_pub = D > P ? D : P;
    }
    __threadfence_system();
    if (a.ring_dev) *reinterpret_cast<volatile unsigned long long*>(&a.ring_host->done) = D;
    *reinterpret_cast<volatile unsigned long long*>(&h->seq) = q;
  }
}

}  // namespace tsg
