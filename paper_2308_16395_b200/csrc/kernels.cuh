// Kernel launch interface of the B200 streaming ST-HOSVD engine.
// All launches are asynchronous on the given stream; every launcher bumps
// the launch counter so bench.py can report gpu_launches.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace tsg {

extern long long g_launches;  // per-process launch counter (engine copies it per handle)

// ---------------------------------------------------------------- linalg
// Jacobi eigendecomposition of a symmetric n x n matrix (column-major, ld n)
// in global memory, one CTA. Outputs eigenvalues (descending, clamped >= 0)
// and eigenvectors (sign rule) exactly as sym_eig_desc (linalg.cpp:120-181)
// specifies, with the cyclic sweep replaced by the round-robin parallel
// ordering (every pair once per sweep). `work` holds 3 n*n + 512 doubles.
void launch_sym_eig(const double* g, int n, double* evals, double* evecs,
                    double* work, int* sweeps_out, cudaStream_t st);

// Truncation of a descending spectrum (linalg.cpp:183-208, sthosvd.cpp:31-35):
// optionally zero sqrt(l) <= 1e-14 sqrt(l_max) first (thin route).
// out_rank[0] = rank, out_disc[0] = trailing sum.
void launch_truncate(double* evals, int n, double delta, int zero_floor,
                     long long* out_rank, double* out_disc, cudaStream_t st);

// G = A A^T (rows x rows) for column-major A (rows x cols), exactly symmetric.
// `partial` must hold splits*rows*rows doubles (see gram_splits()).
int gram_splits(int rows, long long cols);
void launch_gram(const double* a, int rows, long long cols, double* g,
                 double* partial, cudaStream_t st);
// G = A^T A (cols x cols), A column-major rows x cols.
void launch_gram_t(const double* a, long long rows, int cols, double* g,
                   cudaStream_t st);
// C (m x n) = A (m x k, lda) * B (k x n, ldb), all column-major, plain FP64.
void launch_gemm_nn(const double* a, long long lda, const double* b, long long ldb,
                    double* c, long long ldc, long long m, int n, int k, cudaStream_t st);
// Scale column j of A (m x n, lda) by 1/sqrt(evals[j]) (thin-route basis).
void launch_scale_cols_invsqrt(double* a, long long lda, long long m, int n,
                               const double* evals, cudaStream_t st);
// One in-place modified Gram-Schmidt pass (linalg.cpp:64-78), right-looking.
void launch_mgs(double* a, long long lda, long long m, int n, cudaStream_t st);
// max |A^T A - I| (matrix.cpp:118-131) into out[0].
void launch_orth_defect(const double* a, long long lda, long long m, int n,
                        double* out, cudaStream_t st);

// ------------------------------------------------------------- tensors
// Mode-k view of a colexicographic tensor: (left, n, right).
struct ModeView {
  long long left, n, right;
};
// A[i + c n] = T[l + i left + r left n], c = l + r left (tensor.cpp:67-84).
void launch_unfold(const double* t, ModeView v, double* a, cudaStream_t st);
// Zero-pad along the mode: (left, n, right) -> (left, n + extra, right).
void launch_pad(const double* t, ModeView v, long long extra, double* out,
                cudaStream_t st);
// Concatenate (left, na, right) and (left, nb, right) along the mode.
void launch_concat(const double* a, const double* b, long long left,
                   long long na, long long nb, long long right, double* out,
                   cudaStream_t st);

// Fused mode-k projection: P = U^T X_(k), optional residual
// E = X - U P with per-CTA partials of ||E||^2 and ||X||^2.
struct ProjArgs {
  const double* x = nullptr;
  ModeView v{1, 1, 1};
  const double* u = nullptr;   // n x R, column-major, ld = v.n
  int R = 0;
  double* p = nullptr;         // (left, R, right) or nullptr
  double* e = nullptr;         // (left, n, right) or nullptr
  double* partial = nullptr;   // [grid * 2] (res_sq, x_sq) or nullptr
  int residual = 0;
  int stream_in = 0;           // input read once: evict-first loads
  unsigned* tile_counter = nullptr;  // zeroed dynamic tile scheduler (optional)
  const double* upad = nullptr;      // optional pre-padded U image (see pad_u)
  int debug_skip = 0;                // profiling only: 1 skip phase 2, 2 skip reduction, 4 skip DMMA
  int karg0 = 0, karg1 = 0;  // kernel-specific integers (kernels take one ProjArgs parameter so
                             // a graph node's input pointer can be re-pointed in place)
};
// Pre-padded U image for the DMMA projection kernel: rows padded to a
// multiple of 8, row pitch 8*ceil(R/8)+4, zero fill. Returns its size in
// doubles for (N, R); writes it when `out` is non-null.
long long upad_size(long long N, int R);
// Offset (doubles) of the column-owning kernel's U images inside the pad_u
// buffer (N a multiple of 8): [image 1 (N x (8RT+2)) | image 2 (N x (8RT+4))].
long long upad_cols_offset(long long N, int R);
void launch_pad_u(const double* u, long long N, int R, double* out, cudaStream_t st);
// Returns the grid size (number of partial pairs written).
int launch_project(const ProjArgs& a, cudaStream_t st);

// Sum of squares of a device vector into out[0] (two-stage, deterministic).
void launch_sumsq(const double* x, long long n, double* out, double* scratch,
                  cudaStream_t st);

// --------------------------------------------------------- streaming step
struct DecideArgs {
  SliceCtl* slot;
  SliceCtl* host_slot = nullptr;          // mapped host mirror (with seq)
  unsigned long long* seq_counter = nullptr;  // device counter for host_slot->seq
  const double* partial;     // concatenated partial pairs
  int off[kMaxD], cnt[kMaxD];
  int nmodes;                // d-1
  int first_mode;            // first mode evaluated by this decide call
  double tau;
  int order;
  int keep_delta = 0;        // use slot->delta as given (process_nonstreaming_mode)
  // insertion records: copied from the device ring to the mapped host ring
  // under the decision's system fence (keeps that fence off the insertion chain)
  const RecRing* ring_dev = nullptr;
  RecRing* ring_host = nullptr;
  unsigned long long* ring_pub = nullptr;  // device: records already copied
};
void launch_decide(const DecideArgs& a, cudaStream_t st);

// Fused tail: modes [m0, m1) of one slice (each N_k <= 512, R_k <= 32) and
// the decision, one cooperative kernel. Mode k reads the output of mode k-1
// (`x` for k = m0) viewed as (left[k], N[k], right[k]) and writes out[k].
// da carries the partial pairs of the modes [da.first_mode, m0) projected by
// the stand-alone kernels. Returns the grid size, or -1 if not applicable.
struct TailArgs {
  const double* x;
  double* out[kMaxD];
  const double* u[kMaxD];  // U_k, N_k x R_k column-major (ld N_k)
  long long N[kMaxD], left[kMaxD], right[kMaxD];
  int R[kMaxD];
  int m0, m1;
  double* part;            // kMaxD * grid per-CTA partials
  unsigned* done;          // arrival counter (zero between launches)
  DecideArgs da;
  unsigned long long* clk = nullptr;  // debug: per-CTA globaltimer stamps (16 per CTA)
};
bool tail_eligible(long long n, long long r);
int launch_tail(const TailArgs& t, cudaStream_t st);
// Ledger commit for modes [m0, m1): nonstream += ||E_k||^2 as rn*rn;
// with_total adds slice_norm^2 to total_input_sq (streaming.cpp:168-169).
void launch_commit_modes(Ctrl* ctrl, const SliceCtl* slot, int m0, int m1, int with_total,
                         cudaStream_t st);
void launch_ledger_add_nonstream(Ctrl* ctrl, const double* value, cudaStream_t st);

struct SpatialRanks {
  long long v[kMaxD];
};

struct IsvdBufs {
  Ctrl* ctrl;
  const SliceCtl* slot;  // this slice's decisions (delta, norms)
  const double* b;     // projected slice, length n
  const double* q;     // n x r (ld n)
  double* qn;          // n x r' out (ld n)
  const double* c;     // core n x r (ld n)
  double* cn;          // core out
  double* e;           // length n scratch
  const double* sigma; // r
  double* sigma_new;   // r'
  const double* left;  // n_d x r row-major, ld capr
  double* left_new;
  double* pgram;       // capr*capr
  double* inner;       // scratch for the inner SVD (see engine)
  double* partial;     // per-CTA partials
  RecRing* ring;       // mapped host ring of per-insertion records
  long long n;
  long long cap_rows;  // left capacity (n_d itself is read from ctrl)
  int capr;
  int order;
  int r_hint;          // streaming rank before the insertion (host mirror)
  int commit_modes;    // > 0: commit this slice's ledgers first (modes [0, commit_modes))
  int stage_core;      // small path: stage the old core in shared memory
  double* hand;        // grid path: leader -> followers handoff (kHandDoubles)
  unsigned* gsync;     // grid path: [0] epoch, [1] flag, [2] arrivals (zero-initialised)
  long long spatial_ranks[kMaxD];
};
void launch_isvd(const IsvdBufs& b, cudaStream_t st);
// MGS re-orthogonalization of the streaming factor (row-major, ld capr,
// ctrl->n_d rows) and of Q (n x ctrl->r): ISVDOptions::reorthogonalize_every.
void launch_reorth(const Ctrl* ctrl, double* left, int capr, double* q, long long n, cudaStream_t st);
constexpr int kHandDoubles = 3 * 33 * 33 + 8 * 33 + 16;
int isvd_inner_scratch(int capr);
int read_isvd_clocks(long long* out);

// Zero slice (streaming.cpp:171-185).
void launch_zero_slice(Ctrl* ctrl, const SliceCtl* slot, double* left, int capr, RecRing* ring,
                       int order, const long long* spatial, cudaStream_t st);

// stream_init helpers
void launch_init_isvd(Ctrl* ctrl, const double* core, long long n, int r,
                      const double* evals_last, double* q, double* sigma,
                      const double* left_cm, long long n_init, double* left_rm,
                      int capr, cudaStream_t st);
void launch_coupling_check(Ctrl* ctrl, const double* core, const double* q,
                           const double* sigma, long long n, int r,
                           double* partial, cudaStream_t st);

int measure_fp64_peaks(int device, double* dmma_tflops, double* dfma_tflops);

// ------------------------------------------------- reconstruction (recon.cu)
// z (n x count) = core_mat (n x r) * left[t0 .. t0+count)^T (left row-major, ld capr)
void launch_recon_core(const double* core, long long n, int r, const double* left, int capr,
                       long long t0, long long count, double* z, cudaStream_t st);
// out (left, N, right) = U (N x R) along the middle mode of z (left, R, right)
void launch_recon_expand(const double* z, long long left, int R, long long right, const double* u,
                         long long N, double* out, cudaStream_t st);
// out[0] = ||x - y||^2, out[1] = ||x||^2 (part: 4 * kNumSMs doubles)
void launch_diff_sumsq(const double* x, const double* y, long long n, double* part, double* out,
                       cudaStream_t st);

// ------------------------------------------------------ sharded update
constexpr int kMaxShards = 64;
// Partial pairs of the locally projected modes (layout as in DecideArgs).
// Tridiagonal route for the leading eigenpairs of a Gram matrix (tridiag_eig.cu).
bool tri_eig_applicable(int n);
int tri_eig_max_rank(int n);
long long tri_eig_work_doubles(int n, int max_rank);
bool launch_tri_eigvals(const double* g, int n, double* evals, double* work, cudaStream_t st);
void launch_tri_eigvecs(int n, int rank, double* work, double* evecs, cudaStream_t st);

struct ShardPairs {
  const double* partial;
  int off[kMaxD], cnt[kMaxD];
  int nmodes;
};
// out[2k], out[2k+1] = (sum res_sq, sum x_sq) of mode k, fixed order.
void launch_shard_pack_pairs(const ShardPairs& p, double* out, cudaStream_t st);
// Gathered buffer: rank g's block starts at g * count and holds `header`
// doubles of pairs, then its part of the tensor, inner x nloc[g] x outer
// (rows [lo[g], lo[g] + nloc[g]) of the shard mode, which has ns rows in
// all): element (i, j, o) lands at z[i + inner * (lo[g] + j + ns * o)].
// pairs_out (may be null) receives the pairs grouped per mode:
// [k * 2 * world + 2 g + j].
struct ShardLayout {
  int world;
  int header;
  long long count, inner, outer, ns;
  long long lo[kMaxShards], nloc[kMaxShards];
};
void launch_shard_unpack(const ShardLayout& L, const double* recv, double* z, double* pairs_out,
                         cudaStream_t st);

}  // namespace tsg
