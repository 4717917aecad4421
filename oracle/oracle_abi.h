/* TEST INFRASTRUCTURE ONLY — never linked into the product library.
 *
 * C ABI shared by the two CPU checkers under oracle/:
 *   - liboracle.so   (prefix tko_): this repo's plain-C restatement of the
 *                    reference's streaming ST-HOSVD path (tucker_oracle.c);
 *   - _ref/libtucker_ref.so (prefix tkr_): the reference's own C++ sources
 *                    compiled in place from /root/reference by oracle/Makefile,
 *                    wrapped by ref_shim.cpp.
 * Both export the same functions so the tests can drive either one (and the
 * product's tsg_* ABI, include/tsg.h) with identical inputs and compare.
 *
 * Status codes mirror the reference's exception classes:
 *   0 = ok, 1 = std::invalid_argument, 2 = std::runtime_error (coupling drift),
 *   3 = other. */
#ifndef TUCKER_ORACLE_ABI_H
#define TUCKER_ORACLE_ABI_H
#include <stdint.h>

#ifndef ORC
#define ORC(name) tko_##name
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAXD 8

typedef struct orc_state orc_state;

/* Dimensions of a state (filled by query). */
typedef struct {
  int32_t order;                  /* d */
  int64_t n_d;                    /* rows of the streaming factor */
  int64_t rank;                   /* R_{d-1} */
  int64_t insertions;             /* add_row calls */
  int64_t core_dims[ORC_MAXD];    /* R_0..R_{d-1} */
  int64_t slice_dims[ORC_MAXD];   /* N_0..N_{d-2} */
  double tau, squared_error, total_input_sq, nonstream_discarded_sq;
} orc_dims;

/* Per-slice record (SliceMetrics, streaming.hpp:13-22). */
typedef struct {
  int64_t slice_index;
  int64_t ranks[ORC_MAXD];
  double slice_norm, projected_norm, error_estimate;
  double mode_residuals[ORC_MAXD];
  int32_t expanded_mask; /* bit k set when mode k grew this slice */
} orc_metrics;

int ORC(stream_init)(const double* x, int32_t order, const int64_t* dims,
                     double tau, orc_state** out);
int ORC(stream_update)(orc_state* s, const double* y);
/* process_nonstreaming_mode on a caller tensor y (dims ydims, order d-1);
 * y_out receives the carried tensor (capacity y_out_cap doubles), its dims
 * go to ydims_out; *res receives ||E||_F. */
int ORC(process_mode)(orc_state* s, const double* y, const int64_t* ydims,
                      int32_t mode, double delta, double* y_out,
                      int64_t y_out_cap, int64_t* ydims_out, double* res);
int ORC(query)(const orc_state* s, orc_dims* out);
/* Arrays sized from query: core prod(core_dims); factors concat of the d-1
 * column-major N_k x R_k; sigma r; left n_d x r column-major; right n x r
 * column-major (n = prod R_0..R_{d-2}). Any pointer may be NULL. */
int ORC(export_state)(const orc_state* s, double* core, double* factors,
                      double* sigma, double* left, double* right);
int ORC(last_metrics)(const orc_state* s, orc_metrics* out);
int64_t ORC(metrics_count)(const orc_state* s);
int ORC(metrics_at)(const orc_state* s, int64_t i, orc_metrics* out);
/* assemble_streaming_state (streaming.cpp:242-263) from exported pieces. */
int ORC(assemble)(const orc_dims* dims, const double* core,
                  const double* factors, const double* sigma,
                  const double* left, const double* right, orc_state** out);
/* ISVDOptions::reorthogonalize_every of the state's ISVD (isvd.hpp:62-67). */
int ORC(set_reorthogonalize_every)(orc_state* s, int64_t k);
void ORC(destroy)(orc_state* s);
const char* ORC(last_error)(void);

/* Building blocks, exposed for unit-level parity. Column-major buffers. */
int ORC(sym_eig_desc)(int64_t n, const double* g, double* evals,
                      double* evecs);
int64_t ORC(truncation_rank)(int64_t n, const double* evals, double delta);
/* small_svd_truncated: m x n input; left (m x n cap), sigma (n cap),
 * right (n x n cap); returns rank via *rank, discarded via *disc. */
int ORC(small_svd_truncated)(int64_t m, int64_t n, const double* a,
                             double thr, double* left, double* sigma,
                             double* right, int64_t* rank, double* disc);
/* mode_subspace on tensor t (order, dims): basis (N_k x rank cap N_k),
 * eigenvalues (N_k). */
int ORC(mode_subspace)(const double* t, int32_t order, const int64_t* dims,
                       int32_t mode, double delta, double* basis,
                       int64_t* rank, double* evals, double* disc);
/* ttm (tensor.cpp:106-162): out dims = dims with dims[mode] replaced. */
int ORC(ttm)(const double* t, int32_t order, const int64_t* dims,
             int32_t mode, const double* a, int64_t a_rows, int64_t a_cols,
             int32_t transpose_a, double* out);
double ORC(sum_of_squares)(const double* p, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
