/* tsg.h — C ABI of the B200-native streaming ST-HOSVD update.
 *
 * This is the drop-in boundary for the reference's streaming API
 * (reference proj/include/tucker/streaming.hpp). The reference exposes C++
 * only; each entry point below replaces one reference call and keeps its
 * argument meaning, layouts and error behaviour:
 *
 *   tsg_init            <- tucker::stream_init               streaming.hpp:55
 *   tsg_update          <- tucker::stream_update             streaming.hpp:63
 *   tsg_process_mode    <- tucker::process_nonstreaming_mode streaming.hpp:69-70
 *   tsg_estimate_relative_error
 *                       <- tucker::estimate_relative_error   streaming.hpp:79
 *   tsg_import_state    <- tucker::assemble_streaming_state  streaming.hpp:85-87
 *   tsg_export_state    <- StreamingState fields + streaming_factor()
 *                                                            streaming.hpp:34-49
 *   tsg_reconstruct / tsg_error_sums
 *                       <- reconstruct / relative_error     sthosvd.hpp:51,55
 *                          of StreamingState::full_model()  streaming.hpp:48-49
 *   tsg_shard_setup / tsg_shard_begin / tsg_shard_continue
 *                       <- stream_update split over G GPUs (no reference
 *                          counterpart; see the sharded section below)
 *   tsg_metrics_at / tsg_last_metrics
 *                       <- StreamingState::metrics (SliceMetrics, streaming.hpp:13-22)
 *   tsg_sym_eig_desc, tsg_small_svd_truncated, tsg_mode_subspace, tsg_ttm
 *                       <- linalg.hpp:42,54; sthosvd.hpp:38; tensor.hpp:66
 *                          (device implementations; exposed for parity tests)
 *
 * Error behaviour: every function returns a status. TSG_EINVAL mirrors
 * std::invalid_argument / std::out_of_range, TSG_EDRIFT mirrors the
 * std::runtime_error thrown when the core / ISVD coupling drifts
 * (streaming.cpp:39-64), TSG_EDEVICE reports a CUDA failure. The message is
 * available from tsg_last_error(h) (or tsg_last_error(NULL) for handle-less
 * calls).
 *
 * Layouts (identical to the reference): tensors colexicographic
 * (mode 0 fastest); factor matrices column-major N_k x R_k; the core
 * R_0 x ... x R_{d-1}; right (Q) column-major n x r, n = R_0...R_{d-2};
 * the streaming factor ("left") exported column-major n_d x r as
 * StreamingState::streaming_factor() returns it.
 *
 * Memory: TSG_MEM_HOST slices are copied to device staging on a copy
 * stream; TSG_MEM_DEVICE pointers must be device-resident fp64 buffers. The
 * handle's stream (tsg_cuda_stream) is a blocking stream: device reads of a
 * slice are ordered after work queued earlier on the legacy default stream;
 * a producer on another non-blocking stream must synchronise first. In
 * the default synchronous mode a slice may be reused as soon as tsg_update
 * returns. With TSG_ASYNC the engine acts on a slice's decision two calls
 * later (slices t+1 and t+2 are projected while slice t is inserted): a HOST
 * slice must stay unchanged until the following tsg_update returns (its
 * staging copy is then complete), a DEVICE slice until the second following
 * tsg_update (or tsg_synchronize) returns.
 * The handle owns all device memory; one host thread drives a handle.
 */
#ifndef TSG_H
#define TSG_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSG_MAXD 8

enum tsg_status {
  TSG_OK = 0,
  TSG_EINVAL = 1,   /* std::invalid_argument */
  TSG_EDRIFT = 2,   /* coupling drift: std::runtime_error */
  TSG_EOTHER = 3,
  TSG_EDEVICE = 4,  /* CUDA error */
  TSG_EIO = 5       /* checkpoint file error: tucker::IoError (io.hpp:24-33) */
};

enum tsg_mem_kind { TSG_MEM_HOST = 0, TSG_MEM_DEVICE = 1 };

enum tsg_flags {
  /* tsg_update returns once the work is enqueued; drift and device errors
   * surface at the next call. Default: synchronous, like the reference. */
  TSG_ASYNC = 1,
  /* Record CUDA events around the update phases (read with tsg_profile). */
  TSG_PROFILE = 2,
  /* Only the mode-0 projection kernel's events (its duration for roofline
   * accounting) — no event nodes on the tail / insertion streams. */
  TSG_PROFILE_MODE0 = 4
};

typedef struct tsg_stream tsg_stream;

typedef struct {
  int32_t device;            /* CUDA ordinal */
  int32_t flags;             /* tsg_flags */
  int64_t rank_capacity;     /* initial streaming-rank capacity (0 = auto) */
  int64_t row_capacity;      /* initial n_d capacity (0 = auto) */
  int64_t reorthogonalize_every; /* ISVDOptions (isvd.hpp:62-67): MGS of both factors every K insertions, 0 = off */
} tsg_config;

/* Same layout as oracle/oracle_abi.h orc_dims. */
typedef struct {
  int32_t order;
  int64_t n_d;
  int64_t rank;
  int64_t insertions;
  int64_t core_dims[TSG_MAXD];
  int64_t slice_dims[TSG_MAXD];
  double tau, squared_error, total_input_sq, nonstream_discarded_sq;
} tsg_dims;

/* SliceMetrics (streaming.hpp:13-22) plus parity diagnostics. */
typedef struct {
  int64_t slice_index;
  int64_t ranks[TSG_MAXD];
  double slice_norm, projected_norm, error_estimate;
  double mode_residuals[TSG_MAXD];
  int32_t expanded_mask;     /* bit k: mode k grew on this slice */
  int64_t peak_bytes;        /* device high-water mark of this handle */
  double wall_ms;            /* host wall time of the call */
  double trunc_margin;       /* |trailing - delta^2| / delta^2 of the ISVD cut */
  int32_t jacobi_sweeps;     /* inner-SVD sweeps */
} tsg_slice_metrics;

int tsg_create(const tsg_config* cfg, tsg_stream** out);
void tsg_destroy(tsg_stream* h);
const char* tsg_last_error(const tsg_stream* h);

int tsg_init(tsg_stream* h, const double* x, int32_t order,
             const int64_t* dims, double tau, int32_t mem_kind);
int tsg_update(tsg_stream* h, const double* slice, int32_t mem_kind);
int tsg_synchronize(tsg_stream* h);

int tsg_process_mode(tsg_stream* h, const double* y, const int64_t* ydims,
                     int32_t mode, double delta, double* y_out,
                     int64_t y_out_cap, int64_t* ydims_out, double* res);

/* add_row (isvd.hpp:110-111; isvd.cpp:163-250) on the device-resident ISVD of
 * the handle, together with the core rotation stream_update applies around it
 * (streaming.cpp:199-222): b holds n = R_0 * ... * R_{d-2} doubles (the
 * vectorised projected slice), abs_tol is the explicit truncation threshold
 * (stream_update passes delta = tau ||y|| / sqrt(d)), slice_norm_sq >= 0 is
 * added to total_input_sq (streaming.cpp:169; pass 0 to leave it alone).
 * One stream_update equals tsg_process_mode for every non-streaming mode
 * followed by this call. The result mirrors AddRowResult (isvd.hpp:97-104)
 * without inner_left, whose only use — the core rotation — is done here.
 * isvd_init (isvd.hpp:91-93) is tsg_import_state: a 2-way state whose single
 * factor is the identity is exactly a stand-alone ISVDState (left, singular
 * values, right = the core's column space), see INTEGRATION.md. */
typedef struct {
  int64_t r_old, r_new;
  int32_t degenerate;        /* residual too small to add a direction */
  double added_error_sq;     /* energy the inner truncation discarded */
} tsg_add_row_result;
int tsg_add_row(tsg_stream* h, const double* b, int32_t mem_kind, double abs_tol,
                double slice_norm_sq, tsg_add_row_result* out);

int tsg_query(tsg_stream* h, tsg_dims* out);
int tsg_export_state(tsg_stream* h, double* core, double* factors,
                     double* sigma, double* left, double* right);
int tsg_import_state(tsg_stream* h, const tsg_dims* dims, const double* core,
                     const double* factors, const double* sigma,
                     const double* left, const double* right);
double tsg_estimate_relative_error(tsg_stream* h);

/* TUCKCKPT v1 checkpoint of the streaming state, byte-compatible with the
 * reference's save_checkpoint / load_checkpoint + from_checkpoint
 * (io.cpp:268-423, io.hpp): written atomically (path.tmp, then rename).
 * Load validates the header like load_checkpoint (TSG_EIO on a bad magic,
 * version, truncation or shape; TSG_EINVAL for a batch model) and assembles
 * the state into h (TSG_EDRIFT if the core is not v x diag(s)). */
int tsg_save_checkpoint(tsg_stream* h, const char* path);
int tsg_load_checkpoint(tsg_stream* h, const char* path);

int64_t tsg_metrics_count(tsg_stream* h);
int tsg_metrics_at(tsg_stream* h, int64_t i, tsg_slice_metrics* out);
int tsg_last_metrics(tsg_stream* h, tsg_slice_metrics* out);

/* ---- Reconstruction (reconstruct / relative_error, sthosvd.hpp:51,55, of
 * StreamingState::full_model(), streaming.hpp:48-49), slice range by slice
 * range so full-size streams can be verified on sampled slices.
 * tsg_reconstruct writes slices [t0, t0+count) of the model, colexicographic
 * N_0 x ... x N_{d-2} x count, to `out` (host or device per mem_kind).
 * tsg_error_sums returns ||x - X||^2 and ||x||^2 over those slices for the
 * caller's slices x (same layout); relative_error over the whole stream is
 * sqrt(sum num / sum den) (zero-norm rules as in sthosvd.cpp:151-156). */
int tsg_reconstruct(tsg_stream* h, int64_t t0, int64_t count, double* out,
                    int32_t mem_kind);
int tsg_error_sums(tsg_stream* h, const double* x, int64_t t0, int64_t count,
                   int32_t mem_kind, double* num_sq, double* den_sq);

/* ---- Sharded update (one process per GPU).
 *
 * The reference has no distributed mode: this splits ONE stream_update
 * (streaming.hpp:63) across G ranks. Every rank holds the full state (same
 * tsg_init input on every rank, or tsg_import_state of the same state) and
 * rows [bounds[g], bounds[g+1]) of ONE spatial mode s of each slice, passed
 * as a dense colexicographic tensor N_0 x .. x (bounds[g+1]-bounds[g]) x ..
 * x N_{d-2} (a contiguous chunk of the slice when s is the last spatial
 * mode). tsg_shard_setup picks the largest spatial mode (the last one on
 * ties); tsg_shard_setup_mode names it (e.g. BASELINE configs[2]: mode 1).
 *
 *   tsg_shard_setup(h, g, G, bounds)            once, after init/import
 *   per slice:
 *     tsg_shard_begin(h, slab, mem_kind, &ex)   local projections of modes < s
 *     while (ex.pending) {
 *       ex.op == TSG_XCHG_ALLGATHER:
 *         allgather(ex.send -> ex.recv, ex.count doubles per rank, rank order)
 *       ex.op == TSG_XCHG_ALLREDUCE_SUM:
 *         recv[i] = sum over ranks of send[i], i < ex.count, the SAME bytes on
 *         every rank (NCCL allreduce, or a rank-ordered sum)
 *       tsg_shard_continue(h, &ex)
 *     }
 *
 * The exchange buffers are device memory owned by the handle. The request is
 * returned once the local pass is ENQUEUED on tsg_cuda_stream(h): the
 * collective must be enqueued on that stream (or follow a synchronisation),
 * and be complete or enqueued there when tsg_shard_continue is called. In steady state there is exactly one
 * exchange per slice (the compressed local tensor plus partial norms).
 * Growth of a local basis k < s adds ONE all-reduce of the N_k x N_k partial
 * Gram of the rank's residual (sthosvd.cpp:45-59 split over the ranks; the
 * eigensolve runs redundantly, K = W^T E stays local) and one more
 * compressed-tensor allgather for the modes after k. Every reduction over
 * ranks runs on identical bytes, so all ranks end bitwise identical. */
#define TSG_XCHG_ALLGATHER 0
#define TSG_XCHG_ALLREDUCE_SUM 1
typedef struct {
  int32_t pending;   /* 1: a collective is requested; 0: the update is done */
  int32_t op;        /* TSG_XCHG_ALLGATHER or TSG_XCHG_ALLREDUCE_SUM */
  int64_t count;     /* doubles contributed by each rank */
  double* send;      /* device: this rank's count doubles */
  double* recv;      /* device: allgather: world * count doubles, rank g's block
                        at g * count; allreduce: count doubles */
} tsg_exchange;

int tsg_shard_setup(tsg_stream* h, int32_t rank, int32_t world, const int64_t* bounds);
/* mode: the spatial mode (0 .. d-2) whose rows are split; -1 = the default. */
int tsg_shard_setup_mode(tsg_stream* h, int32_t rank, int32_t world, int32_t mode,
                         const int64_t* bounds);
int tsg_shard_begin(tsg_stream* h, const double* slab, int32_t mem_kind, tsg_exchange* ex);
int tsg_shard_continue(tsg_stream* h, tsg_exchange* ex);

/* Profiling harness: average ms of the fused projection kernel over `reps`
 * launches on device buffers (flags: 1 skip the residual phase, 2 skip the
 * cross-warp reduction; results are then not meaningful). */
int tsg_debug_project(const double* x, int64_t left, int64_t n, int64_t right,
                      const double* u, int32_t R, double* p, int32_t flags,
                      int32_t reps, double* ms_out);
/* Bytes the engine reads back per absorbed slice (decision slot, control
 * block snapshot, metrics record). */
int64_t tsg_readback_bytes_per_update(void);
/* Number of kernels this handle has launched (for launch accounting). */
int64_t tsg_kernel_launches(tsg_stream* h);
/* The CUDA stream the handle enqueues on (cudaStream_t as void*). */
void* tsg_cuda_stream(tsg_stream* h);
/* Device pointer to an internal scratch slice buffer of slice size
 * (for callers that synthesize slices on the device). */
double* tsg_slice_buffer(tsg_stream* h, int32_t which);

/* Phase timing (TSG_PROFILE): out[0] = updates timed, out[1] = mode-0
 * projection kernel ms (summed), out[2] = remaining projections + decision
 * ms, out[3] = ISVD + core rotation ms, out[4] = host gap ms (decision
 * readback), out[5] = mode-0 kernel launches. n >= 6. Resets when reset != 0. */
int tsg_profile(tsg_stream* h, double* out, int32_t n, int32_t reset);
/* Per-slice timeline (TSG_PROFILE, since the last tsg_profile reset): five
 * times in ms per profiled slice — mode-0 start, mode-0 end, decision (tail
 * end), insertion start, insertion end. Returns the rows written, -1 on error. */
int64_t tsg_profile_timeline(tsg_stream* h, double* out, int64_t cap);
/* FP64 pipe peaks on a device, TFLOP/s: DMMA (mma.sync f64) and DFMA. */
int tsg_measure_fp64_peaks(int32_t device, double* dmma_tflops, double* dfma_tflops);

/* Device building blocks on host buffers (column-major). */
int tsg_sym_eig_desc(int64_t n, const double* g, double* evals, double* evecs);
int tsg_small_svd_truncated(int64_t m, int64_t n, const double* a, double thr,
                            double* left, double* sigma, double* right,
                            int64_t* rank, double* disc);
int tsg_mode_subspace(const double* t, int32_t order, const int64_t* dims,
                      int32_t mode, double delta, double* basis,
                      int64_t* rank, double* evals, double* disc);
int tsg_ttm(const double* t, int32_t order, const int64_t* dims, int32_t mode,
            const double* a, int64_t a_rows, int64_t a_cols,
            int32_t transpose_a, double* out);

#ifdef __cplusplus
}
#endif
#endif /* TSG_H */
