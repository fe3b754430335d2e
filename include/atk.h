/*
 * atk.h — C ABI of the B200-native a-Tucker st-HOSVD engine (libatk_cuda.so).
 *
 * The reference (a-Tucker, /root/reference/proj) has no FFI layer: its hot
 * path is a header-only C++ API in namespace `atucker`.  Every entry point
 * below replaces one reference function 1:1 (cited per declaration); the C++
 * wrapper include/atucker_b200.hpp restores the reference's exact C++
 * signatures on top of this ABI, and paper_2010_10131_b200/_lib.py binds it
 * with ctypes.  No torch types, no C++ types, no exceptions cross this ABI.
 *
 * Conventions
 *  - Layout (tensor.hpp:99-156): column-major; element (i_1..i_N) at
 *    i_1 + I_1*i_2 + I_1*I_2*i_3 + ...; matrices column-major (i + rows*j).
 *  - Big tensors live on the device behind `atk_tensor` handles; small
 *    matrices (Gram I x I, factors I x R, U R x I) cross as host double arrays,
 *    exactly like the reference returns them as DenseMatrix values.
 *  - Inputs are never mutated; every output is a new object owned by the
 *    caller (reference ownership rule, sthosvd.hpp:126-194 / SPEC.md).
 *  - Calls are synchronous at return (stream-ordered inside).  One atk_ctx
 *    per host thread.
 *  - Errors: a status code 1:1 with the reference exception types
 *    (errors.hpp:9-25) plus CUDA/NCCL/OOM; atk_last_error() returns the
 *    thread-local message (sthosvd rewraps with "mode n: ", sthosvd.hpp:177-183).
 *  - There is no CPU fallback: without a CUDA device every compute call
 *    returns ATK_CUDA_ERROR.
 */
#ifndef ATK_H_
#define ATK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ATK_MAX_ORDER 8

/* errors.hpp:9-25 (Error + subclasses), then engine-specific codes. */
typedef enum atk_status {
    ATK_OK = 0,
    ATK_ERROR = 1,               /* atucker::Error                 */
    ATK_MODE_OUT_OF_RANGE = 2,   /* atucker::ModeOutOfRange        */
    ATK_SHAPE_MISMATCH = 3,      /* atucker::ShapeMismatch         */
    ATK_RANK_EXCEEDS_DIM = 4,    /* atucker::RankExceedsDim        */
    ATK_NOT_SQUARE = 5,          /* atucker::NotSquare             */
    ATK_RANK_TOO_LARGE = 6,      /* atucker::RankTooLarge          */
    ATK_NO_CONVERGENCE = 7,      /* atucker::NoConvergence         */
    ATK_RANK_DEFICIENT = 8,      /* atucker::RankDeficient         */
    ATK_NOT_SPD = 9,             /* atucker::NotSPD                */
    ATK_ZERO_NORM_INPUT = 10,    /* atucker::ZeroNormInput         */
    ATK_EMPTY_DATASET = 11,      /* atucker::EmptyDataset (selector trainer; not raised here) */
    ATK_FEATURE_VERSION = 12,    /* atucker::FeatureVersionMismatch */
    ATK_SCHEMA_MISMATCH = 13,    /* atucker::SchemaMismatch        */
    ATK_IO_FAILURE = 14,         /* atucker::IoFailure (.dten I/O) */
    ATK_CUDA_ERROR = 20,
    ATK_NCCL_ERROR = 21,
    ATK_OOM = 22,
    ATK_INVALID_ARGUMENT = 23,
    ATK_UNSUPPORTED = 24
} atk_status;

/* Storage type of a device tensor.  The reference is fp64-only
 * (tensor.hpp:99-156); fp32 storage is the engine's large-tensor mode
 * (contractions on tcgen05 kind::tf32, reductions / eig in fp64). */
typedef enum atk_dtype { ATK_F32 = 0, ATK_F64 = 1 } atk_dtype;

/* solver_kind.hpp:11 — label encoding of the selector (0 = EIG, 1 = ALS). */
typedef enum atk_solver { ATK_SOLVER_EIG = 0, ATK_SOLVER_ALS = 1, ATK_SOLVER_SVD = 2 } atk_solver;

typedef struct atk_ctx atk_ctx;
typedef struct atk_tensor atk_tensor;

/* The solver-selector hook, Strategy::decide (sthosvd.hpp:64-80): called once
 * per mode, host-side, with the already-shrunk J (sthosvd.hpp:149-153,166).
 * Returns an atk_solver value, or a negative number to abort the run. */
typedef int (*atk_selector_fn)(void* user, int mode, uint64_t i, uint64_t r, uint64_t j);

/* AlsOptions (solvers.hpp:18-22). */
typedef struct atk_als_opts {
    int num_iters;     /* default 5 */
    double rel_tol;    /* 0 disables early stop */
    uint64_t seed;     /* L0 ~ N(0,1) from mt19937_64(mix_seed(seed, mode)) */
} atk_als_opts;

/* Device-side per-stage times of one solve (CUDA events, milliseconds). */
typedef struct atk_stage_times {
    double gram_ms;
    double eig_ms;
    double ttm_ms;
    double als_ms;
    double comm_ms;
    double total_ms;
} atk_stage_times;

/* ModeReport (sthosvd.hpp:25-34) + the per-stage split the reference lacks. */
typedef struct atk_mode_report {
    int mode;
    int solver_used;
    int iterations_run;
    int eig_method;               /* 0 = Jacobi (dense), 1 = Chebyshev-filtered Rayleigh-Ritz,
                                     2 = tridiagonal (Householder + bisection + inverse iteration) */
    double selector_decision_time; /* seconds, host */
    double solver_time;            /* seconds, host wall incl. sync */
    double predicted_cost_eig;
    double predicted_cost_als;
    uint64_t dims_before[ATK_MAX_ORDER];
    uint64_t dims_after[ATK_MAX_ORDER];
    atk_stage_times times;
} atk_mode_report;

/* ------------------------------------------------ allocation tracking
 * instr::AllocTracker / AllocScope (instrumentation.hpp:39-150): live device
 * tensor payloads while enabled; `watched` counts buffers of exactly
 * watch_elems elements (the input's size), so acceptance criterion 12
 * (acceptance.cpp:428-458, "memory discipline") can be asserted on the engine. */
typedef struct atk_alloc_stats {
    int64_t alloc_count;   /* registered allocations */
    int64_t live_elems;    /* currently live tracked elements */
    int64_t peak_elems;    /* high-water mark of live elements */
    int64_t live_watched;  /* live buffers with exactly watch_elems elements */
    int64_t peak_watched;  /* high-water mark of the above */
} atk_alloc_stats;
void atk_alloc_tracking_enable(uint64_t watch_elems);
void atk_alloc_tracking_disable(void);
atk_status atk_alloc_tracking_stats(atk_alloc_stats* out);

/* ------------------------------------------------------------ context */
const char* atk_version(void);
const char* atk_last_error(void);
atk_status atk_ctx_create(int device, atk_ctx** out);
atk_status atk_ctx_destroy(atk_ctx* ctx);
/* Run on a caller-provided cudaStream_t (0 = the context's own stream).  Switching streams
   synchronises the previous one (the context's scratch is ordered by its stream). */
atk_status atk_ctx_set_stream(atk_ctx* ctx, void* cuda_stream);
atk_status atk_ctx_synchronize(atk_ctx* ctx);
/* Kernels this context launched so far (for bench accounting). */
uint64_t atk_ctx_launch_count(const atk_ctx* ctx);
/* Engine tuning knobs (unknown keys -> ATK_INVALID_ARGUMENT):
 *   "simt"          1 = CUDA-core contractions for every shape (default 0: tcgen05 / DMMA)
 *   "eig_method"   -1 auto (tridiagonal for n <= 200, else ChFSI handing over to the dense solver
 *                  after "eig_dense_passes" filter passes), 0 dense Jacobi (n <= 112; also the
 *                  Rayleigh-Ritz solver), 1 ChFSI only, 2 / 3 exact dense tridiagonal (any n <= 4096)
 *   "svd_explicit"  1 = fp64 SVD modes on the explicit unfolding (Gram-preconditioned one-sided
 *                  Jacobi; default), 0 = the Gram route (sigma = sqrt(lambda))
 *   "eig_dense_passes" ChFSI filter passes before the exact dense solver takes over (default 3;
 *                  skipped while the measured rate predicts convergence within ~2 more passes,
 *                  always after twice the budget; -1 = never)
 *   "chfsi_tol"     relative Ritz-residual target of ChFSI (default 1e-12; fp32 Grams use >= 1e-9)
 *   "cheb_fused"    1 = each Chebyshev filter pass is one cooperative launch (default), 0 = per-step launches
 *   "als_head"      -1 = one-pass ALS: phase 1 and phase 2 of a tile in turn (default); k >= 0 interleaves
 *                   tile t+1's phase 1 with t's phase 2, k K-blocks first (measured slower)
 *   "chfsi_lock"    1 = ChFSI locks converged Ritz pairs and filters the rest with a deflated S (default)
 *   "cheb_dataflow" 0 = resident Chebyshev steps end in a grid barrier (default); 1 = per-CTA ready flags
 *                   (each CTA waits only for the producers of its K slice; measured slower)
 *   "lanczos_tiles" 1 = the ChFSI bounds Lanczos keeps S in a 16-CTA cluster's shared memory (n <= ~1250;
 *                   default), 0 = re-read S from L2 every step
 *   "als_fused"     1 = an ALS iteration on mode 0 (fp32, R <= 32) reads Y once: rfac, YR and GR
 *                   from one tcgen05 pass (default), 0 = the two-pass TTM + TTT schedule
 *   "trd_tiles"     1 = tridiagonalise n <= 128 with one to four warps and n <= 192 on 32 x 32 tiles (default),
 *                   2 = tiles for every n <= 192, 0 = column-slot kernel
 *   "chfsi_k"       ChFSI block size (0 = r + max(16, r/4); measured: larger blocks only slow C2's
 *                   flat spectra down)
 *   "eig_assume_psd" 1 = atk_sym_eig_top_r inputs are Grams (Cholesky-preconditioned Jacobi)
 *   "tma_tf32"      1 = round-to-nearest tf32 operand loads (default), 0 = hardware truncation
 *   "gram_2cta"     1 = CTA-pair (cta_group::2) Gram where supported (default)
 *   "als_gram"      1 = ALS iterations on the mode's Gram (YR = S M^T, GR = M S M^T; rfac formed
 *                  once) when the roofline favours it, fp32 (default); 0 = passes over Y
 *   "gram_small"    1 = mode-0 fp32 Grams with I <= 128 stage one operand tile per K-block, read as
 *                  both operands, in a 12-deep ring (default); 0 = the general 4-stage ring
 *   "invit_smem"    1 = inverse iteration (n <= 128) with its iterates and LU factors in shared
 *                  memory, one warp per CTA (default); 0 = the global-memory kernel
 *   "chol_reg"      1 = the k <= 112 Cholesky + inverse (CholeskyQR, ALS solves) with the matrix in
 *                  register tiles, one barrier per pivot (default; 40 us at k = 80); 0 = the
 *                  shared-memory column kernel (67 us)
 *   "ttm_split"     1 = the TTM factor enters the tensor cores as tf32 hi + lo parts (two MMAs per
 *                  K step, ~2^-22 instead of 2^-12; the TTM stays HBM-bound; default), 0 = one tf32 part
 *   "gram_wide"     1 = 2-CTA Gram units of two 256 x 256 tiles of one tile row sharing the staged A
 *                  operand (default; 1/8 fewer shared-memory bytes per flop), 0 = one tile per unit
 *   "gram_chunk_kb" K-blocks per fp32 accumulation chain before the fp64 drain
 *   "gram_launch_kb" 2-CTA Gram: K-blocks per unit per launch (default 4096; 0 = one launch)
 *   "gram_lockstep" 1 = drift limiter in the 1-CTA Gram (default 0) */
atk_status atk_ctx_set_option(atk_ctx* ctx, const char* key, double value);

/* Multi-GPU (one process per GPU): sthosvd shards the input along the LAST
 * mode; each mode's Gram partial sums are combined with one NCCL allreduce
 * (SURVEY §8(e)).  `unique_id` is the 128-byte ncclUniqueId from
 * atk_nccl_unique_id() on rank 0, broadcast by the caller. */
atk_status atk_nccl_unique_id(void* out128);
atk_status atk_comm_init(atk_ctx* ctx, const void* unique_id, int rank, int world);
atk_status atk_comm_destroy(atk_ctx* ctx);

/* Host-staged collectives: the same sharded schedule with the two exchange
 * primitives supplied by the caller (e.g. torch.distributed / gloo), staged
 * through host memory.  It lets N > 1 ranks share ONE GPU (NCCL refuses two
 * ranks on the same device), so the multi-rank schedule — Gram allreduce per
 * mode, the ALS YR/GR allreduce per iteration, the last-mode all-gather — is
 * testable on a single B200.  Callbacks return 0 on success. */
typedef struct atk_host_collectives {
    int (*allreduce_f64)(void* user, double* host_buf, uint64_t count); /* in-place sum */
    int (*broadcast)(void* user, void* host_buf, uint64_t bytes, int root);
    void* user;
} atk_host_collectives;
atk_status atk_comm_init_host(atk_ctx* ctx, const atk_host_collectives* coll, int rank, int world);

/* Collective accounting of this rank since the last reset (either backend):
 * allreduces (the sizes exchange, the packed Gram triangle per sharded EIG
 * mode, YR and GR per sharded ALS iteration) and the last-mode all-gather /
 * broadcasts, with their payload bytes.  No reference counterpart (the
 * reference is single-process); it backs the SURVEY §8(e) schedule tests. */
typedef struct atk_comm_stats {
    uint64_t allreduce_calls, allreduce_bytes;
    uint64_t gather_calls, gather_bytes;
} atk_comm_stats;
atk_status atk_comm_get_stats(const atk_ctx* ctx, atk_comm_stats* out);
atk_status atk_comm_reset_stats(atk_ctx* ctx);

/* ------------------------------------------------------------ tensors */
/* DenseTensor(dims) (tensor.hpp:103-107) — device allocation, NOT zero-filled. */
atk_status atk_tensor_create(atk_ctx* ctx, atk_dtype dtype, int order, const uint64_t* dims,
                             atk_tensor** out);
/* Non-owning view of caller device memory (16-byte aligned). */
atk_status atk_tensor_wrap(atk_ctx* ctx, atk_dtype dtype, int order, const uint64_t* dims,
                           void* device_ptr, atk_tensor** out);
atk_status atk_tensor_from_host(atk_ctx* ctx, atk_dtype dtype, int order, const uint64_t* dims,
                                const void* host, atk_tensor** out);
atk_status atk_tensor_to_host(atk_ctx* ctx, const atk_tensor* t, void* host);
atk_status atk_tensor_free(atk_tensor* t);
atk_status atk_tensor_info(const atk_tensor* t, atk_dtype* dtype, int* order, uint64_t* dims,
                           void** device_ptr);
/* Counter-hash uniform [-1,1) on a 2^-23 grid, x[k] = f(seed, offset + k):
 * the bit-exact device twin of the oracle's or_hash_uniform. */
atk_status atk_fill_uniform(atk_ctx* ctx, atk_tensor* t, uint64_t seed, uint64_t offset);
/* x += alpha * y (same shape/dtype). */
atk_status atk_axpy(atk_ctx* ctx, atk_tensor* x, double alpha, const atk_tensor* y);
/* frobenius_norm (tensor.hpp:158-168), fp64 accumulation. */
atk_status atk_frobenius_norm(atk_ctx* ctx, const atk_tensor* t, double* out);

/* ------------------------------------------------------------ kernels.hpp */
/* kernels::gram (kernels.hpp:127-138): S = X_(n) X_(n)^T, exactly symmetric,
 * I_n x I_n column-major doubles written to host `s_out`. */
atk_status atk_gram(atk_ctx* ctx, const atk_tensor* x, int mode, double* s_out);
/* kernels::ttm (kernels.hpp:88-118): Y = X x_n U with U R x I_n (host,
 * column-major doubles); *y_out is a new device tensor with dim n -> R. */
atk_status atk_ttm(atk_ctx* ctx, const atk_tensor* x, const double* u, uint64_t r, uint64_t i,
                   int mode, atk_tensor** y_out);
/* kernels::ttt_mode (kernels.hpp:122-124): Z = X_(n) Y_(n)^T, I_n x R_n host. */
atk_status atk_ttt(atk_ctx* ctx, const atk_tensor* x, const atk_tensor* y, int mode,
                   double* z_out);

/* ------------------------------------------------------------ linalg.hpp */
/* linalg::sym_eig_top_r (linalg.hpp:101-123): top-r eigenpairs of the
 * symmetrized S (n x n host), values descending, sign rule fix_signs
 * (linalg.hpp:34-50).  `vectors` is n x r. */
atk_status atk_sym_eig_top_r(atk_ctx* ctx, const double* s, uint64_t n, uint64_t r,
                             double* values, double* vectors);
/* linalg::thin_qr (linalg.hpp:126-149): q rows x cols, r cols x cols. */
atk_status atk_thin_qr(atk_ctx* ctx, const double* a, uint64_t rows, uint64_t cols, double* q,
                       double* r);
/* linalg::spd_solve (linalg.hpp:169-177): A X = B via Cholesky. */
atk_status atk_spd_solve(atk_ctx* ctx, const double* a, uint64_t n, const double* b,
                         uint64_t nrhs, double* x);

/* ------------------------------------------------------------ solvers.hpp */
/* eig_mode_solver (solvers.hpp:64-73). factor_out: I_n x r host doubles. */
atk_status atk_eig_mode(atk_ctx* ctx, const atk_tensor* y, int mode, uint64_t r,
                        double* factor_out, atk_tensor** shrunk_out, atk_stage_times* times);
/* als_mode_solver (solvers.hpp:122-138).  l0 (I_n x r host) may be NULL, in
 * which case the reference seeding rule is used.  *iters_run may be NULL. */
atk_status atk_als_mode(atk_ctx* ctx, const atk_tensor* y, int mode, uint64_t r,
                        const atk_als_opts* opts, const double* l0, double* factor_out,
                        atk_tensor** shrunk_out, int* iters_run, atk_stage_times* times);
/* als_iterate (solvers.hpp:88-118): L (I_n x r host) and rfac (device). */
atk_status atk_als_iterate(atk_ctx* ctx, const atk_tensor* y, int mode, const double* l0,
                           uint64_t r, const atk_als_opts* opts, double* l_out,
                           atk_tensor** rfac_out, int* iters_run);
/* svd_mode_solver (solvers.hpp:142-162).  Device route: leading left singular
 * vectors of Y_(n) via the Gram eigenproblem (sigma = sqrt(lambda)); the
 * shrunk tensor diag(sigma) V^T equals U^T Y_(n) exactly in exact arithmetic. */
atk_status atk_svd_mode(atk_ctx* ctx, const atk_tensor* y, int mode, uint64_t r,
                        double* factor_out, atk_tensor** shrunk_out, atk_stage_times* times);

/* ------------------------------------------------------------ sthosvd.hpp */
/* sthosvd (sthosvd.hpp:126-194).  `x` is the whole tensor (single GPU) or,
 * after atk_comm_init, this rank's contiguous slab of the last mode.
 * factors_out: concatenation of the I_n x R_n column-major factors (host).
 * *core_out: new device tensor R_1 x ... x R_N (replicated on every rank).
 * reports: `order` entries, may be NULL.  decide == NULL means fixed EIG. */
atk_status atk_sthosvd(atk_ctx* ctx, const atk_tensor* x, const uint64_t* ranks,
                       atk_selector_fn decide, void* user, const atk_als_opts* opts,
                       atk_tensor** core_out, double* factors_out, atk_mode_report* reports);
/* Host-buffer entry (the e2e path): H2D of `x_host`, sthosvd, D2H of the
 * core into `core_out_host` (prod(ranks) elements of `dtype`). */
atk_status atk_sthosvd_host(atk_ctx* ctx, atk_dtype dtype, int order, const uint64_t* dims,
                            const void* x_host, const uint64_t* ranks, atk_selector_fn decide,
                            void* user, const atk_als_opts* opts, void* core_out_host,
                            double* factors_out, atk_mode_report* reports);
/* reconstruct (sthosvd.hpp:197-209). */
atk_status atk_reconstruct(atk_ctx* ctx, const atk_tensor* core, const double* factors,
                           const uint64_t* original_dims, atk_tensor** out);
/* relative_error (sthosvd.hpp:212-223). */
atk_status atk_relative_error(atk_ctx* ctx, const atk_tensor* x, const atk_tensor* core,
                              const double* factors, double* out);

/* ------------------------------------------------------------ .dten I/O
 * The reference's tensor file (tensor_io.hpp:15-99: "DTEN", u32 version 1,
 * u32 order, order x u64 dims, f64 LE column-major payload) streamed straight
 * to / from device memory through double-buffered pinned chunks; fp32 tensors
 * are narrowed / widened on the device.  Errors: ATK_IO_FAILURE with
 * read_dten's messages (bad magic, version, empty header, zero dimension,
 * > 2^40 elements, truncated payload).  SURVEY §8(f) row 3. */
atk_status atk_dten_info(const char* path, int* order, uint64_t* dims /* ATK_MAX_ORDER */);
/* read_dten (tensor_io.hpp:62-91) into a new device tensor of `dtype`. */
atk_status atk_tensor_read_dten(atk_ctx* ctx, const char* path, atk_dtype dtype, atk_tensor** out);
/* write_dten (tensor_io.hpp:39-52) of a device tensor (payload always f64). */
atk_status atk_tensor_write_dten(atk_ctx* ctx, const atk_tensor* t, const char* path);

/* ------------------------------------------------------------ instrumentation.hpp */
/* Logical GEMM counters (instrumentation.hpp:13-34): one record per logical
 * contraction with the reference's flop charge, not per CUDA launch. */
void atk_reset_gemm_counters(void);
long long atk_gemm_calls(void);
long long atk_gemm_flops(void);
/* Selector cost model (selector.hpp:36-58), exported for the hook. */
double atk_cost_eig(double i, double r, double j);
double atk_cost_als(double i, double r, double j, int num_iters);

/* B200 roofline cost model for the selector hook.  The
 * reference's model (selector.hpp:41-58) counts flops only, calibrated on a
 * CPU, and routes C2/C5 to ALS; on B200 the Gram is tensor-core bound and ALS
 * makes ~2 HBM passes over Y per iteration, so each stage is timed as
 * max(flops / peak, bytes / HBM bandwidth) plus measured fixed costs:
 *   EIG = max(I^2 J / P, s I J / BW) + eig(I) + max(2 I R J / P, s (I+R) J / BW)
 *   ALS = (iters (2 I + 5 R) + 2 R) s J / BW + iters * als_iter_overhead
 *   (mode 0, fp32, R <= 32, I % 128 == 0, I <= 1024 runs the one-pass iteration:
 *    iters * (als_fused_factor * s I J / BW + als_fused_overhead))
 * (s = element bytes, P = tf32 or fp64 tensor rate).  Times in seconds. */
typedef struct atk_roofline_params {
    double hbm_gbs;              /* measured copy bandwidth (MEASURED_PEAKS.json hbm_gbs) */
    double tf32_tflops;          /* measured sustained tf32 rate (profiles/peaks_r2.json) */
    double fp64_tflops;          /* effective DMMA fp64 contraction rate */
    double eig_small_ms;         /* dense tridiagonal eig, I <= 200 */
    double eig_large_ms;         /* ChFSI eig, I > 200 (gapped Gram spectra) */
    double als_iter_overhead_ms; /* R x R solves + host syncs per ALS iteration */
    int dtype;                   /* atk_dtype of the tensor */
    int num_iters;               /* AlsOptions::num_iters */
    double als_fused_factor;     /* one-pass ALS (mode 0, fp32, R <= 32): measured time / (s I J / BW) */
    double als_fused_overhead_ms; /* its per-iteration fixed cost */
    int num_sms;                 /* SMs of the run's device: the one-pass ALS shape gate (per-CTA columns) */
} atk_roofline_params;
void atk_roofline_params_default(atk_roofline_params* p, int dtype, int num_iters);
double atk_roofline_time_eig(const atk_roofline_params* p, double i, double r, double j);
double atk_roofline_time_als(const atk_roofline_params* p, double i, double r, double j);
/* The same for a given mode (the one-pass ALS applies to mode 0 only). */
double atk_roofline_time_als_mode(const atk_roofline_params* p, int mode, double i, double r, double j);
/* An atk_selector_fn: `user` is a const atk_roofline_params*; EIG iff its
 * modelled time is <= ALS's (ties to EIG, as heuristic_choice). */
int atk_roofline_selector(void* user, int mode, uint64_t i, uint64_t r, uint64_t j);

#ifdef __cplusplus
}
#endif
#endif /* ATK_H_ */
