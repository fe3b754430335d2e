// atk_internal.cuh — shared plumbing of libatk_cuda.so: context, tensor
// handles, error mapping, device workspace, launch accounting.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/atk.h"

namespace atk {

// errors.hpp:9-25 -> atk_status.  Thrown inside the library, converted to a
// status code + thread-local message at the C boundary (api.cu).
struct Error : std::runtime_error {
    atk_status code;
    Error(atk_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(atk_status c, const std::string& m) { throw Error(c, m); }

#define ATK_CUDA(expr)                                                                        \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess) {                                                              \
            ::atk::fail(_e == cudaErrorMemoryAllocation ? ATK_OOM : ATK_CUDA_ERROR,           \
                        std::string(#expr) + ": " + cudaGetErrorString(_e) + " at " +         \
                            __FILE__ + ":" + std::to_string(__LINE__));                       \
        }                                                                                     \
    } while (0)

#define ATK_LAUNCHED(ctx)                                                                     \
    do {                                                                                      \
        (ctx)->launches++;                                                                    \
        cudaError_t _e = cudaGetLastError();                                                  \
        if (_e != cudaSuccess)                                                                \
            ::atk::fail(ATK_CUDA_ERROR, std::string("kernel launch: ") +                      \
                                            cudaGetErrorString(_e) + " at " + __FILE__ + ":" + \
                                            std::to_string(__LINE__));                        \
    } while (0)

struct Comm;  // dist.cu

}  // namespace atk

namespace atk {
struct DeferredTiming {
    cudaEvent_t a, b;
    int mode, field;
};
}  // namespace atk

struct atk_ctx {
    int device = 0;
    bool defer_timing = false;  // StageTimer hands its events to `deferred` (sthosvd)
    int timing_mode = 0;
    std::vector<atk::DeferredTiming> deferred;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    uint64_t launches = 0;
    int force_simt = 0;        // option "simt": portable CUDA-core contractions
    int eig_method = -1;       // option "eig_method": -1 auto, 0 dense Jacobi, 1 ChFSI, 2 tridiagonal,
                               // 3 tridiagonal at every n (the grid-wide reduction above 200)
    int svd_explicit = 1;      // option "svd_explicit": SVD mode on the explicit unfolding (fp64)
    int eig_dense_passes = 3;  // option "eig_dense_passes": ChFSI filter passes before the exact dense
                               // solver takes over (n > 200; -1 never)
    double chfsi_tol = 1e-12;  // option "chfsi_tol": relative Ritz residual target
    int cheb_fused = 1;        // option "cheb_fused": whole Chebyshev filter in one cooperative launch
    int als_head = -1;         // option "als_head": one-pass ALS, >= 0 interleaves tile t+1's phase 1 with t's phase 2
                               // (that many K-blocks first); measured slower (C2: 1.63 vs 1.31 ms per iteration)
    int chfsi_lock = 1;        // option "chfsi_lock": lock converged Ritz pairs, filter a deflated S
    int cheb_dataflow = 0;     // option "cheb_dataflow": resident Chebyshev steps synchronised by per-CTA ready
                               // flags instead of a grid barrier (measured slower: 14.0 vs 12.5 us per step)
    int lanczos_tiles = 1;     // option "lanczos_tiles": S resident in a 16-CTA cluster's smem for the bounds
    int als_gram = 1;          // option "als_gram": ALS iterations on the mode's Gram when the roofline says
                               // Gram + one TTM beats the iterations' passes over Y (fp32)
    int als_fused = 1;         // option "als_fused": one pass over Y per ALS iteration (mode 0, fp32)
    int trd_tiles = 1;         // option "trd_tiles": 32 x 32-tile tridiagonalisation for n <= 192
    int chfsi_k = 0;           // option "chfsi_k": ChFSI block size override (0 = r + max(16, r/4))
    bool replicated = false;   // sthosvd's last mode under a comm: the work tensor is whole on every rank
    uint64_t global_last = 0;  // sthosvd under a comm: the global size of the sharded (last) mode
    bool eig_assume_psd = false;  // option "eig_assume_psd": atk_sym_eig_top_r input is a Gram
    int tma_tf32 = 1;          // option "tma_tf32": TMA converts fp32 -> tf32 with round-to-nearest
                               // (the MMA itself truncates: measured 6e-4 bias vs 1e-6, test_gpu_tc.py)
    int gram_chunk_kb = 0;     // option "gram_chunk_kb": K-blocks per fp64 drain (0 = default)
    int gram_small = 1;        // option "gram_small": mode-0 Grams with I <= 128 stage one operand tile per
                               // K-block (read as A and B) in a 12-deep ring; 0 = the general 4-stage ring
    int gram_2cta = 1;         // option "gram_2cta": 256x256 Gram tiles on CTA pairs (cta_group::2)
    int invit_smem = 1;        // option "invit_smem": inverse iteration with its iterates and LU factors in
                               // shared memory (n <= 128); 0 = the global-memory kernel
    int chol_reg = 1;          // option "chol_reg": register-tile Cholesky + inverse (k <= 112): C5's k = 80
                               // in 40 us per call against 67 us for the shared-memory column kernel
    int ttm_split = 1;         // option "ttm_split": TTM factor as tf32 hi + lo (two MMAs per K step)
    int gram_wide = 1;         // option "gram_wide": 2-CTA Gram units of two tiles sharing the A operand
    int gram_lockstep = 0;     // option "gram_lockstep": bound CTA drift so X streams from HBM once
    int gram_launch_kb = 1024; // option "gram_launch_kb": 2-CTA Gram K-blocks per unit per launch (0 = one launch);
                               // C5 mode 0, ncu DRAM per Gram: 4096 -> 48.4 GB, 2048 -> 38.5, 1024 -> 36.8 (1.07x
                               // the 34.4 GB of X), 512 -> 39.2; step time equal within noise (A/B, 3 x 10 steps)
                               // (off: lockstep hot-spots L2 slices, 45 ms vs 34 ms at C5, r1)
    atk::Comm* comm = nullptr;
    cudaEvent_t ev[8] = {};
    void* pinned = nullptr;    // page-locked staging for the end-of-call factor download (grown on demand)
    size_t pinned_bytes = 0;
    // device scratch kept across calls (atk::ScratchScope): the ChFSI block buffers, so a converged
    // eigensolve returns without a burst of stream-ordered frees between its last check and the TTM
    char* scratch = nullptr;
    size_t scratch_bytes = 0, scratch_used = 0;
};

struct atk_tensor {
    atk_ctx* ctx = nullptr;
    atk_dtype dtype = ATK_F64;
    int order = 0;
    uint64_t dims[ATK_MAX_ORDER] = {};
    void* data = nullptr;
    bool owned = false;
    uint64_t track_epoch = 0;  // AllocTracker ticket (0 = untracked)

    uint64_t numel() const {
        uint64_t p = 1;
        for (int m = 0; m < order; ++m) p *= dims[m];
        return p;
    }
    size_t elem_bytes() const { return dtype == ATK_F32 ? 4 : 8; }
    size_t bytes() const { return size_t(numel()) * elem_bytes(); }
};

namespace atk {

// ------------------------------------------------------------------ memory
// Stream-ordered allocations from the device's default pool; the pool keeps
// freed blocks (release threshold = max) so repeated sthosvd calls reuse them.
void* dev_alloc(atk_ctx* ctx, size_t bytes);
// The context's page-locked host staging buffer, at least `bytes` long (kept across calls: a
// fresh pageable vector cost ~1.4 ms of page faults per C5 sthosvd with the GPU idle).
void* pinned_host(atk_ctx* ctx, size_t bytes);
void dev_free(atk_ctx* ctx, void* p);

// ScratchScope: the context's persistent scratch, carved in 256-byte aligned pieces for the
// scope's lifetime (one scope at a time; the context's stream orders every use).  Grown on
// demand; released by atk_ctx_destroy.
struct ScratchScope {
    atk_ctx* ctx;
    ScratchScope(atk_ctx* c, size_t bytes);
    ~ScratchScope() { ctx->scratch_used = 0; }
    ScratchScope(const ScratchScope&) = delete;
    ScratchScope& operator=(const ScratchScope&) = delete;
    void* take(size_t bytes);
    static size_t round(size_t bytes) { return (bytes + 255) / 256 * 256; }
};

template <class T>
struct DevBuf {
    atk_ctx* ctx = nullptr;
    T* p = nullptr;
    size_t n = 0;
    bool own = true;
    DevBuf() = default;
    DevBuf(atk_ctx* c, size_t count) : ctx(c), n(count) {
        p = count ? static_cast<T*>(dev_alloc(c, count * sizeof(T))) : nullptr;
    }
    // borrowed from a ScratchScope (not freed)
    DevBuf(ScratchScope& s, size_t count) : ctx(s.ctx), n(count), own(false) {
        p = count ? static_cast<T*>(s.take(count * sizeof(T))) : nullptr;
    }
    // a view of someone else's memory (not freed)
    DevBuf(atk_ctx* c, T* borrowed, size_t count) : ctx(c), p(borrowed), n(count), own(false) {}
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : ctx(o.ctx), p(o.p), n(o.n), own(o.own) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            reset();
            ctx = o.ctx; p = o.p; n = o.n; own = o.own;
            o.p = nullptr; o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { reset(); }
    void reset() {
        if (p && own) dev_free(ctx, p);
        p = nullptr;
        n = 0;
    }
    T* get() const { return p; }
};

// ------------------------------------------------------------------ tensors
atk_tensor* new_tensor(atk_ctx* ctx, atk_dtype dt, int order, const uint64_t* dims);
void check_tensor(const atk_tensor* t, const char* what);

// LoopSplit (tensor.hpp:175-187) of a device tensor at `mode`.
struct Split {
    uint64_t P = 1, I = 1, O = 1;
};
inline Split loop_split(const uint64_t* dims, int order, int mode) {
    Split s;
    for (int m = 0; m < mode; ++m) s.P *= dims[m];
    s.I = dims[mode];
    for (int m = mode + 1; m < order; ++m) s.O *= dims[m];
    return s;
}

void check_mode(int order, int mode);

// ------------------------------------------------------------------ counters
void record_gemm(long long charge);

// ------------------------------------------------------------------ timing
// Per-stage device time.  stop_ms(field) synchronizes on the stop event,
// unless the context defers timing (sthosvd does): then the event pair is
// handed to ctx->deferred and resolved after the call's final sync, so no
// stage boundary blocks the host (the next stage is enqueued while the GPU
// still runs this one).
enum StageField { kStageGram = 0, kStageEig = 1, kStageTtm = 2, kStageAls = 3, kStageComm = 4 };
struct StageTimer {
    atk_ctx* ctx;
    cudaEvent_t a = nullptr, b = nullptr;
    explicit StageTimer(atk_ctx* c);
    ~StageTimer();
    void start();
    double stop_ms(int field = -1);
};

// ------------------------------------------------------------------ kernels
// gen.cu
void fill_uniform(atk_ctx* ctx, atk_tensor* t, uint64_t seed, uint64_t offset);
double norm2_sq(atk_ctx* ctx, const void* x, atk_dtype dt, uint64_t n);  // sum of squares, fp64
void axpy(atk_ctx* ctx, void* x, const void* y, atk_dtype dt, uint64_t n, double alpha);
void convert(atk_ctx* ctx, void* dst, atk_dtype ddt, const void* src, atk_dtype sdt, uint64_t n);
double diff_norm2_sq(atk_ctx* ctx, const void* x, const void* y, atk_dtype dt, uint64_t n);

// contract.cu — matricization-free contractions (kernels.hpp:34-138).
// Z (I x R, fp64, device, column-major) = X_(n) Y_(n)^T, X viewed as
// (P, I, O), Y as (P, R, O).  `sym` = Gram (X == Y): exact symmetric output.
void ttt(atk_ctx* ctx, const void* x, const void* y, atk_dtype dt, Split s, uint64_t R,
         double* z_dev, bool sym);
// Y (P, R, O) = X (P, I, O) x_n U, U R x I fp64 device (column-major).
void ttm(atk_ctx* ctx, const void* x, atk_dtype dt, Split s, const double* u_dev, uint64_t R,
         void* y);

// dense.cu — small fp64 device linear algebra.
// C(m x n) = alpha op(A) op(B) + beta C, column-major with leading dims.
// The degree-`deg` Chebyshev recurrence of ChFSI in one cooperative launch:
// Y1 = a1 S V + b1 V, Y_{j+1} = a S Y_j + b Y_j + c Y_{j-1}; y = {V, 3 scratch
// n x k blocks}.  Returns the index into y of Y_deg, or -1 if the grid cannot
// be co-resident (the caller then runs the per-step launches).
int cheb_filter(atk_ctx* ctx, const double* S, int n, int k, int deg, double* const y[4], double a1, double b1,
                double a, double b, double c);
void dgemm(atk_ctx* ctx, bool ta, bool tb, int m, int n, int k, double alpha, const double* a,
           int lda, const double* b, int ldb, double beta, double* c, int ldc);
// C (n x n, n <= 160) = alpha op(A) op(A)^T (op(A) n x k): the upper 32 x 32 blocks on DMMA from a
// shared-memory panel that serves as both operands, both triangles written (dgemm.cu).
void dsyrk_upper(atk_ctx* ctx, bool ta, int n, int k, double alpha, const double* a, int lda, double* c, int ldc);
// C = op(A) op(B) (m x n, n = R <= 64, one pass over A, no split-K) for the fp64 first / last-mode
// TTM; tout stores C^T (c[j + ldc i]).
void dgemm_ttm(atk_ctx* ctx, bool ta, bool tb, int m, int n, int k, const double* a, int lda, const double* b,
               int ldb, double* c, int ldc, bool tout);
// Dense symmetric eigensolver for n <= kJacobiMax (one CTA, smem Jacobi):
// all eigenpairs of A (n x n, lda), values descending, vectors n x n.  psd:
// A is known positive semi-definite (Cholesky-preconditioned, vector-free path).
constexpr int kJacobiMax = 112;
// PSD inputs up to this size still fit (U only): sweeps_dev = -1 if the
// Cholesky preconditioning fails (caller falls back to ChFSI).
constexpr int kJacobiPsdMax = 152;
void jacobi_eig(atk_ctx* ctx, const double* a, int n, int lda, double* values, double* vectors,
                int ldv, int* sweeps_dev, bool psd = false);
// tridiag.cu — dense symmetric eigensolver by Householder tridiagonalisation,
// bisection and inverse iteration (one CTA holds the packed lower triangle):
// the top `nvals` (>= nwant) eigenvalues of A (n x n, lda), descending, and
// the vectors of the top `nwant` (n x nwant, ldv), signs NOT fixed.
// Bit-reproducible (no atomics).
constexpr int kTridiagMax = 200;
// All eigenvalues (descending) of a symmetric tridiagonal (d: m, e: m - 1) and the
// eigenvectors of the largest and the smallest (vectors: m x 2).
void tridiag_extreme_eig(atk_ctx* ctx, const double* d, const double* e, int m, double* values, double* vectors);
void tridiag_eig(atk_ctx* ctx, const double* a, int n, int lda, int nwant, double* values, double* vectors,
                 int ldv, int nvals = 0);
// Bisection (top nvals, descending) + inverse iteration (top nwant vectors of T,
// X: n x nwant, wk: 5 n nwant doubles) on the tridiagonal (d, e).
void tridiag_tail(atk_ctx* ctx, const double* d, const double* e, int n, int nvals, int nwant, double* values,
                  double* X, double* wk);
// trd_big.cu — the same solver for kTridiagMax < n <= kBigEigMax with the
// reduction spread over every SM (one persistent cooperative CTA per SM):
// bounded time on any spectrum; vectors n x nwant (ldv), signs NOT fixed.
constexpr int kBigEigMax = 4096;
void dense_eig_big(atk_ctx* ctx, const double* a, int n, int lda, int nwant, double* values, double* vectors,
                   int ldv, bool exact_sym);
size_t smem_cap_bytes();  // opt-in shared memory per block
// Cholesky factorization in place (lower), status written to *info_dev (0 ok, k>0 pivot k).
void cholesky(atk_ctx* ctx, double* a, int n, int* info_dev);
// Shared-memory Cholesky of G (k x k, k <= kJacobiMax) fused with X = L^{-T};
// *info_dev = 0 or 1 + failing pivot.
// identity_tol > 0: if max |G - I| <= identity_tol, X = I exactly (the last
// CholeskyQR pass on an already orthonormal block)
void cholesky_inv_t(atk_ctx* ctx, const double* g, int k, double* x, int* info_dev, double identity_tol = 0.0);
// Q (m x n, n <= kJacobiMax) = orthonormal basis of span(A) by shifted
// CholeskyQR3; false if a Cholesky pivot failed (caller falls back).
bool orthonormal_basis_cholqr(atk_ctx* ctx, const double* a, int m, int n, double* q);
// Zero the strictly lower triangle of the n x n column-major matrix r.
void zero_lower(atk_ctx* ctx, double* r, int n);
// X = A^{-1} B given the Cholesky factor L (lower) of A: B overwritten.
void cholesky_solve(atk_ctx* ctx, const double* l, int n, double* b, int nrhs);
// Householder thin QR of A (m x n, m >= n): Q (m x n), R (n x n), diag(R) >= 0.
void householder_qr(atk_ctx* ctx, const double* a, int m, int n, double* q, double* r);
// fix_signs (linalg.hpp:34-50) on the columns of V (n x r), optional coupled rows.
void fix_signs(atk_ctx* ctx, double* v, int n, int r, int ldv);
void symmetrize(atk_ctx* ctx, double* a, int n);
void set_identity(atk_ctx* ctx, double* a, int n);
void transpose(atk_ctx* ctx, const double* a, int rows, int cols, double* at);

// eig.cu — sym_eig_top_r on device (linalg.hpp:101-123).
struct EigInfo {
    int method = 0;      // 0 dense Jacobi, 1 ChFSI, 2 tridiagonal, 3 dense (n > 200), 4 explicit SVD
    int iterations = 0;  // ChFSI outer iterations
    double residual = 0;
};
// `psd`: the caller guarantees S is positive semidefinite (a Gram), which
// clamps the filter's lower spectrum bound at 0.  `tol` <= 0: ctx->chfsi_tol.
// `exact_sym`: S is bitwise symmetric (the engine's mirrored Grams): no copy.
EigInfo sym_eig_top_r(atk_ctx* ctx, const double* s_dev, int n, int r, double* values_dev,
                      double* vectors_dev, bool psd = false, double tol = 0.0, bool exact_sym = false);
// Power-of-two range scaling of an engine-owned symmetric S in place (only when max|S| lies
// outside [2^-200, 2^200]; psd: the diagonal bounds every entry); fac_dev (2 doubles): the
// eigenvalue factor and the applied scale.  eig_unscale_values multiplies eigenvalues back.
void eig_scale(atk_ctx* ctx, double* s, int n, bool psd, double* fac_dev);
void eig_unscale_values(atk_ctx* ctx, double* values, int count, const double* fac_dev);

}  // namespace atk
