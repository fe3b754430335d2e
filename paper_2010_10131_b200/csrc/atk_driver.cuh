// atk_driver.cuh — declarations shared by the solver driver, the C ABI and
// the tensor-core / distributed back ends.
#pragma once

#include <vector>

#include "atk_internal.cuh"

namespace atk {

// tensor.hpp:33-39
inline uint64_t mix_seed(uint64_t seed, uint64_t salt) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// selector.hpp:36-52
inline double f_eig(double i) { return 9.0 * i * i * i; }
inline double f_qr(double i, double r) { return 2.0 * i * r * r - (2.0 / 3.0) * r * r * r; }
inline double f_inv(double r) { return 2.0 * r * r * r; }
inline double cost_eig(double i, double r, double j) { return i * i * j + 2.0 * i * r * j + f_eig(i); }
inline double cost_als(double i, double r, double j, int num_iters) {
    const double per_iter = 2.0 * i * j * r + 2.0 * j * r * r + 2.0 * i * j * r + 2.0 * j * r * r +
                            4.0 * i * r * r + 2.0 * f_inv(r);
    return per_iter * num_iters + 2.0 * j * r * r + f_qr(i, r);
}

// contract_simt.cu
void ttt_simt(atk_ctx* ctx, const void* x, const void* y, atk_dtype dt, Split s, uint64_t R,
              double* z_dev, bool sym);
void ttm_simt(atk_ctx* ctx, const void* x, atk_dtype dt, Split s, const double* u_dev, uint64_t R,
              void* y);

// contract_tc.cu — tcgen05 (fp32 storage, kind::tf32) / DMMA (fp64) paths.
bool tc_ttt_supported(atk_ctx* ctx, const atk_tensor* x, const atk_tensor* y, int mode, bool sym);
void tc_ttt(atk_ctx* ctx, const atk_tensor* x, const atk_tensor* y, int mode, double* z_dev, bool sym);
bool tc_ttm_supported(atk_ctx* ctx, const atk_tensor* x, uint64_t R, int mode);
void tc_ttm(atk_ctx* ctx, const atk_tensor* x, const double* u_dev, uint64_t R, int mode,
            atk_tensor* y);

// driver.cu
struct ModeOut {
    std::vector<double> factor;  // I x r host (filled by factor_to_host, or by the ALS path)
    DevBuf<double> factor_dev;   // I x r device: EIG / SVD factors stay resident until the caller needs them
    atk_tensor* shrunk = nullptr;
    int iterations = 0;
    int solver = ATK_SOLVER_EIG;
    EigInfo eig;
    atk_stage_times times{};
};
struct AlsOut {
    std::vector<double> l;  // I x r host
    atk_tensor* rfac = nullptr;
    int iterations_run = 0;
    double comm_ms = 0.0;  // per-iteration YR/GR allreduce (sharded runs)
};
// Host copy of a mode's factor (one D2H + sync; no-op when already on the host).
void factor_to_host(atk_ctx* ctx, ModeOut& m, uint64_t count);
// svd.cu — svd_mode_solver on the explicit unfolding (fp64; one-sided Jacobi)
bool svd_explicit_supported(atk_ctx* ctx, const atk_tensor* y, int mode);
ModeOut svd_mode_explicit(atk_ctx* ctx, const atk_tensor* y, int mode, uint64_t r);
void contract_ttt(atk_ctx* ctx, const atk_tensor* x, const atk_tensor* y, int mode, double* z_dev,
                  bool sym);
// als_tc.cu — one ALS iteration's contractions in one pass over Y (mode 0, fp32, R <= 32)
// Shape gate of the one-pass kernel (I x J unfolding, rank R, num_sms CTAs), shared with the
// roofline selector (api.cu) so the selector prices exactly the schedule that will run.
// fp32 tensors below this many elements take the fp32 CUDA-core contractions instead of tcgen05's
// tf32 operands: at that size every path is launch-bound, and full fp32 keeps tiny slowly-converging
// ALS modes within the 1e-4 parity bar (sweep seed 5339: 22 x 10 x 7, 1.3e-4 on tf32, 2.5e-8 fp32)
constexpr uint64_t kTcMinElems = 8192;
inline bool als_fused_shape_ok(uint64_t I, uint64_t R, uint64_t J, int num_sms) {
    constexpr uint64_t kNB = 32, kJT = 128;  // als_tc.cu NB / JT
    if (R < 1 || R > kNB || I % 128 != 0 || I > 1024 || I < 128) return false;
    if ((2 + I / 128) * kNB > 512) return false;  // TMEM columns
    // per-CTA fp32 chains of at most 16K columns (the other kernels' drain bound)
    const uint64_t per_cta = (J + uint64_t(num_sms) - 1) / uint64_t(num_sms);
    return J >= kJT && per_cta <= 16384 && J < (1ull << 31);
}
bool als_fused_supported(atk_ctx* ctx, const atk_tensor* y, int mode, uint64_t R);
void als_fused_pass(atk_ctx* ctx, const atk_tensor* y, const double* m_dev, uint64_t R, double* yr_dev,
                    double* gr_dev, atk_tensor* rfac_out);
atk_tensor* contract_ttm(atk_ctx* ctx, const atk_tensor* x, const double* u_dev, uint64_t R,
                         int mode);
uint64_t j_of(const atk_tensor* t, int mode);
void check_truncation(const atk_tensor* y, int mode, uint64_t r);
// gram_pre: the mode's Gram already on the device (the host entry streams the
// input and overlaps the mode-0 Gram with the copy); gram_pre_ms its device time.
ModeOut eig_mode(atk_ctx* ctx, const atk_tensor* y, int mode, uint64_t r, int solver_kind,
                 const double* gram_pre = nullptr, double gram_pre_ms = 0.0);
ModeOut als_mode(atk_ctx* ctx, const atk_tensor* y, int mode, uint64_t r, const atk_als_opts& opts,
                 const double* l0_host);
AlsOut als_iterate(atk_ctx* ctx, const atk_tensor* y, int mode, const double* l0_host, uint64_t r,
                   const atk_als_opts& opts);
std::vector<double> als_initial_guess(uint64_t rows, uint64_t r, uint64_t seed, uint64_t mode);
void thin_qr_dev(atk_ctx* ctx, const double* a_dev, uint64_t rows, uint64_t cols, double* q_dev,
                 double* r_dev, double fro_a);
// Mode 0 already decided (and, for EIG/SVD, its Gram computed) by the caller.
struct ModeZeroPre {
    int choice = -1;
    double decide_time = 0.0;
    const double* gram = nullptr;
    double gram_ms = 0.0;
};
atk_tensor* sthosvd(atk_ctx* ctx, const atk_tensor* x, const uint64_t* ranks, atk_selector_fn decide,
                    void* user, const atk_als_opts& opts, double* factors_out,
                    atk_mode_report* reports, const ModeZeroPre* pre = nullptr);
// H2D of the host input into x (device, allocated) in chunks along the last
// mode on a side stream, with the mode-0 Gram of every landed chunk computed
// on the context stream meanwhile (fp64 sum of the chunk Grams into s_dev).
// Returns the Gram's device time (ms).
double upload_with_gram0(atk_ctx* ctx, atk_tensor* x, const void* host, double* s_dev);
atk_tensor* reconstruct(atk_ctx* ctx, const atk_tensor* core, const double* factors,
                        const uint64_t* odims);
double relative_error(atk_ctx* ctx, const atk_tensor* x, const atk_tensor* core,
                      const double* factors);

// dten_io.cu — .dten files (tensor_io.hpp) streamed to / from the device.
struct DtenHeader {
    int order = 0;
    uint64_t dims[ATK_MAX_ORDER] = {};
    uint64_t numel = 0;
};
// Validates the header; with `keep` the open FILE* (positioned at the payload) is returned.
DtenHeader dten_header(const char* path, FILE** keep = nullptr);
atk_tensor* dten_read(atk_ctx* ctx, const char* path, atk_dtype dt);
void dten_write(atk_ctx* ctx, const atk_tensor* t, const char* path);

// dist.cu — NCCL over NVLink (one process per GPU).
void comm_init(atk_ctx* ctx, const void* unique_id, int rank, int world);
void comm_destroy(atk_ctx* ctx);
void nccl_unique_id(void* out128);
void comm_init_host(atk_ctx* ctx, const atk_host_collectives* coll, int rank, int world);
void allreduce_sum(atk_ctx* ctx, double* buf, uint64_t count, double* comm_ms);
void allreduce_sum2(atk_ctx* ctx, double* a, uint64_t na, double* b, uint64_t nb, double* comm_ms);
atk_tensor* allgather_last_mode(atk_ctx* ctx, const atk_tensor* local);
uint64_t comm_global_last(atk_ctx* ctx, const atk_tensor* local);
void allreduce_sym(atk_ctx* ctx, double* s, uint64_t n, double* comm_ms);  // packed upper triangle
void comm_end_call(atk_ctx* ctx);
void comm_stats(const atk_ctx* ctx, atk_comm_stats* out);
void comm_stats_reset(atk_ctx* ctx);

}  // namespace atk
