// driver.cu — the per-mode solvers (solvers.hpp) and the st-HOSVD mode loop
// (sthosvd.hpp) orchestrated on the device.  Host code here only sequences
// kernels, calls the selector hook and moves small results; every
// contraction, factorisation and reduction runs in the CUDA kernels.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <random>
#include <string>
#include <vector>

#include "atk_driver.cuh"

namespace atk {

// ------------------------------------------------------------------ contractions
void contract_ttt(atk_ctx* ctx, const atk_tensor* x, const atk_tensor* y, int mode, double* z_dev,
                  bool sym) {
    const Split s = loop_split(x->dims, x->order, mode);
    const uint64_t R = y->dims[mode];
    if (s.P * s.O == 0 || s.I == 0 || R == 0) return;
    if (!ctx->force_simt && x->numel() >= kTcMinElems && tc_ttt_supported(ctx, x, y, mode, sym)) {
        tc_ttt(ctx, x, y, mode, z_dev, sym);
        return;
    }
    // fp64, first or last mode: the unfolding is a plain column-major matrix
    // (kernels.hpp:49-58), so the pipelined DMMA GEMM (cp.async ring, split-K
    // with a fixed-order reduction) applies directly; Grams are symmetrised
    // exactly afterwards (kernels.hpp:127-138)
    if (!ctx->force_simt && x->dtype == ATK_F64 && y->dtype == ATK_F64 && (s.P == 1 || s.O == 1) &&
        s.I <= 0x7fffffffULL && R <= 0x7fffffffULL && s.P * s.O <= 0x7fffffffULL) {
        const auto* xd = static_cast<const double*>(x->data);
        const auto* yd = static_cast<const double*>(y->data);
        if (sym && x == y && s.I <= 160) {  // the Gram as a SYRK: upper blocks only, both triangles written
            if (s.P == 1) dsyrk_upper(ctx, false, int(s.I), int(s.O), 1.0, xd, int(s.I), z_dev, int(s.I));
            else dsyrk_upper(ctx, true, int(s.I), int(s.P), 1.0, xd, int(s.P), z_dev, int(s.I));
            return;
        }
        if (s.P == 1)  // Z = X(I x J) Y(R x J)^T
            dgemm(ctx, false, true, int(s.I), int(R), int(s.O), 1.0, xd, int(s.I), yd, int(R), 0.0, z_dev, int(s.I));
        else  // Z = X(P x I)^T Y(P x R)
            dgemm(ctx, true, false, int(s.I), int(R), int(s.P), 1.0, xd, int(s.P), yd, int(s.P), 0.0, z_dev, int(s.I));
        if (sym) symmetrize(ctx, z_dev, int(s.I));
        return;
    }
    ttt_simt(ctx, x->data, y->data, x->dtype, s, R, z_dev, sym);
}

atk_tensor* contract_ttm(atk_ctx* ctx, const atk_tensor* x, const double* u_dev, uint64_t R,
                         int mode) {
    uint64_t od[ATK_MAX_ORDER];
    for (int m = 0; m < x->order; ++m) od[m] = x->dims[m];
    od[mode] = R;
    atk_tensor* y = new_tensor(ctx, x->dtype, x->order, od);
    const Split s = loop_split(x->dims, x->order, mode);
    if (!ctx->force_simt && x->numel() >= kTcMinElems && tc_ttm_supported(ctx, x, R, mode)) {
        tc_ttm(ctx, x, u_dev, R, mode, y);
    } else {
        ttm_simt(ctx, x->data, x->dtype, s, u_dev, R, y->data);
    }
    return y;
}

uint64_t j_of(const atk_tensor* t, int mode) {
    uint64_t j = 1;
    for (int m = 0; m < t->order; ++m)
        if (m != mode) j *= t->dims[m];
    return j;
}

// solvers.hpp:35-41
void check_truncation(const atk_tensor* y, int mode, uint64_t r) {
    check_mode(y->order, mode);
    if (r < 1 || r > y->dims[mode])
        fail(ATK_RANK_EXCEEDS_DIM, "truncation " + std::to_string(r) + " invalid for mode " +
                                       std::to_string(mode) + " of dimension " +
                                       std::to_string(y->dims[mode]));
}

// ------------------------------------------------------------------ EIG / SVD
// eig_mode_solver (solvers.hpp:64-73): gram -> sym_eig_top_r -> ttm(Y, U^T).
ModeOut eig_mode(atk_ctx* ctx, const atk_tensor* y, int mode, uint64_t r, int solver_kind,
                 const double* gram_pre, double gram_pre_ms) {
    check_truncation(y, mode, r);
    const uint64_t I = y->dims[mode], J = j_of(y, mode);
    // the unfolding's column count: under a sharded sthosvd the local J scaled to the global last
    // mode (every rank then checks the same bound and fails alike)
    uint64_t Jg = J;
    if (ctx->comm && !ctx->replicated && ctx->global_last && mode != y->order - 1)
        Jg = J / y->dims[y->order - 1] * ctx->global_last;
    if (solver_kind == ATK_SOLVER_SVD && r > std::min(I, Jg))
        fail(ATK_RANK_TOO_LARGE, "truncation exceeds the rank bound of the unfolding");
    // the reference's SVD works on the explicit unfolding (solvers.hpp:142-162);
    // fp32 data carries no more than the Gram route's precision (sqrt(eps64)
    // relative sigma), sharded modes have J spread over the ranks: Gram route
    if (solver_kind == ATK_SOLVER_SVD && !gram_pre && svd_explicit_supported(ctx, y, mode))
        return svd_mode_explicit(ctx, y, mode, r);
    ModeOut out;
    out.solver = solver_kind;
    StageTimer tm(ctx);
    DevBuf<double> S(ctx, gram_pre ? 0 : I * I);
    const double* Sg = gram_pre;
    if (!gram_pre) {
        tm.start();
        contract_ttt(ctx, y, y, mode, S.get(), true);
        if (ctx->comm && !ctx->replicated) allreduce_sym(ctx, S.get(), I, &out.times.comm_ms);
        out.times.gram_ms = tm.stop_ms(kStageGram);
        Sg = S.get();
    } else {
        out.times.gram_ms = gram_pre_ms;
    }
    record_gemm((long long)(I * I) * (long long)J);

    DevBuf<double> vals(ctx, r), vecs(ctx, I * r), ut(ctx, I * r);
    tm.start();
    // S is a Gram (PSD).  A tf32-computed Gram carries ~1e-6 relative error, so
    // resolving its eigenpairs beyond a 1e-9 Ritz residual buys nothing (the
    // factor error is ~residual / gap, far below the tf32 Gram error); fp64 keeps 1e-12.
    out.eig = sym_eig_top_r(ctx, Sg, int(I), int(r), vals.get(), vecs.get(), true,
                            y->dtype == ATK_F32 ? std::max(1e-9, ctx->chfsi_tol) : ctx->chfsi_tol,
                            // the engine's Grams are mirrored (bitwise symmetric); an allreduce
                            // may sum (i, j) and (j, i) in different orders, so sharded modes symmetrise
                            /*exact_sym=*/!ctx->comm || ctx->replicated);
    out.times.eig_ms = tm.stop_ms(kStageEig);

    tm.start();
    transpose(ctx, vecs.get(), int(I), int(r), ut.get());  // U^T : r x I
    out.shrunk = contract_ttm(ctx, y, ut.get(), r, mode);
    record_gemm(2LL * (long long)(r * J) * (long long)I);
    out.times.ttm_ms = tm.stop_ms(kStageTtm);
    // the factor stays on the device: sthosvd downloads all of them once at the
    // end, so no host round trip sits between one mode and the next
    out.factor_dev = std::move(vecs);
    out.times.total_ms = out.times.gram_ms + out.times.eig_ms + out.times.ttm_ms;
    return out;
}

void factor_to_host(atk_ctx* ctx, ModeOut& m, uint64_t count) {
    if (!m.factor.empty() || !m.factor_dev.get()) return;
    m.factor.resize(count);
    ATK_CUDA(cudaMemcpyAsync(m.factor.data(), m.factor_dev.get(), count * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    ATK_CUDA(cudaStreamSynchronize(ctx->stream));
}

// ------------------------------------------------------------------ ALS
// spd_solve(A, I) (linalg.hpp:169-177) on the device: returns A^{-1}.
// (A)^{-1} for SPD A, as the reference's spd_solve(A, I) (solvers.hpp:104,109;
// linalg.hpp:169-177, NotSPD on a non-positive pivot).  n <= 112: one-CTA
// Cholesky fused with X = L^{-T}, then A^{-1} = X X^T (two launches instead of
// a column-serial triangular solve).
// With `info_slot` (n <= 112) the pivot status is left on the device for the
// caller to check later (als_iterate checks all of its solves once, after the
// loop: no host round trip per iteration); otherwise it is checked here.
static void spd_inverse(atk_ctx* ctx, const double* a, int n, double* inv, int* info_slot = nullptr) {
    DevBuf<int> info(ctx, info_slot ? 0 : 1);
    int h = 0;
    if (n <= kJacobiMax) {
        DevBuf<double> x(ctx, size_t(n) * n);
        cholesky_inv_t(ctx, a, n, x.get(), info_slot ? info_slot : info.get());
        dgemm(ctx, false, true, n, n, n, 1.0, x.get(), n, x.get(), n, 0.0, inv, n);
        if (info_slot) return;
        ATK_CUDA(cudaMemcpyAsync(&h, info.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        ATK_CUDA(cudaStreamSynchronize(ctx->stream));
        if (h != 0) fail(ATK_NOT_SPD, "Cholesky factorization hit a non-positive pivot");
        return;
    }
    if (info_slot) {  // the large path reports through its own sync below
        ATK_CUDA(cudaMemsetAsync(info_slot, 0, sizeof(int), ctx->stream));
        info = DevBuf<int>(ctx, 1);
    }
    DevBuf<double> l(ctx, size_t(n) * n);
    ATK_CUDA(cudaMemcpyAsync(l.get(), a, size_t(n) * n * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
    cholesky(ctx, l.get(), n, info.get());
    ATK_CUDA(cudaMemcpyAsync(&h, info.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ATK_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h != 0) fail(ATK_NOT_SPD, "Cholesky factorization hit a non-positive pivot");
    set_identity(ctx, inv, n);
    cholesky_solve(ctx, l.get(), n, inv, n);
}

std::vector<double> als_initial_guess(uint64_t rows, uint64_t r, uint64_t seed, uint64_t mode) {
    // solvers.hpp:125-128 — same libstdc++ engine + distribution as the reference.
    std::vector<double> l0(rows * r);
    std::mt19937_64 rng(mix_seed(seed, mode));
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (auto& v : l0) v = gauss(rng);
    return l0;
}

// The Gram route for ALS (see als_iterate): fp32 tensors whose Gram runs on tcgen05, 2 <= iters,
// and the roofline says Gram + one TTM beats the iterations' passes over Y (the one-pass kernel
// when it applies, else the two-pass TTM + TTT schedule).
bool als_gram_route(atk_ctx* ctx, const atk_tensor* y, int mode, uint64_t r, int iters) {
    if (!ctx->als_gram || ctx->force_simt || y->dtype != ATK_F32 || iters < 2) return false;
    // sharded: the local J differs between ranks with uneven slabs, and every rank must take the
    // same schedule (its collectives); the per-iteration allreduce path stays
    if (ctx->comm && !ctx->replicated) return false;
    const uint64_t I = y->dims[mode], J = j_of(y, mode);
    if (I > 4096 || r > I || y->numel() < kTcMinElems || !tc_ttt_supported(ctx, y, y, mode, true)) return false;
    atk_roofline_params p;
    atk_roofline_params_default(&p, ATK_F32, iters);
    const double bw = p.hbm_gbs * 1e9, P = p.tf32_tflops * 1e12;
    const double t_gram = std::max(double(I) * I * J / P, 4.0 * I * J / bw) + 4.0 * (I + r) * J / bw;
    const double t_als = atk_roofline_time_als_mode(&p, mode, double(I), double(r), double(J));
    return t_gram < t_als;
}

// als_iterate (solvers.hpp:88-118).  L stays on the device; rfac is returned.
AlsOut als_iterate(atk_ctx* ctx, const atk_tensor* y, int mode, const double* l0_host, uint64_t r,
                   const atk_als_opts& opts) {
    check_mode(y->order, mode);
    if (opts.num_iters < 1) fail(ATK_ERROR, "num_iters must be at least 1");
    const uint64_t I = y->dims[mode], J = j_of(y, mode);
    AlsOut out;
    DevBuf<double> L(ctx, I * r), Lt(ctx, I * r), GL(ctx, r * r), GLi(ctx, r * r), YR(ctx, I * r),
        GR(ctx, r * r), GRi(ctx, r * r), nxt(ctx, I * r);
    DevBuf<int> infos(ctx, 2 * size_t(opts.num_iters));  // NotSPD status of every solve
    ATK_CUDA(cudaMemsetAsync(infos.get(), 0, 2 * size_t(opts.num_iters) * sizeof(int), ctx->stream));
    auto check_spd = [&](int upto) {  // linalg.hpp:169-177 NotSPD, in iteration order
        std::vector<int> h(2 * size_t(upto));
        ATK_CUDA(cudaMemcpyAsync(h.data(), infos.get(), h.size() * sizeof(int), cudaMemcpyDeviceToHost,
                                 ctx->stream));
        ATK_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int v : h)
            if (v != 0) fail(ATK_NOT_SPD, "Cholesky factorization hit a non-positive pivot");
    };
    ATK_CUDA(cudaMemcpyAsync(L.get(), l0_host, I * r * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    static const bool trace = std::getenv("ATK_TRACE") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto mark = [&](const char* what, int it) {
        if (!trace) return;
        cudaStreamSynchronize(ctx->stream);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[atk als I=%llu r=%llu J=%llu it=%d] %-8s %8.3f ms\n", (unsigned long long)I,
                     (unsigned long long)r, (unsigned long long)J, it, what,
                     std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    mark("start", -1);
    // ALS on the mode's Gram (option "als_gram"): with S = Y_(n) Y_(n)^T formed once, every
    // iteration's contractions collapse to I x I x R products, YR = Y rfac^T = S M^T and
    // GR = rfac rfac^T = M S M^T (M = (L^T L)^{-1} L^T, rfac = M Y_(n)), the same iterates in
    // exact arithmetic (solvers.hpp:88-118); rfac itself is formed once, after the loop.  On
    // B200 the Gram runs on the tensor cores while every ALS pass is HBM-bound, so this wins
    // whenever I^2 J / P + s I J / BW (Gram + final TTM) < iters x (one-pass ALS time).
    if (als_gram_route(ctx, y, mode, r, opts.num_iters)) {
        DevBuf<double> S(ctx, I * I), M(ctx, I * r);
        contract_ttt(ctx, y, y, mode, S.get(), true);
        mark("gram", -1);
        for (int k = 0; k < opts.num_iters; ++k) {
            dgemm(ctx, true, false, int(r), int(r), int(I), 1.0, L.get(), int(I), L.get(), int(I), 0.0, GL.get(),
                  int(r));
            record_gemm(2LL * (long long)(r * r) * (long long)I);
            spd_inverse(ctx, GL.get(), int(r), GLi.get(), infos.get() + 2 * k);
            dgemm(ctx, false, true, int(r), int(I), int(r), 1.0, GLi.get(), int(r), L.get(), int(I), 0.0, M.get(),
                  int(r));
            // YR = S M^T (I x R), GR = M YR (R x R)
            dgemm(ctx, false, true, int(I), int(r), int(I), 1.0, S.get(), int(I), M.get(), int(r), 0.0, YR.get(),
                  int(I));
            dgemm(ctx, false, false, int(r), int(r), int(I), 1.0, M.get(), int(r), YR.get(), int(I), 0.0, GR.get(),
                  int(r));
            symmetrize(ctx, GR.get(), int(r));
            // the reference's logical contractions: W = ttm, rfac = ttm, YR = ttt, GR = ttt
            record_gemm(2LL * (long long)(r * J) * (long long)I);
            record_gemm(2LL * (long long)(r * J) * (long long)r);
            record_gemm(2LL * (long long)(I * r) * (long long)J);
            record_gemm(2LL * (long long)(r * r) * (long long)J);
            spd_inverse(ctx, GR.get(), int(r), GRi.get(), infos.get() + 2 * k + 1);
            dgemm(ctx, false, false, int(I), int(r), int(r), 1.0, YR.get(), int(I), GRi.get(), int(r), 0.0,
                  nxt.get(), int(I));
            record_gemm(2LL * (long long)(I * r) * (long long)r);
            out.iterations_run = k + 1;
            mark("iter", k);
            double change = 0.0;
            if (opts.rel_tol > 0.0) {
                check_spd(k + 1);
                const double diff = diff_norm2_sq(ctx, nxt.get(), L.get(), ATK_F64, I * r);
                const double base = norm2_sq(ctx, L.get(), ATK_F64, I * r);
                change = base > 0.0 ? std::sqrt(diff / base) : 0.0;
            }
            std::swap(L, nxt);
            if (opts.rel_tol > 0.0 && change <= opts.rel_tol) break;
        }
        // rfac of the last iteration (its M): one pass over Y
        out.rfac = contract_ttm(ctx, y, M.get(), r, mode);
        mark("rfac", -1);
    } else if (als_fused_supported(ctx, y, mode, r)) {
        // One pass over Y per iteration (als_tc.cu): rfac = M Y_(0) with
        // M = (L^T L)^{-1} L^T, and YR / GR, from the same streamed tiles.  The
        // update order, seeding, NotSPD checks and early stop are those below.
        uint64_t rdims[ATK_MAX_ORDER];
        for (int m = 0; m < y->order; ++m) rdims[m] = y->dims[m];
        rdims[mode] = r;
        DevBuf<double> M(ctx, I * r);
        out.rfac = new_tensor(ctx, y->dtype, y->order, rdims);
        for (int k = 0; k < opts.num_iters; ++k) {
            dgemm(ctx, true, false, int(r), int(r), int(I), 1.0, L.get(), int(I), L.get(), int(I), 0.0, GL.get(),
                  int(r));
            record_gemm(2LL * (long long)(r * r) * (long long)I);
            spd_inverse(ctx, GL.get(), int(r), GLi.get(), infos.get() + 2 * k);
            dgemm(ctx, false, true, int(r), int(I), int(r), 1.0, GLi.get(), int(r), L.get(), int(I), 0.0, M.get(),
                  int(r));
            // rfac is only consumed after the last iteration (shrunk = rfac x_n R): with a
            // fixed count only that pass writes it; with an early stop every pass does
            const bool keep = opts.rel_tol > 0.0 || k + 1 == opts.num_iters;
            als_fused_pass(ctx, y, M.get(), r, YR.get(), GR.get(), keep ? out.rfac : nullptr);
            // the reference's logical contractions: W = ttm, rfac = ttm, YR = ttt, GR = ttt
            record_gemm(2LL * (long long)(r * J) * (long long)I);
            record_gemm(2LL * (long long)(r * J) * (long long)r);
            record_gemm(2LL * (long long)(I * r) * (long long)J);
            record_gemm(2LL * (long long)(r * r) * (long long)J);
            mark("fused", k);
            if (ctx->comm && !ctx->replicated)
                allreduce_sum2(ctx, YR.get(), I * r, GR.get(), r * r, &out.comm_ms);
            spd_inverse(ctx, GR.get(), int(r), GRi.get(), infos.get() + 2 * k + 1);
            dgemm(ctx, false, false, int(I), int(r), int(r), 1.0, YR.get(), int(I), GRi.get(), int(r), 0.0,
                  nxt.get(), int(I));
            record_gemm(2LL * (long long)(I * r) * (long long)r);
            out.iterations_run = k + 1;
            double change = 0.0;
            if (opts.rel_tol > 0.0) {
                check_spd(k + 1);
                const double diff = diff_norm2_sq(ctx, nxt.get(), L.get(), ATK_F64, I * r);
                const double base = norm2_sq(ctx, L.get(), ATK_F64, I * r);
                change = base > 0.0 ? std::sqrt(diff / base) : 0.0;
            }
            std::swap(L, nxt);
            if (opts.rel_tol > 0.0 && change <= opts.rel_tol) break;
        }
    } else
    for (int k = 0; k < opts.num_iters; ++k) {
        transpose(ctx, L.get(), int(I), int(r), Lt.get());
        atk_tensor* w = contract_ttm(ctx, y, Lt.get(), r, mode);  // W = Y x_n L^T
        mark("ttm_w", k);
        record_gemm(2LL * (long long)(r * J) * (long long)I);
        dgemm(ctx, true, false, int(r), int(r), int(I), 1.0, L.get(), int(I), L.get(), int(I), 0.0,
              GL.get(), int(r));
        record_gemm(2LL * (long long)(r * r) * (long long)I);
        spd_inverse(ctx, GL.get(), int(r), GLi.get(), infos.get() + 2 * k);
        mark("gl_inv", k);
        if (out.rfac) atk_tensor_free(out.rfac);
        mark("free", k);
        out.rfac = contract_ttm(ctx, w, GLi.get(), r, mode);  // rfac = W x_n (L^T L)^{-1}
        record_gemm(2LL * (long long)(r * J) * (long long)r);
        atk_tensor_free(w);
        mark("rfac", k);
        contract_ttt(ctx, y, out.rfac, mode, YR.get(), false);  // YR = Y_(n) rfac_(n)^T
        record_gemm(2LL * (long long)(I * r) * (long long)J);
        mark("ttt_yr", k);
        contract_ttt(ctx, out.rfac, out.rfac, mode, GR.get(), true);  // symmetric: the Gram kernels
        record_gemm(2LL * (long long)(r * r) * (long long)J);
        mark("gram_gr", k);
        // Sharded (SURVEY §8(e) "ALS modes"): YR and GR are sums over J, so the
        // local partials are combined with one grouped allreduce per iteration;
        // L, its Gram and every R x R solve are then replicated bit-identically.
        if (ctx->comm && !ctx->replicated) allreduce_sum2(ctx, YR.get(), I * r, GR.get(), r * r, &out.comm_ms);
        spd_inverse(ctx, GR.get(), int(r), GRi.get(), infos.get() + 2 * k + 1);
        dgemm(ctx, false, false, int(I), int(r), int(r), 1.0, YR.get(), int(I), GRi.get(), int(r),
              0.0, nxt.get(), int(I));
        record_gemm(2LL * (long long)(I * r) * (long long)r);
        mark("solves", k);
        out.iterations_run = k + 1;
        double change = 0.0;
        if (opts.rel_tol > 0.0) {
            check_spd(k + 1);
            const double diff = diff_norm2_sq(ctx, nxt.get(), L.get(), ATK_F64, I * r);
            const double base = norm2_sq(ctx, L.get(), ATK_F64, I * r);
            change = base > 0.0 ? std::sqrt(diff / base) : 0.0;
        }
        std::swap(L, nxt);
        if (opts.rel_tol > 0.0 && change <= opts.rel_tol) break;
    }
    check_spd(out.iterations_run);
    out.l.resize(I * r);
    ATK_CUDA(cudaMemcpyAsync(out.l.data(), L.get(), I * r * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    ATK_CUDA(cudaStreamSynchronize(ctx->stream));
    return out;
}

// thin_qr (linalg.hpp:126-149) on the device.  Q R with diag(R) >= 0 is
// unique for a full-rank A, so any stable method reproduces the reference's
// Householder result: n <= 112 uses shifted CholeskyQR3 (GEMM-shaped) and
// R = Q^T A; a failed Cholesky (numerically rank-deficient input) falls back to
// the one-CTA Householder kernel, which reports RankDeficient exactly as the
// reference does (|r_kk| < 1e-12 ||A||_F).
void thin_qr_dev(atk_ctx* ctx, const double* a_dev, uint64_t rows, uint64_t cols, double* q_dev,
                 double* r_dev, double fro_a) {
    if (rows < cols) fail(ATK_SHAPE_MISMATCH, "thin_qr expects rows >= cols");
    if (orthonormal_basis_cholqr(ctx, a_dev, int(rows), int(cols), q_dev)) {
        dgemm(ctx, true, false, int(cols), int(cols), int(rows), 1.0, q_dev, int(rows), a_dev, int(rows), 0.0, r_dev,
              int(cols));
        zero_lower(ctx, r_dev, int(cols));
    } else {
        householder_qr(ctx, a_dev, int(rows), int(cols), q_dev, r_dev);
    }
    std::vector<double> rh(cols * cols);
    ATK_CUDA(cudaMemcpyAsync(rh.data(), r_dev, cols * cols * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    ATK_CUDA(cudaStreamSynchronize(ctx->stream));
    const double floor = 1e-12 * fro_a;
    for (uint64_t k = 0; k < cols; ++k)
        if (std::fabs(rh[k + cols * k]) < floor)
            fail(ATK_RANK_DEFICIENT, "QR diagonal " + std::to_string(k) + " below tolerance");
}

// als_mode_solver (solvers.hpp:122-138).
ModeOut als_mode(atk_ctx* ctx, const atk_tensor* y, int mode, uint64_t r, const atk_als_opts& opts,
                 const double* l0_host) {
    check_truncation(y, mode, r);
    const uint64_t I = y->dims[mode], J = j_of(y, mode);
    std::vector<double> seeded;
    if (!l0_host) {
        seeded = als_initial_guess(I, r, opts.seed, uint64_t(mode));
        l0_host = seeded.data();
    }
    ModeOut out;
    out.solver = ATK_SOLVER_ALS;
    StageTimer tm(ctx);
    tm.start();
    AlsOut it = als_iterate(ctx, y, mode, l0_host, r, opts);
    DevBuf<double> L(ctx, I * r), Q(ctx, I * r), Rm(ctx, r * r);
    ATK_CUDA(cudaMemcpyAsync(L.get(), it.l.data(), I * r * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    double fro = 0.0;
    for (double v : it.l) fro += v * v;
    thin_qr_dev(ctx, L.get(), I, r, Q.get(), Rm.get(), std::sqrt(fro));
    out.shrunk = contract_ttm(ctx, it.rfac, Rm.get(), r, mode);  // shrunk = rfac x_n R
    record_gemm(2LL * (long long)(r * J) * (long long)r);
    atk_tensor_free(it.rfac);
    out.factor.resize(I * r);
    ATK_CUDA(cudaMemcpyAsync(out.factor.data(), Q.get(), I * r * sizeof(double),
                             cudaMemcpyDeviceToHost, ctx->stream));
    ATK_CUDA(cudaStreamSynchronize(ctx->stream));
    out.times.als_ms = tm.stop_ms(kStageAls);
    out.times.comm_ms = it.comm_ms;
    out.times.total_ms = out.times.als_ms;
    out.iterations = it.iterations_run;
    return out;
}

// ------------------------------------------------------------------ st-HOSVD
static double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// sthosvd (sthosvd.hpp:126-194).  The input is never copied: mode 0 reads x
// directly and every later mode reads the previous shrunk tensor.
atk_tensor* sthosvd(atk_ctx* ctx, const atk_tensor* x, const uint64_t* ranks, atk_selector_fn decide,
                    void* user, const atk_als_opts& opts, double* factors_out,
                    atk_mode_report* reports, const ModeZeroPre* pre) {
    check_tensor(x, "sthosvd input");
    const int order = x->order;
    // sharded input: the last mode's GLOBAL size, from one collective up front
    // (every rank reaches it, so a bad rank fails on all ranks alike); the
    // global J of every sharded mode follows from it without further exchange
    const uint64_t g_last = ctx->comm ? comm_global_last(ctx, x) : x->dims[order - 1];
    struct GlobalLastScope {  // the mode solvers' view of the global last-mode size
        atk_ctx* c;
        GlobalLastScope(atk_ctx* cc, uint64_t g) : c(cc) { c->global_last = g; }
        ~GlobalLastScope() { c->global_last = 0; }
    } global_last_scope(ctx, ctx->comm ? g_last : 0);
    for (int n = 0; n < order; ++n) {
        const uint64_t dn = n == order - 1 ? g_last : x->dims[n];
        if (ranks[n] < 1 || ranks[n] > dn)
            fail(ATK_RANK_EXCEEDS_DIM, "truncation " + std::to_string(ranks[n]) +
                                           " invalid for mode " + std::to_string(n) +
                                           " of dimension " + std::to_string(dn));
    }
    const atk_tensor* work = x;
    atk_tensor* owned = nullptr;
    size_t foff = 0;
    size_t ftotal = 0;
    for (int n = 0; n < order; ++n) ftotal += (n == order - 1 ? g_last : x->dims[n]) * ranks[n];
    DevBuf<double> fdev(ctx, ftotal);  // every device-resident factor, downloaded once at the end
    std::vector<std::pair<size_t, size_t>> dev_segs;
    // stage times are resolved from their events after the final sync
    struct DeferScope {
        atk_ctx* c;
        explicit DeferScope(atk_ctx* cc) : c(cc) {
            for (auto& d : c->deferred) { cudaEventDestroy(d.a); cudaEventDestroy(d.b); }
            c->deferred.clear();
            c->defer_timing = true;
        }
        ~DeferScope() {
            c->defer_timing = false;
            for (auto& d : c->deferred) { cudaEventDestroy(d.a); cudaEventDestroy(d.b); }
            c->deferred.clear();
        }
    } defer_scope(ctx);
    try {
        for (int n = 0; n < order; ++n) {
            ctx->timing_mode = n;
            // after the all-gather the last mode runs on the full (replicated)
            // tensor: its Gram / YR / GR are complete on every rank, no allreduce
            ctx->replicated = ctx->comm && n == order - 1;
            if (ctx->comm && n == order - 1) {
                // the shard mode: gather the (small) shrunk tensor, finish replicated
                atk_tensor* full = allgather_last_mode(ctx, work);
                if (owned) atk_tensor_free(owned);
                owned = full;
                work = full;
            }
            const uint64_t I = work->dims[n], r = ranks[n];
            uint64_t J = j_of(work, n);
            if (ctx->comm && n < order - 1) J = J / work->dims[order - 1] * g_last;
            atk_mode_report rep{};
            rep.mode = n;
            for (int m = 0; m < order; ++m) rep.dims_before[m] = work->dims[m];
            rep.predicted_cost_eig = cost_eig(double(I), double(r), double(J));
            rep.predicted_cost_als = cost_als(double(I), double(r), double(J), opts.num_iters);
            const bool use_pre = n == 0 && pre && pre->choice >= 0;
            const auto td = std::chrono::steady_clock::now();
            const int choice = use_pre ? pre->choice : (decide ? decide(user, n, I, r, J) : ATK_SOLVER_EIG);
            rep.selector_decision_time = use_pre ? pre->decide_time : seconds_since(td);
            if (choice < 0 || choice > 2) fail(ATK_INVALID_ARGUMENT, "selector callback failed");
            const auto ts = std::chrono::steady_clock::now();
            ModeOut mo;
            try {
                if (choice == ATK_SOLVER_ALS)
                    mo = als_mode(ctx, work, n, r, opts, nullptr);
                else if (use_pre && pre->gram)
                    mo = eig_mode(ctx, work, n, r, choice, pre->gram, pre->gram_ms);
                else
                    mo = eig_mode(ctx, work, n, r, choice);
            } catch (const Error& e) {
                // sthosvd.hpp:177-183: NotSPD / NoConvergence keep their type,
                // every other library error becomes a plain Error, all prefixed.
                atk_status code = e.code;
                if (code != ATK_NOT_SPD && code != ATK_NO_CONVERGENCE && code != ATK_CUDA_ERROR &&
                    code != ATK_OOM && code != ATK_NCCL_ERROR)
                    code = ATK_ERROR;
                fail(code, "mode " + std::to_string(n + 1) + ": " + e.what());
            }
            rep.solver_time = seconds_since(ts);
            rep.solver_used = mo.solver;
            rep.iterations_run = mo.iterations;
            rep.eig_method = mo.eig.method;
            rep.times = mo.times;
            const uint64_t fcount = work->dims[n] * r;
            if (mo.factor_dev.get()) {
                ATK_CUDA(cudaMemcpyAsync(fdev.get() + foff, mo.factor_dev.get(), fcount * sizeof(double),
                                         cudaMemcpyDeviceToDevice, ctx->stream));
                dev_segs.push_back({foff, fcount});
            } else {
                std::copy(mo.factor.begin(), mo.factor.end(), factors_out + foff);  // ALS: already on the host
            }
            foff += fcount;
            if (owned) atk_tensor_free(owned);
            owned = mo.shrunk;
            work = owned;
            for (int m = 0; m < order; ++m) rep.dims_after[m] = work->dims[m];
            if (reports) reports[n] = rep;
        }
    } catch (...) {
        ctx->replicated = false;
        comm_end_call(ctx);
        if (owned) atk_tensor_free(owned);
        throw;
    }
    ctx->replicated = false;
    comm_end_call(ctx);
    double* h = dev_segs.empty() ? nullptr : static_cast<double*>(pinned_host(ctx, ftotal * sizeof(double)));
    if (h) ATK_CUDA(cudaMemcpyAsync(h, fdev.get(), ftotal * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ATK_CUDA(cudaStreamSynchronize(ctx->stream));
    for (const auto& sg : dev_segs) std::copy(h + sg.first, h + sg.first + sg.second, factors_out + sg.first);
    if (reports) {
        for (const auto& d : ctx->deferred) {
            float ms = 0.f;
            ATK_CUDA(cudaEventElapsedTime(&ms, d.a, d.b));
            atk_stage_times& t = reports[d.mode].times;
            double* f[] = {&t.gram_ms, &t.eig_ms, &t.ttm_ms, &t.als_ms, &t.comm_ms};
            *f[d.field] += double(ms);
        }
        for (int n = 0; n < order; ++n) {
            atk_stage_times& t = reports[n].times;
            t.total_ms = t.gram_ms + t.eig_ms + t.ttm_ms + t.als_ms;
        }
    }
    return owned;
}

double upload_with_gram0(atk_ctx* ctx, atk_tensor* x, const void* host, double* s_dev) {
    const uint64_t I = x->dims[0], J = j_of(x, 0), esz = x->elem_bytes();
    const uint64_t col_bytes = I * esz;
    // ~32 chunks of >= 256 MB: the copy engine stays saturated, every chunk Gram
    // still fills the SMs, and the last (unhidden) chunk Gram is short
    uint64_t cols = std::max<uint64_t>(1, std::max<uint64_t>((256ull << 20) / col_bytes, (J + 31) / 32));
    cols = std::min(cols, J);
    const uint64_t nchunks = (J + cols - 1) / cols;
    cudaStream_t cs = nullptr;
    ATK_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    std::vector<cudaEvent_t> landed(nchunks, nullptr);
    cudaEvent_t g0 = nullptr, g1 = nullptr;
    double ms = 0.0;
    auto cleanup = [&] {
        for (auto& e : landed)
            if (e) cudaEventDestroy(e);
        if (g0) cudaEventDestroy(g0);
        if (g1) cudaEventDestroy(g1);
        cudaStreamDestroy(cs);
    };
    try {
        for (auto& e : landed) ATK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ATK_CUDA(cudaEventCreate(&g0));
        ATK_CUDA(cudaEventCreate(&g1));
        // the destination must be allocated before the side stream writes into it
        ATK_CUDA(cudaEventRecord(landed[0], ctx->stream));
        ATK_CUDA(cudaStreamWaitEvent(cs, landed[0], 0));
        for (uint64_t c = 0; c < nchunks; ++c) {
            const uint64_t j0 = c * cols, nc = std::min(cols, J - j0);
            ATK_CUDA(cudaMemcpyAsync(static_cast<char*>(x->data) + j0 * col_bytes,
                                     static_cast<const char*>(host) + j0 * col_bytes, nc * col_bytes,
                                     cudaMemcpyHostToDevice, cs));
            ATK_CUDA(cudaEventRecord(landed[c], cs));
        }
        DevBuf<double> part(ctx, I * I);
        bool timing = false;
        for (uint64_t c = 0; c < nchunks; ++c) {
            const uint64_t j0 = c * cols, nc = std::min(cols, J - j0);
            ATK_CUDA(cudaStreamWaitEvent(ctx->stream, landed[c], 0));
            if (!timing) {
                ATK_CUDA(cudaEventRecord(g0, ctx->stream));
                timing = true;
            }
            atk_tensor view;  // mode-0 matricization of the chunk: I x nc, in place
            view.ctx = ctx;
            view.dtype = x->dtype;
            view.order = 2;
            view.dims[0] = I;
            view.dims[1] = nc;
            view.data = static_cast<char*>(x->data) + j0 * col_bytes;
            contract_ttt(ctx, &view, &view, 0, c == 0 ? s_dev : part.get(), true);
            if (c > 0) axpy(ctx, s_dev, part.get(), ATK_F64, I * I, 1.0);
        }
        ATK_CUDA(cudaEventRecord(g1, ctx->stream));
        ATK_CUDA(cudaEventSynchronize(g1));
        float f = 0.f;
        ATK_CUDA(cudaEventElapsedTime(&f, g0, g1));
        ms = f;
    } catch (...) {
        cudaStreamSynchronize(cs);
        cleanup();
        throw;
    }
    cleanup();
    return ms;
}

// reconstruct (sthosvd.hpp:197-209)
atk_tensor* reconstruct(atk_ctx* ctx, const atk_tensor* core, const double* factors,
                        const uint64_t* odims) {
    check_tensor(core, "core");
    const int order = core->order;
    atk_tensor* y = nullptr;
    const atk_tensor* cur = core;
    size_t off = 0;
    for (int n = 0; n < order; ++n) {
        const uint64_t In = odims[n], Rn = core->dims[n];
        DevBuf<double> u(ctx, In * Rn);
        ATK_CUDA(cudaMemcpyAsync(u.get(), factors + off, In * Rn * sizeof(double),
                                 cudaMemcpyHostToDevice, ctx->stream));
        off += In * Rn;
        atk_tensor* nxt = contract_ttm(ctx, cur, u.get(), In, n);  // U_n is I_n x R_n ("R x I")
        record_gemm(2LL * (long long)(In * j_of(cur, n)) * (long long)Rn);
        if (y) atk_tensor_free(y);
        y = nxt;
        cur = y;
    }
    return y;
}

// relative_error (sthosvd.hpp:212-223)
double relative_error(atk_ctx* ctx, const atk_tensor* x, const atk_tensor* core,
                      const double* factors) {
    const double nx2 = norm2_sq(ctx, x->data, x->dtype, x->numel());
    if (nx2 == 0.0) fail(ATK_ZERO_NORM_INPUT, "relative error is undefined for a zero tensor");
    atk_tensor* xh = reconstruct(ctx, core, factors, x->dims);
    for (int m = 0; m < x->order; ++m)
        if (xh->dims[m] != x->dims[m]) {
            atk_tensor_free(xh);
            fail(ATK_SHAPE_MISMATCH, "reconstruction shape differs from input");
        }
    if (xh->dtype != x->dtype) {  // e.g. fp32 core against an fp64 copy of the input
        atk_tensor* cv = new_tensor(ctx, x->dtype, x->order, x->dims);
        convert(ctx, cv->data, x->dtype, xh->data, xh->dtype, x->numel());
        atk_tensor_free(xh);
        xh = cv;
    }
    const double d2 = diff_norm2_sq(ctx, xh->data, x->data, x->dtype, x->numel());
    atk_tensor_free(xh);
    return std::sqrt(d2) / std::sqrt(nx2);
}

}  // namespace atk
