// svd.cu — svd_mode_solver on the explicit unfolding (solvers.hpp:142-162,
// linalg.hpp:153-166): the reference matricizes Y_(n) and runs a thin SVD, so
// its left singular vectors keep their accuracy where the Gram route
// (sigma = sqrt(lambda of Y Y^T)) squares the condition number and loses the
// vectors of sigma_k / sigma_1 < ~1e-8.
//
// Device algorithm (fp64 input):
//   1. S = Y_(n) Y_(n)^T (the Gram kernels) and ALL its eigenvectors Q
//      (tridiagonal / grid-wide dense solver): a preconditioner, exact for the
//      large singular values;
//   2. M = Q^T Y_(n), materialised row-major (I x J, the explicit unfolding,
//      column j = p + P o as matricize orders it, tensor.hpp);
//   3. one-sided (Hestenes) Jacobi on the ROWS of M: round-robin tournaments of
//      I/2 disjoint row pairs per launch, one CTA per pair, fp64 dot products
//      in a fixed order; each rotation is also applied to the columns of
//      W (= Q at the start), so Y_(n) = W M throughout.  With the Q start only
//      the small-sigma clusters still rotate: 2-4 sweeps.  A tall unfolding
//      (I > J, e.g. a last mode after the others shrank) is the mirror image:
//      V from S' = Y^T Y, the J columns of M = Y V rotated, U = column / sigma.
//   4. sigma_k = |row k of M| (rows are sigma_k v_k^T once orthogonal),
//      sorted descending; U = the matching columns of W with the reference's
//      sign rule (largest |u_i| positive, first on ties; linalg.hpp:34-50),
//      and the shrunk tensor = those rows of M with the same signs
//      (= diag(sigma) V^T, solvers.hpp:155-160), tensorized.
// Relative accuracy follows one-sided Jacobi's (Demmel-Veselic): the sigma
// of a row is resolved to ~eps relative to itself, not to sigma_1.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>
#include <vector>

#include "atk_driver.cuh"

namespace atk {
namespace {

constexpr int kSvdThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int k = 0; k < int(blockDim.x >> 5); ++k) t += sh[k];  // fixed order: bit-reproducible
    return t;
}

// M[i * J + p + P o] = B[p + P (i + I o)]
__global__ void unfold_rows(const double* __restrict__ b, uint64_t P, uint64_t I, uint64_t O,
                            double* __restrict__ m) {
    const uint64_t tot = P * I * O, J = P * O;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t p = e % P, t = e / P, i = t % I, o = t / I;
        m[i * J + p + P * o] = b[e];
    }
}

// One tournament round: pair slot blockIdx.x of round t (players 0..N-1, N even;
// players >= I are byes).  Rotates rows (p, q) of M and columns (p, q) of W.
__global__ void __launch_bounds__(kSvdThreads) jacobi_rows_round(double* __restrict__ m, uint64_t J,
                                                                  double* __restrict__ w, int I, int N, int t,
                                                                  double tol, const double* __restrict__ negl,
                                                                  int* __restrict__ rotated) {
    __shared__ double sh[kSvdThreads / 32];
    const int j = blockIdx.x;
    auto player = [&](int k) { return k == 0 ? 0 : (t + k - 1) % (N - 1) + 1; };
    int p = player(j), q = player(N - 1 - j);
    if (p > q) { const int s = p; p = q; q = s; }
    if (q >= I) return;  // bye
    double* mp = m + uint64_t(p) * J;
    double* mq = m + uint64_t(q) * J;
    double a = 0.0, b = 0.0, c = 0.0;
    for (uint64_t k = threadIdx.x; k < J; k += blockDim.x) {
        const double x = mp[k], y = mq[k];
        a = fma(x, x, a);
        b = fma(y, y, b);
        c = fma(x, y, c);
    }
    a = block_sum(a, sh);
    b = block_sum(b, sh);
    c = block_sum(c, sh);
    // a row at rounding level of the whole matrix (|row|^2 <= *negl) is converged as it is: rows
    // that are exact multiples of one vector (a constant tensor's unfolding) would otherwise
    // rotate forever, every rotation leaving an exactly parallel residue (dgesvj skips them too)
    if (a <= *negl || b <= *negl) return;
    if (!(c != 0.0) || !(fabs(c) > tol * sqrt(a) * sqrt(b))) return;
    // rows made orthogonal: tan(2 theta) = 2c / (b - a), t = the small root
    const double zeta = (b - a) / (2.0 * c);
    const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
    const double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
    for (uint64_t k = threadIdx.x; k < J; k += blockDim.x) {
        const double x = mp[k], y = mq[k];
        mp[k] = cs * x - sn * y;
        mq[k] = sn * x + cs * y;
    }
    double* wp = w + uint64_t(p) * I;
    double* wq = w + uint64_t(q) * I;
    for (int k = threadIdx.x; k < I; k += blockDim.x) {
        const double x = wp[k], y = wq[k];
        wp[k] = cs * x - sn * y;
        wq[k] = sn * x + cs * y;
    }
    if (threadIdx.x == 0) atomicAdd(rotated, 1);
}

__global__ void __launch_bounds__(kSvdThreads) row_norms(const double* __restrict__ m, uint64_t J,
                                                          double* __restrict__ out) {
    __shared__ double sh[kSvdThreads / 32];
    const double* r = m + uint64_t(blockIdx.x) * J;
    double s = 0.0;
    for (uint64_t k = threadIdx.x; k < J; k += blockDim.x) s = fma(r[k], r[k], s);
    s = block_sum(s, sh);
    if (threadIdx.x == 0) out[blockIdx.x] = sqrt(s);
}

// negl = (16 eps)^2 sum_k |row k|^2 (= (16 eps ||M||_F)^2), one CTA
__global__ void __launch_bounds__(kSvdThreads) negligible_threshold(const double* __restrict__ norms, int count,
                                                                     double* __restrict__ negl) {
    __shared__ double sh[kSvdThreads / 32];
    double t = 0.0;
    for (int k = threadIdx.x; k < count; k += blockDim.x) t = fma(norms[k], norms[k], t);
    t = block_sum(t, sh);
    if (threadIdx.x == 0) *negl = 256.0 * 2.220446049250313e-16 * 2.220446049250313e-16 * t;
}

// U(:, k) = sign_k W(:, perm[k]); sign_k makes the largest |entry| (first on
// ties) positive.  One CTA per output column.
__global__ void __launch_bounds__(kSvdThreads) gather_left(const double* __restrict__ w, int I,
                                                            const int* __restrict__ perm, double* __restrict__ u,
                                                            double* __restrict__ sign) {
    __shared__ double sb[kSvdThreads / 32];
    __shared__ int si[kSvdThreads / 32];
    const double* c = w + uint64_t(perm[blockIdx.x]) * I;
    double best = -1.0;
    int bi = 0;
    for (int i = threadIdx.x; i < I; i += blockDim.x) {
        const double a = fabs(c[i]);
        if (a > best) { best = a; bi = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    if (lane == 0) { sb[wp] = best; si[wp] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < int(blockDim.x >> 5); ++k)
            if (sb[k] > sb[0] || (sb[k] == sb[0] && si[k] < si[0])) { sb[0] = sb[k]; si[0] = si[k]; }
        sign[blockIdx.x] = c[si[0]] < 0.0 ? -1.0 : 1.0;
    }
    __syncthreads();
    const double s = sign[blockIdx.x];
    for (int i = threadIdx.x; i < I; i += blockDim.x) u[uint64_t(blockIdx.x) * I + i] = s * c[i];
}

// shrunk[p + P (k + r o)] = sign_k M[perm[k] * J + p + P o]
__global__ void tensorize_rows(const double* __restrict__ m, uint64_t P, uint64_t O, int r,
                               const int* __restrict__ perm, const double* __restrict__ sign,
                               double* __restrict__ out) {
    const uint64_t J = P * O, tot = P * uint64_t(r) * O;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t p = e % P, t = e / P, k = t % r, o = t / r;
        out[e] = sign[k] * m[uint64_t(perm[k]) * J + p + P * o];
    }
}

// Tall unfoldings (I > J): the J columns of M = Q^T Y_(n) are rotated instead
// (I - J rows of M cannot become mutually orthogonal without vanishing
// exactly).  A[j * I + i] = B[p + P (i + I o)], j = p + P o.
__global__ void unfold_cols(const double* __restrict__ b, uint64_t P, uint64_t I, uint64_t O,
                            double* __restrict__ a) {
    const uint64_t tot = P * I * O;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t p = e % P, t = e / P, i = t % I, o = t / I;
        a[(p + P * o) * I + i] = b[e];
    }
}

// T(:, k) = M(:, perm[k]) / sigma_perm[k]  (M: I x n column-major), the left vectors of a
// column-rotated tall unfolding.
__global__ void scale_cols(const double* __restrict__ m, int I, const int* __restrict__ perm,
                           const double* __restrict__ sig, int r, double* __restrict__ t) {
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < uint64_t(I) * r;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const int i = int(e % I), k = int(e / I);
        const double sg = sig[perm[k]];
        t[e] = sg > 0.0 ? m[uint64_t(perm[k]) * I + i] / sg : 0.0;
    }
}

// Columns of T whose sigma is at rounding level (sigma^2 <= *negl: a rank-deficient tall unfolding)
// carry no direction; replace each, in order, by the unit vector of e_j's component orthogonal to
// the columns kept so far, j the row where that component is largest (>= (I - r) / I), twice
// projected.  One CTA; the core slices they multiply are zero, so only orthonormality matters.
__global__ void __launch_bounds__(kSvdThreads) complete_null_cols(double* __restrict__ t, int I, int r,
                                                                   const int* __restrict__ perm,
                                                                   const double* __restrict__ sig,
                                                                   const double* __restrict__ negl) {
    __shared__ double sh[kSvdThreads / 32];
    __shared__ double sb[kSvdThreads / 32];
    __shared__ int si[kSvdThreads / 32];
    const double thr = *negl;
    auto kept = [&](int c, int k) { return c < k || sig[perm[c]] * sig[perm[c]] > thr; };
    for (int k = 0; k < r; ++k) {
        if (sig[perm[k]] * sig[perm[k]] > thr) continue;
        double* v = t + uint64_t(k) * I;
        // pick j = argmax_j 1 - sum_{kept c} T(j, c)^2 (first on ties)
        double best = -1.0;
        int bj = 0;
        for (int j = threadIdx.x; j < I; j += blockDim.x) {
            double q = 1.0;
            for (int c = 0; c < r; ++c)
                if (c != k && kept(c, k)) q -= t[uint64_t(c) * I + j] * t[uint64_t(c) * I + j];
            if (q > best) { best = q; bj = j; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if (ob > best || (ob == best && oj < bj)) { best = ob; bj = oj; }
        }
        const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
        __syncthreads();
        if (lane == 0) { sb[wp] = best; si[wp] = bj; }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int q = 1; q < int(blockDim.x >> 5); ++q)
                if (sb[q] > sb[0] || (sb[q] == sb[0] && si[q] < si[0])) { sb[0] = sb[q]; si[0] = si[q]; }
        __syncthreads();
        const int j = si[0];
        for (int i = threadIdx.x; i < I; i += blockDim.x) v[i] = i == j ? 1.0 : 0.0;
        for (int pass = 0; pass < 2; ++pass)
            for (int c = 0; c < r; ++c) {
                if (c == k || !kept(c, k)) continue;
                const double* u = t + uint64_t(c) * I;
                double d = 0.0;
                for (int i = threadIdx.x; i < I; i += blockDim.x) d = fma(u[i], v[i], d);
                d = block_sum(d, sh);
                for (int i = threadIdx.x; i < I; i += blockDim.x) v[i] = fma(-d, u[i], v[i]);
            }
        double n2 = 0.0;
        for (int i = threadIdx.x; i < I; i += blockDim.x) n2 = fma(v[i], v[i], n2);
        const double inv = 1.0 / sqrt(block_sum(n2, sh));
        for (int i = threadIdx.x; i < I; i += blockDim.x) v[i] *= inv;
        __syncthreads();
    }
}

// shrunk[p + P (k + r o)] = sign_k sigma_k W(p + P o, perm[k]), W (J x J) column-major
__global__ void tensorize_cols(const double* __restrict__ w, uint64_t P, uint64_t O, int r,
                               const int* __restrict__ perm, const double* __restrict__ sign,
                               const double* __restrict__ sig, double* __restrict__ out) {
    const uint64_t J = P * O, tot = P * uint64_t(r) * O;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t p = e % P, t = e / P, k = t % r, o = t / r;
        out[e] = sign[k] * sig[perm[k]] * w[uint64_t(perm[k]) * J + p + P * o];
    }
}

__global__ void iota_fill(int* __restrict__ v, int n) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) v[e] = e;
}

int grid_for(atk_ctx* ctx, uint64_t n) {
    return int(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, uint64_t(ctx->num_sms) * 16)));
}

}  // namespace

bool svd_explicit_supported(atk_ctx* ctx, const atk_tensor* y, int mode) {
    if (!ctx->svd_explicit || y->dtype != ATK_F64) return false;
    if (ctx->comm && !ctx->replicated) return false;  // J is spread over the ranks: Gram route
    const uint64_t I = y->dims[mode], J = j_of(y, mode);
    if (I > uint64_t(kBigEigMax) || I < 2) return false;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return 2.0 * double(I) * double(J) * 8.0 + 8.0 * double(I) * double(I) * 4.0 < 0.5 * double(free_b);
}

ModeOut svd_mode_explicit(atk_ctx* ctx, const atk_tensor* y, int mode, uint64_t r) {
    const Split s = loop_split(y->dims, y->order, mode);
    const uint64_t I = s.I, J = s.P * s.O;
    cudaStream_t st = ctx->stream;
    ModeOut out;
    out.solver = ATK_SOLVER_SVD;
    StageTimer tm(ctx);
    // Wide (I <= J): precondition with the eigenvectors Q of S = Y Y^T (I x I), rotate the I
    // rows of M = Q^T Y (row-graded: rows ~ sigma_k v_k^T), accumulating W = Q.
    // Tall (I > J): precondition with the eigenvectors V of S' = Y^T Y (J x J), rotate the J
    // columns of M = Y V (column-graded: columns ~ sigma_k u_k), accumulating W = V.  Either
    // way one-sided Jacobi sees a graded matrix and resolves each sigma to ~eps relative to
    // itself; I - J rows could never become mutually orthogonal without vanishing exactly.
    const bool tall = I > J;
    const uint64_t nrot = tall ? J : I, len = tall ? I : J;  // rotated vectors and their length
    DevBuf<double> M(ctx, I * J), W(ctx, nrot * nrot);
    tm.start();
    {
        DevBuf<double> S(ctx, nrot * nrot), vals(ctx, nrot);
        if (tall) {
            // M <- Y_(n) column-major (I x J); S' = M^T M; W = V; M <- M V
            unfold_cols<<<grid_for(ctx, I * J), 256, 0, st>>>(static_cast<const double*>(y->data), s.P, I, s.O,
                                                              M.get());
            ATK_LAUNCHED(ctx);
            dgemm(ctx, true, false, int(J), int(J), int(I), 1.0, M.get(), int(I), M.get(), int(I), 0.0, S.get(),
                  int(J));
            symmetrize(ctx, S.get(), int(J));
        } else {
            contract_ttt(ctx, y, y, mode, S.get(), true);
        }
        out.times.gram_ms = tm.stop_ms(kStageGram);
        record_gemm((long long)(I * I) * (long long)J);
        tm.start();
        DevBuf<double> fac(ctx, 2);
        eig_scale(ctx, S.get(), int(nrot), true, fac.get());  // huge / tiny data: the preconditioner's range
        if (nrot <= uint64_t(kTridiagMax))
            tridiag_eig(ctx, S.get(), int(nrot), int(nrot), int(nrot), vals.get(), W.get(), int(nrot));
        else
            dense_eig_big(ctx, S.get(), int(nrot), int(nrot), int(nrot), vals.get(), W.get(), int(nrot), true);
    }
    if (tall) {
        DevBuf<double> MV(ctx, I * J);
        dgemm(ctx, false, false, int(I), int(J), int(J), 1.0, M.get(), int(I), W.get(), int(J), 0.0, MV.get(), int(I));
        M = std::move(MV);
    } else {
        // M = Q^T Y_(n), row-major (row i contiguous over j = p + P o)
        DevBuf<double> Qt(ctx, I * I);
        transpose(ctx, W.get(), int(I), int(I), Qt.get());
        atk_tensor* B = contract_ttm(ctx, y, Qt.get(), I, mode);
        Qt.reset();
        unfold_rows<<<grid_for(ctx, I * J), 256, 0, st>>>(static_cast<const double*>(B->data), s.P, I, s.O, M.get());
        ATK_LAUNCHED(ctx);
        atk_tensor_free(B);
    }
    // one-sided Jacobi on the nrot contiguous vectors of M
    const int N = int(nrot + (nrot & 1));
    const double tol = 2.220446049250313e-16 * std::max(1.0, std::sqrt(double(len)));
    DevBuf<int> rot(ctx, 1);
    DevBuf<double> negl(ctx, 1), norms0(ctx, nrot);
    row_norms<<<unsigned(nrot), kSvdThreads, 0, st>>>(M.get(), len, norms0.get());
    ATK_LAUNCHED(ctx);
    negligible_threshold<<<1, kSvdThreads, 0, st>>>(norms0.get(), int(nrot), negl.get());
    ATK_LAUNCHED(ctx);
    int sweeps = 0, last = -1;
    const int max_sweeps = 30;
    for (; sweeps < max_sweeps; ++sweeps) {
        ATK_CUDA(cudaMemsetAsync(rot.get(), 0, sizeof(int), st));
        for (int t = 0; t < N - 1; ++t) {
            jacobi_rows_round<<<N / 2, kSvdThreads, 0, st>>>(M.get(), len, W.get(), int(nrot), N, t, tol, negl.get(),
                                                             rot.get());
            ATK_LAUNCHED(ctx);
        }
        ATK_CUDA(cudaMemcpyAsync(&last, rot.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
        ATK_CUDA(cudaStreamSynchronize(st));
        if (last == 0) break;
    }
    if (last != 0) fail(ATK_NO_CONVERGENCE, "singular value decomposition failed");
    // sigma, order, U with the sign rule, shrunk = diag(sigma) V^T rows
    DevBuf<double> sig(ctx, nrot);
    row_norms<<<unsigned(nrot), kSvdThreads, 0, st>>>(M.get(), len, sig.get());
    ATK_LAUNCHED(ctx);
    std::vector<double> hs(nrot);
    ATK_CUDA(cudaMemcpyAsync(hs.data(), sig.get(), nrot * sizeof(double), cudaMemcpyDeviceToHost, st));
    ATK_CUDA(cudaStreamSynchronize(st));
    std::vector<int> perm(nrot);
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return hs[a] > hs[b]; });
    perm.resize(r);
    DevBuf<int> dperm(ctx, r);
    DevBuf<double> U(ctx, I * r), sign(ctx, r);
    ATK_CUDA(cudaMemcpyAsync(dperm.get(), perm.data(), r * sizeof(int), cudaMemcpyHostToDevice, st));
    if (tall) {
        DevBuf<double> T(ctx, I * r);
        DevBuf<int> ident(ctx, r);
        scale_cols<<<grid_for(ctx, I * r), 256, 0, st>>>(M.get(), int(I), dperm.get(), sig.get(), int(r), T.get());
        ATK_LAUNCHED(ctx);
        if (hs[perm[r - 1]] * hs[perm[r - 1]] <= 256.0 * 4.93038065763132e-32 * std::accumulate(
                hs.begin(), hs.end(), 0.0, [](double acc, double x) { return acc + x * x; }) * 2.0) {
            complete_null_cols<<<1, kSvdThreads, 0, st>>>(T.get(), int(I), int(r), dperm.get(), sig.get(), negl.get());
            ATK_LAUNCHED(ctx);
        }
        iota_fill<<<1, 256, 0, st>>>(ident.get(), int(r));
        ATK_LAUNCHED(ctx);
        gather_left<<<unsigned(r), kSvdThreads, 0, st>>>(T.get(), int(I), ident.get(), U.get(), sign.get());
        ATK_LAUNCHED(ctx);
    } else {
        gather_left<<<unsigned(r), kSvdThreads, 0, st>>>(W.get(), int(I), dperm.get(), U.get(), sign.get());
        ATK_LAUNCHED(ctx);
    }
    out.times.eig_ms = tm.stop_ms(kStageEig);
    tm.start();
    uint64_t od[ATK_MAX_ORDER];
    for (int m = 0; m < y->order; ++m) od[m] = y->dims[m];
    od[mode] = r;
    out.shrunk = new_tensor(ctx, ATK_F64, y->order, od);
    if (tall)
        tensorize_cols<<<grid_for(ctx, s.P * r * s.O), 256, 0, st>>>(W.get(), s.P, s.O, int(r), dperm.get(),
                                                                     sign.get(), sig.get(),
                                                                     static_cast<double*>(out.shrunk->data));
    else
        tensorize_rows<<<grid_for(ctx, s.P * r * s.O), 256, 0, st>>>(M.get(), s.P, s.O, int(r), dperm.get(),
                                                                     sign.get(), static_cast<double*>(out.shrunk->data));
    ATK_LAUNCHED(ctx);
    out.times.ttm_ms = tm.stop_ms(kStageTtm);
    out.factor_dev = std::move(U);
    out.eig.method = 4;
    out.eig.iterations = sweeps + 1;  // Jacobi sweeps
    out.times.total_ms = out.times.gram_ms + out.times.eig_ms + out.times.ttm_ms;
    return out;
}

}  // namespace atk
