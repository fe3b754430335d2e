// eig.cu — linalg::sym_eig_top_r (linalg.hpp:101-123) on the device, fp64.
//
// The reference computes ALL eigenpairs with Eigen's SelfAdjointEigenSolver
// and keeps the top r.  On the device:
//   n <= kJacobiMax : dense one-CTA Jacobi (dense.cu), all pairs, keep top r.
//   n  > kJacobiMax : Chebyshev-filtered subspace iteration (ChFSI) on a
//                     block of k = min(n, max(r+16, 3r/2)) vectors with a
//                     Rayleigh-Ritz step solved by the dense Jacobi, run until
//                     every wanted Ritz pair has relative residual
//                     ||S v - theta v|| <= tol * max|spectrum| (fp64).
// Both paths finish with descending order + fix_signs (linalg.hpp:34-50), so
// factors are comparable entry-wise with the reference when the spectrum is
// gapped.  Spectrum bounds for the filter come from an m-step Lanczos run
// (device), its tridiagonal solved by the same Jacobi kernel.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "atk_internal.cuh"

namespace atk {
namespace {

__global__ void lanczos_step(const double* __restrict__ sq, double* __restrict__ q,
                             double* __restrict__ qprev, int n, int j, double* __restrict__ alpha,
                             double* __restrict__ beta) {
    // q holds q_j, sq = S q_j.  w = sq - beta_{j-1} q_{j-1} - alpha_j q_j,
    // beta_j = ||w||, q_{j-1} <- q_j, q_j <- w / beta_j.
    __shared__ double red[33];
    const int tid = threadIdx.x, nt = blockDim.x;
    const double bprev = j > 0 ? beta[j - 1] : 0.0;
    double d = 0.0;
    for (int i = tid; i < n; i += nt) d += sq[i] * q[i];
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if ((tid & 31) == 0) red[tid >> 5] = d;
    __syncthreads();
    if (tid == 0) {
        double t = 0;
        for (int w = 0; w < (nt >> 5); ++w) t += red[w];
        red[32] = t;
    }
    __syncthreads();
    const double a = red[32];
    double ss = 0.0;
    for (int i = tid; i < n; i += nt) {
        const double w = sq[i] - bprev * qprev[i] - a * q[i];
        ss += w * w;
    }
    __syncthreads();
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((tid & 31) == 0) red[tid >> 5] = ss;
    __syncthreads();
    if (tid == 0) {
        double t = 0;
        for (int w = 0; w < (nt >> 5); ++w) t += red[w];
        red[32] = sqrt(t);
        alpha[j] = a;
        beta[j] = red[32];
    }
    __syncthreads();
    const double b = red[32];
    const double inv = b > 0 ? 1.0 / b : 0.0;
    for (int i = tid; i < n; i += nt) {
        const double w = sq[i] - bprev * qprev[i] - a * q[i];
        qprev[i] = q[i];
        q[i] = w * inv;
    }
}

__global__ void tridiag_dense(const double* __restrict__ alpha, const double* __restrict__ beta,
                              int m, double* __restrict__ t) {
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int i = e % m, j = e / m;
        double v = 0.0;
        if (i == j) v = alpha[i];
        else if (i == j + 1) v = beta[j];
        else if (j == i + 1) v = beta[i];
        t[e] = v;
    }
}

__global__ void fill_normalish(double* __restrict__ v, size_t n, uint64_t seed) {
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += size_t(gridDim.x) * blockDim.x) {
        uint64_t x = (e + 1) * 0x9e3779b97f4a7c15ULL ^ seed;
        x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
        x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
        x ^= x >> 31;
        v[e] = double(int64_t(x >> 11) - (int64_t(1) << 52)) * (1.0 / 4503599627370496.0);
    }
}

// ynew = g1 * y + g2 * yprev  (elementwise; dgemm then adds a * S y)
__global__ void cheb_combine(double* __restrict__ ynew, const double* __restrict__ y,
                             const double* __restrict__ yprev, size_t n, double g1, double g2) {
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += size_t(gridDim.x) * blockDim.x)
        ynew[e] = g1 * y[e] + (yprev ? g2 * yprev[e] : 0.0);
}

// res[j] = || W(:, j) - theta_j V(:, j) ||, j < r   (one warp per column)
__global__ void ritz_residual(const double* __restrict__ w, const double* __restrict__ v,
                              const double* __restrict__ theta, int n, int r,
                              double* __restrict__ res) {
    const int col = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (col >= r) return;
    const double th = theta[col];
    double s = 0.0;
    for (int i = lane; i < n; i += 32) {
        const double d = w[i + size_t(n) * col] - th * v[i + size_t(n) * col];
        s += d * d;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) res[col] = sqrt(s);
}

inline unsigned nblk(size_t n) { return unsigned(std::min<size_t>((n + 255) / 256, 4096)); }

struct Bounds {
    double lo, hi;
};

// m-step Lanczos on S (n x n): extreme Ritz values widened by the last beta.
Bounds lanczos_bounds(atk_ctx* ctx, const double* S, int n) {
    cudaStream_t st = ctx->stream;
    const int m = std::min(n, 40);
    DevBuf<double> q(ctx, n), qp(ctx, n), sq(ctx, n), al(ctx, m), be(ctx, m), tm(ctx, size_t(m) * m),
        tv(ctx, m), tz(ctx, size_t(m) * m);
    DevBuf<int> sweeps(ctx, 1);
    fill_normalish<<<nblk(n), 256, 0, st>>>(q.get(), n, 0x5eed1234ULL);
    ATK_LAUNCHED(ctx);
    ATK_CUDA(cudaMemsetAsync(qp.get(), 0, n * sizeof(double), st));
    const double nq = std::sqrt(norm2_sq(ctx, q.get(), ATK_F64, n));
    axpy(ctx, q.get(), q.get(), ATK_F64, n, 1.0 / nq - 1.0);  // q <- q / ||q||
    for (int j = 0; j < m; ++j) {
        dgemm(ctx, false, false, n, 1, n, 1.0, S, n, q.get(), n, 0.0, sq.get(), n);
        lanczos_step<<<1, 1024, 0, st>>>(sq.get(), q.get(), qp.get(), n, j, al.get(), be.get());
        ATK_LAUNCHED(ctx);
    }
    tridiag_dense<<<1, 256, 0, st>>>(al.get(), be.get(), m, tm.get());
    ATK_LAUNCHED(ctx);
    jacobi_eig(ctx, tm.get(), m, m, tv.get(), tz.get(), m, sweeps.get());
    std::vector<double> hv(m), hb(m);
    ATK_CUDA(cudaMemcpyAsync(hv.data(), tv.get(), m * sizeof(double), cudaMemcpyDeviceToHost, st));
    ATK_CUDA(cudaMemcpyAsync(hb.data(), be.get(), m * sizeof(double), cudaMemcpyDeviceToHost, st));
    ATK_CUDA(cudaStreamSynchronize(st));
    const double bm = std::fabs(hb[m - 1]);
    return {hv[m - 1] - bm, hv[0] + bm};  // hv is descending
}

// Rayleigh-Ritz on the orthonormal block V (n x k): W = S V, T = V^T W,
// T = Z diag(theta) Z^T (Jacobi, descending), V <- V Z, W <- W Z.
void rayleigh_ritz(atk_ctx* ctx, const double* S, int n, int k, double* V, double* W, double* T,
                   double* Z, double* theta, double* tmp, int* sweeps) {
    const size_t nk = size_t(n) * k;
    dgemm(ctx, false, false, n, k, n, 1.0, S, n, V, n, 0.0, W, n);
    dgemm(ctx, true, false, k, k, n, 1.0, V, n, W, n, 0.0, T, k);
    jacobi_eig(ctx, T, k, k, theta, Z, k, sweeps);
    dgemm(ctx, false, false, n, k, k, 1.0, V, n, Z, k, 0.0, tmp, n);
    ATK_CUDA(cudaMemcpyAsync(V, tmp, nk * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    dgemm(ctx, false, false, n, k, k, 1.0, W, n, Z, k, 0.0, tmp, n);
    ATK_CUDA(cudaMemcpyAsync(W, tmp, nk * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
}

}  // namespace

EigInfo sym_eig_top_r(atk_ctx* ctx, const double* s_dev, int n, int r, double* values_dev,
                      double* vectors_dev) {
    EigInfo info;
    cudaStream_t st = ctx->stream;
    const bool dense = n <= kJacobiMax && ctx->eig_method != 1;
    if (dense) {
        DevBuf<double> vals(ctx, n), vecs(ctx, size_t(n) * n);
        DevBuf<int> sweeps(ctx, 1);
        jacobi_eig(ctx, s_dev, n, n, vals.get(), vecs.get(), n, sweeps.get());
        ATK_CUDA(cudaMemcpyAsync(values_dev, vals.get(), r * sizeof(double), cudaMemcpyDeviceToDevice, st));
        ATK_CUDA(cudaMemcpyAsync(vectors_dev, vecs.get(), size_t(n) * r * sizeof(double),
                                 cudaMemcpyDeviceToDevice, st));
        fix_signs(ctx, vectors_dev, n, r, n);
        int sw = 0;
        ATK_CUDA(cudaMemcpyAsync(&sw, sweeps.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
        ATK_CUDA(cudaStreamSynchronize(st));
        if (sw >= 60) fail(ATK_NO_CONVERGENCE, "symmetric eigendecomposition failed (Jacobi sweeps)");
        info.method = 0;
        info.iterations = sw;
        return info;
    }

    // ---------------- ChFSI
    int k = std::min(n, std::max(r + 16, (3 * r + 1) / 2));
    k = std::min(k, kJacobiMax);
    if (k < r) fail(ATK_UNSUPPORTED, "sym_eig_top_r: r > 112 with n > 112 is not supported");
    const size_t nn = size_t(n) * n, nk = size_t(n) * k;
    DevBuf<double> S(ctx, nn), V(ctx, nk), W(ctx, nk), Ya(ctx, nk), Yb(ctx, nk), Yc(ctx, nk),
        T(ctx, size_t(k) * k), Z(ctx, size_t(k) * k), theta(ctx, k), Rm(ctx, size_t(k) * k),
        res(ctx, k);
    DevBuf<int> sweeps(ctx, 1);
    static const bool trace = std::getenv("ATK_TRACE") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto mark = [&](const char* what, int a = -1, double v = 0.0) {
        if (!trace) return;
        cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[atk eig n=%d r=%d k=%d] %-10s %8.3f ms  %d %.3e\n", n, r, k, what,
                     std::chrono::duration<double, std::milli>(now - t_last).count(), a, v);
        t_last = now;
    };
    ATK_CUDA(cudaMemcpyAsync(S.get(), s_dev, nn * sizeof(double), cudaMemcpyDeviceToDevice, st));
    symmetrize(ctx, S.get(), n);
    mark("prep");
    const Bounds b = lanczos_bounds(ctx, S.get(), n);
    mark("lanczos", 0, b.lo);

    // random orthonormal start
    fill_normalish<<<nblk(nk), 256, 0, st>>>(Ya.get(), nk, 0xc0ffee11ULL);
    ATK_LAUNCHED(ctx);
    householder_qr(ctx, Ya.get(), n, k, V.get(), Rm.get());
    mark("qr0");
    rayleigh_ritz(ctx, S.get(), n, k, V.get(), W.get(), T.get(), Z.get(), theta.get(), Ya.get(),
                  sweeps.get());
    mark("rr0");

    const int max_outer = 100;
    std::vector<double> hth(k), hres(r);
    double scale = std::max(std::fabs(b.lo), std::fabs(b.hi));
    int it = 0;
    double worst = 0.0;
    for (;; ++it) {
        ritz_residual<<<(r + 7) / 8, 256, 0, st>>>(W.get(), V.get(), theta.get(), n, r, res.get());
        ATK_LAUNCHED(ctx);
        ATK_CUDA(cudaMemcpyAsync(hth.data(), theta.get(), k * sizeof(double), cudaMemcpyDeviceToHost, st));
        ATK_CUDA(cudaMemcpyAsync(hres.data(), res.get(), r * sizeof(double), cudaMemcpyDeviceToHost, st));
        ATK_CUDA(cudaStreamSynchronize(st));
        scale = std::max(scale, std::fabs(hth[0]));
        worst = 0.0;
        for (int j = 0; j < r; ++j) worst = std::max(worst, hres[j]);
        if (!(scale > 0.0) || worst <= ctx->chfsi_tol * scale || it >= max_outer) break;
        // Chebyshev filter on the unwanted interval [lo, cut]
        const double cut = hth[k - 1];
        const double lo = std::min(b.lo, cut - 1e-12 * scale);
        double e = 0.5 * (cut - lo), c = 0.5 * (cut + lo);
        if (!(e > 0.0)) e = 1e-12 * scale;
        const double smax = std::max(1.0, (std::max(b.hi, hth[0]) - c) / e);
        const double g = 1.0 / (2.0 * smax + 1.0);  // per-step rescale, keeps the recurrence linear
        // degree: enough to separate [lo, cut] from the top by ~1e30, capped at 16
        const double ac = std::acosh(std::max(1.0 + 1e-12, smax));
        const int degree = std::max(2, std::min(16, int(std::ceil(69.0 / ac))));
        // Y1 = g (S V - c V) / e ; Y_{j+1} = g (2/e)(S Y_j - c Y_j) - g^2 Y_{j-1}
        double* yprev = V.get();
        double* ycur = Ya.get();
        double* ynext = Yb.get();
        cheb_combine<<<nblk(nk), 256, 0, st>>>(ycur, V.get(), nullptr, nk, -g * c / e, 0.0);
        ATK_LAUNCHED(ctx);
        dgemm(ctx, false, false, n, k, n, g / e, S.get(), n, V.get(), n, 1.0, ycur, n);
        // first Y_{j-1} is V scaled consistently: V_hat_0 = V (g^0)
        for (int j = 1; j < degree; ++j) {
            cheb_combine<<<nblk(nk), 256, 0, st>>>(ynext, ycur, yprev, nk, -2.0 * g * c / e, -g * g);
            ATK_LAUNCHED(ctx);
            dgemm(ctx, false, false, n, k, n, 2.0 * g / e, S.get(), n, ycur, n, 1.0, ynext, n);
            double* spare = (yprev == V.get()) ? Yc.get() : yprev;
            yprev = ycur;
            ycur = ynext;
            ynext = spare;
        }
        mark("filter", degree, worst / scale);
        householder_qr(ctx, ycur, n, k, V.get(), Rm.get());
        mark("qr");
        rayleigh_ritz(ctx, S.get(), n, k, V.get(), W.get(), T.get(), Z.get(), theta.get(),
                      ynext == V.get() ? Yc.get() : ynext, sweeps.get());
        mark("rr", it);
    }
    mark("done", it, worst / scale);
    ATK_CUDA(cudaMemcpyAsync(values_dev, theta.get(), r * sizeof(double), cudaMemcpyDeviceToDevice, st));
    ATK_CUDA(cudaMemcpyAsync(vectors_dev, V.get(), size_t(n) * r * sizeof(double),
                             cudaMemcpyDeviceToDevice, st));
    fix_signs(ctx, vectors_dev, n, r, n);
    info.method = 1;
    info.iterations = it;
    info.residual = scale > 0 ? worst / scale : 0.0;
    if (it >= max_outer && worst > 1e3 * ctx->chfsi_tol * scale)
        fail(ATK_NO_CONVERGENCE, "symmetric eigendecomposition failed (ChFSI did not converge)");
    return info;
}

}  // namespace atk
