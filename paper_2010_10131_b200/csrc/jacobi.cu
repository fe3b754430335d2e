// jacobi.cu — small dense symmetric eigensolver (n <= kJacobiMax), one CTA.
//
// One-sided (Hestenes) Jacobi on A itself: U = A V is orthogonalised column
// pair by column pair; at convergence A V = U with orthogonal columns, i.e.
// A = (U Sigma^-1) Sigma V^T, and for symmetric A the eigenvalues are
// lambda_j = v_j^T A v_j = u_j . v_j, eigenvectors v_j.  Each round rotates
// the n/2 disjoint column pairs of a round-robin tournament, one 16-lane group
// per pair (three group-reduced dot products, then the pair's columns of U and
// V updated in place).  Pairs touch disjoint columns, so a round costs one
// __syncthreads; the CTA has exactly 16 * n/2 threads so no lane idles.
// U and V live in shared memory (2 n^2 doubles).
// Used for: the dense eig of small Grams (n <= 112), the Rayleigh-Ritz
// problems of ChFSI and the Lanczos tridiagonal.  Output sorted descending
// (linalg.hpp:101-123 keeps the top r of the full spectrum).
#include <algorithm>
#include <cmath>

#include "atk_internal.cuh"

namespace atk {
namespace {

constexpr int kGroup = 16;                        // lanes per column pair
constexpr int kMaxThreads = kGroup * ((kJacobiMax + 1) / 2);  // 896

__device__ __forceinline__ int rr_player(int t, int k, int N) {
    return k == 0 ? 0 : (t + k - 1) % (N - 1) + 1;
}

__global__ void __launch_bounds__(kMaxThreads, 1)
    jacobi1s_kernel(const double* __restrict__ ain, int n, int lda, double* __restrict__ values,
                    double* __restrict__ vout, int ldv, int* __restrict__ sweeps_out) {
    extern __shared__ double sm[];
    const int ld = n + 1;  // odd leading dimension: column accesses hit distinct banks
    double* U = sm;
    double* V = U + size_t(ld) * n;
    double* lam = V + size_t(ld) * n;  // n
    __shared__ int rotated;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int N = n + (n & 1);
    const double tol = fmax(1e-15, 4.0 * n * 2.220446049250313e-16);
    // tournament schedule precomputed once: sched[t * N/2 + j] = p | q << 8 (p < q)
    uint16_t* sched = reinterpret_cast<uint16_t*>(lam + n);
    for (int e = tid; e < (N - 1) * (N / 2); e += nt) {
        const int t = e / (N / 2), j = e % (N / 2);
        int p = rr_player(t, j, N), q = rr_player(t, N - 1 - j, N);
        if (p > q) { const int x = p; p = q; q = x; }
        sched[e] = uint16_t(p | (q << 8));
    }

    for (int e = tid; e < n * n; e += nt) {
        const int i = e % n, j = e / n;
        U[i + ld * j] = 0.5 * (ain[i + size_t(lda) * j] + ain[j + size_t(lda) * i]);
        V[i + ld * j] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();

    const int grp = tid / kGroup, gl = tid % kGroup;
    int sweep = 0;
    for (; sweep < 40 && n > 1; ++sweep) {
        if (tid == 0) rotated = 0;
        __syncthreads();
        for (int t = 0; t < N - 1; ++t) {
            bool active = grp < N / 2;
            int p = 0, q = 0;
            if (active) {
                const int pq = sched[t * (N / 2) + grp];
                p = pq & 255;
                q = pq >> 8;
                active = q < n;  // dummy player when n is odd
            }
            double* up = U + ld * p;
            double* uq = U + ld * q;
            double a = 0.0, b = 0.0, g = 0.0;
            if (active) {
#pragma unroll 4
                for (int i = gl; i < n; i += kGroup) {
                    const double x = up[i], y = uq[i];
                    a = fma(x, x, a);
                    b = fma(y, y, b);
                    g = fma(x, y, g);
                }
            }
#pragma unroll
            for (int o = kGroup / 2; o > 0; o >>= 1) {
                a += __shfl_xor_sync(0xffffffffu, a, o);
                b += __shfl_xor_sync(0xffffffffu, b, o);
                g += __shfl_xor_sync(0xffffffffu, g, o);
            }
            // rounding in the length-n dot products is ~n eps sqrt(ab): a tighter
            // threshold never converges (measured: 40 sweeps at n = 96 with 1e-15)
            if (active && g != 0.0 && fabs(g) > tol * sqrt(a * b)) {
                // t = tan(theta) is the small root of t^2 + 2 zeta t - 1 = 0.  A fast
                // fp32 estimate (the fp64 chain div -> sqrt -> div dominated the round
                // latency) is polished by one fp64 Newton step whose reciprocal comes
                // from fp32 rcp: the error squares, ~1e-14.  The angle must be fp64-
                // accurate: an error eps leaves g'/sqrt(a b) ~ eps sqrt(a/b), which for
                // a/b ~ 1e12 (RR blocks of gapped Grams) is ~1e-1 with a bare fp32 angle
                // (measured: 13 sweeps at n = 96 instead of ~7).  (c, s) are normalised
                // in fp64, so the rotation stays orthogonal.
                const double zeta = (b - a) / (2.0 * g);
                double tt;
                if (fabs(zeta) < 1e15) {
                    const float zf = float(zeta);
                    const double t0 = double(copysignf(1.0f, zf) / (fabsf(zf) + sqrtf(fmaf(zf, zf, 1.0f))));
                    const double f = fma(t0, t0, fma(2.0 * zeta, t0, -1.0));
                    const double fp = 2.0 * (t0 + zeta);
                    tt = t0 - f * double(__frcp_rn(float(fp)));
                } else {
                    tt = 0.5 / zeta;
                }
                const double c = rsqrt(fma(tt, tt, 1.0)), s = c * tt;
                double* vp = V + ld * p;
                double* vq = V + ld * q;
#pragma unroll 4
                for (int i = gl; i < n; i += kGroup) {
                    const double x = up[i], y = uq[i];
                    up[i] = c * x - s * y;
                    uq[i] = fma(s, x, c * y);
                    const double xv = vp[i], yv = vq[i];
                    vp[i] = c * xv - s * yv;
                    vq[i] = fma(s, xv, c * yv);
                }
                if (gl == 0) rotated = 1;
            }
            __syncthreads();
        }
        const bool done = !rotated;
        __syncthreads();  // everyone has read the flag before thread 0 resets it
        if (done) break;
    }
    // lambda_j = u_j . v_j  (sign-correct for indefinite A), one group per column
    for (int j0 = 0; j0 < n; j0 += nt / kGroup) {  // uniform trip count: shuffles stay converged
        const int j = j0 + grp;
        double d = 0.0;
        if (j < n)
            for (int i = gl; i < n; i += kGroup) d = fma(U[i + ld * j], V[i + ld * j], d);
        for (int o = kGroup / 2; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        if (j < n && gl == 0) lam[j] = d;
    }
    __syncthreads();
    for (int i = tid; i < n; i += nt) {
        const double li = lam[i];
        int rank = 0;
        for (int j = 0; j < n; ++j) {
            const double lj = lam[j];
            rank += (lj > li) || (lj == li && j < i);
        }
        values[rank] = li;
        for (int r = 0; r < n; ++r) vout[r + size_t(ldv) * rank] = V[r + ld * i];
    }
    if (tid == 0 && sweeps_out) *sweeps_out = sweep;
}

}  // namespace

size_t jacobi1s_smem_bytes(int n) {
    const int N = n + (n & 1);
    return (size_t(2) * (n + 1) * n + n) * sizeof(double) + size_t(N) * (N / 2) * sizeof(uint16_t) + 64;
}

void jacobi_eig(atk_ctx* ctx, const double* a, int n, int lda, double* values, double* vectors, int ldv,
                int* sweeps_dev) {
    if (n > kJacobiMax) fail(ATK_UNSUPPORTED, "jacobi_eig: n exceeds the shared-memory capacity");
    const size_t smem = jacobi1s_smem_bytes(n);
    static bool attr = false;
    if (!attr) {
        ATK_CUDA(cudaFuncSetAttribute(jacobi1s_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(jacobi1s_smem_bytes(kJacobiMax))));
        attr = true;
    }
    const int N = n + (n & 1);
    const int threads = ((kGroup * std::max(1, N / 2)) + 31) / 32 * 32;
    jacobi1s_kernel<<<1, threads, smem, ctx->stream>>>(a, n, lda, values, vectors, ldv, sweeps_dev);
    ATK_LAUNCHED(ctx);
}

}  // namespace atk

namespace atk {
namespace {

// X = L^{-T} for G = L L^T, entirely in shared memory, by symmetric Gauss-Jordan
// elimination on [G | I]: step c subtracts (A(i,c)/d_c) row_c from every row
// i > c of both blocks (trailing upper triangle of A, columns <= c of W).  The
// row scalings by 1/sqrt(d_c) are deferred to the output pass, so each step
// reads only row c (final after step c-1) and writes rows > c: ONE barrier per
// step, and no separate triangular inverse (W ends as L^{-1}, X = W^T).
// One CTA, k <= 112.  info = 0 on success, else 1 + the failing pivot
// (linalg.hpp:169-177 NotSPD).
__global__ void __launch_bounds__(1024) chol_inv_kernel(const double* __restrict__ g, int k,
                                                        double* __restrict__ x, int* __restrict__ info) {
    extern __shared__ double sm[];
    const int ld = k + 1;
    double* A = sm;                  // k x k, upper triangle live
    double* W = A + size_t(ld) * k;  // k x k, becomes L^{-1} (unscaled rows)
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int e = tid; e < k * k; e += nt) {
        const int i = e % k, j = e / k;
        A[i + ld * j] = g[e];
        W[i + ld * j] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    int bad = 0;
    for (int c = 0; c < k; ++c) {
        const double d = A[c + ld * c];
        if (!(d > 0.0)) {  // uniform: every thread read the same pivot
            bad = c + 1;
            break;
        }
        const double inv = 1.0 / d;
        const int m = k - c - 1;
        for (int e = tid; e < m * k; e += nt) {
            const int i = c + 1 + e % m, j = e / m;
            const double f = A[c + ld * i] * inv;  // A(i, c) / d_c via symmetry
            if (j <= c) W[i + ld * j] = fma(-f, W[c + ld * j], W[i + ld * j]);
            else if (j >= i) A[i + ld * j] = fma(-f, A[c + ld * j], A[i + ld * j]);
        }
        __syncthreads();
    }
    if (bad) {
        if (tid == 0) *info = bad;
        return;
    }
    for (int e = tid; e < k * k; e += nt) {
        const int r = e % k, c = e / k;
        x[e] = (r <= c) ? W[c + ld * r] * rsqrt(A[c + ld * c]) : 0.0;
    }
    if (tid == 0) *info = 0;
}

}  // namespace

void cholesky_inv_t(atk_ctx* ctx, const double* g, int k, double* x, int* info_dev) {
    if (k > kJacobiMax) fail(ATK_UNSUPPORTED, "cholesky_inv_t: k too large");
    const size_t smem = size_t(2) * (k + 1) * k * sizeof(double);
    static bool attr = false;
    if (!attr) {
        ATK_CUDA(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(size_t(2) * (kJacobiMax + 1) * kJacobiMax * sizeof(double))));
        attr = true;
    }
    const int threads = std::min(1024, std::max(64, (k * k / 8 + 31) / 32 * 32));
    chol_inv_kernel<<<1, threads, smem, ctx->stream>>>(g, k, x, info_dev);
    ATK_LAUNCHED(ctx);
}

}  // namespace atk
