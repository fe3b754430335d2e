// jacobi.cu — small dense symmetric eigensolver (n <= kJacobiMax), one CTA.
//
// One-sided (Hestenes) Jacobi: the columns of a working matrix U are
// orthogonalised pair by pair.  Each round rotates the n/2 disjoint column
// pairs of a round-robin tournament, one 16-lane group per pair (three
// group-reduced dot products from register-resident column slices, then the
// pair's columns updated in place).  Pairs touch disjoint columns, so a round
// costs one __syncthreads.  Two variants, chosen per call:
//
//  * PSD input (Grams, Rayleigh-Ritz blocks of a Gram): Cholesky-preconditioned
//    and vector-free.  T + sigma I = L L^T (sigma = 2 n eps max diag keeps the
//    factorisation positive definite; eigenvectors are unchanged by a shift),
//    then U = L is rotated to U = L J with orthogonal columns.  T + sigma I =
//    L J J^T L^T = sum_j u_j u_j^T, so lambda_j = |u_j|^2 - sigma with
//    eigenvector u_j / |u_j|: no accumulated V, half the shared-memory traffic
//    per round, and the triangular factor converges in fewer sweeps than T
//    itself (measured offline on gapped RR blocks: 11 sweeps instead of 16).
//    A failed pivot falls back to the general variant.
//  * General symmetric input: U = A V on A itself, V accumulated; lambda_j =
//    u_j . v_j (sign-correct for indefinite A), eigenvectors v_j.
//
// U (and V) live in shared memory.  Used for: the dense eig of small Grams
// (n <= 112), the Rayleigh-Ritz and SVQB problems of ChFSI and the Lanczos
// tridiagonal.  Output sorted descending (linalg.hpp:101-123 keeps the top r
// of the full spectrum).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "atk_internal.cuh"

namespace atk {
namespace {

// kJacobiGroup lanes per column pair.  Measured at n = 96 (PSD path): 16 lanes
// 1.29 ms, 8 lanes 1.55 ms, 4 lanes 2.34 ms (n = 152: 4.3 vs 5.6 ms at 8).
constexpr int kJacobiGroup = 16;

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ int rr_player(int t, int k, int N) {
    return k == 0 ? 0 : (t + k - 1) % (N - 1) + 1;
}

// MAXN <= kJacobiMax: U and V in shared memory (both variants).  MAXN up to
// kJacobiPsdMax: U only, PSD variant only (a failed Cholesky reports
// sweeps = -1 and the caller falls back to ChFSI).  Column pairs are dealt to
// the nt / G groups in ceil(pairs / groups) passes per round.
template <int G, int MAXN, int MAXT>
__global__ void __launch_bounds__(MAXT, 1)
    jacobi1s_kernel(const double* __restrict__ ain, int n, int lda, bool psd, double* __restrict__ values,
                    double* __restrict__ vout, int ldv, int* __restrict__ sweeps_out) {
    constexpr bool kHasV = MAXN <= kJacobiMax;
    extern __shared__ double sm[];
    const int ld = n + 1;  // odd leading dimension: column accesses hit distinct banks
    double* U = sm;
    double* V = kHasV ? U + size_t(ld) * n : nullptr;
    double* lam = U + size_t(ld) * n * (kHasV ? 2 : 1);  // n
    double* scl = lam + n;                                // n: 1 / |u_j| (PSD variant)
    __shared__ int rotated;
    __shared__ double sh_sigma;
    constexpr int kGroup = G, kVals = (MAXN + G - 1) / G;  // column slice per lane
    const int tid = threadIdx.x, nt = blockDim.x;
    const int N = n + (n & 1);
    const double eps = 2.220446049250313e-16;
    const double tol = fmax(1e-15, 4.0 * n * eps);
    const double tol2 = tol * tol;
    // tournament schedule precomputed once: sched[t * N/2 + j] = p | q << 8 (p < q)
    uint16_t* sched = reinterpret_cast<uint16_t*>(scl + n);
    for (int e = tid; e < (N - 1) * (N / 2); e += nt) {
        const int t = e / (N / 2), j = e % (N / 2);
        int p = rr_player(t, j, N), q = rr_player(t, N - 1 - j, N);
        if (p > q) { const int x = p; p = q; q = x; }
        sched[e] = uint16_t(p | (q << 8));
    }
    for (int e = tid; e < n * n; e += nt) {
        const int i = e % n, j = e / n;
        U[i + ld * j] = 0.5 * (ain[i + size_t(lda) * j] + ain[j + size_t(lda) * i]);
    }
    __syncthreads();

    bool usev = !psd;
    double sigma = 0.0;
    if (psd) {
        if (tid < 32) {
            double m = 0.0;
            for (int i = tid; i < n; i += 32) m = fmax(m, fabs(U[i + ld * i]));
            for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (tid == 0) sh_sigma = 2.0 * n * eps * m;
        }
        __syncthreads();
        sigma = sh_sigma;
        for (int i = tid; i < n; i += nt) U[i + ld * i] += sigma;
        __syncthreads();
        // right-looking Cholesky, lower triangle, one barrier per step: column c
        // is final (unscaled) after step c-1; the 1/sqrt(d_c) scaling is deferred.
        __shared__ int chol_ok;
        const int cw = nt;
        {
            int okw = 1;
            for (int c = 0; c < n; ++c) {
                const double d = U[c + ld * c];
                if (!(d > 0.0)) {  // uniform: every worker read the same pivot
                    okw = 0;
                    break;
                }
                const double inv = 1.0 / d;
                // warps over columns, lanes over rows (no integer division in the loop)
                for (int j = c + 1 + (tid >> 5); j < n; j += cw >> 5) {
                    const double ljc = U[j + ld * c] * inv;
                    for (int i = j + (tid & 31); i < n; i += 32)
                        U[i + ld * j] = fma(-U[i + ld * c], ljc, U[i + ld * j]);
                }
                __syncthreads();
            }
            if (tid == 0) chol_ok = okw;
        }
        __syncthreads();
        const bool ok = chol_ok != 0;
        if (ok) {
            for (int j = tid; j < n; j += nt) lam[j] = rsqrt(U[j + ld * j]);
            __syncthreads();
            for (int e = tid; e < n * n; e += nt) {
                const int i = e % n, j = e / n;
                U[i + ld * j] = (i >= j) ? U[i + ld * j] * lam[j] : 0.0;
            }
        } else if constexpr (!kHasV) {  // no room for V: let the caller fall back
            if (tid == 0 && sweeps_out) *sweeps_out = -1;
            return;
        } else {  // not numerically PSD: the general variant on A itself
            usev = true;
            sigma = 0.0;
            for (int e = tid; e < n * n; e += nt) {
                const int i = e % n, j = e / n;
                U[i + ld * j] = 0.5 * (ain[i + size_t(lda) * j] + ain[j + size_t(lda) * i]);
            }
        }
    }
    if (kHasV && usev)
        for (int e = tid; e < n * n; e += nt) V[e % n + ld * (e / n)] = (e % n == e / n) ? 1.0 : 0.0;
    __syncthreads();

    const int grp = tid / kGroup, gl = tid % kGroup;
    int sweep = 0;
    for (; sweep < 40 && n > 1; ++sweep) {
        // column norms |u_j|^2 into lam[], exact at every sweep start; within the
        // sweep they are updated analytically (a' = a - t g, b' = b + t g), so a
        // round reduces only the one dot product g
        for (int j0 = 0; j0 < n; j0 += nt / kGroup) {  // uniform trip count
            const int j = j0 + grp;
            double d = 0.0;
            if (j < n)
                for (int i = gl; i < n; i += kGroup) d = fma(U[i + ld * j], U[i + ld * j], d);
            for (int o = kGroup / 2; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            if (j < n && gl == 0) lam[j] = d;
        }
        if (tid == 0) rotated = 0;
        __syncthreads();
        for (int t = 0; t < N - 1; ++t) {
          for (int base = 0; base < N / 2; base += nt / kGroup) {  // uniform trip count
            const int pr = base + grp;
            bool active = pr < N / 2;
            int p = 0, q = 0;
            if (active) {
                const int pq = sched[t * (N / 2) + pr];
                p = pq & 255;
                q = pq >> 8;
                active = q < n;  // dummy player when n is odd
            }
            double* up = U + ld * p;
            double* uq = U + ld * q;
            double xr[kVals], yr[kVals];
            double g = 0.0;
#pragma unroll
            for (int s = 0; s < kVals; ++s) {
                const int i = gl + kGroup * s;
                xr[s] = yr[s] = 0.0;
                if (active && i < n) {
                    xr[s] = up[i];
                    yr[s] = uq[i];
                }
                g = fma(xr[s], yr[s], g);
            }
            // read before the full-warp shuffles: no lane can reach the lam[] update
            // below before every lane of the warp has read its old values
            const double a = active ? lam[p] : 1.0, b = active ? lam[q] : 1.0;
#pragma unroll
            for (int o = kGroup / 2; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
            // rounding in the length-n dot products is ~n eps sqrt(ab): a tighter
            // threshold never converges (measured: 40 sweeps at n = 96 with 1e-15)
            if (active && g * g > tol2 * (a * b)) {
                // t = tan(theta) is the small root of t^2 + 2 zeta t - 1 = 0.  Only
                // MUFU approximations seed it (no fp64 division/sqrt routines, no
                // IEEE slow paths): zeta = (b - a) / 2g uses rcp.approx + one fp64
                // Newton step, t0 an approximate fp32 formula, then one fp64 Newton
                // step on the quadratic; both errors square (~1e-14).  (c, s) are
                // normalised in fp64: the rotation stays orthogonal to fp64 precision.
                double zeta;
                const double g2 = 2.0 * g;
                if (fabs(g2) > 1e-30 && fabs(g2) < 1e30) {
                    const double r0 = double(rcp_approx(float(g2)));
                    zeta = (b - a) * (r0 * fma(-g2, r0, 2.0));
                } else {
                    zeta = (b - a) / g2;
                }
                double tt;
                if (fabs(zeta) < 1e15) {
                    const float zf = float(zeta);
                    const float az = fabsf(zf);
                    const double t0 = double(copysignf(rcp_approx(az + sqrt_approx(fmaf(az, az, 1.0f))), zf));
                    const double f = fma(t0, t0, fma(2.0 * zeta, t0, -1.0));
                    tt = t0 - f * double(rcp_approx(float(2.0 * (t0 + zeta))));
                } else {
                    tt = 0.5 / zeta;
                }
                const double c = rsqrt(fma(tt, tt, 1.0)), s = c * tt;
#pragma unroll
                for (int k = 0; k < kVals; ++k) {
                    const int i = gl + kGroup * k;
                    if (i < n) {
                        up[i] = c * xr[k] - s * yr[k];
                        uq[i] = fma(s, xr[k], c * yr[k]);
                    }
                }
                if (kHasV && usev) {
                    double* vp = V + ld * p;
                    double* vq = V + ld * q;
                    for (int i = gl; i < n; i += kGroup) {
                        const double xv = vp[i], yv = vq[i];
                        vp[i] = c * xv - s * yv;
                        vq[i] = fma(s, xv, c * yv);
                    }
                }
                if (gl == 0) {
                    lam[p] = fma(-tt, g, a);
                    lam[q] = fma(tt, g, b);
                    rotated = 1;
                }
            }
          }
            __syncthreads();
        }
        const bool done = !rotated;
        __syncthreads();  // everyone has read the flag before thread 0 resets it
        if (done) break;
    }
    // eigenvalues: u_j . v_j (general) or |u_j|^2 - sigma (PSD); in the PSD
    // variant V's first row keeps 1/|u_j| for the normalisation below
    for (int j0 = 0; j0 < n; j0 += nt / kGroup) {  // uniform trip count: shuffles stay converged
        const int j = j0 + grp;
        double d = 0.0;
        if (j < n) {
            const double* w = (kHasV && usev) ? V + ld * j : U + ld * j;
            for (int i = gl; i < n; i += kGroup) d = fma(U[i + ld * j], w[i], d);
        }
        for (int o = kGroup / 2; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        if (j < n && gl == 0) {
            lam[j] = d - sigma;
            scl[j] = d > 0.0 ? rsqrt(d) : 0.0;
        }
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
        if (kHasV && usev) {
            for (int r = 0; r < n; ++r) vout[r + size_t(ldv) * rank] = V[r + ld * i];
        } else {
            const double sc = scl[i];
            for (int r = 0; r < n; ++r) vout[r + size_t(ldv) * rank] = U[r + ld * i] * sc;
        }
    }
    if (tid == 0 && sweeps_out) *sweeps_out = sweep;
}

size_t jacobi1s_smem_bytes(int n, bool with_v) {
    const int N = n + (n & 1);
    return (size_t(with_v ? 2 : 1) * (n + 1) * n + 2 * n) * sizeof(double) + size_t(N) * (N / 2) * sizeof(uint16_t) +
           64;
}

template <int G, int MAXN, int MAXT>
void launch_jacobi(atk_ctx* ctx, const double* a, int n, int lda, double* values, double* vectors, int ldv,
                   int* sweeps_dev, bool psd) {
    constexpr bool kHasV = MAXN <= kJacobiMax;
    static bool attr = false;
    if (!attr) {
        ATK_CUDA(cudaFuncSetAttribute(jacobi1s_kernel<G, MAXN, MAXT>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(jacobi1s_smem_bytes(MAXN, kHasV))));
        attr = true;
    }
    const int N = n + (n & 1);
    const int threads = std::min(MAXT, ((G * std::max(1, N / 2)) + 31) / 32 * 32);
    jacobi1s_kernel<G, MAXN, MAXT><<<1, threads, jacobi1s_smem_bytes(n, kHasV), ctx->stream>>>(
        a, n, lda, psd, values, vectors, ldv, sweeps_dev);
    ATK_LAUNCHED(ctx);
}

}  // namespace

void jacobi_eig(atk_ctx* ctx, const double* a, int n, int lda, double* values, double* vectors, int ldv,
                int* sweeps_dev, bool psd) {
    if (n <= kJacobiMax) {
        launch_jacobi<kJacobiGroup, kJacobiMax, kJacobiGroup * ((kJacobiMax + 1) / 2)>(ctx, a, n, lda, values,
                                                                                       vectors, ldv, sweeps_dev, psd);
    } else if (psd && n <= kJacobiPsdMax) {
        launch_jacobi<kJacobiGroup, kJacobiPsdMax, 768>(ctx, a, n, lda, values, vectors, ldv, sweeps_dev, psd);
    } else {
        fail(ATK_UNSUPPORTED, "jacobi_eig: n exceeds the shared-memory capacity");
    }
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
                                                        double* __restrict__ x, int* __restrict__ info,
                                                        double identity_tol) {
    extern __shared__ double sm[];
    const int ld = k + 1;
    double* A = sm;                  // k x k, upper triangle live
    double* W = A + size_t(ld) * k;  // k x k, becomes L^{-1} (unscaled rows)
    const int tid = threadIdx.x, nt = blockDim.x;
    if (identity_tol > 0.0) {  // uniform
        double dev = 0.0;
        for (int e = tid; e < k * k; e += nt) dev = fmax(dev, fabs(g[e] - ((e % k) == (e / k) ? 1.0 : 0.0)));
        for (int o = 16; o > 0; o >>= 1) dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
        if ((tid & 31) == 0) sm[tid >> 5] = dev;
        __syncthreads();
        dev = 0.0;
        for (int q = 0; q < (nt >> 5); ++q) dev = fmax(dev, sm[q]);
        __syncthreads();
        if (dev <= identity_tol) {
            for (int e = tid; e < k * k; e += nt) x[e] = ((e % k) == (e / k)) ? 1.0 : 0.0;
            if (tid == 0) *info = 0;
            return;
        }
    }
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
        // warps over columns, lanes over rows i > c; A(i, c) = A[c + ld i] (symmetry).
        // At most 4 columns per warp (k <= 112 <= 4 x 32 warps... or 4 x nw):
        // unrolled, so the per-column set-up is not a loop-carried chain.
        const int nw = nt >> 5, w0 = tid >> 5, lane = tid & 31;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int j = w0 + q * nw;
            if (j >= k) break;
            if (j <= c) {
                const double wcj = W[c + ld * j] * inv;
                double* wc = W + ld * j;
                for (int i = c + 1 + lane; i < k; i += 32) wc[i] = fma(-A[c + ld * i], wcj, wc[i]);
            } else {
                const double acj = A[c + ld * j] * inv;
                double* ac = A + ld * j;
                for (int i = c + 1 + lane; i <= j; i += 32) ac[i] = fma(-A[c + ld * i], acj, ac[i]);
            }
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

// The same factorisation with the working set in REGISTERS, at compile-time
// positions: thread (warp w of 8, lane l) owns entries (i, j), i = l + 32 m
// (m < MR), j = w + 8 n (n < NC).  G is first scaled to unit diagonal
// (G' = D^-1/2 G D^-1/2, so every pivot d_c lies in (0, 1]).  Position (i, j)
// holds C = A + W, the Gauss-Jordan pair [A | W] superimposed: A's eliminated
// columns are 0 and W (= L'^{-1}, unit lower) is 0 above its diagonal, so the
// row operation row_i -= mult_i row_c is ONE uniform update of every entry,
// C(i, :) -= mult_i C(c, :), mult_i = A(c, i) / d_c for rows i > c (0 for
// finished rows): no per-entry predicates.  The published row c carries
// d_c + 1 at its diagonal (A(c, c) + W(c, c)), which turns column c into
// W(i, c) = -mult_i (error <= ~3 eps relative since d_c <= 1).  Rows are
// processed in groups of 32 with the group index a template parameter, so row
// c + 1's owners (lane (c + 1) mod 32 of every warp) publish their registers
// without run-time register selection: one barrier per step.  (A first layout
// with 32 warps and per-entry live-range predicates issued ~500 instructions
// per warp per step: 120 us at k = 80, slower than the shared-memory column
// kernel.)  Same outputs as chol_inv_kernel: X = L^{-T} with A = L L^T,
// info = 0 or 1 + the failing pivot (a non-positive diagonal entry of G is
// reported as its own pivot).
constexpr int kCtWarps = 8;

template <int MR, int NC, int MM>
__device__ __forceinline__ void chol_tile_step(double (&v)[MR][NC], int c, int k, int lane, int w,
                                               double (*row)[128], double* dinv, double* dpiv, int* bad_sh) {
    const int cb = c & 1, nb = cb ^ 1;
    const double inv = dinv[c];
    double mult[MR], rv[NC];
#pragma unroll
    for (int m = 0; m < MR; ++m) {
        const int i = lane + 32 * m;
        mult[m] = i > c ? row[cb][i] * inv : 0.0;  // A(i, c) = A(c, i); the row is 0 beyond k
    }
#pragma unroll
    for (int n = 0; n < NC; ++n) rv[n] = row[cb][w + kCtWarps * n];
#pragma unroll
    for (int m = 0; m < MR; ++m)
#pragma unroll
        for (int n = 0; n < NC; ++n) v[m][n] = fma(-mult[m], rv[n], v[m][n]);
    const int r1 = c + 1;
    if (r1 < k && lane == (r1 & 31)) {  // publish row c + 1 (final after this step): register row MM
#pragma unroll
        for (int n = 0; n < NC; ++n) row[nb][w + kCtWarps * n] = v[MM][n];
        if (w == (r1 & (kCtWarps - 1))) {  // the diagonal's owner
            const double d = row[nb][r1];   // its own store
            row[nb][r1] = d + 1.0;
            dpiv[r1] = d;
            dinv[r1] = 1.0 / d;
            if (!(d > 0.0)) *bad_sh = r1 + 1;
        }
    }
    __syncthreads();
}

template <int MR, int NC>
__global__ void __launch_bounds__(kCtWarps * 32, 1)
    chol_inv_tile_kernel(const double* __restrict__ g, int k, double* __restrict__ x, int* __restrict__ info,
                         double identity_tol) {
    __shared__ double row[2][128], dinv[128], dpiv[128], sdiag[128];
    __shared__ int bad_sh;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5;
    if (identity_tol > 0.0) {  // uniform
        double dev = 0.0;
        for (int e = tid; e < k * k; e += nt) dev = fmax(dev, fabs(g[e] - ((e % k) == (e / k) ? 1.0 : 0.0)));
        for (int o = 16; o > 0; o >>= 1) dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
        if (lane == 0) row[0][w] = dev;
        __syncthreads();
        dev = 0.0;
        for (int q = 0; q < (nt >> 5); ++q) dev = fmax(dev, row[0][q]);
        __syncthreads();
        if (dev <= identity_tol) {
            for (int e = tid; e < k * k; e += nt) x[e] = ((e % k) == (e / k)) ? 1.0 : 0.0;
            if (tid == 0) *info = 0;
            return;
        }
    }
    if (tid == 0) bad_sh = 0x7fffffff;
    __syncthreads();
    for (int j = tid; j < 128; j += nt) {
        row[0][j] = row[1][j] = 0.0;
        const double gd = j < k ? g[j + size_t(k) * j] : 1.0;
        if (!(gd > 0.0)) atomicMin(&bad_sh, j + 1);  // the first non-positive diagonal entry
        sdiag[j] = gd > 0.0 ? rsqrt(gd) : 0.0;
    }
    __syncthreads();
    if (bad_sh != 0x7fffffff) {  // uniform
        if (tid == 0) *info = bad_sh;
        return;
    }
    __syncthreads();
    if (tid == 0) bad_sh = 0;
    double v[MR][NC];
#pragma unroll
    for (int m = 0; m < MR; ++m)
#pragma unroll
        for (int n = 0; n < NC; ++n) {
            const int i = lane + 32 * m, j = w + kCtWarps * n;
            v[m][n] = (i < k && j < k) ? g[i + size_t(k) * j] * sdiag[i] * sdiag[j] : 0.0;  // both triangles
        }
    if (lane == 0) {  // row 0 (register row 0)
#pragma unroll
        for (int n = 0; n < NC; ++n) row[0][w + kCtWarps * n] = v[0][n];
        if (w == 0) {
            const double d = v[0][0];
            row[0][0] = d + 1.0;
            dpiv[0] = d;
            dinv[0] = 1.0 / d;
        }
    }
    __syncthreads();
    // steps c whose next row c + 1 lies in register row MM: c in [32 MM - 1, 32 MM + 31)
    int bad = 0;
#pragma unroll
    for (int mm = 0; mm < MR; ++mm) {
        const int c_lo = mm == 0 ? 0 : 32 * mm - 1, c_hi = min(k, 32 * mm + 31);
        for (int c = c_lo; c < c_hi && !bad; ++c) {
            if (bad_sh) {  // uniform (read after the barrier that published it)
                bad = bad_sh;
                break;
            }
            if (mm == 0) chol_tile_step<MR, NC, 0>(v, c, k, lane, w, row, dinv, dpiv, &bad_sh);
            else if (mm == 1) chol_tile_step<MR, NC, (MR > 1 ? 1 : 0)>(v, c, k, lane, w, row, dinv, dpiv, &bad_sh);
            else if (mm == 2) chol_tile_step<MR, NC, (MR > 2 ? 2 : 0)>(v, c, k, lane, w, row, dinv, dpiv, &bad_sh);
            else chol_tile_step<MR, NC, (MR > 3 ? 3 : 0)>(v, c, k, lane, w, row, dinv, dpiv, &bad_sh);
        }
    }
    if (!bad && bad_sh) bad = bad_sh;  // the last published pivot
    if (bad) {
        if (tid == 0) *info = bad;
        return;
    }
    // X(j, i) = W(i, j) / sqrt(d_i) / sqrt(g_jj), W(i, i) = 1, W(i, j) = C(i, j) for j < i
#pragma unroll
    for (int m = 0; m < MR; ++m) {
        const int i = lane + 32 * m;
        if (i >= k) continue;
        const double r = rsqrt(dpiv[i]);
#pragma unroll
        for (int n = 0; n < NC; ++n) {
            const int j = w + kCtWarps * n;
            if (j < k) x[j + size_t(k) * i] = j > i ? 0.0 : (j == i ? r : v[m][n] * r) * sdiag[j];
        }
    }
    if (tid == 0) *info = 0;
}

}  // namespace

void cholesky_inv_t(atk_ctx* ctx, const double* g, int k, double* x, int* info_dev, double identity_tol) {
    if (k > kJacobiMax) fail(ATK_UNSUPPORTED, "cholesky_inv_t: k too large");
    const size_t smem = size_t(2) * (k + 1) * k * sizeof(double);
    static bool attr = false;
    if (!attr) {
        ATK_CUDA(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(size_t(2) * (kJacobiMax + 1) * kJacobiMax * sizeof(double))));
        attr = true;
    }
    if (ctx->chol_reg) {
        // 8 warps: warp w owns columns w + 8 n, lanes own rows (chol_inv_tile_kernel)
        constexpr int T = kCtWarps * 32;
        if (k <= 32) chol_inv_tile_kernel<1, 4><<<1, T, 0, ctx->stream>>>(g, k, x, info_dev, identity_tol);
        else if (k <= 64) chol_inv_tile_kernel<2, 8><<<1, T, 0, ctx->stream>>>(g, k, x, info_dev, identity_tol);
        else if (k <= 96) chol_inv_tile_kernel<3, 12><<<1, T, 0, ctx->stream>>>(g, k, x, info_dev, identity_tol);
        else chol_inv_tile_kernel<4, 14><<<1, T, 0, ctx->stream>>>(g, k, x, info_dev, identity_tol);
        ATK_LAUNCHED(ctx);
        return;
    }
    int threads = std::min(1024, std::max(64, 32 * k));  // one warp per column (measured: 128 threads 4x slower)
    static const int th_env = std::getenv("ATK_CHOL_THREADS") ? std::atoi(std::getenv("ATK_CHOL_THREADS")) : 0;
    if (th_env >= 32 && th_env <= 1024) threads = th_env / 32 * 32;  // probe knob
    threads = std::max(threads, 32 * ((k + 3) / 4));                  // <= 4 columns per warp (kernel unroll)
    chol_inv_kernel<<<1, threads, smem, ctx->stream>>>(g, k, x, info_dev, identity_tol);
    ATK_LAUNCHED(ctx);
}

}  // namespace atk
