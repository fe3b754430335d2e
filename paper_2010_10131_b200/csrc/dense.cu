// dense.cu — small fp64 device linear algebra behind linalg.hpp.
//
//  dgemm           : tiled CUDA-core fp64 GEMM (column-major, transposes).
//  jacobi_eig      : one-CTA cyclic two-sided Jacobi with the matrix resident
//                    in shared memory (n <= kJacobiMax): every round rotates
//                    n/2 disjoint pairs (round-robin tournament ordering) and
//                    updates A' = J^T A J as independent 2x2 blocks, so a round
//                    costs two __syncthreads.  Output sorted descending
//                    (linalg.hpp:101-123 keeps the top r of the full spectrum).
//  cholesky*       : linalg::spd_solve (linalg.hpp:169-177), NotSPD on a
//                    non-positive pivot.
//  householder_qr  : linalg::thin_qr (linalg.hpp:126-149) incl. the diag(R)>=0
//                    sign normalisation.
//  fix_signs       : linalg.hpp:34-50.
#include <algorithm>
#include <cmath>

#include "atk_internal.cuh"

namespace atk {
namespace {

// ------------------------------------------------------------------ Jacobi
// Round-robin tournament: position k of round t holds player
//   0                       if k == 0
//   (t + k - 1) % (N-1) + 1 otherwise
// and pairs are (pos[j], pos[N-1-j]).
__device__ __forceinline__ int rr_player(int t, int k, int N) {
    return k == 0 ? 0 : (t + k - 1) % (N - 1) + 1;
}

constexpr int kJacobiThreads = 1024;

__global__ void __launch_bounds__(kJacobiThreads) jacobi_kernel(const double* __restrict__ ain,
                                                                int n, int lda,
                                                                double* __restrict__ values,
                                                                double* __restrict__ vout, int ldv,
                                                                int* __restrict__ sweeps_out) {
    extern __shared__ double sm[];
    const int N = n + (n & 1);  // even number of players (dummy = n when n odd)
    const int ld = n + 1;       // padded smem leading dim
    double* A = sm;             // n x n, A[i + ld*j]
    double* V = A + size_t(ld) * n;
    double* cs = V + size_t(ld) * n;        // 2 * (N/2): c, s per pair
    int* pp = reinterpret_cast<int*>(cs + N);  // p, q per pair
    uint16_t* tab = reinterpret_cast<uint16_t*>(pp + N);  // packed (a << 8 | b), b <= a
    __shared__ int rotated;
    __shared__ double red[33];
    const int tid = threadIdx.x, nt = blockDim.x;
    {
        const int np = N / 2;
        for (int e = tid; e < np * (np + 1) / 2; e += nt) {
            int a = int((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
            while ((a + 1) * (a + 2) / 2 <= e) ++a;
            while (a * (a + 1) / 2 > e) --a;
            tab[e] = uint16_t((a << 8) | (e - a * (a + 1) / 2));
        }
    }

    double fro = 0.0;
    for (int e = tid; e < n * n; e += nt) {
        const int i = e % n, j = e / n;
        const double v = 0.5 * (ain[i + size_t(lda) * j] + ain[j + size_t(lda) * i]);
        A[i + ld * j] = v;
        V[i + ld * j] = (i == j) ? 1.0 : 0.0;
        fro += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
    if ((tid & 31) == 0) red[tid >> 5] = fro;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < (nt >> 5); ++w) t += red[w];
        red[32] = sqrt(t);
    }
    __syncthreads();
    const double floor_abs = 1e-17 * red[32];

    const int npairs = N / 2;
    int sweep = 0;
    for (; sweep < 60 && N > 1; ++sweep) {
        if (tid == 0) rotated = 0;
        __syncthreads();
        for (int t = 0; t < N - 1; ++t) {
            // phase A: rotation per pair
            for (int j = tid; j < npairs; j += nt) {
                int p = rr_player(t, j, N), q = rr_player(t, N - 1 - j, N);
                if (p > q) { const int tmp = p; p = q; q = tmp; }
                double c = 1.0, s = 0.0;
                if (q < n) {
                    const double apq = A[p + ld * q];
                    const double app = A[p + ld * p], aqq = A[q + ld * q];
                    if (fabs(apq) > floor_abs && fabs(apq) > 1e-16 * sqrt(fabs(app * aqq))) {
                        const double theta = (aqq - app) / (2.0 * apq);
                        const double tt = (theta >= 0 ? 1.0 : -1.0) /
                                          (fabs(theta) + sqrt(1.0 + theta * theta));
                        c = 1.0 / sqrt(1.0 + tt * tt);
                        s = tt * c;
                        rotated = 1;
                    }
                }
                cs[2 * j] = c;
                cs[2 * j + 1] = s;
                pp[2 * j] = p;
                pp[2 * j + 1] = q;
            }
            __syncthreads();
            // phase B: 2x2 block updates of A (upper block pairs, mirrored) and V columns
            const int nblk = npairs * (npairs + 1) / 2;
            for (int e = tid; e < nblk + n * npairs; e += nt) {
                if (e < nblk) {
                    const int a = tab[e] >> 8, b = tab[e] & 255;  // b <= a
                    const double ca = cs[2 * a], sa = cs[2 * a + 1];
                    const double cb = cs[2 * b], sb = cs[2 * b + 1];
                    if (sa == 0.0 && sb == 0.0) continue;
                    const int pa = pp[2 * a], qa = pp[2 * a + 1];
                    const int pb = pp[2 * b], qb = pp[2 * b + 1];
                    const bool qa_ok = qa < n, qb_ok = qb < n;
                    // block rows {pa, qa} x cols {pb, qb}
                    const double x11 = A[pa + ld * pb];
                    const double x12 = qb_ok ? A[pa + ld * qb] : 0.0;
                    const double x21 = qa_ok ? A[qa + ld * pb] : 0.0;
                    const double x22 = (qa_ok && qb_ok) ? A[qa + ld * qb] : 0.0;
                    const double m11 = x11 * cb - x12 * sb, m12 = x11 * sb + x12 * cb;
                    const double m21 = x21 * cb - x22 * sb, m22 = x21 * sb + x22 * cb;
                    double n11 = ca * m11 - sa * m21, n12 = ca * m12 - sa * m22;
                    double n21 = sa * m11 + ca * m21, n22 = sa * m12 + ca * m22;
                    if (a == b) {  // diagonal block: the rotation annihilates (pa, qa)
                        n12 = 0.0;
                        n21 = 0.0;
                    }
                    A[pa + ld * pb] = n11;
                    A[pb + ld * pa] = n11;
                    if (qb_ok) { A[pa + ld * qb] = n12; A[qb + ld * pa] = n12; }
                    if (qa_ok) { A[qa + ld * pb] = n21; A[pb + ld * qa] = n21; }
                    if (qa_ok && qb_ok) { A[qa + ld * qb] = n22; A[qb + ld * qa] = n22; }
                } else {
                    const int f = e - nblk;
                    const int i = f % n, a = f / n;
                    const double ca = cs[2 * a], sa = cs[2 * a + 1];
                    if (sa == 0.0) continue;
                    const int pa = pp[2 * a], qa = pp[2 * a + 1];
                    const double vp = V[i + ld * pa], vq = V[i + ld * qa];
                    V[i + ld * pa] = ca * vp - sa * vq;
                    V[i + ld * qa] = sa * vp + ca * vq;
                }
            }
            __syncthreads();
        }
        if (!rotated) break;
        __syncthreads();
    }
    // sort descending by rank (ties broken by index) and emit
    for (int i = tid; i < n; i += nt) {
        const double li = A[i + ld * i];
        int rank = 0;
        for (int j = 0; j < n; ++j) {
            const double lj = A[j + ld * j];
            rank += (lj > li) || (lj == li && j < i);
        }
        values[rank] = li;
        for (int r = 0; r < n; ++r) vout[r + size_t(ldv) * rank] = V[r + ld * i];
    }
    if (tid == 0 && sweeps_out) *sweeps_out = sweep;
}

// ------------------------------------------------------------------ Cholesky
// Right-looking, one CTA, in place on a (n x n, lower).  info = 0 or k+1.
__global__ void cholesky_kernel(double* __restrict__ a, int n, int* __restrict__ info) {
    __shared__ int bad;
    const int tid = threadIdx.x, nt = blockDim.x;
    if (tid == 0) bad = 0;
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        const double d = a[k + size_t(n) * k];
        if (!(d > 0.0)) {
            if (tid == 0) bad = k + 1;
            break;
        }
        const double l = sqrt(d);
        __syncthreads();
        if (tid == 0) a[k + size_t(n) * k] = l;
        for (int i = k + 1 + tid; i < n; i += nt) a[i + size_t(n) * k] /= l;
        __syncthreads();
        const int m = n - k - 1;
        for (int e = tid; e < m * m; e += nt) {
            const int i = k + 1 + e % m, j = k + 1 + e / m;
            if (i >= j) a[i + size_t(n) * j] -= a[i + size_t(n) * k] * a[j + size_t(n) * k];
        }
        __syncthreads();
    }
    __syncthreads();
    if (tid == 0) *info = bad;
    // zero the strict upper triangle (factor is L)
    if (bad == 0)
        for (int e = tid; e < n * n; e += nt) {
            const int i = e % n, j = e / n;
            if (i < j) a[e] = 0.0;
        }
}

// B <- A^{-1} B with A = L L^T: forward then backward substitution, one thread per rhs column.
__global__ void cholesky_solve_kernel(const double* __restrict__ l, int n, double* __restrict__ b,
                                      int nrhs) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nrhs) return;
    double* x = b + size_t(n) * c;
    for (int i = 0; i < n; ++i) {
        double s = x[i];
        for (int k = 0; k < i; ++k) s -= l[i + size_t(n) * k] * x[k];
        x[i] = s / l[i + size_t(n) * i];
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = x[i];
        for (int k = i + 1; k < n; ++k) s -= l[k + size_t(n) * i] * x[k];
        x[i] = s / l[i + size_t(n) * i];
    }
}

// ------------------------------------------------------------------ QR
__device__ double block_reduce_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double t = 0;
    if (w == 0) {
        t = (l < int(blockDim.x >> 5)) ? sh[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (l == 0) sh[32] = t;
    }
    __syncthreads();
    return sh[32];
}

// Householder QR of W (m x n, in place, global), tau[n]; then Q (m x n) and
// R (n x n) with diag(R) >= 0.  One CTA.
__global__ void __launch_bounds__(1024) householder_qr_kernel(double* __restrict__ w, int m,
                                                              int n, double* __restrict__ tau,
                                                              double* __restrict__ q,
                                                              double* __restrict__ r) {
    __shared__ double sh[33];
    extern __shared__ double dots[];  // n column dot products
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nw = nt >> 5;
    for (int k = 0; k < n; ++k) {
        double* col = w + size_t(m) * k;
        double ss = 0.0;
        for (int i = k + 1 + tid; i < m; i += nt) ss += col[i] * col[i];
        const double sigma = block_reduce_sum(ss, sh);
        const double alpha = col[k];
        double beta, t, vscale;
        if (sigma == 0.0) {
            t = 0.0;
            beta = alpha;
            vscale = 0.0;
        } else {
            const double nrm = sqrt(alpha * alpha + sigma);
            beta = alpha <= 0 ? nrm : -nrm;  // beta = -sign(alpha) * ||x||
            t = (beta - alpha) / beta;
            vscale = 1.0 / (alpha - beta);
        }
        __syncthreads();
        // v = [1; col[k+1:] * vscale]; store v below the diagonal, beta on it
        for (int i = k + 1 + tid; i < m; i += nt) col[i] *= vscale;
        if (tid == 0) {
            tau[k] = t;
            col[k] = beta;
        }
        __syncthreads();
        // apply H = I - t v v^T to trailing columns j > k: A_j -= t v (v^T A_j)
        for (int j = k + 1 + warp; j < n; j += nw) {
            const double* cj = w + size_t(m) * j;
            double d = (lane == 0) ? cj[k] : 0.0;
            for (int i = k + 1 + lane; i < m; i += 32) d += col[i] * cj[i];
            for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            if (lane == 0) dots[j] = d;
        }
        __syncthreads();
        for (int j = k + 1; j < n; ++j) {
            double* cj = w + size_t(m) * j;
            const double f = t * dots[j];
            if (f != 0.0) {
                for (int i = k + tid; i < m; i += nt) cj[i] -= f * (i == k ? 1.0 : col[i]);
            }
        }
        __syncthreads();
    }
    // R (upper of w) with sign normalisation, Q = H_0 ... H_{n-1} [I; 0]
    for (int e = tid; e < n * n; e += nt) {
        const int i = e % n, j = e / n;
        r[e] = (i <= j) ? w[i + size_t(m) * j] : 0.0;
    }
    for (int e = tid; e < m * n; e += nt) {
        const int i = e % m, j = e / m;
        q[e] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int k = n - 1; k >= 0; --k) {
        const double t = tau[k];
        const double* col = w + size_t(m) * k;
        for (int j = k + warp; j < n; j += nw) {
            const double* qj = q + size_t(m) * j;
            double d = (lane == 0) ? qj[k] : 0.0;
            for (int i = k + 1 + lane; i < m; i += 32) d += col[i] * qj[i];
            for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            if (lane == 0) dots[j] = d;
        }
        __syncthreads();
        for (int j = k; j < n; ++j) {
            double* qj = q + size_t(m) * j;
            const double f = t * dots[j];
            if (f != 0.0)
                for (int i = k + tid; i < m; i += nt) qj[i] -= f * (i == k ? 1.0 : col[i]);
        }
        __syncthreads();
    }
    // diag(R) >= 0: flip row k of R and column k of Q (linalg.hpp:137-142)
    for (int k = 0; k < n; ++k) {
        if (r[k + size_t(n) * k] < 0.0) {
            for (int c = tid; c < n; c += nt) r[k + size_t(n) * c] = -r[k + size_t(n) * c];
            for (int i = tid; i < m; i += nt) q[i + size_t(m) * k] = -q[i + size_t(m) * k];
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ misc
// fix_signs: one warp per column; largest |v| with the first index on ties.
// One CTA per column (a warp per column was a 64-deep chain of L2 round trips
// at n = 2048): largest |v_i|, ties to the lowest i, then flip if negative.
__global__ void __launch_bounds__(256) fix_signs_kernel(double* __restrict__ v, int n, int r, int ldv) {
    __shared__ double sb[8];
    __shared__ int si[8];
    __shared__ int flip_sh;
    const int col = blockIdx.x;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    double* c = v + size_t(ldv) * col;
    double best = -1.0;
    int bi = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double a = fabs(c[i]);
        if (a > best) { best = a; bi = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (lane == 0) {
        sb[wp] = best;
        si[wp] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = sb[0];
        int ib = si[0];
        for (int q = 1; q < int(blockDim.x >> 5); ++q)
            if (sb[q] > b || (sb[q] == b && si[q] < ib)) { b = sb[q]; ib = si[q]; }
        flip_sh = c[ib] < 0.0;
    }
    __syncthreads();
    if (flip_sh)
        for (int i = threadIdx.x; i < n; i += blockDim.x) c[i] = -c[i];
}

__global__ void symmetrize_kernel(double* a, int n) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * n) return;
    const int i = e % n, j = e / n;
    if (i < j) {
        const double v = 0.5 * (a[i + size_t(n) * j] + a[j + size_t(n) * i]);
        a[i + size_t(n) * j] = v;
        a[j + size_t(n) * i] = v;
    }
}

__global__ void identity_kernel(double* a, int n) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * n) return;
    a[e] = (e % n == e / n) ? 1.0 : 0.0;
}

__global__ void transpose_kernel(const double* a, int rows, int cols, double* at) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * cols) return;
    const int i = e % rows, j = e / rows;
    at[j + size_t(cols) * i] = a[e];
}

inline unsigned blocks_for(size_t n, int t) { return unsigned((n + t - 1) / t); }

}  // namespace

size_t jacobi_smem_bytes(int n) {
    const int N = n + (n & 1);
    const int np = N / 2;
    return size_t(2) * (n + 1) * n * sizeof(double) + size_t(N) * sizeof(double) +
           size_t(N) * sizeof(int) + size_t(np) * (np + 1) / 2 * sizeof(uint16_t) + 64;
}

// Two-sided variant kept for A/B checks (option "jacobi2s"); the default is jacobi.cu.
void jacobi2s_eig(atk_ctx* ctx, const double* a, int n, int lda, double* values, double* vectors,
                  int ldv, int* sweeps_dev) {
    if (n > kJacobiMax) fail(ATK_UNSUPPORTED, "jacobi_eig: n exceeds the shared-memory capacity");
    const size_t smem = jacobi_smem_bytes(n);
    ATK_CUDA(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    jacobi_kernel<<<1, kJacobiThreads, smem, ctx->stream>>>(a, n, lda, values, vectors, ldv, sweeps_dev);
    ATK_LAUNCHED(ctx);
}

void cholesky(atk_ctx* ctx, double* a, int n, int* info_dev) {
    cholesky_kernel<<<1, 512, 0, ctx->stream>>>(a, n, info_dev);
    ATK_LAUNCHED(ctx);
}

void cholesky_solve(atk_ctx* ctx, const double* l, int n, double* b, int nrhs) {
    cholesky_solve_kernel<<<blocks_for(nrhs, 64), 64, 0, ctx->stream>>>(l, n, b, nrhs);
    ATK_LAUNCHED(ctx);
}

void householder_qr(atk_ctx* ctx, const double* a, int m, int n, double* q, double* r) {
    // any n (the ALS factor QR for R > 112, where CholeskyQR's one-CTA Cholesky does not fit)
    const size_t smem = size_t(std::max(n, 1)) * sizeof(double);
    if (smem > smem_cap_bytes()) fail(ATK_UNSUPPORTED, "householder_qr: too many columns for one CTA");
    static size_t attr = 48 * 1024;
    if (smem > attr) {
        ATK_CUDA(cudaFuncSetAttribute(householder_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr = smem;
    }
    DevBuf<double> w(ctx, size_t(m) * n + n);
    ATK_CUDA(cudaMemcpyAsync(w.get(), a, size_t(m) * n * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
    householder_qr_kernel<<<1, 1024, smem, ctx->stream>>>(w.get(), m, n, w.get() + size_t(m) * n, q, r);
    ATK_LAUNCHED(ctx);
}

void fix_signs(atk_ctx* ctx, double* v, int n, int r, int ldv) {
    if (r <= 0 || n <= 0) return;
    fix_signs_kernel<<<unsigned(r), 256, 0, ctx->stream>>>(v, n, r, ldv);
    ATK_LAUNCHED(ctx);
}

void symmetrize(atk_ctx* ctx, double* a, int n) {
    symmetrize_kernel<<<blocks_for(size_t(n) * n, 256), 256, 0, ctx->stream>>>(a, n);
    ATK_LAUNCHED(ctx);
}

void set_identity(atk_ctx* ctx, double* a, int n) {
    identity_kernel<<<blocks_for(size_t(n) * n, 256), 256, 0, ctx->stream>>>(a, n);
    ATK_LAUNCHED(ctx);
}

void transpose(atk_ctx* ctx, const double* a, int rows, int cols, double* at) {
    transpose_kernel<<<blocks_for(size_t(rows) * cols, 256), 256, 0, ctx->stream>>>(a, rows, cols, at);
    ATK_LAUNCHED(ctx);
}

namespace {
__global__ void zero_lower_kernel(double* r, int n) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x)
        if (e % n > e / n) r[e] = 0.0;
}
}  // namespace

void zero_lower(atk_ctx* ctx, double* r, int n) {
    zero_lower_kernel<<<std::max(1, std::min(64, (n * n + 255) / 256)), 256, 0, ctx->stream>>>(r, n);
    ATK_LAUNCHED(ctx);
}

}  // namespace atk
