// tridiag.cu — dense symmetric eigensolver for n <= kTridiagMax by reduction
// to tridiagonal form (the structure of LAPACK dsytrd + dstebz + dstein +
// dormtr; the reference's Eigen SelfAdjointEigenSolver, linalg.hpp:101-123,
// also tridiagonalises first, then runs implicit QR).  Four launches:
//
//  1. trd_kernel (one CTA, 1024 threads): Householder reduction A = Q T Q^T
//     of the symmetrised input, packed lower triangle resident in shared memory
//     (n <= 200: 160.8 KB).  Warps own columns (j = w mod 32), lanes own rows
//     (i = lane mod 32) so the symmetric matvec reads each stored element once
//     and the rank-2 update touches it once; the matvec's row partials go
//     through a per-warp buffer summed in a fixed order (no atomics: results
//     are bit-reproducible, which the sharded multi-GPU path relies on).
//     Three barriers per Householder step.
//  2. bisect_kernel (one warp per wanted eigenvalue): Sturm-count
//     multisection, 32 shifts per pass (each pass narrows the bracket 33x).
//  3. invit_kernel (one warp per cluster): inverse iteration on T - lambda I
//     (tridiagonal LU with partial pivoting, dgttrf/dgttrs), 3 iterations from
//     a fixed pseudo-random start.  Eigenvalues closer than 1e-3 ||T||_1 form a
//     cluster (dstein's criterion): the cluster's members are solved in
//     parallel, one lane each, and Gram-Schmidt-orthogonalised in order after
//     every iteration.
//  4. backtr_kernel (one warp per vector): x <- H_0 ... H_{n-3} x with the
//     Householder vectors staged in shared memory.
//
// Only the wanted top `nwant` pairs are formed (the reference computes all n
// and discards n - r).  Values descending; signs are fixed by the caller.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "atk_internal.cuh"

namespace atk {
namespace {

constexpr int kRowSlots = (kTridiagMax + 31) / 32;  // rows per lane

__device__ __forceinline__ int pk(int i, int j, int n) {  // A(i, j), i >= j, packed lower
    return j * n - (j * (j - 1)) / 2 + (i - j);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Publish reflector c (c + 2 < n) from the current column c: every lane of
// the calling warp; writes T's d[c], e[c], tau[c], scal[c] and the dense v
// (zero outside rows c+1..n-1) into vb.  dsytd2 / dlarfg conventions.
template <int S>
__device__ __forceinline__ void publish_reflector(const double* AP, int n, int c, double* vb, double* sh_tau,
                                                  double* d, double* e, double* tau_out, double* scal_out) {
    const int lane = threadIdx.x & 31;
    const int cc = pk(c, c, n) - c;
    const double alpha = AP[cc + c + 1];
    double x[S], xn = 0.0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int i = lane + 32 * s;
        x[s] = (i >= c + 2 && i < n) ? AP[cc + i] : 0.0;
        xn = fma(x[s], x[s], xn);
    }
    xn = warp_sum(xn);
    double tau = 0.0, scal = 0.0, beta = alpha;
    if (xn > 0.0) {
        beta = -copysign(sqrt(fma(alpha, alpha, xn)), alpha);
        scal = 1.0 / (alpha - beta);
        tau = (beta - alpha) / beta;
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int i = lane + 32 * s;
        vb[i] = (i == c + 1) ? 1.0 : x[s] * scal;
    }
    if (lane == 0) {
        d[c] = AP[cc + c];
        e[c] = beta;
        tau_out[c] = tau;
        scal_out[c] = scal;
        *sh_tau = tau;
    }
}

// hh: packed lower triangle after the reduction (column k below the diagonal =
// the unscaled Householder vector k); d, e: T; tau, scal: reflector k is
// H_k = I - tau_k v v^T with v_{k+1} = 1, v_i = hh(i, k) * scal_k (i > k + 1).
// S = ceil(n / 32) row slots per lane (a template: no dead slots for small n).
template <int S, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
    trd_kernel(const double* __restrict__ a, int n, int lda, double* __restrict__ hh, double* __restrict__ d,
               double* __restrict__ e, double* __restrict__ tau_out, double* __restrict__ scal_out,
               long long* __restrict__ prof) {
    extern __shared__ double sm[];
    long long t_mark = clock64(), t_acc[6] = {0, 0, 0, 0, 0, 0};  // ATK_TRD_PROFILE: cycles per phase
    auto lap = [&](int ph) {
        if (prof) {
            const long long t = clock64();
            t_acc[ph] += t - t_mark;
            t_mark = t;
        }
    };
    constexpr int NR = 32 * S;             // padded rows
    const int np = n * (n + 1) / 2;
    double* AP = sm;                       // np + NR zero pad (reads past the end stay finite)
    double* part = AP + np + NR;           // NW x n row partials of the matvec
    double* dots = part + NW * n;          // n: column dots of the matvec
    double* p = dots + n;                  // NR
    double* vbuf = p + NR;                 // 2 x NR (reflector k in vbuf[k & 1])
    double* vav = vbuf + 2 * NR;           // NW partials of v^T A v
    double* sc = vav + NW;                 // tau[2], K
    constexpr int NT = NW * 32, TPR = NT / 256;  // B2: threads per row (rows <= 256)
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (int j = 0; j < n; ++j)
        for (int i = j + tid; i < n; i += NT)
            AP[pk(i, j, n)] = 0.5 * (a[i + size_t(lda) * j] + a[j + size_t(lda) * i]);
    for (int q = tid; q < NR; q += NT) {
        AP[np + q] = 0.0;
        p[q] = 0.0;
    }
    for (int q = tid; q < NW * n; q += NT) part[q] = 0.0;
    __syncthreads();
    lap(0);
    if (n > 2 && w == 0) publish_reflector<S>(AP, n, 0, vbuf, sc, d, e, tau_out, scal_out);
    __syncthreads();
    lap(0);

    for (int k = 0; k + 2 < n; ++k) {
        const double tau = sc[k & 1];
        const double* vk = vbuf + (k & 1) * NR;
        const int j0 = k + 1 + ((w - (k + 1)) % NW + NW) % NW;
        const bool next = k + 3 < n;  // reflector k+1 exists
        if (tau != 0.0) {  // uniform
            double v[S], acc[S];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                v[s] = vk[lane + 32 * s];
                acc[s] = 0.0;
            }
            // ---- B: symmetric matvec A22 v (warp w: columns j = w mod NW), v^T A v partial.
            //      Four columns per pass with their warp reductions interleaved (the
            //      per-column shuffle chains are the latency that bounds this phase).
            double vav_l = 0.0;
            for (int jb = j0; jb < n; jb += 4 * NW) {
                double dt[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int j = jb + c * NW;
                    dt[c] = 0.0;
                    if (j >= n) continue;  // warp-uniform
                    const double vj = vk[j];
                    const int cj = pk(j, j, n) - j;
                    const int s0 = j >> 5;
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        if (s < s0) continue;  // warp-uniform
                        const int i = lane + 32 * s;
                        const double aij = AP[cj + i];
                        if (s == s0) {  // the diagonal slot: rows i >= j only
                            dt[c] = fma(i >= j ? aij : 0.0, v[s], dt[c]);
                            acc[s] = fma(i > j ? aij : 0.0, vj, acc[s]);
                        } else {
                            dt[c] = fma(aij, v[s], dt[c]);
                            acc[s] = fma(aij, vj, acc[s]);
                        }
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                    for (int c = 0; c < 4; ++c) dt[c] += __shfl_xor_sync(0xffffffffu, dt[c], o);
                if (lane == 0)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int j = jb + c * NW;
                        if (j < n) {
                            dots[j] = dt[c];
                            vav_l = fma(vk[j], dt[c], vav_l);
                        }
                    }
            }
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const int i = lane + 32 * s;
                vav_l = fma(v[s], acc[s], vav_l);
                if (i > k && i < n) part[w * n + i] = acc[s];
            }
            vav_l = warp_sum(vav_l);
            if (lane == 0) vav[w] = vav_l;
            lap(1);
            __syncthreads();
            lap(2);
            // ---- B2: p = tau (dots + sum_w part[w]) in a fixed order, TPR threads per row;
            //      K = (tau / 2) p^T v = (tau^2 / 2) v^T A v
            {
                const int row = k + 1 + tid / TPR, q0 = tid % TPR;
                double s0 = 0.0;
                if (row < n)
#pragma unroll
                    for (int q = q0; q < NW; q += TPR) s0 += part[q * n + row];
#pragma unroll
                for (int o = 1; o < TPR; o <<= 1) s0 += __shfl_xor_sync(0xffffffffu, s0, o);
                if (row < n && q0 == 0) p[row] = tau * (dots[row] + s0);
                if (tid == NT - 1) {
                    double t = 0.0;
                    for (int q = 0; q < NW; ++q) t += vav[q];
                    sc[2] = 0.5 * tau * tau * t;
                }
            }
            __syncthreads();
            lap(3);
            // ---- C: w = p - K v ; A22 -= v w^T + w v^T (owned columns); the owner of
            //      column k+1 then publishes reflector k+1 from the updated column
            const double K = sc[2];
            double wr[S];
#pragma unroll
            for (int s = 0; s < S; ++s) wr[s] = fma(-K, v[s], p[lane + 32 * s]);
            // two columns per pass: all loads issued before the stores (ILP)
            for (int jb = j0; jb < n; jb += 2 * NW) {
                double nv[2][S];
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int j = jb + c * NW;
                    if (j >= n) continue;  // warp-uniform
                    const double vj = vk[j];
                    const double wj = fma(-K, vj, p[j]);
                    const int cj = pk(j, j, n) - j;
                    const int s0 = j >> 5;
#pragma unroll
                    for (int s = 0; s < S; ++s)
                        if (s >= s0) nv[c][s] = fma(-v[s], wj, fma(-wr[s], vj, AP[cj + lane + 32 * s]));
                }
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int j = jb + c * NW;
                    if (j >= n) continue;
                    const int cj = pk(j, j, n) - j;
                    const int s0 = j >> 5;
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        if (s < s0) continue;  // warp-uniform
                        const int i = lane + 32 * s;
                        if (s == s0) {
                            if (i >= j && i < n) AP[cj + i] = nv[c][s];
                        } else if (s + 1 < S || i < n) {  // only the last slot can run past n
                            AP[cj + i] = nv[c][s];
                        }
                    }
                    if (j == k + 1 && next) {
                        __syncwarp();
                        publish_reflector<S>(AP, n, k + 1, vbuf + ((k + 1) & 1) * NR, sc + ((k + 1) & 1), d, e,
                                             tau_out, scal_out);
                    }
                }
            }
        } else if (next && w == ((k + 1) & (NW - 1))) {  // H_k = I: column k+1 unchanged
            publish_reflector<S>(AP, n, k + 1, vbuf + ((k + 1) & 1) * NR, sc + ((k + 1) & 1), d, e, tau_out,
                                 scal_out);
        }
        lap(4);
        __syncthreads();
        lap(5);
    }
    if (tid == 0) {
        if (n >= 2) {
            d[n - 2] = AP[pk(n - 2, n - 2, n)];
            e[n - 2] = AP[pk(n - 1, n - 2, n)];
            tau_out[n - 2] = 0.0;
            scal_out[n - 2] = 0.0;
        }
        d[n - 1] = AP[pk(n - 1, n - 1, n)];
        tau_out[n - 1] = 0.0;
        scal_out[n - 1] = 0.0;
    }
    for (int q = tid; q < np; q += NT) hh[q] = AP[q];
    if (prof && (lane == 0))
        for (int q = 0; q < 6; ++q) atomicAdd(reinterpret_cast<unsigned long long*>(prof + q), (unsigned long long)t_acc[q]);
}

// ||T||_1 (= ||T||_inf) and the Gershgorin interval, warp-cooperative.
struct TNorm {
    double lo, hi, norm;
};
__device__ TNorm tnorm_warp(const double* d, const double* e, int n) {
    const int lane = threadIdx.x & 31;
    double lo = DBL_MAX, hi = -DBL_MAX, nm = 0.0;
    for (int i = lane; i < n; i += 32) {
        const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0);
        lo = fmin(lo, d[i] - r);
        hi = fmax(hi, d[i] + r);
        nm = fmax(nm, fabs(d[i]) + r);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        nm = fmax(nm, __shfl_xor_sync(0xffffffffu, nm, o));
    }
    return {lo, hi, nm};
}

// Number of eigenvalues of T below x (Sturm sequence of the LDL^T pivots).
__device__ __forceinline__ int sturm_count(const double* __restrict__ d, const double* __restrict__ e2, int n,
                                           double x, double pivmin) {
    double q = d[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    int c = q < 0.0;
    for (int i = 1; i < n; ++i) {
        // e2 / q by rcp.approx + one Newton step (relative error ~2^-44: the count is
        // exact for e2 perturbed by ~1e-13 relative, far inside the 1e-12 bars; the
        // second step cost a fifth of the serial chain)
        double r;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
        r = r * fma(-q, r, 2.0);
        q = fma(-e2[i - 1], r, d[i] - x);
        if (fabs(q) < pivmin) q = -pivmin;
        c += q < 0.0;
    }
    return c;
}

// C Sturm counts at once (independent chains interleaved: the serial
// rcp + Newton + fma chain of one count is latency-bound, so C counts cost
// about one).  Same arithmetic per count as sturm_count.
template <int C>
__device__ __forceinline__ void sturm_count_multi(const double* __restrict__ d, const double* __restrict__ e2, int n,
                                                  const double (&x)[C], double pivmin, int (&cnt)[C]) {
    double q[C];
    const double d0 = d[0];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        q[c] = d0 - x[c];
        if (fabs(q[c]) < pivmin) q[c] = -pivmin;
        cnt[c] = q[c] < 0.0;
    }
    for (int i = 1; i < n; ++i) {
        const double di = d[i], e2i = e2[i - 1];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            double r;
            asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q[c]));
            r = r * fma(-q[c], r, 2.0);
            q[c] = fma(-e2i, r, di - x[c]);
            if (fabs(q[c]) < pivmin) q[c] = -pivmin;
            cnt[c] += q[c] < 0.0;
        }
    }
}

// values[j] = the j-th largest eigenvalue of T, j < nwant.  One warp per j:
// multisection with 32 C shifts per pass (C chains per lane), d and e^2 in
// shared memory.  A pass narrows the interval (32 C + 1)x.
template <int kBisC>
__global__ void __launch_bounds__(256) bisect_kernel(const double* __restrict__ d, const double* __restrict__ e,
                                                     int n, int nwant, double* __restrict__ values) {
    extern __shared__ double e2s[];  // e^2 (n - 1), then d (n)
    double* ds = e2s + n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        if (i + 1 < n) e2s[i] = e[i] * e[i];
        ds[i] = d[i];
    }
    __syncthreads();
    const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (j >= nwant) return;
    const TNorm tn = tnorm_warp(ds, e, n);
    double emax2 = 0.0;
    for (int i = lane; i + 1 < n; i += 32) emax2 = fmax(emax2, e2s[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) emax2 = fmax(emax2, __shfl_xor_sync(0xffffffffu, emax2, o));
    const double pivmin = DBL_MIN * fmax(1.0, emax2);
    const double eps = DBL_EPSILON;
    const double slack = 2.0 * eps * tn.norm * n + 2.0 * pivmin;
    double lo = tn.lo - slack, hi = tn.hi + slack;
    const int t = n - 1 - j;  // ascending index
    const double atol = 2.0 * eps * tn.norm;
    constexpr int NS = 32 * kBisC;  // shifts per pass, s = c 32 + lane (increasing x)
    for (int it = 0; it < 64; ++it) {
        const double wdt = hi - lo;
        if (!(wdt > fmax(atol, 2.0 * eps * fmax(fabs(lo), fabs(hi))))) break;
        double x[kBisC];
        int cnt[kBisC];
#pragma unroll
        for (int c = 0; c < kBisC; ++c) x[c] = lo + wdt * double(c * 32 + lane + 1) / double(NS + 1);
        sturm_count_multi<kBisC>(ds, e2s, n, x, pivmin, cnt);
        int first = NS;  // the first shift with count >= t + 1
#pragma unroll
        for (int c = kBisC - 1; c >= 0; --c) {
            const unsigned b = __ballot_sync(0xffffffffu, cnt[c] >= t + 1);
            if (b) first = c * 32 + __ffs(b) - 1;
        }
        auto xs = [&](int s) { return lo + wdt * double(s + 1) / double(NS + 1); };
        if (first < NS) {
            const double nl = first > 0 ? xs(first - 1) : lo;
            hi = xs(first);
            lo = nl;
        } else {
            lo = xs(NS - 1);
        }
    }
    if (lane == 0) values[j] = tn.norm > 0.0 ? 0.5 * (lo + hi) : 0.0;  // T = 0: exactly zero
}

// d and e^2 staged in shared memory: 2 n doubles (n = 4096: 64 KB, above the default 48 KB)
void bisect_launch(atk_ctx* ctx, const double* d, const double* e, int n, int nvals, double* values) {
    // 2 warps per CTA (the wanted values spread over ~nvals / 2 SMs: the fp64 reciprocal pipe, not
    // the chain latency, bounds 8 warps per SM) and 2 interleaved chains per lane (64 shifts per
    // pass): C5's n = 80 block 41 -> 35 us, n = 2048 876 -> 707 us (profiles/bisect_sweep.sh)
    static const int wpb = std::getenv("ATK_BIS_WPB") ? std::atoi(std::getenv("ATK_BIS_WPB")) : 2;  // probe knobs
    static const int nc = std::getenv("ATK_BIS_C") ? std::atoi(std::getenv("ATK_BIS_C")) : 2;
    const size_t smem = 2 * size_t(n) * sizeof(double);
    static size_t attr = 48 * 1024;
    if (smem > attr) {
        ATK_CUDA(cudaFuncSetAttribute(bisect_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        ATK_CUDA(cudaFuncSetAttribute(bisect_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        ATK_CUDA(cudaFuncSetAttribute(bisect_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr = smem;
    }
    const dim3 g((nvals + wpb - 1) / wpb), b(32 * wpb);
    if (nc == 1) bisect_kernel<1><<<g, b, smem, ctx->stream>>>(d, e, n, nvals, values);
    else if (nc == 2) bisect_kernel<2><<<g, b, smem, ctx->stream>>>(d, e, n, nvals, values);
    else bisect_kernel<4><<<g, b, smem, ctx->stream>>>(d, e, n, nvals, values);
}

__device__ __forceinline__ double hash_unit(uint64_t x) {  // splitmix64 -> (-1, 1)
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return double(int64_t(x >> 11) - (int64_t(1) << 52)) * (1.0 / 4503599627370496.0);
}

// Inverse iteration for the wanted eigenvalues (descending, lam[0..nwant)).
// X: n x nwant (ld n) eigenvectors of T.  wk: 5 n doubles per member.
__global__ void __launch_bounds__(256) invit_kernel(const double* __restrict__ d, const double* __restrict__ e,
                                                    int n, const double* __restrict__ lam, int nwant,
                                                    double* __restrict__ X, double* __restrict__ wk,
                                                    const int* __restrict__ skip = nullptr) {
    const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (j >= nwant || (skip && *skip)) return;
    const TNorm tn = tnorm_warp(d, e, n);
    const double ortol = 1e-3 * tn.norm;
    if (j > 0 && lam[j - 1] - lam[j] <= ortol) return;  // not a cluster leader
    int end = j + 1;
    while (end < nwant && lam[end - 1] - lam[end] <= ortol) ++end;
    const double pertol = 10.0 * DBL_EPSILON * fmax(tn.norm, DBL_MIN);
    const double tiny = tn.norm > 0.0 ? DBL_EPSILON * tn.norm : 1.0;  // pivot floor
    for (int cb = j; cb < end; cb += 32) {
        const int mm = cb + lane;
        const bool mine = mm < end;
        double* x = X + size_t(n) * (mine ? mm : j);
        // the chunk's factors interleaved by member (lane): array a, row i at
        // base[(a n + i) cs + lane], so a warp's accesses are contiguous
        const int cs = min(32, end - cb);
        double* base = wk + size_t(5) * n * cb + (mine ? lane : 0);
        const size_t st = size_t(cs);
        double* dl = base;                  // L multipliers
        double* dd = base + size_t(n) * st;  // 1 / U(i, i)
        double* du = dd + size_t(n) * st;
        double* du2 = du + size_t(n) * st;
        double* pv = du2 + size_t(n) * st;  // 1.0 where rows i, i + 1 were interchanged
        if (mine) {
            // shift, kept >= pertol below the previous member (dstein)
            double sh = lam[j];
            for (int q = j + 1; q <= mm; ++q) sh = fmin(lam[q], sh - pertol);
            // dgttrf on T - sh I (one division per row: f = l * (1 / pivot))
            double di = d[0] - sh, ui = n > 1 ? e[0] : 0.0;
            for (int i = 0; i + 1 < n; ++i) {
                const double li = e[i], dn = d[i + 1] - sh, un = i + 2 < n ? e[i + 1] : 0.0;
                if (fabs(di) >= fabs(li)) {
                    if (fabs(di) < tiny) di = copysign(tiny, di);
                    const double r = 1.0 / di;
                    const double f = li * r;
                    dl[i * st] = f;
                    dd[i * st] = r;
                    du[i * st] = ui;
                    du2[i * st] = 0.0;
                    pv[i * st] = 0.0;
                    di = fma(-f, ui, dn);
                    ui = un;
                } else {
                    const double r = 1.0 / li;
                    const double f = di * r;
                    dl[i * st] = f;
                    dd[i * st] = r;
                    du[i * st] = dn;
                    du2[i * st] = un;
                    pv[i * st] = 1.0;
                    di = fma(-f, dn, ui);
                    ui = -f * un;
                }
            }
            if (fabs(di) < tiny) di = copysign(tiny, di);
            dd[(n - 1) * st] = 1.0 / di;
            for (int i = 0; i < n; ++i) x[i] = hash_unit(uint64_t(mm) * 1000003ULL + i);
        }
        for (int it = 0; it < 3; ++it) {
            if (mine) {
                // dgttrs: L (with interchanges; the running entry stays in a register) then U
                double cr = x[0];
                for (int i = 0; i + 1 < n; ++i) {
                    const double nx = x[i + 1];
                    if (pv[i * st] != 0.0) {
                        x[i] = nx;
                        cr = fma(-dl[i * st], nx, cr);
                    } else {
                        x[i] = cr;
                        cr = fma(-dl[i * st], cr, nx);
                    }
                }
                x[n - 1] = cr;
                double x2 = 0.0, x1 = x[n - 1] * dd[(n - 1) * st];
                x[n - 1] = x1;
                for (int i = n - 2; i >= 0; --i) {
                    const double xi = (x[i] - du[i * st] * x1 - du2[i * st] * x2) * dd[i * st];
                    x[i] = xi;
                    x2 = x1;
                    x1 = xi;
                }
            }
            __syncwarp();
            // Gram-Schmidt of this chunk's members, in order, against every
            // earlier member of the cluster (orthonormal already), then normalise
            const int cend = min(end, cb + 32);
            for (int q = cb; q < cend; ++q) {
                double* xq = X + size_t(n) * q;
                double mx = 0.0;
                for (int i = lane; i < n; i += 32) mx = fmax(mx, fabs(xq[i]));
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                const double sc = mx > 0.0 ? 1.0 / mx : 1.0;  // pre-scale: the solve grows x by ~1/eps
                for (int i = lane; i < n; i += 32) xq[i] *= sc;
                __syncwarp();
                for (int u = j; u < q; ++u) {
                    const double* xu = X + size_t(n) * u;
                    double dt = 0.0;
                    for (int i = lane; i < n; i += 32) dt = fma(xu[i], xq[i], dt);
                    dt = warp_sum(dt);
                    for (int i = lane; i < n; i += 32) xq[i] = fma(-dt, xu[i], xq[i]);
                    __syncwarp();
                }
                double nr = 0.0;
                for (int i = lane; i < n; i += 32) nr = fma(xq[i], xq[i], nr);
                nr = warp_sum(nr);
                const double inv = nr > 0.0 ? 1.0 / sqrt(nr) : 0.0;
                for (int i = lane; i < n; i += 32) xq[i] *= inv;
                __syncwarp();
            }
        }
    }
}

// invit_kernel with the working set in SHARED memory (n <= kIvSmemMax): one
// warp per CTA (CTA j = wanted vector j; non-leaders exit), the chunk's
// iterates x and their tridiagonal LU factors interleaved by member (lane) at
// stride 32.  Same arithmetic and order as invit_kernel.  The global-memory
// version's solve loops were a chain of L2 round trips (a store to x[i] then a
// dependent load of x[i + 1], factors re-read from L2): 70 us for C5's
// Rayleigh-Ritz block (n = 80, 64 vectors).
constexpr int kIvSmemMax = 128;  // 6 n x 32 doubles = 192 KB
__global__ void __launch_bounds__(32) invit_smem_kernel(const double* __restrict__ d, const double* __restrict__ e,
                                                         int n, const double* __restrict__ lam, int nwant,
                                                         double* __restrict__ X, const int* __restrict__ skip) {
    extern __shared__ double sm[];
    const int j = blockIdx.x;
    const int lane = threadIdx.x & 31;
    if (j >= nwant || (skip && *skip)) return;
    const TNorm tn = tnorm_warp(d, e, n);
    const double ortol = 1e-3 * tn.norm;
    if (j > 0 && lam[j - 1] - lam[j] <= ortol) return;  // not a cluster leader
    int end = j + 1;
    while (end < nwant && lam[end - 1] - lam[end] <= ortol) ++end;
    const double pertol = 10.0 * DBL_EPSILON * fmax(tn.norm, DBL_MIN);
    const double tiny = tn.norm > 0.0 ? DBL_EPSILON * tn.norm : 1.0;  // pivot floor
    constexpr int st = 32;
    double* xs = sm;  // member c of the chunk: xs[i st + c]
    double* x = xs + lane;
    double* dl = sm + size_t(n) * st + lane;  // L multipliers
    double* dd = dl + size_t(n) * st;         // 1 / U(i, i)
    double* du = dd + size_t(n) * st;
    double* du2 = du + size_t(n) * st;
    double* pv = du2 + size_t(n) * st;  // 1.0 where rows i, i + 1 were interchanged
    for (int cb = j; cb < end; cb += 32) {
        const int mm = cb + lane;
        const bool mine = mm < end;
        if (mine) {
            // shift, kept >= pertol below the previous member (dstein)
            double sh = lam[j];
            for (int q = j + 1; q <= mm; ++q) sh = fmin(lam[q], sh - pertol);
            // dgttrf on T - sh I (one division per row: f = l * (1 / pivot))
            double di = d[0] - sh, ui = n > 1 ? e[0] : 0.0;
            for (int i = 0; i + 1 < n; ++i) {
                const double li = e[i], dn = d[i + 1] - sh, un = i + 2 < n ? e[i + 1] : 0.0;
                if (fabs(di) >= fabs(li)) {
                    if (fabs(di) < tiny) di = copysign(tiny, di);
                    const double r = 1.0 / di;
                    const double f = li * r;
                    dl[i * st] = f;
                    dd[i * st] = r;
                    du[i * st] = ui;
                    du2[i * st] = 0.0;
                    pv[i * st] = 0.0;
                    di = fma(-f, ui, dn);
                    ui = un;
                } else {
                    const double r = 1.0 / li;
                    const double f = di * r;
                    dl[i * st] = f;
                    dd[i * st] = r;
                    du[i * st] = dn;
                    du2[i * st] = un;
                    pv[i * st] = 1.0;
                    di = fma(-f, dn, ui);
                    ui = -f * un;
                }
            }
            if (fabs(di) < tiny) di = copysign(tiny, di);
            dd[(n - 1) * st] = 1.0 / di;
            for (int i = 0; i < n; ++i) x[i * st] = hash_unit(uint64_t(mm) * 1000003ULL + i);
        }
        const int cend = min(end, cb + 32);
        for (int it = 0; it < 3; ++it) {
            if (mine) {
                double cr = x[0];
                for (int i = 0; i + 1 < n; ++i) {
                    const double nx = x[(i + 1) * st];
                    if (pv[i * st] != 0.0) {
                        x[i * st] = nx;
                        cr = fma(-dl[i * st], nx, cr);
                    } else {
                        x[i * st] = cr;
                        cr = fma(-dl[i * st], cr, nx);
                    }
                }
                x[(n - 1) * st] = cr;
                double x2 = 0.0, x1 = x[(n - 1) * st] * dd[(n - 1) * st];
                x[(n - 1) * st] = x1;
                for (int i = n - 2; i >= 0; --i) {
                    const double xi = (x[i * st] - du[i * st] * x1 - du2[i * st] * x2) * dd[i * st];
                    x[i * st] = xi;
                    x2 = x1;
                    x1 = xi;
                }
            }
            __syncwarp();
            // Gram-Schmidt of the chunk's members in order against every earlier
            // member of the cluster (earlier chunks: final, in X), then normalise
            for (int q = cb; q < cend; ++q) {
                double* xq = xs + (q - cb);
                double mx = 0.0;
                for (int i = lane; i < n; i += 32) mx = fmax(mx, fabs(xq[i * st]));
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                const double sc = mx > 0.0 ? 1.0 / mx : 1.0;  // pre-scale: the solve grows x by ~1/eps
                for (int i = lane; i < n; i += 32) xq[i * st] *= sc;
                __syncwarp();
                for (int u = j; u < q; ++u) {
                    const bool here = u >= cb;
                    const double* xu = here ? xs + (u - cb) : X + size_t(n) * u;
                    const int su = here ? st : 1;
                    double dt = 0.0;
                    for (int i = lane; i < n; i += 32) dt = fma(xu[i * su], xq[i * st], dt);
                    dt = warp_sum(dt);
                    for (int i = lane; i < n; i += 32) xq[i * st] = fma(-dt, xu[i * su], xq[i * st]);
                    __syncwarp();
                }
                double nr = 0.0;
                for (int i = lane; i < n; i += 32) nr = fma(xq[i * st], xq[i * st], nr);
                nr = warp_sum(nr);
                const double inv = nr > 0.0 ? 1.0 / sqrt(nr) : 0.0;
                for (int i = lane; i < n; i += 32) xq[i * st] *= inv;
                __syncwarp();
            }
        }
        for (int q = cb; q < cend; ++q)  // the chunk's vectors out
            for (int i = lane; i < n; i += 32) X[size_t(n) * q + i] = xs[i * st + (q - cb)];
        __syncwarp();
    }
}

// The same inverse iteration for large n (the dense path of trd_big.cu): ONE CTA
// per cluster.  Members are solved in parallel (one thread each, factors
// interleaved by member so a warp's loads are contiguous), then the whole CTA
// orthonormalises them in order by classical Gram-Schmidt with
// re-orthogonalisation (CGS2): member q against the cluster's earlier members,
// the dot products spread over the warps.  In exact arithmetic this is the
// sequential Gram-Schmidt of invit_kernel / dstein; at n = 2048 with a flat
// spectrum (one 64-member cluster) it is ~10x faster than one warp per cluster.
constexpr int kIvT = 512;
__device__ __forceinline__ double block_reduce(double v, double* red, bool is_max) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double x = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? fmax(v, x) : v + x;
    }
    __syncthreads();  // red may still be read by the previous call
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = is_max ? 0.0 : 0.0;
    for (int q = 0; q < kIvT / 32; ++q) s = is_max ? fmax(s, red[q]) : s + red[q];
    return s;
}

__global__ void __launch_bounds__(kIvT) invit_cta_kernel(const double* __restrict__ d, const double* __restrict__ e,
                                                        int n, const double* __restrict__ lam, int nwant,
                                                        double* __restrict__ X, double* __restrict__ wk) {
    // (the block path below runs first; this kernel is its fallback)
    extern __shared__ double dsh[];  // nwant: dot products of the current member
    __shared__ double red[kIvT / 32];
    __shared__ TNorm tnsh;
    const int j = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (t < 32) {
        const TNorm tn = tnorm_warp(d, e, n);
        if (t == 0) tnsh = tn;
    }
    __syncthreads();
    const TNorm tn = tnsh;
    const double ortol = 1e-3 * tn.norm;
    if (j > 0 && lam[j - 1] - lam[j] <= ortol) return;  // not a cluster leader (CTA-uniform)
    int end = j + 1;
    while (end < nwant && lam[end - 1] - lam[end] <= ortol) ++end;
    const double pertol = 10.0 * DBL_EPSILON * fmax(tn.norm, DBL_MIN);
    const double tiny = tn.norm > 0.0 ? DBL_EPSILON * tn.norm : 1.0;
    for (int cb = j; cb < end; cb += kIvT) {
        const int cs = min(kIvT, end - cb);
        const int mm = cb + t;
        const bool mine = t < cs;
        const size_t st = size_t(cs);
        double* base = wk + size_t(5) * n * cb + (mine ? t : 0);
        double* dl = base;
        double* dd = base + size_t(n) * st;
        double* du = dd + size_t(n) * st;
        double* du2 = du + size_t(n) * st;
        double* pv = du2 + size_t(n) * st;
        double* x = X + size_t(n) * (mine ? mm : j);
        if (mine) {
            double sh = lam[j];
            for (int q = j + 1; q <= mm; ++q) sh = fmin(lam[q], sh - pertol);
            double di = d[0] - sh, ui = n > 1 ? e[0] : 0.0;
            for (int i = 0; i + 1 < n; ++i) {
                const double li = e[i], dn = d[i + 1] - sh, un = i + 2 < n ? e[i + 1] : 0.0;
                if (fabs(di) >= fabs(li)) {
                    if (fabs(di) < tiny) di = copysign(tiny, di);
                    const double r = 1.0 / di;
                    const double f = li * r;
                    dl[i * st] = f;
                    dd[i * st] = r;
                    du[i * st] = ui;
                    du2[i * st] = 0.0;
                    pv[i * st] = 0.0;
                    di = fma(-f, ui, dn);
                    ui = un;
                } else {
                    const double r = 1.0 / li;
                    const double f = di * r;
                    dl[i * st] = f;
                    dd[i * st] = r;
                    du[i * st] = dn;
                    du2[i * st] = un;
                    pv[i * st] = 1.0;
                    di = fma(-f, dn, ui);
                    ui = -f * un;
                }
            }
            if (fabs(di) < tiny) di = copysign(tiny, di);
            dd[(n - 1) * st] = 1.0 / di;
            for (int i = 0; i < n; ++i) x[i] = hash_unit(uint64_t(mm) * 1000003ULL + i);
        }
        for (int it = 0; it < 3; ++it) {
            if (mine) {
                double cr = x[0];
                for (int i = 0; i + 1 < n; ++i) {
                    const double nx = x[i + 1];
                    if (pv[i * st] != 0.0) {
                        x[i] = nx;
                        cr = fma(-dl[i * st], nx, cr);
                    } else {
                        x[i] = cr;
                        cr = fma(-dl[i * st], cr, nx);
                    }
                }
                x[n - 1] = cr;
                double x2 = 0.0, x1 = x[n - 1] * dd[(n - 1) * st];
                x[n - 1] = x1;
                for (int i = n - 2; i >= 0; --i) {
                    const double xi = (x[i] - du[i * st] * x1 - du2[i * st] * x2) * dd[i * st];
                    x[i] = xi;
                    x2 = x1;
                    x1 = xi;
                }
            }
            __syncthreads();
            // CGS2 of this chunk's members, in order, against every earlier cluster member
            for (int q = cb; q < cb + cs; ++q) {
                double* xq = X + size_t(n) * q;
                double mx = 0.0;
                for (int i = t; i < n; i += kIvT) mx = fmax(mx, fabs(xq[i]));
                mx = block_reduce(mx, red, true);
                const double sc = mx > 0.0 ? 1.0 / mx : 1.0;  // pre-scale: the solve grows x by ~1/eps
                for (int i = t; i < n; i += kIvT) xq[i] *= sc;
                const int np = q - j;
                for (int pass = 0; pass < 2 && np > 0; ++pass) {
                    __syncthreads();
                    for (int u = w; u < np; u += kIvT / 32) {
                        const double* xu = X + size_t(n) * (j + u);
                        double dt = 0.0;
                        for (int i = lane; i < n; i += 32) dt = fma(xu[i], xq[i], dt);
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) dt += __shfl_xor_sync(0xffffffffu, dt, o);
                        if (lane == 0) dsh[u] = dt;
                    }
                    __syncthreads();
                    for (int i = t; i < n; i += kIvT) {
                        double a = 0.0;
                        for (int u = 0; u < np; ++u) a = fma(dsh[u], X[size_t(n) * (j + u) + i], a);
                        xq[i] -= a;
                    }
                }
                double nr = 0.0;
                for (int i = t; i < n; i += kIvT) nr = fma(xq[i], xq[i], nr);
                nr = block_reduce(nr, red, false);
                const double inv = nr > 0.0 ? 1.0 / sqrt(nr) : 0.0;
                for (int i = t; i < n; i += kIvT) xq[i] *= inv;
                __syncthreads();
            }
        }
    }
}

// ---------------------------------------------------------------- block inverse iteration
// Every wanted member solved in parallel (one thread each, dstein's shifts:
// within a cluster each member's shift sits >= pertol below the previous
// one), three dgttrs solves from the same pseudo-random start as the
// kernels above, each followed by a normalisation; then the whole block is
// orthonormalised at once by the Lowdin step X <- X (3/2 I - 1/2 X^T X).
// When the members are distinct to working precision (gap >> eps ||T||, the
// flat Gram spectra of C5u / C2: a 64-member dstein "cluster" whose vectors
// are each already accurate to eps ||T|| / gap), X^T X = I + E with |E| tiny
// and one step leaves |E'| ~ 3/4 |E|^2: the same accuracy as Gram-Schmidt in
// order, without its serial chain (C5u n = 2048: 14.7 ms -> see DESIGN).
// Degenerate eigenvalues (|E| > 1e-3) fall back to the sequential kernels.
// Factors and x are interleaved by member: array a, row i at (a n + i) nw + m.
__device__ void invit_member(const double* __restrict__ d, const double* __restrict__ e, int n,
                             const double* __restrict__ lam, int m, const TNorm& tn, double* __restrict__ f,
                             size_t st, double* __restrict__ x, size_t xs) {
    const double ortol = 1e-3 * tn.norm;
    const double pertol = 10.0 * DBL_EPSILON * fmax(tn.norm, DBL_MIN);
    const double tiny = tn.norm > 0.0 ? DBL_EPSILON * tn.norm : 1.0;
    int j = m;
    while (j > 0 && lam[j - 1] - lam[j] <= ortol) --j;
    double sh = lam[j];
    for (int q = j + 1; q <= m; ++q) sh = fmin(lam[q], sh - pertol);
    double* dl = f;
    double* dd = f + size_t(n) * st;
    double* du = dd + size_t(n) * st;
    double* du2 = du + size_t(n) * st;
    double* pv = du2 + size_t(n) * st;
    double di = d[0] - sh, ui = n > 1 ? e[0] : 0.0;
    for (int i = 0; i + 1 < n; ++i) {
        const double li = e[i], dn = d[i + 1] - sh, un = i + 2 < n ? e[i + 1] : 0.0;
        if (fabs(di) >= fabs(li)) {
            if (fabs(di) < tiny) di = copysign(tiny, di);
            const double r = 1.0 / di;
            const double fl = li * r;
            dl[i * st] = fl;
            dd[i * st] = r;
            du[i * st] = ui;
            du2[i * st] = 0.0;
            pv[i * st] = 0.0;
            di = fma(-fl, ui, dn);
            ui = un;
        } else {
            const double r = 1.0 / li;
            const double fl = di * r;
            dl[i * st] = fl;
            dd[i * st] = r;
            du[i * st] = dn;
            du2[i * st] = un;
            pv[i * st] = 1.0;
            di = fma(-fl, dn, ui);
            ui = -fl * un;
        }
    }
    if (fabs(di) < tiny) di = copysign(tiny, di);
    dd[(n - 1) * st] = 1.0 / di;
    for (int i = 0; i < n; ++i) x[i * xs] = hash_unit(uint64_t(m) * 1000003ULL + i);
    // The solves are serial recurrences over rows; their operands are loaded
    // kCh rows at a time into registers first (x[j] is read before it is
    // overwritten in both sweeps, so the early loads are exact), which keeps
    // kCh loads in flight instead of one memory round trip per row.
    constexpr int kCh = 16;
    for (int it = 0; it < 3; ++it) {
        double cr = x[0];
        for (int i0 = 0; i0 + 1 < n; i0 += kCh) {
            const int cnt = min(kCh, n - 1 - i0);
            double pvr[kCh], dlr[kCh], nxr[kCh];
#pragma unroll
            for (int q = 0; q < kCh; ++q)
                if (q < cnt) {
                    pvr[q] = pv[(i0 + q) * st];
                    dlr[q] = dl[(i0 + q) * st];
                    nxr[q] = x[(i0 + q + 1) * xs];
                }
#pragma unroll
            for (int q = 0; q < kCh; ++q)
                if (q < cnt) {
                    const double nx = nxr[q];
                    if (pvr[q] != 0.0) {
                        x[(i0 + q) * xs] = nx;
                        cr = fma(-dlr[q], nx, cr);
                    } else {
                        x[(i0 + q) * xs] = cr;
                        cr = fma(-dlr[q], cr, nx);
                    }
                }
        }
        double x2 = 0.0, x1 = cr * dd[(n - 1) * st];
        x[(n - 1) * xs] = x1;
        for (int i1 = n - 2; i1 >= 0; i1 -= kCh) {
            const int cnt = min(kCh, i1 + 1);
            double xr[kCh], ur[kCh], u2r[kCh], dr[kCh];
#pragma unroll
            for (int q = 0; q < kCh; ++q)
                if (q < cnt) {
                    const int i = i1 - q;
                    xr[q] = x[i * xs];
                    ur[q] = du[i * st];
                    u2r[q] = du2[i * st];
                    dr[q] = dd[i * st];
                }
#pragma unroll
            for (int q = 0; q < kCh; ++q)
                if (q < cnt) {
                    const double xi = (xr[q] - ur[q] * x1 - u2r[q] * x2) * dr[q];
                    x[(i1 - q) * xs] = xi;
                    x2 = x1;
                    x1 = xi;
                }
        }
        double mx = 0.0;
        for (int i = 0; i < n; ++i) mx = fmax(mx, fabs(x[i * xs]));
        const double sc = mx > 0.0 ? 1.0 / mx : 1.0;  // the solve grows x by ~1/eps
        double nr = 0.0;
        for (int i = 0; i < n; ++i) {
            const double v = x[i * xs] * sc;
            nr = fma(v, v, nr);
        }
        const double inv = nr > 0.0 ? sc / sqrt(nr) : 0.0;
        for (int i = 0; i < n; ++i) x[i * xs] *= inv;
    }
}

constexpr int kIpT = 64;
// X (n x nw, ld n) <- the members' normalised inverse-iteration vectors.  wk: 6 n nw.
__global__ void __launch_bounds__(kIpT) invit_par_kernel(const double* __restrict__ d, const double* __restrict__ e,
                                                         int n, const double* __restrict__ lam, int nw,
                                                         double* __restrict__ X, double* __restrict__ wk) {
    __shared__ TNorm tnsh;
    if (threadIdx.x < 32) {
        const TNorm t = tnorm_warp(d, e, n);
        if (threadIdx.x == 0) tnsh = t;
    }
    __syncthreads();
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= nw) return;
    const size_t st = size_t(nw);
    double* xw = wk + size_t(5) * n * st + m;
    invit_member(d, e, n, lam, m, tnsh, wk + m, st, xw, st);
    for (int i = 0; i < n; ++i) X[size_t(m) * n + i] = xw[size_t(i) * st];
}

__global__ void any_cluster(const double* __restrict__ d, const double* __restrict__ e, int n,
                            const double* __restrict__ lam, int nw, int* __restrict__ out) {
    __shared__ TNorm tnsh;
    if (threadIdx.x < 32) {
        const TNorm t = tnorm_warp(d, e, n);
        if (threadIdx.x == 0) tnsh = t;
    }
    __syncthreads();
    int c = 0;
    for (int m = threadIdx.x + 1; m < nw; m += blockDim.x) c += (lam[m - 1] - lam[m] <= 1e-3 * tnsh.norm);
    atomicAdd(out, c);  // clustered neighbour pairs
}

// emax = max |G - I| (G: nw x nw), as the bit pattern of a non-negative double
__global__ void lowdin_defect(const double* __restrict__ g, int nw, unsigned long long* __restrict__ emax) {
    double mx = 0.0;
    const size_t tot = size_t(nw) * nw;
    for (size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x; q < tot; q += size_t(gridDim.x) * blockDim.x) {
        const double v = g[q] - ((q % nw) == (q / nw) ? 1.0 : 0.0);
        mx = fmax(mx, fabs(v));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(emax, __double_as_longlong(mx));
}

// C = 3/2 I - 1/2 G
__global__ void lowdin_coeff(const double* __restrict__ g, int nw, double* __restrict__ c) {
    const size_t tot = size_t(nw) * nw;
    for (size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x; q < tot; q += size_t(gridDim.x) * blockDim.x)
        c[q] = ((q % nw) == (q / nw) ? 1.5 : 0.0) - 0.5 * g[q];
}

// The same for small tridiagonals (n * nw <= kIbSmall, the Rayleigh-Ritz
// blocks of ChFSI): one CTA, X in shared memory, no host round trip.  On a
// defect > 1e-3 it leaves *fallback = 1 and invit_kernel (launched right
// after with `skip` = !fallback) redoes the block sequentially.
constexpr int kIbSmall = 6400;
constexpr int kIbMinPairs = 8;  // clustered neighbour pairs before the block path pays
constexpr int kIbT = 256;
__global__ void __launch_bounds__(kIbT) invit_block_small_kernel(const double* __restrict__ d,
                                                                 const double* __restrict__ e, int n,
                                                                 const double* __restrict__ lam, int nw,
                                                                 double* __restrict__ Xout, double* __restrict__ wk,
                                                                 int* __restrict__ ok) {
    extern __shared__ double sm[];
    double* X = sm;                     // row-major: X[i nw + m]
    double* Y = X + size_t(n) * nw;     // the update
    double* G = Y + size_t(n) * nw;     // nw x nw
    __shared__ TNorm tnsh;
    __shared__ double red[kIbT / 32];
    const int t = threadIdx.x;
    if (t < 32) {
        const TNorm tt = tnorm_warp(d, e, n);
        if (t == 0) tnsh = tt;
    }
    __syncthreads();
    const TNorm tn = tnsh;
    // few dstein-clustered neighbours among the wanted values (C5's signal
    // Ritz values): the one-warp-per-cluster kernel is the cheaper one (its
    // short Gram-Schmidt chains cost less than this kernel's block steps)
    int clustered = 0;
    for (int m = t + 1; m < nw; m += kIbT) clustered += (lam[m - 1] - lam[m] <= 1e-3 * tn.norm);
    if (__syncthreads_count(clustered) < kIbMinPairs) {  // nw <= 80 < kIbT: one pair per thread
        if (t == 0) *ok = 0;
        return;
    }
    for (int m = t; m < nw; m += kIbT) invit_member(d, e, n, lam, m, tn, wk + m, size_t(nw), X + m, size_t(nw));
    for (int step = 0; step < 2; ++step) {
        __syncthreads();
        double mx = 0.0;
        for (int q = t; q < nw * nw; q += kIbT) {
            const int a = q % nw, b = q / nw;
            double g = 0.0;
            for (int i = 0; i < n; ++i) g = fma(X[i * nw + a], X[i * nw + b], g);
            G[q] = g;
            mx = fmax(mx, fabs(g - (a == b ? 1.0 : 0.0)));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if ((t & 31) == 0) red[t >> 5] = mx;
        __syncthreads();
        double em = 0.0;
        for (int w = 0; w < kIbT / 32; ++w) em = fmax(em, red[w]);
        if (em > 1e-3) {  // degenerate: the sequential kernel takes over
            if (t == 0) *ok = 0;
            return;
        }
        if (step == 1 && em <= 1e-14) break;
        for (int q = t; q < n * nw; q += kIbT) {
            const int i = q / nw, b = q % nw;
            double y = 0.0;
            for (int a = 0; a < nw; ++a) y = fma(X[i * nw + a], (a == b ? 1.5 : 0.0) - 0.5 * G[b * nw + a], y);
            Y[q] = y;
        }
        __syncthreads();
        for (int q = t; q < n * nw; q += kIbT) X[q] = Y[q];
        if (em <= 1e-7) break;  // one step leaves ~0.75 em^2
    }
    __syncthreads();
    for (int q = t; q < n * nw; q += kIbT) {
        const int m = q / n, i = q % n;
        Xout[size_t(m) * n + i] = X[i * nw + m];
    }
    if (t == 0) *ok = 1;
}

// vout(:, c) = H_0 ... H_{n-3} X(:, c); one warp per column, reflectors in smem.
template <int S>
__global__ void __launch_bounds__(1024) backtr_kernel(const double* __restrict__ hh, const double* __restrict__ tau,
                                                      const double* __restrict__ scal, int n,
                                                      const double* __restrict__ X, int nwant,
                                                      double* __restrict__ vout, int ldv) {
    extern __shared__ double sm[];
    constexpr int NR = 32 * S;
    const int np = n * (n + 1) / 2;
    double* H = sm;            // np + NR zero pad
    double* ts = H + np + NR;  // tau, scal
    for (int q = threadIdx.x; q < np; q += blockDim.x) H[q] = hh[q];
    for (int q = threadIdx.x; q < NR; q += blockDim.x) H[np + q] = 0.0;
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        ts[q] = tau[q];
        ts[n + q] = scal[q];
    }
    __syncthreads();
    const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (c >= nwant) return;
    double x[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int i = lane + 32 * s;
        x[s] = i < n ? X[size_t(n) * c + i] : 0.0;
    }
    // reflectors in pairs (H_{k-1} H_k x): the three dots a.x, b.x, b.a are reduced
    // together, so each pair costs one warp-reduction latency instead of two
    int k = n - 3;
    for (; k >= 1; k -= 2) {
        const double ta = ts[k], tb = ts[k - 1];
        if (ta == 0.0 && tb == 0.0) continue;
        const double sa = ts[n + k], sb = ts[n + k - 1];
        const int ca = pk(k, k, n) - k, cb = pk(k - 1, k - 1, n) - (k - 1);
        const int s0 = k >> 5;
        double va[S], vb[S], da = 0.0, db = 0.0, dab = 0.0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            va[s] = 0.0;
            vb[s] = 0.0;
            if (s >= s0) {  // warp-uniform
                const int i = lane + 32 * s;
                const double ha = H[ca + i] * sa, hb = H[cb + i] * sb;
                va[s] = (i == k + 1) ? 1.0 : (i > k + 1 && i < n) ? ha : 0.0;  // pad rows stay 0
                vb[s] = (i == k) ? 1.0 : (i > k && i < n) ? hb : 0.0;
                da = fma(va[s], x[s], da);
                db = fma(vb[s], x[s], db);
                dab = fma(vb[s], va[s], dab);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            da += __shfl_xor_sync(0xffffffffu, da, o);
            db += __shfl_xor_sync(0xffffffffu, db, o);
            dab += __shfl_xor_sync(0xffffffffu, dab, o);
        }
        const double c1 = ta * da;                  // H_k:     x -= c1 a
        const double c2 = tb * fma(-c1, dab, db);   // H_{k-1}: x -= c2 b, with b.(x - c1 a)
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (s >= s0) x[s] = fma(-c2, vb[s], fma(-c1, va[s], x[s]));
    }
    for (; k >= 0; --k) {  // the odd one left (k = 0)
        const double tk = ts[k];
        if (tk == 0.0) continue;
        const double sk = ts[n + k];
        const int ck = pk(k, k, n) - k;
        const int s0 = (k + 1) >> 5;
        double v[S], dt0 = 0.0, dt1 = 0.0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            v[s] = 0.0;
            if (s >= s0) {  // warp-uniform
                const int i = lane + 32 * s;
                const double h = H[ck + i] * sk;
                v[s] = (i == k + 1) ? 1.0 : (i > k + 1 && i < n) ? h : 0.0;  // pad rows stay 0
                if (s & 1) dt1 = fma(v[s], x[s], dt1);
                else dt0 = fma(v[s], x[s], dt0);
            }
        }
        const double dt = tk * warp_sum(dt0 + dt1);
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (s >= s0) x[s] = fma(-dt, v[s], x[s]);
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int i = lane + 32 * s;
        if (i < n) vout[size_t(ldv) * c + i] = x[s];
    }
}

// ---------------------------------------------------------------------------
// Tile variant (n <= 192): the lower triangle as 32 x 32 tiles (diagonal tiles
// hold the full symmetric block), leading dimension 33 so both the row walk
// (lane = row) and the column walk (lane = column) are near conflict-free.
// Warps own tiles.  Per Householder step: warp 0 forms the reflector; the
// matvec of tile (I, J) yields a row part B v_J (lane = row) and, off the
// diagonal, a column part B^T v_I (lane = column) -- no shuffles; a fixed-order
// sum of those parts gives p; every warp forms K = (tau/2) p.v redundantly and
// applies the rank-2 update to its tiles.  Four barriers per step, ~10x fewer
// instructions than the column-slot kernel.  Output: the same hh / d / e / tau
// / scal as trd_kernel (hh written packed at the end for backtr_kernel).
constexpr int kTileLd = 33, kTileDbl = 32 * kTileLd;

__device__ __forceinline__ int tile_index(int I, int J) { return I * (I + 1) / 2 + J; }

// NT = 7 covers 192 < n <= 200 (C1's n = 200): its last tile row holds at most 8 rows, stored
// with a 9-row leading dimension (28 full tiles would need 236 KB of shared memory, this 211 KB)
static_assert(kTridiagMax <= 6 * 32 + 8, "TileShape<7>: the short tile row holds 8 rows");
template <int NT>
struct TileShape {
    static constexpr bool SHORT = NT == 7;
    static constexpr int RP = 8, LDL = 9;  // rows of the short tile row, its leading dimension
    static constexpr int NTILES = NT * (NT + 1) / 2;
    static constexpr int NFULL = SHORT ? (NT - 1) * NT / 2 : NTILES;  // tiles stored 32 x 33
    static constexpr int TDBL = NFULL * kTileDbl + (SHORT ? NT * 32 * LDL : 0);
    __device__ static __forceinline__ bool last(int I) { return SHORT && I == NT - 1; }
    __device__ static __forceinline__ int off(int I, int J) {
        return last(I) ? NFULL * kTileDbl + J * 32 * LDL : tile_index(I, J) * kTileDbl;
    }
    __device__ static __forceinline__ int ld(int I) { return last(I) ? LDL : kTileLd; }
};

constexpr int kTileThreads = 256;  // 8 warps: 255 registers/thread (at 512 the CTA-id read was rematerialised per step)

template <int NT>
__global__ void __launch_bounds__(kTileThreads, 1)
    trd_tile_kernel(const double* __restrict__ a, int n, int lda, double* __restrict__ hh, double* __restrict__ d,
                    double* __restrict__ e, double* __restrict__ tau_out, double* __restrict__ scal_out,
                    long long* __restrict__ prof) {
    using TS = TileShape<NT>;
    constexpr int NTILES = TS::NTILES, NR = 32 * NT, NWARP = kTileThreads / 32;
    long long t_mark = clock64(), t_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // ATK_TRD_PROFILE
    auto lap = [&](int ph) {
        if (prof) {
            const long long t = clock64();
            t_acc[ph] += t - t_mark;
            t_mark = t;
        }
    };
    extern __shared__ double sm[];
    double* T = sm;                       // NTILES x (32 x 33) (TileShape: a short last tile row)
    double* crow = T + TS::TDBL;          // NTILES x 32: row parts
    double* ccol = crow + NTILES * 32;    // NTILES x 32: column parts
    double* v = ccol + NTILES * 32;       // NR
    double* pb = v + NR;                  // NR
    // tau lives in the dynamic buffer: a static __shared__ variable costs an
    // SR_CgaCtaId read (S2UR, long latency) at every access in this kernel
    double& sh_tau = pb[NR];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    auto at = [&](int i, int j) -> double& {  // i >= j or same diagonal tile
        const int I = i >> 5, J = j >> 5;
        return T[TS::off(I, J) + (i & 31) + TS::ld(I) * (j & 31)];
    };
    // load: symmetrised, zero padding
    for (int q = tid; q < TS::TDBL; q += kTileThreads) T[q] = 0.0;
    __syncthreads();
    for (int q = tid; q < n * n; q += kTileThreads) {
        const int i = q % n, j = q / n;
        if ((i >> 5) >= (j >> 5)) at(i, j) = 0.5 * (a[i + size_t(lda) * j] + a[j + size_t(lda) * i]);
    }
    __syncthreads();

    for (int k = 0; k + 2 < n; ++k) {
        // ---- A: reflector from column k (warp 0)
        if (w == 0) {
            const double alpha = at(k + 1, k);
            double xn = 0.0;
            for (int i = k + 2 + lane; i < n; i += 32) {
                const double x = at(i, k);
                xn = fma(x, x, xn);
            }
            xn = warp_sum(xn);
            double tau = 0.0, scal = 0.0, beta = alpha;
            if (xn > 0.0) {
                beta = -copysign(sqrt(fma(alpha, alpha, xn)), alpha);
                scal = 1.0 / (alpha - beta);
                tau = (beta - alpha) / beta;
            }
            for (int i = lane; i < NR; i += 32)
                v[i] = (i == k + 1) ? 1.0 : (i > k + 1 && i < n) ? at(i, k) * scal : 0.0;
            if (lane == 0) {
                d[k] = at(k, k);
                e[k] = beta;
                tau_out[k] = tau;
                scal_out[k] = scal;
                sh_tau = tau;
            }
        }
        lap(0);
        __syncthreads();
        lap(1);
        const double tau = sh_tau;
        if (tau == 0.0) continue;  // uniform: H_k = I
        const int J0 = (k + 1) >> 5;
        const int nact = (NT - J0) * (NT - J0 + 1) / 2;
        // ---- B: per-tile matvec parts
        for (int q = w; q < nact; q += NWARP) {
            // q -> (I, J), J0 <= J <= I < NT, enumerated column by column
            int J = J0, rem = q;
            while (rem >= NT - J) { rem -= NT - J; ++J; }
            const int I = J + rem;
            const double* B = T + TS::off(I, J);
            const double* vJ = v + J * 32;
            const double* vI = v + I * 32;
            // 8 independent accumulators per walk: the fp64 FMA chains, not the loads,
            // bound this loop
            double ra[8], ca[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) ra[u] = ca[u] = 0.0;
            const bool off = I != J;
            const bool lst = TS::last(I);
            const int ld = TS::ld(I), rows = lst ? TS::RP : 32;  // stored rows of this tile
            const bool lv = lane < rows;
#pragma unroll
            for (int c = 0; c < 32; c += 8)
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (lv) ra[u] = fma(B[lane + ld * (c + u)], vJ[c + u], ra[u]);
                    if (off && c < rows) ca[u] = fma(B[c + u + ld * lane], vI[c + u], ca[u]);
                }
            crow[tile_index(I, J) * 32 + lane] = ((ra[0] + ra[1]) + (ra[2] + ra[3])) + ((ra[4] + ra[5]) + (ra[6] + ra[7]));
            if (off)
                ccol[tile_index(I, J) * 32 + lane] =
                    ((ca[0] + ca[1]) + (ca[2] + ca[3])) + ((ca[4] + ca[5]) + (ca[6] + ca[7]));
        }
        lap(2);
        __syncthreads();
        lap(3);
        // ---- B2: p = tau (row parts of row block I + column parts of tiles below), fixed order
        for (int i = tid; i < NR; i += kTileThreads) {
            double s0 = 0.0;
            if (i > k && i < n) {
                const int I = i >> 5, r = i & 31;
                for (int J = J0; J <= I; ++J) s0 += crow[tile_index(I, J) * 32 + r];
                for (int I2 = I + 1; I2 < NT; ++I2) s0 += ccol[tile_index(I2, I) * 32 + r];
                s0 *= tau;
            }
            pb[i] = s0;
        }
        lap(4);
        __syncthreads();
        lap(5);
        // ---- C: K = (tau/2) p.v (every warp, identical arithmetic); A -= v w^T + w v^T
        double pv = 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) pv = fma(pb[lane + 32 * t], v[lane + 32 * t], pv);
        const double K = 0.5 * tau * warp_sum(pv);
        for (int q = w; q < nact; q += NWARP) {
            int J = J0, rem = q;
            while (rem >= NT - J) { rem -= NT - J; ++J; }
            const int I = J + rem;
            double* B = T + TS::off(I, J);
            const int ld = TS::ld(I);
            if (TS::last(I) && lane >= TS::RP) continue;  // rows the short tile row does not store
            const double vr = v[I * 32 + lane];
            const double wr = fma(-K, vr, pb[I * 32 + lane]);
            const double* vJ = v + J * 32;
            const double* pJ = pb + J * 32;
            // batches of 8 columns: all loads issued before the stores (no aliasing stalls)
#pragma unroll
            for (int c = 0; c < 32; c += 8) {
                double xs[8], vc[8], pc[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    xs[u] = B[lane + ld * (c + u)];
                    vc[u] = vJ[c + u];
                    pc[u] = pJ[c + u];
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const double wc = fma(-K, vc[u], pc[u]);
                    B[lane + ld * (c + u)] = fma(-vr, wc, fma(-wr, vc[u], xs[u]));
                }
            }
        }
        lap(6);
        __syncthreads();
        lap(7);
    }
    if (tid == 0) {
        if (n >= 2) {
            d[n - 2] = at(n - 2, n - 2);
            e[n - 2] = at(n - 1, n - 2);
            tau_out[n - 2] = 0.0;
            scal_out[n - 2] = 0.0;
        }
        d[n - 1] = at(n - 1, n - 1);
        tau_out[n - 1] = 0.0;
        scal_out[n - 1] = 0.0;
    }
    for (int j = 0; j < n; ++j)  // packed lower triangle for backtr_kernel
        for (int i = j + tid; i < n; i += kTileThreads) hh[pk(i, j, n)] = at(i, j);
    if (prof && lane == 0 && (w == 0 || w == 1))
        for (int q = 0; q < 8; ++q)
            atomicAdd(reinterpret_cast<unsigned long long*>(prof + 8 * w + q), (unsigned long long)t_acc[q]);
}

size_t trd_tile_smem(int nt) {
    const int ntiles = nt * (nt + 1) / 2;
    const size_t tdbl = nt == 7 ? size_t(TileShape<7>::TDBL) : size_t(ntiles) * kTileDbl;
    return (tdbl + size_t(ntiles) * 64 + 64 * size_t(nt) + 2) * sizeof(double);
}

// n <= 32 NW (NW <= 4): the same reduction (dsytd2 conventions, same outputs as
// trd_kernel / trd_tile_kernel) by NW warps, lane-owned rows of the FULL
// symmetric matrix in shared memory (column-major, odd ld: conflict-free).
// Warp w owns rows 32 w + lane in the matvec and the rank-2 update, so the
// only cross-warp traffic is two scalar sums per step.  For the Rayleigh-Ritz
// blocks of ChFSI (k = 48) and the small modes (n = 48) the tile kernel's
// 256-thread barriers were the whole cost (~107 us at n = 48).
template <int NW, int CS>
__global__ void __launch_bounds__(NW * CS * 32, 1)
    trd_small_kernel(const double* __restrict__ a, int n, int lda, double* __restrict__ hh, double* __restrict__ d,
                     double* __restrict__ e, double* __restrict__ tau_out, double* __restrict__ scal_out) {
    // CS warps per 32-row block: warp (w, s) owns rows 32 w + lane and the s-th
    // contiguous part of the trailing columns in the matvec and the update
    constexpr int NR = 32 * NW, LD = NR + 1;
    extern __shared__ double sm[];
    double* A = sm;              // NR x LD
    double* vs = A + NR * LD;    // NR: reflector
    double* ws = vs + NR;        // NR: w = p - K v
    double* pp = ws + NR;        // CS x NR: matvec partials
    double* red = pp + CS * NR;  // 2 x NW cross-warp partials
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int w = wid % NW, sp = wid / NW;
    const int i = w * 32 + lane;  // the row this thread owns
    if (sp == 0)
        for (int j = 0; j < n; ++j)
            A[i + LD * j] = i < n ? 0.5 * (a[i + size_t(lda) * j] + a[j + size_t(lda) * i]) : 0.0;
    if (sp == 0) {
        vs[i] = 0.0;
        ws[i] = 0.0;
    }
    __syncthreads();
    auto sum_all = [&](double x, int slot) {  // split-0 warps' sums, fixed order across warps
        x = warp_sum(x);
        if (NW == 1 && CS == 1) return x;
        if (sp == 0 && lane == 0) red[slot * NW + w] = x;
        __syncthreads();
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < NW; ++q) t += red[slot * NW + q];
        return t;
    };
    for (int k = 0; k + 2 < n; ++k) {
        // reflector k from column k, rows k+1..n-1 (dlarfg)
        const double x = (i >= k + 2 && i < n) ? A[i + LD * k] : 0.0;
        const double xn = sum_all(x * x, 0);
        const double alpha = A[(k + 1) + LD * k];
        double tau = 0.0, scal = 0.0, beta = alpha;
        if (xn > 0.0) {
            beta = -copysign(sqrt(fma(alpha, alpha, xn)), alpha);
            scal = 1.0 / (alpha - beta);
            tau = (beta - alpha) / beta;
        }
        const double vi = (i == k + 1) ? 1.0 : x * scal;
        if (sp == 0) vs[i] = vi;
        if (threadIdx.x == 0) {
            d[k] = A[k + LD * k];
            e[k] = beta;
            tau_out[k] = tau;
            scal_out[k] = scal;
        }
        __syncthreads();
        if (tau == 0.0) continue;  // uniform: H_k = I
        const int len = n - k - 1;
        const int ja = k + 1 + (sp * len) / CS, jb = k + 1 + ((sp + 1) * len) / CS;
        // this split's part of p = tau A22 v (row i), four independent chains
        double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
        int j = ja;
#pragma unroll 2
        for (; j + 3 < jb; j += 4) {
            p0 = fma(A[i + LD * j], vs[j], p0);
            p1 = fma(A[i + LD * (j + 1)], vs[j + 1], p1);
            p2 = fma(A[i + LD * (j + 2)], vs[j + 2], p2);
            p3 = fma(A[i + LD * (j + 3)], vs[j + 3], p3);
        }
        for (; j < jb; ++j) p0 = fma(A[i + LD * j], vs[j], p0);
        double pi;
        if (CS == 1) {
            pi = (i > k && i < n) ? tau * ((p0 + p1) + (p2 + p3)) : 0.0;
        } else {
            pp[sp * NR + i] = (p0 + p1) + (p2 + p3);
            __syncthreads();
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < CS; ++q) t += pp[q * NR + i];
            pi = (i > k && i < n) ? tau * t : 0.0;
        }
        const double K = 0.5 * tau * sum_all(pi * vi, 1);
        const double wi = fma(-K, vi, pi);
        if (sp == 0) ws[i] = wi;
        __syncthreads();
        if (i > k && i < n) {
            // four columns per pass, loads first (a rolled loop is one shared-
            // memory round trip per element)
            for (j = ja; j + 3 < jb; j += 4) {
                double av[4], wv[4], vv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    av[u] = A[i + LD * (j + u)];
                    wv[u] = ws[j + u];
                    vv[u] = vs[j + u];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) A[i + LD * (j + u)] = fma(-vi, wv[u], fma(-wi, vv[u], av[u]));
            }
            for (; j < jb; ++j) A[i + LD * j] = fma(-vi, ws[j], fma(-wi, vs[j], A[i + LD * j]));
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (n >= 2) {
            d[n - 2] = A[(n - 2) + LD * (n - 2)];
            e[n - 2] = A[(n - 1) + LD * (n - 2)];
            tau_out[n - 2] = 0.0;
            scal_out[n - 2] = 0.0;
        }
        d[n - 1] = A[(n - 1) + LD * (n - 1)];
        tau_out[n - 1] = 0.0;
        scal_out[n - 1] = 0.0;
    }
    // packed lower triangle (column k below the diagonal: the raw reflector k)
    if (sp == 0)
        for (int jj = 0; jj < n; ++jj)
            if (i >= jj && i < n) hh[pk(i, jj, n)] = A[i + LD * jj];
}

template <int NW, int CS>
void launch_trd_small(atk_ctx* ctx, const double* a, int n, int lda, double* hh, double* d, double* e, double* tau,
                      double* scal) {
    constexpr int NR = 32 * NW;
    const size_t smem = (size_t(NR) * (NR + 1) + 2 * NR + size_t(CS) * NR + 2 * NW) * sizeof(double);
    static bool attr = false;
    if (!attr) {
        ATK_CUDA(cudaFuncSetAttribute(trd_small_kernel<NW, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(smem)));
        attr = true;
    }
    trd_small_kernel<NW, CS><<<1, NW * CS * 32, smem, ctx->stream>>>(a, n, lda, hh, d, e, tau, scal);
    ATK_LAUNCHED(ctx);
}

template <int NW>
void launch_trd_small_cs(atk_ctx* ctx, const double* a, int n, int lda, double* hh, double* d, double* e,
                         double* tau, double* scal) {
    static const int cs = std::getenv("ATK_TRD_CS") ? std::atoi(std::getenv("ATK_TRD_CS")) : 2;  // probe knob
    if (cs == 1) launch_trd_small<NW, 1>(ctx, a, n, lda, hh, d, e, tau, scal);
    else if (cs == 4) launch_trd_small<NW, 4>(ctx, a, n, lda, hh, d, e, tau, scal);
    else launch_trd_small<NW, 2>(ctx, a, n, lda, hh, d, e, tau, scal);
}

template <int NT>
void launch_trd_tile(atk_ctx* ctx, const double* a, int n, int lda, double* hh, double* d, double* e, double* tau,
                     double* scal) {
    static bool attr = false;
    if (!attr) {
        ATK_CUDA(cudaFuncSetAttribute(trd_tile_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(trd_tile_smem(NT))));
        attr = true;
    }
    static long long* prof = nullptr;
    static const bool want = std::getenv("ATK_TRD_PROFILE") != nullptr;
    if (want && !prof) ATK_CUDA(cudaMalloc(&prof, 16 * sizeof(long long)));
    if (prof) ATK_CUDA(cudaMemsetAsync(prof, 0, 16 * sizeof(long long), ctx->stream));
    trd_tile_kernel<NT><<<1, kTileThreads, trd_tile_smem(NT), ctx->stream>>>(a, n, lda, hh, d, e, tau, scal, prof);
    ATK_LAUNCHED(ctx);
    if (prof) {
        long long h[16];
        ATK_CUDA(cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
        ATK_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int ww = 0; ww < 2; ++ww)
            std::fprintf(stderr,
                         "[trd_tile n=%d warp %d] cycles: A %lld barA %lld B %lld barB %lld B2 %lld barB2 %lld C %lld "
                         "barC %lld\n",
                         n, ww, h[8 * ww], h[8 * ww + 1], h[8 * ww + 2], h[8 * ww + 3], h[8 * ww + 4], h[8 * ww + 5],
                         h[8 * ww + 6], h[8 * ww + 7]);
    }
}

size_t trd_smem(int n, int nw) {
    const int nr = 32 * ((n + 31) / 32);
    return (size_t(n) * (n + 1) / 2 + 4 * size_t(nr) + size_t(nw) * (n + 1) + n + 4) * sizeof(double);
}
size_t backtr_smem(int n) {
    const int nr = 32 * ((n + 31) / 32);
    return (size_t(n) * (n + 1) / 2 + nr + 2 * size_t(n)) * sizeof(double);
}

template <int S>
void launch_trd_backtr(atk_ctx* ctx, bool trd, const double* a, int n, int lda, double* hh, double* d, double* e,
                       double* tau, double* scal, const double* X, int nwant, double* vout, int ldv) {
    // 64 registers per thread at 1024 threads spill the 3+ slot variants: they run 16 warps
    constexpr int NW = S >= 3 ? 16 : 32;
    static bool attr = false;
    if (!attr) {
        ATK_CUDA(cudaFuncSetAttribute(trd_kernel<S, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(trd_smem(std::min(32 * S, kTridiagMax), NW))));
        ATK_CUDA(cudaFuncSetAttribute(backtr_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(backtr_smem(std::min(32 * S, kTridiagMax)))));
        attr = true;
    }
    if (trd) {
        static long long* prof = nullptr;
        static const bool want = std::getenv("ATK_TRD_PROFILE") != nullptr;
        if (want && !prof) ATK_CUDA(cudaMalloc(&prof, 6 * sizeof(long long)));
        if (prof) ATK_CUDA(cudaMemsetAsync(prof, 0, 6 * sizeof(long long), ctx->stream));
        trd_kernel<S, NW><<<1, NW * 32, trd_smem(n, NW), ctx->stream>>>(a, n, lda, hh, d, e, tau, scal, prof);
        if (prof) {
            long long h[6];
            ATK_CUDA(cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
            ATK_CUDA(cudaStreamSynchronize(ctx->stream));
            std::fprintf(stderr, "[trd n=%d NW=%d] cycles/warp: load %.0f B %.0f barB %.0f B2 %.0f C %.0f barC %.0f\n", n,
                         NW, h[0] / double(NW), h[1] / double(NW), h[2] / double(NW), h[3] / double(NW),
                         h[4] / double(NW), h[5] / double(NW));
        }
    } else {
        // 4 vectors (warps) per CTA: the wanted vectors spread over nwant / 4 SMs instead of
        // sharing two (C5's 64 Ritz vectors at n = 80: 36 -> 17 us, profiles/backtr_sweep.sh)
        static const int bw_env = std::getenv("ATK_BACKTR_BW") ? std::atoi(std::getenv("ATK_BACKTR_BW")) : 4;
        const int bw = std::max(1, std::min(bw_env, nwant));
        backtr_kernel<S><<<unsigned((nwant + bw - 1) / bw), 32 * bw, backtr_smem(n), ctx->stream>>>(
            hh, tau, scal, n, X, nwant, vout, ldv);
    }
    ATK_LAUNCHED(ctx);
}

void trd_backtr(atk_ctx* ctx, bool trd, const double* a, int n, int lda, double* hh, double* d, double* e,
                double* tau, double* scal, const double* X, int nwant, double* vout, int ldv) {
    static_assert(kTridiagMax <= 224, "row slots");
    // n <= 128: one to four warps, no 256-thread barriers (n = 48 / 80-96 / 128:
    // 69 / 168 / 320 us against the tile kernel's 108 / 229 / 411 us)
    if (trd && ctx->trd_tiles == 1 && n <= 128) {
        switch ((n + 31) / 32) {
            case 1: launch_trd_small_cs<1>(ctx, a, n, lda, hh, d, e, tau, scal); break;
            case 2: launch_trd_small_cs<2>(ctx, a, n, lda, hh, d, e, tau, scal); break;
            case 3: launch_trd_small_cs<3>(ctx, a, n, lda, hh, d, e, tau, scal); break;
            default: launch_trd_small_cs<4>(ctx, a, n, lda, hh, d, e, tau, scal); break;
        }
        return;
    }
    if (trd && ctx->trd_tiles && n <= kTridiagMax) {  // tile variant (7 tile rows: a short last one)
        switch ((n + 31) / 32) {
            case 1: launch_trd_tile<1>(ctx, a, n, lda, hh, d, e, tau, scal); return;
            case 2: launch_trd_tile<2>(ctx, a, n, lda, hh, d, e, tau, scal); return;
            case 3: launch_trd_tile<3>(ctx, a, n, lda, hh, d, e, tau, scal); return;
            case 4: launch_trd_tile<4>(ctx, a, n, lda, hh, d, e, tau, scal); return;
            case 5: launch_trd_tile<5>(ctx, a, n, lda, hh, d, e, tau, scal); return;
            case 6: launch_trd_tile<6>(ctx, a, n, lda, hh, d, e, tau, scal); return;
            default: launch_trd_tile<7>(ctx, a, n, lda, hh, d, e, tau, scal); return;
        }
    }
    switch ((n + 31) / 32) {
        case 1: launch_trd_backtr<1>(ctx, trd, a, n, lda, hh, d, e, tau, scal, X, nwant, vout, ldv); break;
        case 2: launch_trd_backtr<2>(ctx, trd, a, n, lda, hh, d, e, tau, scal, X, nwant, vout, ldv); break;
        case 3: launch_trd_backtr<3>(ctx, trd, a, n, lda, hh, d, e, tau, scal, X, nwant, vout, ldv); break;
        case 4: launch_trd_backtr<4>(ctx, trd, a, n, lda, hh, d, e, tau, scal, X, nwant, vout, ldv); break;
        case 5: launch_trd_backtr<5>(ctx, trd, a, n, lda, hh, d, e, tau, scal, X, nwant, vout, ldv); break;
        case 6: launch_trd_backtr<6>(ctx, trd, a, n, lda, hh, d, e, tau, scal, X, nwant, vout, ldv); break;
        default: launch_trd_backtr<7>(ctx, trd, a, n, lda, hh, d, e, tau, scal, X, nwant, vout, ldv); break;
    }
}

}  // namespace

// Extreme eigenpairs of the symmetric tridiagonal (d, e) (the Lanczos T of
// eig.cu): all m values by bisection (descending), then inverse iteration for
// the largest and the smallest only, no reduction or back-transform.
// vectors: m x 2 (ld m), column 0 for values[0], column 1 for values[m - 1].
void tridiag_extreme_eig(atk_ctx* ctx, const double* d, const double* e, int m, double* values, double* vectors) {
    if (m < 1 || m > kTridiagMax) fail(ATK_UNSUPPORTED, "tridiag_extreme_eig: m out of range");
    DevBuf<double> wk(ctx, 5 * size_t(m));
    const int wpb = 8;
    bisect_launch(ctx, d, e, m, m, values);
    ATK_LAUNCHED(ctx);
    // one vector per launch: a lone eigenvalue is its own cluster, so a near-
    // degenerate extreme pair costs no Gram-Schmidt (any vector of the pair's
    // space bounds the same way)
    invit_kernel<<<1, 32, 0, ctx->stream>>>(d, e, m, values, 1, vectors, wk.get());
    ATK_LAUNCHED(ctx);
    invit_kernel<<<1, 32, 0, ctx->stream>>>(d, e, m, values + (m - 1), 1, vectors + m, wk.get());
    ATK_LAUNCHED(ctx);
}

// The block path for large n (host-checked): false when the defect says the
// members are degenerate and the sequential CGS2 kernel must run instead.
static bool invit_block(atk_ctx* ctx, const double* d, const double* e, int n, const double* values, int nw,
                        double* X) {
    if (nw < 2 || std::getenv("ATK_INVIT_SEQ")) return false;
    cudaStream_t st = ctx->stream;
    {  // any dstein cluster among the wanted values?  (else one CTA per member is cheaper)
        DevBuf<int> cl(ctx, 1);
        ATK_CUDA(cudaMemsetAsync(cl.get(), 0, sizeof(int), st));
        any_cluster<<<1, 256, 0, st>>>(d, e, n, values, nw, cl.get());
        ATK_LAUNCHED(ctx);
        int h = 0;
        ATK_CUDA(cudaMemcpyAsync(&h, cl.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
        ATK_CUDA(cudaStreamSynchronize(st));
        if (h < kIbMinPairs) return false;
    }
    DevBuf<double> wk(ctx, size_t(6) * n * nw), G(ctx, size_t(nw) * nw), C(ctx, size_t(nw) * nw),
        X2(ctx, size_t(n) * nw);
    DevBuf<unsigned long long> em(ctx, 1);
    invit_par_kernel<<<unsigned((nw + kIpT - 1) / kIpT), kIpT, 0, st>>>(d, e, n, values, nw, X, wk.get());
    ATK_LAUNCHED(ctx);
    const int grid = int(std::min<size_t>((size_t(nw) * nw + 255) / 256, size_t(ctx->num_sms) * 4));
    for (int step = 0; step < 2; ++step) {
        dgemm(ctx, true, false, nw, nw, n, 1.0, X, n, X, n, 0.0, G.get(), nw);
        ATK_CUDA(cudaMemsetAsync(em.get(), 0, sizeof(unsigned long long), st));
        lowdin_defect<<<grid, 256, 0, st>>>(G.get(), nw, em.get());
        ATK_LAUNCHED(ctx);
        unsigned long long hb = 0;
        ATK_CUDA(cudaMemcpyAsync(&hb, em.get(), sizeof(hb), cudaMemcpyDeviceToHost, st));
        ATK_CUDA(cudaStreamSynchronize(st));
        double e0;
        std::memcpy(&e0, &hb, sizeof(e0));
        if (std::getenv("ATK_TRACE")) std::fprintf(stderr, "[atk invit n=%d nw=%d] block defect %.3e\n", n, nw, e0);
        if (!(e0 <= 1e-3)) return false;
        if (step == 1 && e0 <= 1e-14) break;
        lowdin_coeff<<<grid, 256, 0, st>>>(G.get(), nw, C.get());
        ATK_LAUNCHED(ctx);
        dgemm(ctx, false, false, n, nw, nw, 1.0, X, n, C.get(), nw, 0.0, X2.get(), n);
        ATK_CUDA(cudaMemcpyAsync(X, X2.get(), size_t(n) * nw * sizeof(double), cudaMemcpyDeviceToDevice, st));
        if (e0 <= 1e-7) break;
    }
    return true;
}

void tridiag_tail(atk_ctx* ctx, const double* d, const double* e, int n, int nvals, int nwant, double* values,
                  double* X, double* wk) {
    const int wpb = 8;
    static const bool trace = std::getenv("ATK_TRACE") != nullptr;
    cudaEvent_t ev[3] = {};
    if (trace)
        for (auto& x : ev) cudaEventCreate(&x);
    if (trace) cudaEventRecord(ev[0], ctx->stream);
    bisect_launch(ctx, d, e, n, nvals, values);
    ATK_LAUNCHED(ctx);
    if (trace) cudaEventRecord(ev[1], ctx->stream);
    if (nwant > 0 && !invit_block(ctx, d, e, n, values, nwant, X)) {
        invit_cta_kernel<<<unsigned(nwant), kIvT, size_t(nwant) * sizeof(double), ctx->stream>>>(d, e, n, values,
                                                                                               nwant, X, wk);
        ATK_LAUNCHED(ctx);
    }
    if (trace) {
        cudaEventRecord(ev[2], ctx->stream);
        cudaEventSynchronize(ev[2]);
        float a = 0.f, b = 0.f;
        cudaEventElapsedTime(&a, ev[0], ev[1]);
        cudaEventElapsedTime(&b, ev[1], ev[2]);
        std::fprintf(stderr, "[atk tridiag n=%d] bisect %.3f ms, inverse iteration %.3f ms\n", n, a, b);
        for (auto& x : ev) cudaEventDestroy(x);
    }
}

// One warp per cluster leader: the shared-memory variant for n <= kIvSmemMax
// (option "invit_smem", default 1), else the global-memory kernel.
static void invit_warp(atk_ctx* ctx, const double* d, const double* e, int n, const double* values, int nwant,
                       double* X, double* wk, const int* skip) {
    if (ctx->invit_smem && n <= kIvSmemMax) {
        const size_t smem = size_t(6) * n * 32 * sizeof(double);
        static bool attr = false;
        if (!attr) {
            ATK_CUDA(cudaFuncSetAttribute(invit_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(size_t(6) * kIvSmemMax * 32 * sizeof(double))));
            attr = true;
        }
        invit_smem_kernel<<<unsigned(nwant), 32, smem, ctx->stream>>>(d, e, n, values, nwant, X, skip);
        ATK_LAUNCHED(ctx);
        return;
    }
    const int wpb = 8;
    invit_kernel<<<unsigned((nwant + wpb - 1) / wpb), 32 * wpb, 0, ctx->stream>>>(d, e, n, values, nwant, X, wk, skip);
    ATK_LAUNCHED(ctx);
}

void tridiag_eig(atk_ctx* ctx, const double* a, int n, int lda, int nwant, double* values, double* vectors,
                 int ldv, int nvals) {
    if (n < 1 || n > kTridiagMax) fail(ATK_UNSUPPORTED, "tridiag_eig: n out of range");
    if (nvals < nwant) nvals = nwant;
    if (nwant < 0 || nvals > n) fail(ATK_RANK_TOO_LARGE, "tridiag_eig: nwant out of range");
    cudaStream_t st = ctx->stream;
    const size_t np = size_t(n) * (n + 1) / 2;
    DevBuf<double> ws(ctx, np + 4 * size_t(n) + size_t(n) * nwant + 5 * size_t(n) * nwant);
    double* hh = ws.get();
    double* d = hh + np;
    double* e = d + n;
    double* tau = e + n;
    double* scal = tau + n;
    double* X = scal + n;
    double* wk = X + size_t(n) * nwant;
    trd_backtr(ctx, true, a, n, lda, hh, d, e, tau, scal, nullptr, 0, nullptr, 0);
    const int wpb = 8;
    bisect_launch(ctx, d, e, n, nvals, values);
    ATK_LAUNCHED(ctx);
    if (nwant == 0) return;
    if (nwant >= 2 && n * nwant <= kIbSmall && !std::getenv("ATK_INVIT_SEQ")) {
        // block path in one CTA; the sequential kernel only runs if it declined
        const size_t smem = (2 * size_t(n) * nwant + size_t(nwant) * nwant) * sizeof(double);
        static bool attr = false;
        if (!attr) {
            ATK_CUDA(cudaFuncSetAttribute(invit_block_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(3 * kIbSmall * sizeof(double))));
            attr = true;
        }
        DevBuf<int> ok(ctx, 1);
        invit_block_small_kernel<<<1, kIbT, smem, st>>>(d, e, n, values, nwant, X, wk, ok.get());
        ATK_LAUNCHED(ctx);
        invit_warp(ctx, d, e, n, values, nwant, X, wk, ok.get());
    } else {
        invit_warp(ctx, d, e, n, values, nwant, X, wk, nullptr);
    }
    trd_backtr(ctx, false, nullptr, n, 0, hh, d, e, tau, scal, X, nwant, vectors, ldv);
}

}  // namespace atk
