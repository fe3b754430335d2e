// trd_big.cu — exact dense symmetric eigensolver for kTridiagMax < n <= kBigEigMax:
// linalg::sym_eig_top_r (linalg.hpp:101-123), whose Eigen SelfAdjointEigenSolver
// (:108) tridiagonalises and then runs implicit QR on ALL eigenpairs.  Here the
// cost is bounded on any spectrum (n - 2 Householder steps, no iteration count
// that depends on eigenvalue gaps), and only the top r vectors are formed.
//
//  1. trd_grid_kernel — one persistent cooperative CTA per SM reduces
//     A = Q T Q^T by Householder steps (LAPACK dsytd2, lower).  Column j of the
//     trailing matrix belongs to CTA j mod G and is stored WHOLE (rows k+1..n-1,
//     both triangles), so p = tau A v needs no cross-CTA reduction: each CTA
//     forms p_j for its own columns.  Columns sit in shared memory (13 slots of
//     n doubles per SM at n = 2048); the first columns of a CTA spill to a global
//     work copy when they do not fit (they retire first, after <= 1 pass over
//     the SMs).  Per step k:
//       wait for reflector k (one published counter, ld.acquire)
//       p_j = tau_k A(:, j)^T v_k for the CTA's live columns; s_c = sum p_j v_j
//       grid barrier (monotone arrival counter)
//       s = sum_c s_c in a fixed order; w = p - (tau_k s / 2) v_k
//       the owner of column k+1 updates it first, forms reflector k+1 and
//       publishes it; every CTA then applies A -= v w^T + w v^T to its columns
//     Fixed-order sums only (no atomics on data): bit-reproducible, which the
//     sharded multi-GPU path relies on (every rank must hold identical factors).
//  2. bisection + inverse iteration on T for the top r (tridiag.cu).
//  3. backtr_big_kernel — x <- H_0 ... H_{n-3} x: one warp per vector, x in
//     shared memory, reflectors read through L1 two at a time (one fused
//     three-dot reduction per pair).
//
// Spin-waits are bounded (~4 s): a grid that is not co-resident reports
// ATK_CUDA_ERROR instead of hanging the device.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "atk_internal.cuh"

namespace atk {
namespace {

constexpr int kBT = 512;  // threads per CTA
constexpr int kBW = kBT / 32;
constexpr long long kSpinCycles = 1ll << 33;  // ~4 s at 1.9 GHz

struct TrdArgs {
    const double* a;
    int lda, n, sym;  // sym: the input is exactly symmetric (else 0.5 (A + A^T))
    double* wk;       // global column storage (columns j < nglob_max * G), ld n
    double* hh;       // n x n: reflector k in column k, rows k+1..n-1, hh(k+1, k) = 1
    double *d, *e, *tau;
    double* pbuf;   // 2 x n: p of the current step (parity-buffered)
    double* spart;  // 2 x G: per-CTA partial p^T v
    unsigned* sync; // [0] barrier arrivals, [1] reflectors published, [2] abort
    int nslots;     // shared-memory column slots per CTA
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Thread 0 only: wait until *p >= target; false (and the abort word set) on timeout.
__device__ bool spin_until(const unsigned* p, unsigned target, unsigned* abort_word) {
    const long long t0 = clock64();
    for (unsigned it = 0;; ++it) {
        if (ld_acquire(p) >= target) return true;
        if ((it & 255u) == 255u) {
            if (ld_acquire(abort_word) != 0u) return false;
            if (clock64() - t0 > kSpinCycles) {
                atomicExch(abort_word, 1u);
                return false;
            }
        }
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Every thread gets the block-wide sum (fixed order).  sh: >= kBW doubles.
__device__ __forceinline__ double block_sum_all(double v, double* sh) {
    v = warp_sum(v);
    __syncthreads();  // sh may still be read by a previous call
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kBW; ++w) s += sh[w];
    return s;
}

// S: row slots per thread (n - 1 <= S * kBT); QM: max columns per CTA.
template <int S, int QM>
__global__ void __launch_bounds__(kBT, 1) trd_grid_kernel(const TrdArgs p) {
    extern __shared__ __align__(16) double sm[];
    const int n = p.n, G = gridDim.x, c = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int nq = c < n ? (n - c + G - 1) / G : 0;  // owned columns j = c + q G
    const int nglob = max(0, nq - p.nslots);           // the first nglob live in global memory
    double* slots = sm;
    double* red = sm + size_t(p.nslots) * n;  // kBW x QM warp partials
    double* psm = red + kBW * QM;             // p_j of the live columns
    double* vsm = psm + QM;                   // v_j
    double* wsm = vsm + QM;                   // w_j
    double* pv = wsm + QM;                    // p_j v_j
    double* misc = pv + QM;                   // [0] tau s / 2, [1] abort flag, [2..] block_sum scratch
    auto col = [&](int q) -> double* {
        return q < nglob ? p.wk + size_t(c + q * G) * n : slots + size_t(q - nglob) * n;
    };

    // load (and symmetrise) the owned columns
    for (int q = 0; q < nq; ++q) {
        const int j = c + q * G;
        double* cj = col(q);
        if (p.sym) {
            for (int i = t; i < n; i += kBT) cj[i] = p.a[i + size_t(p.lda) * j];
        } else {
            for (int i = t; i < n; i += kBT) cj[i] = 0.5 * (p.a[i + size_t(p.lda) * j] + p.a[j + size_t(p.lda) * i]);
        }
    }
    __syncthreads();

    // reflector cc from rows cc+1..n-1 of column cc (dlarfg), published to all CTAs
    auto publish = [&](int cc, const double* cj) {
        double xs = 0.0;
        for (int i = cc + 2 + t; i < n; i += kBT) xs = fma(cj[i], cj[i], xs);
        xs = block_sum_all(xs, misc + 2);
        const double alpha = cj[cc + 1];
        double tau = 0.0, scal = 0.0, beta = alpha;
        if (xs > 0.0) {
            beta = -copysign(sqrt(fma(alpha, alpha, xs)), alpha);
            scal = 1.0 / (alpha - beta);
            tau = (beta - alpha) / beta;
        }
        double* hk = p.hh + size_t(cc) * n;
        for (int i = cc + 1 + t; i < n; i += kBT) __stcg(hk + i, i == cc + 1 ? 1.0 : cj[i] * scal);
        if (t == 0) {
            p.d[cc] = cj[cc];
            p.e[cc] = beta;
            __stcg(p.tau + cc, tau);
        }
        __syncthreads();
        if (t == 0) {
            __threadfence();
            st_release(p.sync + 1, unsigned(cc + 1));
        }
    };

    if (c == 0 && n > 2) publish(0, col(0));

    double vr[S], wr[S];
    for (int k = 0; k + 2 < n; ++k) {
        const int par = k & 1, r0 = k + 1;
        if (t == 0) misc[1] = spin_until(p.sync + 1, unsigned(k + 1), p.sync + 2) ? 0.0 : 1.0;
        __syncthreads();
        if (misc[1] != 0.0) return;
        const double tk = __ldcg(p.tau + k);
        const double* hk = p.hh + size_t(k) * n;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int i = r0 + t + kBT * s;
            vr[s] = i < n ? __ldcg(hk + i) : 0.0;
        }
        // live owned columns: q >= q0 (j = c + q G >= k + 1)
        const int q0 = k + 1 <= c ? 0 : (k + 1 - c + G - 1) / G;
        const int nl = nq - q0;
        double acc[QM];
#pragma unroll
        for (int qq = 0; qq < QM; ++qq) {
            acc[qq] = 0.0;
            if (qq < nl) {
                const double* cj = col(q0 + qq);
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const int i = r0 + t + kBT * s;
                    if (i < n) acc[qq] = fma(cj[i], vr[s], acc[qq]);
                }
            }
        }
#pragma unroll
        for (int qq = 0; qq < QM; ++qq) {
            if (qq < nl) {
                const double v = warp_sum(acc[qq]);
                if (lane == 0) red[w * QM + qq] = v;
            }
        }
        __syncthreads();
        if (t < nl) {
            double sacc = 0.0;
#pragma unroll
            for (int ww = 0; ww < kBW; ++ww) sacc += red[ww * QM + t];
            const int j = c + (q0 + t) * G;
            const double pj = tk * sacc, vj = __ldcg(hk + j);
            psm[t] = pj;
            vsm[t] = vj;
            pv[t] = pj * vj;
            __stcg(p.pbuf + size_t(par) * n + j, pj);
        }
        __syncthreads();
        if (t == 0) {
            double sc = 0.0;
            for (int q = 0; q < nl; ++q) sc += pv[q];
            __stcg(p.spart + size_t(par) * G + c, sc);
            __threadfence();
            atomicAdd(p.sync, 1u);
            misc[1] = spin_until(p.sync, unsigned(G) * unsigned(k + 1), p.sync + 2) ? 0.0 : 1.0;
        }
        __syncthreads();
        if (misc[1] != 0.0) return;
        if (w == 0) {
            double x = 0.0;
            for (int q = lane; q < G; q += 32) x += __ldcg(p.spart + size_t(par) * G + q);
            x = warp_sum(x);
            if (lane == 0) misc[0] = 0.5 * tk * x;
        }
        double pr[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int i = r0 + t + kBT * s;
            pr[s] = i < n ? __ldcg(p.pbuf + size_t(par) * n + i) : 0.0;
        }
        __syncthreads();
        const double hs = misc[0];
#pragma unroll
        for (int s = 0; s < S; ++s) wr[s] = fma(-hs, vr[s], pr[s]);
        if (t < nl) wsm[t] = fma(-hs, vsm[t], psm[t]);
        __syncthreads();
        // the owner of column k + 1 (its first live column) goes first
        const bool own_next = nl > 0 && c + q0 * G == k + 1;
        if (own_next) {
            double* cj = col(q0);
            const double wj = wsm[0], vj = vsm[0];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const int i = r0 + t + kBT * s;
                if (i < n) cj[i] = fma(-vr[s], wj, fma(-wr[s], vj, cj[i]));
            }
            __syncthreads();
            if (k + 1 <= n - 3) {
                publish(k + 1, cj);
            } else if (t == 0) {  // k + 1 == n - 2: the trailing 2 x 2 block
                p.d[n - 2] = cj[n - 2];
                p.e[n - 2] = cj[n - 1];
                p.tau[n - 2] = 0.0;
            }
        }
        for (int qq = own_next ? 1 : 0; qq < nl; ++qq) {
            double* cj = col(q0 + qq);
            const double wj = wsm[qq], vj = vsm[qq];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const int i = r0 + t + kBT * s;
                if (i < n) cj[i] = fma(-vr[s], wj, fma(-wr[s], vj, cj[i]));
            }
        }
    }
    __syncthreads();
    if (t == 0 && c == (n - 1) % G) p.d[n - 1] = col((n - 1 - c) / G)[n - 1];
}

constexpr int kBKW = 4;  // vectors (warps) per back-transformation CTA

// vout(:, c) = H_0 ... H_{n-3} X(:, c), H_k = I - tau_k v_k v_k^T (v_k in hh column k).
__global__ void __launch_bounds__(kBKW * 32) backtr_big_kernel(const double* __restrict__ hh,
                                                              const double* __restrict__ tau, int n,
                                                              const double* __restrict__ X, int nwant,
                                                              double* __restrict__ vout, int ldv) {
    extern __shared__ __align__(16) double xsm[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cidx = blockIdx.x * kBKW + w;
    if (cidx >= nwant) return;  // no block-wide barriers below
    double* x = xsm + size_t(w) * n;
    for (int i = lane; i < n; i += 32) x[i] = X[size_t(n) * cidx + i];
    __syncwarp();
    int k = n - 3;
    for (; k >= 1; k -= 2) {  // H_{k-1} H_k x
        const double ta = __ldg(tau + k), tb = __ldg(tau + k - 1);
        if (ta == 0.0 && tb == 0.0) continue;
        const double* a = hh + size_t(k) * n;      // rows k+1.., a(k+1) = 1
        const double* b = hh + size_t(k - 1) * n;  // rows k..,   b(k) = 1
        double da = 0.0, db = 0.0, dab = 0.0;
        for (int i = k + lane; i < n; i += 32) {
            const double bi = __ldg(b + i), ai = i > k ? __ldg(a + i) : 0.0, xi = x[i];
            da = fma(ai, xi, da);
            db = fma(bi, xi, db);
            dab = fma(bi, ai, dab);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            da += __shfl_xor_sync(0xffffffffu, da, o);
            db += __shfl_xor_sync(0xffffffffu, db, o);
            dab += __shfl_xor_sync(0xffffffffu, dab, o);
        }
        const double c1 = ta * da;                 // H_k:     x -= c1 a
        const double c2 = tb * fma(-c1, dab, db);  // H_{k-1}: x -= c2 b, with b.(x - c1 a)
        for (int i = k + lane; i < n; i += 32) {
            const double bi = __ldg(b + i), ai = i > k ? __ldg(a + i) : 0.0;
            x[i] = fma(-c2, bi, fma(-c1, ai, x[i]));
        }
        __syncwarp();
    }
    for (; k >= 0; --k) {
        const double tk = __ldg(tau + k);
        if (tk == 0.0) continue;
        const double* a = hh + size_t(k) * n;
        double da = 0.0;
        for (int i = k + 1 + lane; i < n; i += 32) da = fma(__ldg(a + i), x[i], da);
        da = tk * warp_sum(da);
        for (int i = k + 1 + lane; i < n; i += 32) x[i] = fma(-da, __ldg(a + i), x[i]);
        __syncwarp();
    }
    for (int i = lane; i < n; i += 32) vout[size_t(ldv) * cidx + i] = x[i];
}

size_t trd_grid_extra(int qm) { return size_t(kBW * qm + 4 * qm + 2 + 2 + kBW) * sizeof(double); }

template <int S, int QM>
void launch_trd_grid(atk_ctx* ctx, TrdArgs& a, int G, size_t smem) {
    static bool attr = false;
    if (!attr) {
        ATK_CUDA(cudaFuncSetAttribute(trd_grid_kernel<S, QM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(smem_cap_bytes())));
        attr = true;
    }
    void* args[] = {&a};
    static const bool noncoop = std::getenv("ATK_PROFILE_NONCOOP") != nullptr;  // ncu replays (1 CTA / SM)
    if (noncoop) {
        trd_grid_kernel<S, QM><<<unsigned(G), kBT, smem, ctx->stream>>>(a);
    } else {
        ATK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(trd_grid_kernel<S, QM>), dim3(unsigned(G)),
                                             dim3(kBT), args, smem, ctx->stream));
    }
    ATK_LAUNCHED(ctx);
}

}  // namespace

size_t smem_cap_bytes() {
    static size_t cap = 0;
    if (!cap) {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cap = v > 0 ? size_t(v) : size_t(227 * 1024);
    }
    return cap;
}

void dense_eig_big(atk_ctx* ctx, const double* a, int n, int lda, int nwant, double* values, double* vectors,
                   int ldv, bool exact_sym) {
    if (n < 3 || n > kBigEigMax) fail(ATK_UNSUPPORTED, "dense_eig_big: n out of range");
    if (nwant < 1 || nwant > n) fail(ATK_RANK_TOO_LARGE, "dense_eig_big: nwant out of range");
    cudaStream_t st = ctx->stream;
    const int G = ctx->num_sms;
    const int qmax = (n + G - 1) / G;
    const int S = (n - 1 + kBT - 1) / kBT;
    int qm = qmax <= 8 ? 8 : qmax <= 16 ? 16 : 32;
    if (qmax > 32 || S > 8) fail(ATK_UNSUPPORTED, "dense_eig_big: n too large for this GPU");
    const size_t extra = trd_grid_extra(qm);
    const size_t cap = smem_cap_bytes();
    int nslots = int(std::min<size_t>(qmax, (cap - extra) / (size_t(n) * sizeof(double))));
    const size_t smem = size_t(nslots) * n * sizeof(double) + extra;
    const int nglob_max = std::max(0, qmax - nslots);
    const size_t wk_cols = std::min<size_t>(n, size_t(nglob_max) * G);
    const size_t nn = size_t(n) * n;
    DevBuf<double> ws(ctx, wk_cols * n + nn + 3 * size_t(n) + 2 * size_t(n) + 2 * size_t(G) + size_t(n) * nwant +
                               5 * size_t(n) * nwant);
    double* wk = ws.get();
    double* hh = wk + wk_cols * n;
    double* d = hh + nn;
    double* e = d + n;
    double* tau = e + n;
    double* pbuf = tau + n;
    double* spart = pbuf + 2 * size_t(n);
    double* X = spart + 2 * size_t(G);
    double* wkinv = X + size_t(n) * nwant;
    DevBuf<unsigned> sync(ctx, 4);
    ATK_CUDA(cudaMemsetAsync(sync.get(), 0, 4 * sizeof(unsigned), st));
    TrdArgs args{a, lda, n, exact_sym ? 1 : 0, wk, hh, d, e, tau, pbuf, spart, sync.get(), nslots};
    // ATK_TRACE: device time of the three phases (events, printed after the final sync)
    static const bool trace = std::getenv("ATK_TRACE") != nullptr;
    cudaEvent_t ev[4] = {};
    if (trace)
        for (auto& x : ev) {
            cudaEventCreate(&x);
        }
    if (trace) cudaEventRecord(ev[0], st);
    if (S <= 2 && qm == 8) launch_trd_grid<2, 8>(ctx, args, G, smem);
    else if (S <= 4 && qm <= 16) launch_trd_grid<4, 16>(ctx, args, G, smem);
    else launch_trd_grid<8, 32>(ctx, args, G, smem);
    if (trace) cudaEventRecord(ev[1], st);
    tridiag_tail(ctx, d, e, n, nwant, nwant, values, X, wkinv);
    if (trace) cudaEventRecord(ev[2], st);
    static bool battr = false;
    if (!battr) {
        ATK_CUDA(cudaFuncSetAttribute(backtr_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(size_t(kBKW) * kBigEigMax * sizeof(double))));
        battr = true;
    }
    backtr_big_kernel<<<unsigned((nwant + kBKW - 1) / kBKW), kBKW * 32, size_t(kBKW) * n * sizeof(double), st>>>(
        hh, tau, n, X, nwant, vectors, ldv);
    ATK_LAUNCHED(ctx);
    if (trace) cudaEventRecord(ev[3], st);
    unsigned abort_word = 0;
    ATK_CUDA(cudaMemcpyAsync(&abort_word, sync.get() + 2, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    ATK_CUDA(cudaStreamSynchronize(st));
    if (trace) {
        float ms[3];
        for (int q = 0; q < 3; ++q) cudaEventElapsedTime(&ms[q], ev[q], ev[q + 1]);
        std::fprintf(stderr, "[atk dense eig n=%d r=%d] trd %.3f ms (%d smem slots/SM) bisect+invit %.3f ms backtr %.3f ms\n",
                     n, nwant, ms[0], nslots, ms[1], ms[2]);
        for (auto& x : ev) cudaEventDestroy(x);
    }
    if (abort_word) fail(ATK_CUDA_ERROR, "dense_eig_big: grid synchronisation timed out (grid not co-resident)");
}

}  // namespace atk
