// trd_big.cu — exact dense symmetric eigensolver for kTridiagMax < n <= kBigEigMax:
// linalg::sym_eig_top_r (linalg.hpp:101-123), whose Eigen SelfAdjointEigenSolver
// (:108) tridiagonalises and then runs implicit QR on ALL eigenpairs.  Here the
// cost is bounded on any spectrum (n - 2 Householder steps, no iteration count
// that depends on eigenvalue gaps), and only the top r vectors are formed.
//
//  1. Householder tridiagonalisation A = Q T Q^T (LAPACK dsytd2, lower) by
//     trd_kernel, in two launches of the same code:
//       grid phase    — one persistent cooperative CTA per SM (G = 148),
//                       exchange through L2 + a software grid barrier
//                       (~1.2 us, measured: profiles/barrier_probe.cu);
//       cluster phase — once the trailing matrix fits 16 SMs' shared memory
//                       (n - k <= ~640), one 16-CTA cluster, exchange through
//                       DSMEM + the hardware cluster barrier (~0.28 us).
//     Column j of the trailing matrix belongs to CTA j mod G and is stored
//     WHOLE (rows k+1..n-1, both triangles), so p = tau A v needs no cross-CTA
//     reduction: each CTA forms p_j for its own columns.  The pivot column's
//     last update and reflector are computed REDUNDANTLY by every CTA from p
//     and the column's pre-update copy, so a step needs one barrier and no
//     other wait, and the update of step k-1 is fused with the matvec of step k
//     (one pass over the columns per step).  Rows are dealt to threads once
//     (row i on thread (i - k0) mod 512), so v and w stay in registers.
//     Fixed-order sums only (no atomics on data): the result is
//     bit-reproducible, which the sharded multi-GPU path relies on (every rank
//     must hold identical factors).
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
#include <type_traits>

#include "atk_internal.cuh"

namespace atk {
namespace {

constexpr int kBT = 512;  // threads per CTA
constexpr int kBW = kBT / 32;
constexpr int kMaxG = 160;  // grid size bound (B200: 148 SMs)
constexpr int kCH = 16;     // columns per accumulation chunk
constexpr int kCS = 16;     // cluster size of the tail phase
constexpr int kCQM = 48;    // columns per CTA in the tail phase (trailing size <= 768)
constexpr long long kSpinCycles = 1ll << 33;  // ~4 s at 1.9 GHz

struct TrdArgs {
    const double* src;  // columns at iteration k0: the input (grid) or the handoff copy (cluster)
    int lds, n, sym;    // sym: src exactly symmetric (else 0.5 (A + A^T))
    int k0, k1;         // iterations [k0, k1); k1 == n - 2 also finishes T
    double* wk;         // grid: columns that do not fit shared memory (column j at wk + j n)
    double* hand;       // k1 < n - 2: trailing matrix after update k1 - 1 (column j at hand + j n)
    double* hh;         // n x n: reflector k in column k, rows k+1..n-1, hh(k+1, k) = 1
    double *d, *e, *tau;
    double* pbuf;    // grid exchange: 2 x n, p by parity
    double* colbuf;  // 2 x n: column k+1 after update k-1
    unsigned* sync;  // [0] barrier arrivals, [2] abort
    int nslots, slot_len;  // shared-memory column slots per CTA and their length (rows k0+1..)
    long long* prof;       // ATK_TRD_PROFILE: CTA 0 thread 0 cycles per phase
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
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

// Block-wide fixed-order sum with one barrier: `sh` (kBW doubles) must not be
// read by a pending earlier call (callers alternate two buffers).
__device__ __forceinline__ double block_sum_1(double v, double* sh) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kBW; ++w) s += sh[w];
    return s;
}

// Warp sums of 16 per-lane values in 16 shuffles (recursive halving): lane l
// returns the full warp sum of acc[l >> 1] (lanes 2c and 2c+1 hold column c).
__device__ __forceinline__ double warp_sum16_t(double (&acc)[16]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int h = 8; h >= 1; h >>= 1) {  // exchange with lane ^ (2 h): keep the half selected by that bit
        const bool up = (lane & (2 * h)) != 0;
#pragma unroll
        for (int q = 0; q < h; ++q) {
            const double send = up ? acc[q] : acc[q + h];
            const double keep = up ? acc[q + h] : acc[q];
            acc[q] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * h);
        }
    }
    return acc[0] + __shfl_xor_sync(0xffffffffu, acc[0], 1);
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ double ld_remote(const double* local, uint32_t rank) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_addr(local)), "r"(rank));
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
    return v;
}

// Exchange through L2 (grid phase).
struct GridEx {
    const TrdArgs& p;
    int G;
    __device__ double pv(int par, int i) const { return __ldcg(p.pbuf + size_t(par) * p.n + i); }
    __device__ double colv(int par, int /*k*/, int i) const { return __ldcg(p.colbuf + size_t(par) * p.n + i); }
    __device__ void put_p(int par, int j, double v) const { __stcg(p.pbuf + size_t(par) * p.n + j, v); }
    __device__ void put_col(int par, int i, double v) const { __stcg(p.colbuf + size_t(par) * p.n + i, v); }
    // every thread, after warp 0 wrote pbuf (the other warps' stores are
    // ordered by the preceding __syncthreads); false on abort
    __device__ bool barrier(int k, double* flag) const {
        if (threadIdx.x < 32) {
            __syncwarp();
            if (threadIdx.x == 0) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.sync) : "memory");
                *flag = spin_until(p.sync, unsigned(G) * unsigned(k + 1 - p.k0), p.sync + 2) ? 0.0 : 1.0;
            }
        }
        __syncthreads();
        return *flag == 0.0;
    }
};

// Exchange through DSMEM (cluster phase): every CTA keeps its own p_j, its
// copy of the next pivot column and its partial in local shared memory; the
// readers load them remotely after the cluster barrier.
struct ClusterEx {
    const TrdArgs& p;
    double* pl;   // 2 x ceil(n / kCS): p_j at j / kCS
    double* cbl;  // 2 x slot_len: pivot column copy, row i at i - (k0 + 1)
    int pl_len;
    __device__ double pv(int par, int i) const { return ld_remote(pl + par * pl_len + i / kCS, uint32_t(i % kCS)); }
    __device__ double colv(int par, int k, int i) const {
        return ld_remote(cbl + par * p.slot_len + (i - p.k0 - 1), uint32_t(k % kCS));
    }
    __device__ void put_p(int par, int j, double v) const { pl[par * pl_len + j / kCS] = v; }
    __device__ void put_col(int par, int i, double v) const { cbl[par * p.slot_len + (i - p.k0 - 1)] = v; }
    __device__ bool barrier(int, double*) const {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        return true;
    }
};

// S: row slots per thread ((n - k0) <= S * kBT); QM: max stored columns per CTA.
//
// Iteration k (k0 <= k < k1), entered after barrier k-1:
//   A. finish column k: every CTA reads p_{k-1}, the partials of
//      p_{k-1}^T v_{k-1} and column k as it stood before update k-1 (copied by
//      its owner), and applies update k-1 to it;
//   B. every CTA forms reflector k from it redundantly (bitwise identical: the
//      same operations in the same order); the owner of column k stores it;
//   C. ONE pass over the CTA's live columns applies update k-1 and accumulates
//      A v_k; the owner of column k+1 also copies it for the next pivot;
//   D. p_k = tau_k A v_k for the owned columns, partial p_k^T v_k; barrier k.
template <int S, int QM, bool CLUSTER>
__global__ void __launch_bounds__(kBT, 1) trd_kernel(const TrdArgs p) {
    extern __shared__ __align__(16) double sm[];
    const int n = p.n, G = gridDim.x, c = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int k0 = p.k0, rb = k0;  // row i lives on thread (i - rb) % kBT, slot (i - rb) / kBT
    // owned stored columns: j = jf + q G >= k0 + 1
    const int jf = k0 + 1 + ((c - (k0 + 1) % G) + G) % G;
    const int nq = jf < n ? (n - jf + G - 1) / G : 0;
    const int nglob = CLUSTER ? 0 : max(0, nq - p.nslots);
    double* slots = sm;
    double* red = slots + size_t(p.nslots) * p.slot_len;  // kBW x QM
    double* wq = red + kBW * QM;                           // QM: w_{k-1} at the owned columns
    double* vq = wq + QM;                                  // 2 x QM: v by parity at the owned columns
    double* misc = vq + 2 * QM;                            // [1] abort, [2] alpha, [3] p_{k-1}(k), [4..] 4 x kBW sums
    double* xtra = misc + 4 + 4 * kBW;                     // cluster: pl, cbl
    const int pl_len = (n + kCS - 1) / kCS;
    using Ex = typename std::conditional<CLUSTER, ClusterEx, GridEx>::type;
    Ex ex = [&] {
        if constexpr (CLUSTER) return ClusterEx{p, xtra, xtra + 2 * pl_len, pl_len};
        else return GridEx{p, G};
    }();
    auto col = [&](int q) -> double* {  // column jf + q G; element i at [i]
        if (!CLUSTER && q < nglob) return p.wk + size_t(jf + q * G) * n;
        return slots + size_t(q - nglob) * p.slot_len - (k0 + 1);
    };
    auto src = [&](int i, int j) -> double {
        return p.sym ? p.src[i + size_t(p.lds) * j] : 0.5 * (p.src[i + size_t(p.lds) * j] + p.src[j + size_t(p.lds) * i]);
    };
    for (int q = 0; q < nq; ++q) {
        const int j = jf + q * G;
        double* cj = col(q);
        for (int i = k0 + 1 + t; i < n; i += kBT) cj[i] = src(i, j);
    }
    // per row slot: the owned-column index of the row (or -1)
    int qrow[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int i = rb + t + kBT * s;
        qrow[s] = (i >= jf && i < n && (i - jf) % G == 0) ? (i - jf) / G : -1;
    }

    long long t_mark = clock64(), t_acc[5] = {0, 0, 0, 0, 0};
    const bool prof = p.prof != nullptr && c == 0 && t == 0;
    auto lap = [&](int ph) {
        if (prof) {
            const long long tt = clock64();
            t_acc[ph] += tt - t_mark;
            t_mark = tt;
        }
    };
    __syncthreads();

    double tprev = 0.0;  // tau_{k-1}
    double vpr[S], wr[S], vn[S], cr[S];
#pragma unroll
    for (int s = 0; s < S; ++s) vpr[s] = wr[s] = 0.0;
    // ---- A for iteration k: column k after update k-1 in cr (rows > k), row k in *ck
    auto finish_column = [&](int k, bool first, double& ck) {
        const int prv = (k & 1) ^ 1;
        if (first) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const int i = rb + t + kBT * s;
                cr[s] = (i > k && i < n) ? src(i, k) : 0.0;
                if (i == k) ck = src(k, k);
            }
            return;
        }
        double pr[S], cb[S], cbk = 0.0, sp = 0.0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int i = rb + t + kBT * s;
            const bool act = i > k && i < n;
            pr[s] = act ? ex.pv(prv, i) : 0.0;
            cb[s] = act ? ex.colv(prv, k, i) : 0.0;
            sp = fma(pr[s], vpr[s], sp);
            if (i == k) {
                cbk = ex.colv(prv, k, k);
                const double pk_ = ex.pv(prv, k);
                misc[3] = pk_;
                sp += pk_;  // v_{k-1}(k) = 1
            }
        }
        // s = p_{k-1}^T v_{k-1} from the p this CTA loads anyway (same order in every CTA)
        const double hs = 0.5 * tprev * block_sum_1(sp, misc + 4 + 2 * kBW + kBW * (k & 1));
        const double pk = misc[3];
        const double wk_ = pk - hs;  // v_{k-1}(k) = 1
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int i = rb + t + kBT * s;
            const bool act = i > k && i < n;
            wr[s] = act ? fma(-hs, vpr[s], pr[s]) : 0.0;
            cr[s] = act ? fma(-vpr[s], wk_, cb[s] - wr[s]) : 0.0;
            if (act && qrow[s] >= 0) wq[qrow[s]] = wr[s];
            if (i == k) ck = fma(-2.0, wk_, cbk);
        }
    };

    int k = k0;
    for (; k < p.k1; ++k) {
        const int par = k & 1, prv = par ^ 1;
        const bool first = k == k0;
        double ck = 0.0;
        finish_column(k, first, ck);
        lap(0);
        // ---- B: reflector k from rows k+1.. of column k (dlarfg), redundantly in every CTA
        double xs = 0.0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int i = rb + t + kBT * s;
            if (i > k + 1 && i < n) xs = fma(cr[s], cr[s], xs);
            if (i == k + 1) misc[2] = cr[s];
        }
        xs = block_sum_1(xs, misc + 4 + kBW * par);
        const double alpha = misc[2];
        double tk = 0.0, scal = 0.0, beta = alpha;
        if (xs > 0.0) {
            beta = -copysign(sqrt(fma(alpha, alpha, xs)), alpha);
            scal = 1.0 / (alpha - beta);
            tk = (beta - alpha) / beta;
        }
        const bool owner_k = (k - c) % G == 0;
        double* hk = p.hh + size_t(k) * n;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int i = rb + t + kBT * s;
            vn[s] = i == k + 1 ? 1.0 : (i > k + 1 && i < n) ? cr[s] * scal : 0.0;
            if (i > k && i < n) {
                if (qrow[s] >= 0) vq[par * QM + qrow[s]] = vn[s];
                if (owner_k) hk[i] = vn[s];
            }
            if (owner_k && i == k) p.d[k] = ck;
        }
        if (owner_k && t == 0) {
            p.e[k] = beta;
            p.tau[k] = tk;
        }
        lap(1);
        // ---- C: update k-1 and A v_k in one pass over the live owned columns (j >= k+1)
        const int qa = jf >= k + 1 ? 0 : (k + 1 - jf + G - 1) / G;
        const int nl = nq - qa;
        const int s_dead = (k + 1 - rb) / kBT;  // slots whose rows are all <= k
        for (int cb0 = 0; cb0 < nl; cb0 += kCH) {
            double acc[kCH];
#pragma unroll
            for (int qq = 0; qq < kCH; ++qq) {
                acc[qq] = 0.0;
                if (cb0 + qq < nl) {
                    const int q = qa + cb0 + qq, j = jf + q * G;
                    double* cj = col(q);
                    const double wj = first ? 0.0 : wq[q], vj = first ? 0.0 : vq[prv * QM + q];
                    const bool to_col = j == k + 1;
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        if (s < s_dead || rb + kBT * s >= n) continue;  // CTA-uniform: whole slot dead
                        const int i = rb + t + kBT * s;
                        if (i > k && i < n) {
                            double a = cj[i];
                            if (!first) {
                                a = fma(-vpr[s], wj, fma(-wr[s], vj, a));
                                cj[i] = a;
                            }
                            if (to_col) ex.put_col(par, i, a);
                            acc[qq] = fma(a, vn[s], acc[qq]);
                        }
                    }
                }
            }
            const double v = warp_sum16_t(acc);
            if ((lane & 1) == 0 && cb0 + (lane >> 1) < nl) red[w * QM + cb0 + (lane >> 1)] = v;
        }
        lap(2);
        __syncthreads();
        // ---- D: p_k = tau_k A v_k for the owned columns, partial p_k^T v_k, barrier k
        if (w == 0) {
            for (int l = lane; l < nl; l += 32) {
                double sacc = 0.0;
#pragma unroll
                for (int ww = 0; ww < kBW; ++ww) sacc += red[ww * QM + l];
                ex.put_p(par, jf + (qa + l) * G, tk * sacc);
            }
        }
        lap(3);
        if (!ex.barrier(k, misc + 1)) return;
        tprev = tk;
#pragma unroll
        for (int s = 0; s < S; ++s) vpr[s] = vn[s];
        lap(4);
    }
    if (prof)
        for (int q = 0; q < 5; ++q) p.prof[q] += t_acc[q];
    if (k + 2 == n) {
        // ---- the trailing 2 x 2 block after update n-3 (k == n - 2)
        double ck = 0.0;
        finish_column(k, k == k0, ck);  // column n-2: cr at row n-1, ck at row n-2
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int i = rb + t + kBT * s;
            if (i == n - 2 && c == 0) {
                p.d[n - 2] = ck;
                p.tau[n - 2] = 0.0;
            }
            if (i == n - 1) {
                if (c == 0) p.e[n - 2] = cr[s];
                if ((n - 1 - c) % G == 0) {  // the owner of column n-1: A(n-1, n-1) after update n-3
                    const double a = col((n - 1 - jf) / G)[n - 1];
                    p.d[n - 1] = k == k0 ? a : fma(-2.0 * vpr[s], wr[s], a);
                }
            }
        }
        // no CTA may exit while another still reads its shared memory remotely
        if constexpr (CLUSTER) ex.barrier(k, misc + 1);
        return;
    }
    // ---- handoff (grid phase, k == k1): the trailing matrix after update k1-1
    double ck = 0.0;
    finish_column(k, false, ck);
    if ((k - c) % G == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int i = rb + t + kBT * s;
            if (i > k && i < n) p.hand[size_t(k) * n + i] = cr[s];
            if (i == k) p.hand[size_t(k) * n + k] = ck;
        }
    }
    __syncthreads();  // wq complete
    const int qa = jf >= k + 1 ? 0 : (k + 1 - jf + G - 1) / G;
    const int prv = (k & 1) ^ 1;
    for (int q = qa; q < nq; ++q) {
        const int j = jf + q * G;
        const double* cj = col(q);
        const double wj = wq[q], vj = vq[prv * QM + q];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int i = rb + t + kBT * s;
            if (i > k && i < n) p.hand[size_t(j) * n + i] = fma(-vpr[s], wj, fma(-wr[s], vj, cj[i]));
        }
    }
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

// ---------------------------------------------------------------------------
// Blocked back-transformation (compact WY, fp64 DMMA): with B_b = H_kb ... H_kb+31
// = I - V_b T_b V_b^T (LAPACK dlarft, forward / columnwise), Q = B_0 ... B_last and
// Z <- B_b Z = Z - V_b (T_b (V_b^T Z)) for b = last..0.  One CTA per 8 vectors
// (Z resident in shared memory); V_b^T Z and V_b W are m8n8k4 DMMA tiles with
// the rows split over the warps, the reflectors read straight from hh (L2).
constexpr int kWYB = 32;  // reflectors per block
constexpr int kWYT = 256;
constexpr int kWYV = 8;  // vectors per CTA (one DMMA n-fragment)

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// V_b(i, q): reflector k = kb + q at row i (zero above its leading 1 and past k = n - 3)
__device__ __forceinline__ double vb_at(const double* hh, int n, int k, int i) {
    return (k <= n - 3 && i >= k + 1 && i < n) ? __ldg(hh + size_t(k) * n + i) : 0.0;
}

__global__ void __launch_bounds__(kWYT) larft_kernel(const double* __restrict__ hh, const double* __restrict__ tau,
                                                    int n, double* __restrict__ tout) {
    __shared__ double G[kWYB][kWYB + 1];   // V^T V (upper)
    __shared__ double Ts[kWYB][kWYB + 1];  // T (upper)
    const int b = blockIdx.x, kb = b * kWYB, t = threadIdx.x, w = t >> 5, lane = t & 31;
    for (int pq = w; pq < kWYB * kWYB; pq += kWYT / 32) {
        const int pp = pq % kWYB, qq = pq / kWYB;
        if (pp > qq) continue;  // warp-uniform
        const int kp = kb + pp, kq = kb + qq;
        double sacc = 0.0;
        if (kq <= n - 3)
            for (int i = kq + 1 + lane; i < n; i += 32) sacc = fma(vb_at(hh, n, kp, i), __ldg(hh + size_t(kq) * n + i), sacc);
        sacc = warp_sum(sacc);
        if (lane == 0) G[pp][qq] = sacc;
    }
    __syncthreads();
    if (w == 0) {
        for (int i = 0; i < kWYB; ++i) {
            const int k = kb + i;
            const double ti = k <= n - 3 ? __ldg(tau + k) : 0.0;
            double y = 0.0;
            if (lane < i)
                for (int q = lane; q < i; ++q) y = fma(Ts[lane][q], G[q][i], y);
            __syncwarp();
            Ts[lane][i] = lane < i ? -ti * y : lane == i ? ti : 0.0;
            __syncwarp();
        }
    }
    __syncthreads();
    for (int e = t; e < kWYB * kWYB; e += kWYT) tout[size_t(b) * kWYB * kWYB + e] = Ts[e % kWYB][e / kWYB];
}

__global__ void __launch_bounds__(kWYT) backtr_wy_kernel(const double* __restrict__ hh, const double* __restrict__ tg,
                                                        int n, int nblk, const double* __restrict__ X, int nwant,
                                                        double* __restrict__ vout, int ldv) {
    extern __shared__ __align__(16) double zs[];  // n x kWYV, row-major (zs[i * 8 + c])
    __shared__ double wp[kWYT / 32][kWYB * kWYV];
    __shared__ double ws[kWYB * kWYV];
    __shared__ double ts[kWYB * kWYB];  // column-major T_b
    const int c0 = blockIdx.x * kWYV, t = threadIdx.x, w = t >> 5, lane = t & 31;
    const int nv = min(kWYV, nwant - c0);
    const int gq = lane >> 2, tq = lane & 3;
    for (int e = t; e < n * kWYV; e += kWYT) {
        const int i = e / kWYV, c = e % kWYV;
        zs[e] = c < nv ? X[size_t(n) * (c0 + c) + i] : 0.0;
    }
    for (int b = nblk - 1; b >= 0; --b) {
        const int kb = b * kWYB, r0 = kb + 1, nrows = n - r0;
        for (int e = t; e < kWYB * kWYB; e += kWYT) ts[e] = __ldg(tg + size_t(b) * kWYB * kWYB + e);
        __syncthreads();
        // 1. W = V^T Z (32 x 8): warps split the rows in 4-row k-steps
        double acc[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
        const int ksteps = (nrows + 3) / 4;
        for (int ks = w; ks < ksteps; ks += kWYT / 32) {
            const int i = r0 + ks * 4 + tq;
            const double bz = i < n ? zs[i * kWYV + gq] : 0.0;
#pragma unroll
            for (int mf = 0; mf < 4; ++mf) dmma884(acc[mf][0], acc[mf][1], vb_at(hh, n, kb + mf * 8 + gq, i), bz);
        }
#pragma unroll
        for (int mf = 0; mf < 4; ++mf) {
            wp[w][(mf * 8 + gq) * kWYV + 2 * tq] = acc[mf][0];
            wp[w][(mf * 8 + gq) * kWYV + 2 * tq + 1] = acc[mf][1];
        }
        __syncthreads();
        double wsum = 0.0;
#pragma unroll
        for (int q = 0; q < kWYT / 32; ++q) wsum += wp[q][t];  // t < 256 = kWYB * kWYV
        ws[t] = wsum;
        __syncthreads();
        // 2. W <- T W (T upper)
        {
            const int m = t / kWYV, cc = t % kWYV;
            double y = 0.0;
            for (int q = m; q < kWYB; ++q) y = fma(ts[q * kWYB + m], ws[q * kWYV + cc], y);
            __syncthreads();
            ws[t] = y;
        }
        __syncthreads();
        // 3. Z -= V W: 8-row m-fragments over the warps, K = 32 reflectors
        const int mfr = (nrows + 7) / 8;
        for (int mf = w; mf < mfr; mf += kWYT / 32) {
            const int row = r0 + mf * 8 + gq;
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int kk = 0; kk < kWYB / 4; ++kk) {
                const int q = kk * 4 + tq;
                dmma884(d0, d1, -vb_at(hh, n, kb + q, row), ws[q * kWYV + gq]);
            }
            if (row < n) {
                zs[row * kWYV + 2 * tq] += d0;
                zs[row * kWYV + 2 * tq + 1] += d1;
            }
        }
        __syncthreads();
    }
    for (int e = t; e < n * kWYV; e += kWYT) {
        const int i = e / kWYV, c = e % kWYV;
        if (c < nv) vout[size_t(ldv) * (c0 + c) + i] = zs[e];
    }
}

template <int S, int QM, bool CL>
void launch_trd(atk_ctx* ctx, TrdArgs& a, size_t smem) {
    static bool attr = false;
    if (!attr) {
        ATK_CUDA(cudaFuncSetAttribute(trd_kernel<S, QM, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(smem_cap_bytes())));
        if (CL) ATK_CUDA(cudaFuncSetAttribute(trd_kernel<S, QM, CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr = true;
    }
    if (CL) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(kCS);
        cfg.blockDim = dim3(kBT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = kCS;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        ATK_CUDA(cudaLaunchKernelEx(&cfg, trd_kernel<S, QM, CL>, a));
    } else {
        void* args[] = {&a};
        static const bool noncoop = std::getenv("ATK_PROFILE_NONCOOP") != nullptr;  // ncu replays (1 CTA / SM)
        if (noncoop)
            trd_kernel<S, QM, CL><<<unsigned(ctx->num_sms), kBT, smem, ctx->stream>>>(a);
        else
            ATK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(trd_kernel<S, QM, CL>),
                                                 dim3(unsigned(ctx->num_sms)), dim3(kBT), args, smem, ctx->stream));
    }
    ATK_LAUNCHED(ctx);
}

// shared memory beside the column slots (doubles)
size_t trd_extra(int n, int qm, bool cl, int slot_len) {
    size_t x = size_t(kBW) * qm + 3 * size_t(qm) + 4 + 4 * kBW;
    if (cl) x += 2 * size_t((n + kCS - 1) / kCS) + 2 * size_t(slot_len);
    return x * sizeof(double);
}

// Can a 16-CTA cluster of trd_kernel<2, kCQM, true> with `smem` bytes run?
bool cluster_ok(size_t smem) {
    static int ok = -1;
    if (ok < 0) {
        cudaFuncSetAttribute(trd_kernel<2, kCQM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(smem_cap_bytes()));
        cudaFuncSetAttribute(trd_kernel<2, kCQM, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(kCS);
        cfg.blockDim = dim3(kBT);
        cfg.dynamicSmemBytes = smem_cap_bytes() - 1024;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = kCS;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nc = 0;
        ok = (cudaOccupancyMaxActiveClusters(&nc, trd_kernel<2, kCQM, true>, &cfg) == cudaSuccess && nc >= 1) ? 1 : 0;
        cudaGetLastError();
    }
    (void)smem;
    return ok == 1;
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
    const size_t cap = smem_cap_bytes();
    // tail phase: the largest trailing size L (rows k0+1..n-1) one 16-CTA cluster holds
    int L = 0;
    if (std::getenv("ATK_TRD_NOCLUSTER") == nullptr) {
        for (int l = std::min(n - 1, std::min(kCQM * kCS, 2 * kBT - 1)); l >= 16; --l) {
            const size_t need = size_t((l + kCS - 1) / kCS) * l * sizeof(double) + trd_extra(n, kCQM, true, l);
            if (need <= cap) {
                L = l;
                break;
            }
        }
        if (L > 0 && !cluster_ok(cap)) L = 0;
    }
    const int ks = L > 0 ? n - 1 - L : n - 2;  // first iteration of the tail phase (n - 2: none)
    const size_t nn = size_t(n) * n;
    // grid phase shape
    const int gslot = n - 1;
    const int qmax = (n - 1 + G - 1) / G;
    const int Sg = (n + kBT - 1) / kBT;
    // the launched instance (below) fixes QM, and with it the kernel's shared-memory layout
    // beside the column slots: size for THAT QM (n > 2048 launches <8, 32> with qmax <= 16)
    const int qm0 = qmax <= 8 ? 8 : qmax <= 16 ? 16 : 32;
    const int qm = (Sg <= 2 && qm0 == 8) ? 8 : (Sg <= 4 && qm0 <= 16) ? 16 : 32;
    if (ks > 0 && (qmax > 32 || Sg > 8 || G > kMaxG)) fail(ATK_UNSUPPORTED, "dense_eig_big: n too large for this GPU");
    const size_t gextra = trd_extra(n, qm, false, gslot);
    const int nslots = int(std::min<size_t>(qmax, (cap - gextra) / (size_t(gslot) * sizeof(double))));
    const size_t gsmem = size_t(nslots) * gslot * sizeof(double) + gextra;
    const int nglob_max = std::max(0, qmax - nslots);
    const size_t wk_cols = ks > 0 ? std::min<size_t>(n, size_t(nglob_max + 1) * G) : 0;
    DevBuf<double> ws(ctx, wk_cols * n + (ks > 0 && L > 0 ? nn : 0) + nn + 3 * size_t(n) + 4 * size_t(n) +
                               size_t(n) * nwant + 5 * size_t(n) * nwant);
    double* wk = ws.get();
    double* hand = wk + wk_cols * n;
    double* hh = hand + (ks > 0 && L > 0 ? nn : 0);
    double* d = hh + nn;
    double* e = d + n;
    double* tau = e + n;
    double* pbuf = tau + n;
    double* colbuf = pbuf + 2 * size_t(n);
    double* X = colbuf + 2 * size_t(n);
    double* wkinv = X + size_t(n) * nwant;
    DevBuf<unsigned> sync(ctx, 4);
    ATK_CUDA(cudaMemsetAsync(sync.get(), 0, 4 * sizeof(unsigned), st));
    static long long* prof = nullptr;
    static const bool want_prof = std::getenv("ATK_TRD_PROFILE") != nullptr;
    if (want_prof && !prof) ATK_CUDA(cudaMalloc(&prof, 8 * sizeof(long long)));
    if (prof) ATK_CUDA(cudaMemsetAsync(prof, 0, 8 * sizeof(long long), st));
    // ATK_TRACE: device time of the phases (events, printed after the final sync)
    static const bool trace = std::getenv("ATK_TRACE") != nullptr;
    cudaEvent_t ev[5] = {};
    if (trace)
        for (auto& x : ev) cudaEventCreate(&x);
    if (trace) cudaEventRecord(ev[0], st);
    if (ks > 0) {
        TrdArgs g{a, lda, n, exact_sym ? 1 : 0, 0, ks, wk, hand, hh, d, e, tau, pbuf, colbuf, sync.get(),
                  nslots, gslot, prof};
        if (qm == 8) launch_trd<2, 8, false>(ctx, g, gsmem);
        else if (qm == 16) launch_trd<4, 16, false>(ctx, g, gsmem);
        else launch_trd<8, 32, false>(ctx, g, gsmem);
    }
    if (trace) cudaEventRecord(ev[1], st);
    if (L > 0) {
        const int k0 = std::max(ks, 0);
        const int slot = n - k0 - 1;
        const int nsl = (slot + kCS - 1) / kCS;
        const size_t csmem = size_t(nsl) * slot * sizeof(double) + trd_extra(n, kCQM, true, slot);
        TrdArgs cl{ks > 0 ? hand : a, ks > 0 ? n : lda, n, (ks > 0 || exact_sym) ? 1 : 0, k0, n - 2, nullptr, nullptr,
                   hh, d, e, tau, nullptr, nullptr, sync.get(), nsl, slot, prof};
        launch_trd<2, kCQM, true>(ctx, cl, csmem);
    }
    if (trace) cudaEventRecord(ev[2], st);
    tridiag_tail(ctx, d, e, n, nwant, nwant, values, X, wkinv);
    if (trace) cudaEventRecord(ev[3], st);
    const size_t wy_smem = size_t(n) * kWYV * sizeof(double);
    if (wy_smem + 32 * 1024 <= cap && std::getenv("ATK_BACKTR_WARP") == nullptr) {
        static bool wattr = false;
        if (!wattr) {
            ATK_CUDA(cudaFuncSetAttribute(backtr_wy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(cap - 32 * 1024)));
            wattr = true;
        }
        const int nblk = (n - 2 + kWYB - 1) / kWYB;
        DevBuf<double> tb(ctx, size_t(nblk) * kWYB * kWYB);
        larft_kernel<<<unsigned(nblk), kWYT, 0, st>>>(hh, tau, n, tb.get());
        ATK_LAUNCHED(ctx);
        backtr_wy_kernel<<<unsigned((nwant + kWYV - 1) / kWYV), kWYT, wy_smem, st>>>(hh, tb.get(), n, nblk, X, nwant,
                                                                                     vectors, ldv);
        ATK_LAUNCHED(ctx);
    } else {
        static bool battr = false;
        if (!battr) {
            ATK_CUDA(cudaFuncSetAttribute(backtr_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(size_t(kBKW) * kBigEigMax * sizeof(double))));
            battr = true;
        }
        backtr_big_kernel<<<unsigned((nwant + kBKW - 1) / kBKW), kBKW * 32, size_t(kBKW) * n * sizeof(double),
                            st>>>(hh, tau, n, X, nwant, vectors, ldv);
        ATK_LAUNCHED(ctx);
    }
    if (trace) cudaEventRecord(ev[4], st);
    unsigned abort_word = 0;
    ATK_CUDA(cudaMemcpyAsync(&abort_word, sync.get() + 2, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    ATK_CUDA(cudaStreamSynchronize(st));
    if (prof) {
        long long h[5];
        ATK_CUDA(cudaMemcpy(h, prof, sizeof(h), cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "[trd n=%d] CTA0 cycles/step: A %.0f B %.0f C %.0f D %.0f barrier %.0f\n", n,
                     h[0] / double(n - 2), h[1] / double(n - 2), h[2] / double(n - 2), h[3] / double(n - 2),
                     h[4] / double(n - 2));
    }
    if (trace) {
        float ms[4];
        for (int q = 0; q < 4; ++q) cudaEventElapsedTime(&ms[q], ev[q], ev[q + 1]);
        std::fprintf(stderr,
                     "[atk dense eig n=%d r=%d] trd grid %.3f ms (%d steps, %d smem slots/SM) cluster %.3f ms (%d steps) "
                     "bisect+invit %.3f ms backtr %.3f ms\n",
                     n, nwant, ms[0], std::max(ks, 0), nslots, ms[1], L > 0 ? n - 2 - std::max(ks, 0) : 0, ms[2],
                     ms[3]);
        for (auto& x : ev) cudaEventDestroy(x);
    }
    if (abort_word) fail(ATK_CUDA_ERROR, "dense_eig_big: grid synchronisation timed out (grid not co-resident)");
}

}  // namespace atk
