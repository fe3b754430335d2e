// dgemm.cu — fp64 GEMM for the eigensolver / ALS small dense algebra.
//
// C(m x n) = alpha op(A) op(B) + beta C, column-major.  128x64 block tile,
// 8-deep K slices in a 4-stage cp.async ring in shared memory, 8 warps each owning a
// 32x32 block computed on the fp64 tensor cores (DMMA m8n8k4, dmma.cuh), and a
// deterministic split-K (fixed-order fp64 partial sums) so that the skinny
// shapes of Chebyshev filtering (2048 x 96 x 2048) still fill all 148 SMs.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "atk_internal.cuh"
#include "dmma.cuh"

namespace atk {
namespace {

constexpr int BM = 128, BN = 64, BK = 8, NT = 256, STAGES = 4;
constexpr int LDA = BM + 4, LDB = BN + 4;   // = 4 (mod 16): conflict-free fragments
constexpr int WM = 4, FM = 4, FN = 4;       // 8 warps: 4 x 2, each 32 x 32
constexpr int STAGE_DOUBLES = BK * (LDA + LDB);
constexpr size_t SMEM_BYTES = size_t(STAGES) * STAGE_DOUBLES * sizeof(double);
// Column-tile variants: BN_ = 16 FN_ (2 warps along N), so an 80- or 96-column
// right operand (the ChFSI blocks) is one tile instead of 64 + a mostly empty one.
template <int FN_>
struct Tile {
    static constexpr int BN_ = 16 * FN_, LDB_ = BN_ + 4;  // = 4 (mod 16)
    static constexpr int STAGE = BK * (LDA + LDB_);
    static constexpr size_t SMEM = size_t(STAGES) * STAGE * sizeof(double);
};

// 8-byte global -> shared async copy; src_bytes = 0 zero-fills (out-of-range).
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// K slices stream through a STAGES-deep cp.async ring (global latency hidden
// behind the DMMA work of the slices already resident; one barrier per slice).
// acc = op(A)[m0:m0+BM, kb:ke] x op(B)[kb:ke, n0:n0+BN]
template <int FN_ = FN>
__device__ __forceinline__ void gemm_block(bool ta, bool tb, int m, int n, int m0, int n0, int kb, int ke,
                                           const double* __restrict__ a, int lda, const double* __restrict__ b,
                                           int ldb, double* dsm, dmma::Acc<FM, FN_>& acc) {
    constexpr int BN_ = Tile<FN_>::BN_, LDB_ = Tile<FN_>::LDB_, STAGE_ = Tile<FN_>::STAGE;
    const int tid = threadIdx.x;
    dmma::zero(acc);
    auto issue = [&](int stage, int k0) {
        double* As = dsm + stage * STAGE_;
        double* Bs = As + BK * LDA;
#pragma unroll
        for (int e = tid; e < BK * BM; e += NT) {
            int kk, mm;
            if (!ta) { mm = e % BM; kk = e / BM; } else { kk = e % BK; mm = e / BK; }
            const int gm = m0 + mm, gk = k0 + kk;
            const bool ok = gm < m && gk < ke;
            cp_async8(As + kk * LDA + mm, ok ? (ta ? a + gk + size_t(lda) * gm : a + gm + size_t(lda) * gk) : a, ok);
        }
#pragma unroll
        for (int e = tid; e < BK * BN_; e += NT) {
            int kk, nn;
            if (tb) { nn = e % BN_; kk = e / BN_; } else { kk = e % BK; nn = e / BK; }
            const int gn = n0 + nn, gk = k0 + kk;
            const bool ok = gn < n && gk < ke;
            cp_async8(Bs + kk * LDB_ + nn, ok ? (tb ? b + gn + size_t(ldb) * gk : b + gk + size_t(ldb) * gn) : b, ok);
        }
    };
    const int nt = (ke > kb) ? (ke - kb + BK - 1) / BK : 0;
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nt) issue(s, kb + s * BK);
        cp_async_commit();
    }
    for (int t = 0; t < nt; ++t) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();  // slice t landed for every thread; slice t-1's buffer is free
        const int tn = t + STAGES - 1;
        if (tn < nt) issue(tn % STAGES, kb + tn * BK);
        cp_async_commit();
        const double* As = dsm + (t % STAGES) * STAGE_;
        dmma::tile_step<LDA, LDB_, WM, FM, FN_>(acc, As, As + BK * LDA, BK);
    }
    cp_async_wait<0>();
    __syncthreads();  // the ring may be refilled by the next call
}

template <int FN_>
__global__ void __launch_bounds__(NT) dgemm_tile(bool ta, bool tb, int m, int n, int k, int kchunk,
                                                 const double* __restrict__ a, int lda,
                                                 const double* __restrict__ b, int ldb,
                                                 double* __restrict__ out, size_t out_split_stride,
                                                 int ldo, double alpha, double beta, bool direct,
                                                 bool tout = false) {
    extern __shared__ __align__(16) double dsm[];
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * Tile<FN_>::BN_;
    const int kb = blockIdx.z * kchunk, ke = min(k, kb + kchunk);
    dmma::Acc<FM, FN_> acc;
    gemm_block<FN_>(ta, tb, m, n, m0, n0, kb, ke, a, lda, b, ldb, dsm, acc);
    double* o = out + size_t(blockIdx.z) * out_split_stride;
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN_; ++j)
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int gm = m0 + dmma::row_of<WM, FM>(i), gn = n0 + dmma::col_of<WM, FN_>(j, t);
                if (gm < m && gn < n) {
                    double* cp = tout ? o + gn + size_t(ldo) * gm : o + gm + size_t(ldo) * gn;  // tout: C^T stored
                    const double v = acc.v[i][j][t];
                    if (direct) *cp = alpha * v + (beta == 0.0 ? 0.0 : beta * *cp);
                    else *cp = v;
                }
            }
}

// ------------------------------------------------------------------ Chebyshev filter
// The whole degree-d three-term recurrence of ChFSI in ONE cooperative launch
// (eig.cu): per step every CTA computes a split-K partial of S Y_j on DMMA,
// a grid barrier, then all CTAs combine Y_{j+1} = a (sum of partials) +
// b Y_j + c Y_{j-1} in a fixed order (deterministic), a second barrier.  S
// (n x n fp64) and the n x k blocks stay L2-resident across steps; the
// per-step cost is the DMMA work spread over ~all SMs plus two grid barriers,
// instead of three launches (combine, GEMM, split-K reduce) per step.
struct ChebArgs {
    const double* S;
    int n, k, deg;
    double* y[4];        // y[0] = V (read-only start), y[1..3] rotating buffers
    double* part;        // splits x n x k
    unsigned* bar;       // [0] count, [1] generation
    int gm, gn, splits, kchunk;
    double a1, b1;       // step 1: Y1 = a1 S V + b1 V
    double a, b, c;      // step j: Y_{j+1} = a S Y_j + b Y_j + c Y_{j-1}
};

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == nblocks - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) __nanosleep(40);
        }
        __threadfence();
    }
    __syncthreads();
}

// Grid barrier with release/acquire atomics instead of full fences: the
// arrival is atom.add.acq_rel (publishes this CTA's writes, ordered before it
// by bar.sync; the last arriver also acquires everyone else's), waiters poll
// the generation word with ld.acquire and no back-off.
__device__ __forceinline__ void grid_barrier_ra(unsigned* bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g, old;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
        if (old == nblocks - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
        } else {
            unsigned cur;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
            } while (cur == g);
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(NT) cheb_filter_kernel(const ChebArgs p) {
    extern __shared__ __align__(16) double dsm[];
    const int ntile = p.gm * p.gn;
    const int tile = blockIdx.x % ntile, split = blockIdx.x / ntile;
    const bool worker = blockIdx.x < unsigned(ntile * p.splits);
    const int m0 = (tile % p.gm) * BM, n0 = (tile / p.gm) * BN;
    const int kb = split * p.kchunk, ke = min(p.n, kb + p.kchunk);
    const size_t nk = size_t(p.n) * p.k;
    int iprev = 0, icur = 0, inext = 1;  // step 1 reads V (y[0])
    for (int step = 0; step < p.deg; ++step) {
        const double* ycur = p.y[icur];
        if (worker) {
            dmma::Acc<FM, FN> acc;
            gemm_block(false, false, p.n, p.k, m0, n0, kb, ke, p.S, p.n, ycur, p.n, dsm, acc);
            double* o = p.part + size_t(split) * nk;
#pragma unroll
            for (int i = 0; i < FM; ++i)
#pragma unroll
                for (int j = 0; j < FN; ++j)
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        const int gm = m0 + dmma::row_of<WM, FM>(i), gn = n0 + dmma::col_of<WM, FN>(j, t);
                        if (gm < p.n && gn < p.k) o[gm + size_t(p.n) * gn] = acc.v[i][j][t];
                    }
        }
        grid_barrier(p.bar, gridDim.x);
        const double a = step == 0 ? p.a1 : p.a, b = step == 0 ? p.b1 : p.b, c = step == 0 ? 0.0 : p.c;
        const double* yprev = p.y[iprev];
        double* ynext = p.y[inext];
        for (size_t e = size_t(blockIdx.x) * NT + threadIdx.x; e < nk; e += size_t(gridDim.x) * NT) {
            double s = 0.0;
            for (int z = 0; z < p.splits; ++z) s += p.part[size_t(z) * nk + e];
            double v = fma(a, s, b * ycur[e]);
            if (c != 0.0) v = fma(c, yprev[e], v);
            ynext[e] = v;
        }
        grid_barrier(p.bar, gridDim.x);
        // rotation as in eig.cu's host loop: yprev <- ycur, ycur <- ynext, ynext <- a free
        // buffer (never V = y[0], which the recurrence only reads)
        if (step == 0) {
            iprev = 0; icur = 1; inext = 2;
        } else {
            const int spare = (iprev == 0) ? 3 : iprev;
            iprev = icur; icur = inext; inext = spare;
        }
    }
}

// ------------------------------------------------------------------ resident-S Chebyshev filter
// Variant for n <= ~1150 (the flat-spectrum ChFSI blocks): S is split into
// strips of `rows` rows, one 8-CTA cluster per strip, CTA r of a cluster
// holding the strip's K range [r kc, (r+1) kc) of S in shared memory for the
// WHOLE filter (S symmetric: the strip's rows are read as contiguous columns).
// The strip height is 8 ceil(n / (8 x co-resident clusters)) (B200: 15 8-CTA
// clusters, so 72 rows at n = 1024).  Per step a CTA streams only its K slice
// of Y_j (cp.async.cg, L2), forms the rows x k split-K partial on DMMA, the
// cluster reduces the 8 partials through DSMEM in a fixed order (CTA r
// finishes rows [r rows/8, (r+1) rows/8) of the strip, applies the three-term
// recurrence and stores Y_{j+1}), and ONE grid barrier publishes Y_{j+1}.
// cheb_filter_kernel re-streams all of S from L2 every step and pays two grid
// barriers per step.
constexpr int RS_CS = 8;   // CTAs per cluster (= K splits)
constexpr int RS_EPT = 4;  // output elements per thread in the cluster reduction

struct ChebResArgs {
    const double* S;
    int n, k, deg, kc, ldk;  // kc = K slice per CTA, ldk = kc + 4 (= 4 mod 16)
    int rows, wm;            // strip rows (8 MF), warps along M (MF = wm FM)
    int ncols;               // padded block width (8 NF, NF = wn FN)
    double* y[4];
    unsigned* bar;
    unsigned* ready;         // per-CTA count of Y steps written (dataflow mode), or null: grid barrier
    double a1, b1, a, b, c;
};

__device__ __forceinline__ void cp_async16_cg(void* dst, const void* src, bool valid) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0) : "memory");
}

// warp tile FM x FN 8x8 fragments; warps (wm, wn) = (warp % p.wm, warp / p.wm)
template <int FM, int FN>
__global__ void __launch_bounds__(512) cheb_resident_kernel(const ChebResArgs p) {
    extern __shared__ __align__(16) double rsm[];
    const int ldk = p.ldk, kc = p.kc, n = p.n, k = p.k, rows = p.rows, ncols = p.ncols;
    double* At = rsm;                  // rows x ldk:  S(m0 + m, kb + kk)
    double* Bt = At + rows * ldk;      // ncols x ldk: Y(kb + kk, c)
    double* Pbuf = Bt + ncols * ldk;   // [2] ncols x rows partials, P[c * rows + m] (by step parity)
    const uint32_t rank = blockIdx.x % RS_CS;
    const int strip = blockIdx.x / RS_CS;
    const int m0 = strip * rows, kb = int(rank) * kc;
    const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31;
    const int hk = kc / 2;
    // S strip slice, once: row m of the strip = column m0 + m of S, contiguous in kk
    for (int e = tid; e < rows * hk; e += nt) {
        const int m = e / hk, kk = 2 * (e % hk);
        const int gm = m0 + m, gk = kb + kk;
        const bool ok = gm < n && gk < n;  // n even (host check): a 16-byte pair is all-in or all-out
        cp_async16_cg(At + m * ldk + kk, ok ? p.S + gk + size_t(n) * gm : p.S, ok);
    }
    cp_async_commit();
    const int wm = warp % p.wm, wn = warp / p.wm;
    const int fr = lane >> 2, fk = lane & 3;
    const int mr = rows / RS_CS;  // rows this CTA finishes
    int iprev = 0, icur = 0, inext = 1;
    // dataflow mode: the CTAs that write rows [kb, kb + kc) of Y (a contiguous
    // id range: row g is finished by CTA (g / rows) * 8 + (g % rows) / mr)
    const int kend = min(n, kb + kc);
    const int prod0 = kb < n ? (kb / rows) * RS_CS + (kb % rows) / mr : 0;
    const int prod1 = kb < n ? ((kend - 1) / rows) * RS_CS + ((kend - 1) % rows) / mr : -1;
    for (int step = 0; step < p.deg; ++step) {
        const double* ycur = step == 0 ? p.y[0] : p.y[icur];
        double* P = Pbuf + size_t(step & 1) * ncols * rows;
        if (p.ready && step > 0) {
            // wait for the producers of this CTA's K slice of Y_step (release/acquire
            // counters); the cluster barrier below then orders this step after every
            // CTA's step - 1 (the union of the cluster's slices is all of Y), which
            // is what the buffer rotation and the partial double-buffer rely on
            if (warp == 0)
                for (int q = prod0 + lane; q <= prod1; q += 32) {
                    unsigned v;
                    do {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.ready + q) : "memory");
                    } while (v < unsigned(step));
                }
            __syncthreads();
        }
        for (int e = tid; e < ncols * hk; e += nt) {
            const int cc = e / hk, kk = 2 * (e % hk);
            const int gk = kb + kk;
            const bool ok = cc < k && gk < n;
            cp_async16_cg(Bt + cc * ldk + kk, ok ? ycur + gk + size_t(n) * cc : ycur, ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        double acc[FM][FN][2];
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
            for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        const double* ap = At + (wm * FM * 8 + fr) * ldk + fk;
        const double* bp = Bt + (wn * FN * 8 + fr) * ldk + fk;
#pragma unroll 4
        for (int kk = 0; kk < kc; kk += 4) {
            double a[FM], bb[FN];
#pragma unroll
            for (int i = 0; i < FM; ++i) a[i] = ap[i * 8 * ldk + kk];
#pragma unroll
            for (int j = 0; j < FN; ++j) bb[j] = bp[j * 8 * ldk + kk];
#pragma unroll
            for (int i = 0; i < FM; ++i)
#pragma unroll
                for (int j = 0; j < FN; ++j) dmma::mma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
        }
        // accumulator (i, j, t): row (wm FM + i) 8 + fr, column (wn FN + j) 8 + 2 fk + t
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
            for (int j = 0; j < FN; ++j)
#pragma unroll
                for (int t = 0; t < 2; ++t)
                    P[((wn * FN + j) * 8 + 2 * fk + t) * rows + (wm * FM + i) * 8 + fr] = acc[i][j][t];
        const double ca = step == 0 ? p.a1 : p.a, cb = step == 0 ? p.b1 : p.b, ccoef = step == 0 ? 0.0 : p.c;
        const double* yprev = p.y[iprev];
        double* ynext = p.y[inext];
        const uint32_t pbase = static_cast<uint32_t>(__cvta_generic_to_shared(P));
        // this thread's (up to RS_EPT) output elements; their Y_j / Y_{j-1}
        // terms are loaded before the cluster barrier so the L2 latency hides
        // behind it
        double base[RS_EPT];
        int off[RS_EPT];  // P offset (cc * rows + m), or -1
#pragma unroll
        for (int u = 0; u < RS_EPT; ++u) {
            const int e = tid + u * nt;
            off[u] = -1;
            base[u] = 0.0;
            if (e < mr * k) {
                const int m = int(rank) * mr + e % mr, cc = e / mr;
                if (m0 + m < n) {
                    const size_t g = (m0 + m) + size_t(n) * cc;
                    off[u] = cc * rows + m;
                    base[u] = cb * __ldcg(ycur + g);
                    if (ccoef != 0.0) base[u] = fma(ccoef, __ldcg(yprev + g), base[u]);
                }
            }
        }
        // every CTA of the cluster has its partial in smem
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        double v[RS_EPT][RS_CS];
#pragma unroll
        for (int u = 0; u < RS_EPT; ++u)
#pragma unroll
            for (int z = 0; z < RS_CS; ++z) {
                v[u][z] = 0.0;
                if (off[u] >= 0) {
                    uint32_t ra;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                                 : "=r"(ra)
                                 : "r"(pbase + uint32_t(off[u]) * 8u), "r"(uint32_t(z)));
                    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v[u][z]) : "r"(ra) : "memory");
                }
            }
#pragma unroll
        for (int u = 0; u < RS_EPT; ++u) {
            if (off[u] < 0) continue;
            double sum = 0.0;
#pragma unroll
            for (int z = 0; z < RS_CS; ++z) sum += v[u][z];  // split order: deterministic
            const int m = off[u] % rows, cc = off[u] / rows;
            ynext[(m0 + m) + size_t(n) * cc] = fma(ca, sum, base[u]);
        }
        if (p.ready) {
            // publish: this CTA's rows of Y_{step+1} are written
            __syncthreads();
            if (tid == 0)
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.ready + blockIdx.x), "r"(unsigned(step + 1))
                             : "memory");
        } else {
            // Y_{j+1} complete everywhere (also frees P and Bt for the next step)
            grid_barrier_ra(p.bar, gridDim.x);
        }
        if (step == 0) {
            iprev = 0; icur = 1; inext = 2;
        } else {
            const int spare = (iprev == 0) ? 3 : iprev;
            iprev = icur; icur = inext; inext = spare;
        }
    }
    // no CTA may exit while a cluster peer can still read its partials through
    // DSMEM (dataflow mode has no closing grid barrier)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Small outputs: G lanes per element (G | 32), lane t sums splits t, t+G, ...
// in order, then a fixed xor tree over the G lanes (deterministic).  The
// one-thread-per-element loop is a chain of `splits` L2 round trips.
__global__ void dgemm_splitk_reduce_g(const double* __restrict__ part, int splits, int m, int n, int G,
                                      double alpha, double beta, double* __restrict__ c, int ldc) {
    const size_t mn = size_t(m) * n;
    const size_t gid = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t e = gid / G;
    const int t = int(gid % G);
    double s = 0.0;
    if (e < mn)
        for (int z = t; z < splits; z += G) s += part[size_t(z) * mn + e];
    for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (e < mn && t == 0) {
        const int i = int(e % m), j = int(e / m);
        double* cp = c + i + size_t(ldc) * j;
        *cp = alpha * s + (beta == 0.0 ? 0.0 : beta * *cp);
    }
}

__global__ void dgemm_splitk_reduce(const double* __restrict__ part, int splits, int m, int n,
                                    double alpha, double beta, double* __restrict__ c, int ldc) {
    const size_t mn = size_t(m) * n;
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < mn; e += size_t(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int z = 0; z < splits; ++z) s += part[size_t(z) * mn + e];
        const int i = int(e % m), j = int(e / m);
        double* cp = c + i + size_t(ldc) * j;
        *cp = alpha * s + (beta == 0.0 ? 0.0 : beta * *cp);
    }
}

}  // namespace

namespace {

template <int FN_>
void dgemm_launch(atk_ctx* ctx, bool ta, bool tb, int m, int n, int k, double alpha, const double* a, int lda,
                  const double* b, int ldb, double beta, double* c, int ldc) {
    constexpr int BN_ = Tile<FN_>::BN_;
    constexpr size_t SMEM_ = Tile<FN_>::SMEM;
    static bool attr = false;
    if (!attr) {
        ATK_CUDA(cudaFuncSetAttribute(dgemm_tile<FN_>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_)));
        attr = true;
    }
    const int gm = (m + BM - 1) / BM, gn = (n + BN_ - 1) / BN_;
    const int tiles = gm * gn;
    int splits = 1;
    // up to 4 resident CTAs per SM (51-59 KB smem each)
    // K chunks of >= 32 (4 slices): the skinny ChFSI GEMMs (k x k over n, n x k x k) were
    // latency-bound on 8-16 CTAs with 128-deep chunks (C2: 1.60 -> 1.00 ms of dgemm per step,
    // with the lane-parallel split-K reduction below); ATK_DGEMM_MIN_CHUNK is a probe knob
    static const int min_chunk = std::getenv("ATK_DGEMM_MIN_CHUNK") ? std::atoi(std::getenv("ATK_DGEMM_MIN_CHUNK")) : 32;
    // (one wave of one CTA per SM for the deep-K ChFSI S-products, 9 splits instead of 37, measured
    // r2: DMMA part +19 us, reduction -13 us per eigensolve: not kept)
    if (tiles < 4 * ctx->num_sms && k >= 2 * min_chunk)
        splits = std::min(std::max(1, (4 * ctx->num_sms + tiles - 1) / tiles), std::max(1, k / min_chunk));
    int kchunk = (k + splits - 1) / splits;
    kchunk = (kchunk + BK - 1) / BK * BK;
    splits = std::max(1, (k + kchunk - 1) / std::max(1, kchunk));
    if (k <= 0) {
        kchunk = 0;
        splits = 1;
    }
    if (splits == 1) {
        dim3 grid{unsigned(gm), unsigned(gn), 1u};
        dgemm_tile<FN_><<<grid, NT, SMEM_, ctx->stream>>>(ta, tb, m, n, std::max(k, 0), std::max(kchunk, BK), a, lda,
                                                          b, ldb, c, 0, ldc, alpha, beta, true);
        ATK_LAUNCHED(ctx);
        return;
    }
    DevBuf<double> part(ctx, size_t(splits) * m * n);
    dim3 grid{unsigned(gm), unsigned(gn), unsigned(splits)};
    dgemm_tile<FN_><<<grid, NT, SMEM_, ctx->stream>>>(ta, tb, m, n, k, kchunk, a, lda, b, ldb, part.get(),
                                                      size_t(m) * n, m, 1.0, 0.0, false);
    ATK_LAUNCHED(ctx);
    const size_t mn = size_t(m) * n;
    // lanes per element: enough threads to cover ~8 waves' worth, at most 32
    int G = 1;
    while (G < 32 && G < splits && mn * size_t(G) < size_t(ctx->num_sms) * 2048) G <<= 1;
    if (G > 1) {
        const size_t threads = mn * size_t(G);
        dgemm_splitk_reduce_g<<<unsigned((threads + 255) / 256), 256, 0, ctx->stream>>>(part.get(), splits, m, n, G,
                                                                                      alpha, beta, c, ldc);
    } else {
        dgemm_splitk_reduce<<<unsigned(std::min<size_t>((mn + 255) / 256, size_t(ctx->num_sms) * 8)), 256, 0,
                              ctx->stream>>>(part.get(), splits, m, n, alpha, beta, c, ldc);
    }
    ATK_LAUNCHED(ctx);
}

}  // namespace

// ------------------------------------------------------------------ SYRK
// The fp64 first / last-mode Gram (kernels.hpp:127-138, the unfolding is a
// plain column-major matrix) as a SYRK: C = op(A) op(A)^T, n <= 160.  A K-slice
// of the n-row panel is staged ONCE in shared memory (cp.async ring) and serves
// as both operands.  The upper 32 x 32 blocks (nb = ceil(n / 32), U = nb (nb + 1)
// / 2 of them) go ONE per warp (U warps, a 4 x 4 grid of DMMA m8n8k4 fragments
// each: 16 independent accumulation chains), so no warp waits on another's
// second block.
// Split-K over CTAs, fixed-order partial sums; the reduction writes both
// triangles.  At n = 128 (C3 mode 0): 10 of the 16 blocks a GEMM computes,
// from half the staged bytes.
constexpr int kSyBK = 16, kSyStages = 4, kSyMaxN = 160;  // 2U <= 30 warps

// FN: 8-column DMMA fragments per warp (2: a 32 x 16 half-block, 4: a whole 32 x 32 block)
template <int FN>
__global__ void __launch_bounds__(FN == 4 ? 512 : 1024) syrk_panel_kernel(bool ta, int n, int k, int kchunk,
                                                          const double* __restrict__ a, int lda,
                                                          double* __restrict__ part) {
    constexpr int HB = 4 / FN;  // warps per 32 x 32 block
    extern __shared__ __align__(16) double ps[];
    const int nb = (n + 31) / 32;
    const int ldp = nb * 32 + 4;  // = 4 (mod 16): conflict-free fragment loads
    const int stage = kSyBK * ldp;
    const int tid = threadIdx.x, nt_ = blockDim.x, warp = tid >> 5, lane = tid & 31;
    const int r = lane & 3, c = lane >> 2;
    const int kb = blockIdx.x * kchunk, ke = min(k, kb + kchunk);
    // warp -> (row block, column block, part), row-major over the upper blocks
    int rb = 0, cb = 0;
    {
        int t = warp / HB;
        for (int i = 0; i < nb; ++i) {
            if (t < nb - i) {
                rb = i;
                cb = i + t;
                break;
            }
            t -= nb - i;
        }
    }
    const int c0 = cb * 32 + (warp % HB) * (8 * FN);
    double acc[4][FN][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    auto issue = [&](int st, int k0) {
        double* P = ps + st * stage;
        for (int e = tid; e < kSyBK * n; e += nt_) {
            int kk, mm;
            if (!ta) { mm = e % n; kk = e / n; } else { kk = e % kSyBK; mm = e / kSyBK; }
            const int gk = k0 + kk;
            const bool ok = gk < ke;
            cp_async8(P + kk * ldp + mm, ok ? (ta ? a + gk + size_t(lda) * mm : a + mm + size_t(lda) * gk) : a, ok);
        }
    };
    const int nt = (ke > kb) ? (ke - kb + kSyBK - 1) / kSyBK : 0;
    // rows n .. 32 nb - 1 of every stage stay 0
    for (int e = tid; e < kSyStages * stage; e += nt_)
        if ((e % ldp) >= n) ps[e] = 0.0;
#pragma unroll
    for (int s = 0; s < kSyStages - 1; ++s) {
        if (s < nt) issue(s, kb + s * kSyBK);
        cp_async_commit();
    }
    const int aoff = r * ldp + rb * 32 + c, boff = r * ldp + c0 + c;
    for (int t = 0; t < nt; ++t) {
        cp_async_wait<kSyStages - 2>();
        __syncthreads();
        const int tn = t + kSyStages - 1;
        if (tn < nt) issue(tn % kSyStages, kb + tn * kSyBK);
        cp_async_commit();
        const double* P = ps + (t % kSyStages) * stage;
#pragma unroll
        for (int kk = 0; kk < kSyBK; kk += 4) {
            double av[4], bv[FN];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = P[aoff + kk * ldp + i * 8];
#pragma unroll
            for (int j = 0; j < FN; ++j) bv[j] = P[boff + kk * ldp + j * 8];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < FN; ++j) dmma::mma_8x8x4(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
        }
    }
    cp_async_wait<0>();
    double* o = part + size_t(blockIdx.x) * size_t(n) * n;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j)
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int gm = rb * 32 + i * 8 + c, gn = c0 + j * 8 + 2 * r + t;
                if (gm < n && gn < n) o[gm + size_t(n) * gn] = acc[i][j][t];
            }
}

// C(i, j) = C(j, i) = alpha sum_z part[z](min, max): the upper triangle of the partials,
// summed in split order, written to both triangles
__global__ void syrk_reduce_kernel(const double* __restrict__ part, int splits, int n, double alpha,
                                   double* __restrict__ cout, int ldc) {
    const size_t tot = size_t(n) * n;
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += size_t(gridDim.x) * blockDim.x) {
        const int i = int(e % n), j = int(e / n);
        const int u = min(i, j), v = max(i, j);
        const size_t off = u + size_t(n) * v;
        double sum = 0.0;
        for (int z = 0; z < splits; ++z) sum += part[size_t(z) * tot + off];
        cout[i + size_t(ldc) * j] = alpha * sum;
    }
}

void dsyrk_upper(atk_ctx* ctx, bool ta, int n, int k, double alpha, const double* a, int lda, double* c, int ldc) {
    if (n <= 0) return;
    if (n > kSyMaxN) fail(ATK_UNSUPPORTED, "dsyrk_upper: n > 160");
    // one whole 32 x 32 block per warp (16 independent DMMA chains: C3 mode 0 2.09 -> 1.62 ms against
    // 32 x 16 halves on twice the warps); ATK_SYRK_HALF: the half-block variant (probe knob)
    static const bool full = std::getenv("ATK_SYRK_HALF") == nullptr;
    const int nb = (n + 31) / 32, warps = full ? nb * (nb + 1) / 2 : nb * (nb + 1);
    const size_t smem = size_t(kSyStages) * kSyBK * (nb * 32 + 4) * sizeof(double);
    static bool attr = false;
    if (!attr) {
        ATK_CUDA(cudaFuncSetAttribute(syrk_panel_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(size_t(kSyStages) * kSyBK * (kSyMaxN + 4) * sizeof(double))));
        ATK_CUDA(cudaFuncSetAttribute(syrk_panel_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(size_t(kSyStages) * kSyBK * (kSyMaxN + 4) * sizeof(double))));
        attr = true;
    }
    // one or two CTAs per SM, K chunks of >= 256
    int splits = std::max(1, std::min(2 * ctx->num_sms, (k + 255) / 256));
    int kchunk = (k + splits - 1) / splits;
    kchunk = (kchunk + kSyBK - 1) / kSyBK * kSyBK;
    splits = std::max(1, (k + kchunk - 1) / kchunk);
    DevBuf<double> part(ctx, size_t(splits) * n * n);
    if (full) syrk_panel_kernel<4><<<splits, 32 * warps, smem, ctx->stream>>>(ta, n, k, kchunk, a, lda, part.get());
    else syrk_panel_kernel<2><<<splits, 32 * warps, smem, ctx->stream>>>(ta, n, k, kchunk, a, lda, part.get());
    ATK_LAUNCHED(ctx);
    syrk_reduce_kernel<<<unsigned(std::min<size_t>((size_t(n) * n + 255) / 256, size_t(ctx->num_sms) * 8)), 256, 0,
                         ctx->stream>>>(part.get(), splits, n, alpha, c, ldc);
    ATK_LAUNCHED(ctx);
}

// C = op(A) op(B) for the fp64 first / last-mode TTM (kernels.hpp:88-118; the unfolding is a
// plain column-major matrix): m = the long dimension (J or P), n = R <= 64, k = I, one pass over
// A through the cp.async ring with a column tile of 16 ceil(R / 16), no split-K (m fills the
// GPU).  tout: C^T is stored (c[j + ldc i]), the mode-0 output layout (R x J).
void dgemm_ttm(atk_ctx* ctx, bool ta, bool tb, int m, int n, int k, const double* a, int lda, const double* b,
               int ldb, double* c, int ldc, bool tout) {
    if (m <= 0 || n <= 0) return;
    if (n > 64) fail(ATK_UNSUPPORTED, "dgemm_ttm: n > 64");
    auto go = [&](auto fnc) {
        constexpr int FN_ = decltype(fnc)::value;
        static bool attr = false;
        if (!attr) {
            ATK_CUDA(cudaFuncSetAttribute(dgemm_tile<FN_>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(Tile<FN_>::SMEM)));
            attr = true;
        }
        dim3 grid{unsigned((m + BM - 1) / BM), unsigned((n + Tile<FN_>::BN_ - 1) / Tile<FN_>::BN_), 1u};
        dgemm_tile<FN_><<<grid, NT, Tile<FN_>::SMEM, ctx->stream>>>(ta, tb, m, n, std::max(k, 0), std::max(k, BK), a,
                                                                    lda, b, ldb, c, 0, ldc, 1.0, 0.0, true, tout);
        ATK_LAUNCHED(ctx);
    };
    if (n <= 16) go(std::integral_constant<int, 1>{});
    else if (n <= 32) go(std::integral_constant<int, 2>{});
    else if (n <= 48) go(std::integral_constant<int, 3>{});
    else go(std::integral_constant<int, 4>{});
}

void dgemm(atk_ctx* ctx, bool ta, bool tb, int m, int n, int k, double alpha, const double* a, int lda,
           const double* b, int ldb, double beta, double* c, int ldc) {
    if (m <= 0 || n <= 0) return;
    // one column tile for the ChFSI block widths (n = 65..96) instead of 64 + a mostly empty one
    if (n > 64 && n <= 80) dgemm_launch<5>(ctx, ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc);
    else if (n > 80 && n <= 96) dgemm_launch<6>(ctx, ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc);
    else dgemm_launch<4>(ctx, ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc);
}

namespace {

template <int FM, int FN>
int cheb_resident_max_clusters() {
    static int max_clusters = -1;
    if (max_clusters < 0) {
        max_clusters = 0;
        if (cudaFuncSetAttribute(cheb_resident_kernel<FM, FN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 200 * 1024) == cudaSuccess) {
            cudaLaunchConfig_t cfg{};
            cudaLaunchAttribute at{};
            at.id = cudaLaunchAttributeClusterDimension;
            at.val.clusterDim.x = RS_CS;
            at.val.clusterDim.y = at.val.clusterDim.z = 1;
            cfg.gridDim = dim3(RS_CS);
            cfg.blockDim = dim3(512);
            cfg.dynamicSmemBytes = 200 * 1024;
            cfg.attrs = &at;
            cfg.numAttrs = 1;
            if (cudaOccupancyMaxActiveClusters(&max_clusters, cheb_resident_kernel<FM, FN>, &cfg) != cudaSuccess)
                max_clusters = 0;
        }
        cudaGetLastError();
    }
    return max_clusters;
}

template <int FM, int FN>
bool cheb_resident_launch(atk_ctx* ctx, ChebResArgs p, int strips, size_t smem, int warps) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[2]{};
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = RS_CS;
    at[0].val.clusterDim.y = at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.gridDim = dim3(unsigned(strips * RS_CS));
    cfg.blockDim = dim3(unsigned(32 * warps));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cfg.attrs = at;
    // ncu cannot replay a cooperative cluster launch (LaunchFailed): under the
    // profiler, ATK_PROFILE_NONCOOP=1 drops the cooperative attribute (the
    // grid is still sized to co-resident clusters, and ncu serialises kernels)
    static const bool noncoop = std::getenv("ATK_PROFILE_NONCOOP") != nullptr;
    cfg.numAttrs = noncoop ? 1 : 2;
    if (const cudaError_t err = cudaLaunchKernelEx(&cfg, cheb_resident_kernel<FM, FN>, p); err != cudaSuccess) {
        cudaGetLastError();  // e.g. cooperative + cluster refused: the split-K kernel instead
        if (std::getenv("ATK_TRACE")) std::fprintf(stderr, "[atk cheb_resident] launch: %s\n", cudaGetErrorString(err));
        return false;
    }
    ATK_LAUNCHED(ctx);
    return true;
}

// Strip height and warp layout for (n, k); false = use cheb_filter_kernel.
bool cheb_resident(atk_ctx* ctx, const double* S, int n, int k, int deg, double* const y[4], double a1, double b1,
                   double a, double b, double c) {
    if (n % 2 != 0 || n < 8 * RS_CS || k < 1 || k > 112) return false;
    const int max_clusters = cheb_resident_max_clusters<3, 2>();  // same resources for every instance
    if (max_clusters < 1) return false;
    int mf = (n + 8 * max_clusters - 1) / (8 * max_clusters);  // 8-row fragments per strip
    if (mf % 2 && mf % 3) ++mf;
    const int fm = (mf % 3 == 0) ? 3 : 2, wm = mf / fm;
    int nf = (k + 7) / 8;
    const int fn = (nf % 3 == 0) ? 3 : 2;
    if (nf % fn) ++nf;
    const int wn = nf / fn, warps = wm * wn;
    const int rows = 8 * mf, strips = (n + rows - 1) / rows;
    if (warps > 16 || strips > max_clusters || rows % RS_CS) return false;
    if ((rows / RS_CS) * k > RS_EPT * 32 * warps) return false;  // reduction: <= RS_EPT elements per thread
    const int kc = ((n + RS_CS - 1) / RS_CS + 3) / 4 * 4;  // K slice per CTA, a multiple of 4
    const int ldk = kc + 4 + (16 - (kc + 4) % 16 + 4) % 16;   // = 4 (mod 16)
    const size_t smem = (size_t(rows) * ldk + size_t(8 * nf) * ldk + size_t(2) * (8 * nf) * rows) * sizeof(double);
    if (std::getenv("ATK_TRACE"))
        std::fprintf(stderr, "[atk cheb_resident n=%d k=%d] clusters %d/%d rows %d warps %dx%d frag %dx%d smem %zu\n",
                     n, k, strips, max_clusters, rows, wm, wn, fm, fn, smem);
    if (smem > 200 * 1024) return false;
    const int ncta = strips * RS_CS;
    DevBuf<unsigned> bar(ctx, 2 + size_t(ncta));
    ATK_CUDA(cudaMemsetAsync(bar.get(), 0, (2 + size_t(ncta)) * sizeof(unsigned), ctx->stream));
    const ChebResArgs p{S,  n,  k,        deg,   kc,    ldk,  rows,
                        wm, 8 * nf,       {y[0], y[1], y[2], y[3]},   bar.get(),
                        ctx->cheb_dataflow ? bar.get() + 2 : nullptr, a1,   b1,   a, b, c};
    if (fm == 3 && fn == 3) return cheb_resident_max_clusters<3, 3>() && cheb_resident_launch<3, 3>(ctx, p, strips, smem, warps);
    if (fm == 3 && fn == 2) return cheb_resident_launch<3, 2>(ctx, p, strips, smem, warps);
    if (fm == 2 && fn == 3) return cheb_resident_max_clusters<2, 3>() && cheb_resident_launch<2, 3>(ctx, p, strips, smem, warps);
    return cheb_resident_max_clusters<2, 2>() && cheb_resident_launch<2, 2>(ctx, p, strips, smem, warps);
}

// final Y_deg sits in the buffer the rotation left as "current"
int cheb_final_buffer(int deg) {
    int iprev = 0, icur = 0, inext = 1;
    for (int step = 0; step < deg; ++step) {
        if (step == 0) {
            iprev = 0; icur = 1; inext = 2;
        } else {
            const int spare = (iprev == 0) ? 3 : iprev;
            iprev = icur; icur = inext; inext = spare;
        }
    }
    return icur;
}

}  // namespace

int cheb_filter(atk_ctx* ctx, const double* S, int n, int k, int deg, double* const y[4], double a1, double b1,
                double a, double b, double c) {
    if (ctx->cheb_fused == 1 && cheb_resident(ctx, S, n, k, deg, y, a1, b1, a, b, c)) return cheb_final_buffer(deg);
    static bool attr = false;
    static int max_blocks = 0;
    if (!attr) {
        ATK_CUDA(cudaFuncSetAttribute(cheb_filter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(SMEM_BYTES)));
        int per_sm = 0;
        ATK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cheb_filter_kernel, NT, SMEM_BYTES));
        max_blocks = per_sm * ctx->num_sms;
        attr = true;
    }
    const int gm = (n + BM - 1) / BM, gn = (k + BN - 1) / BN, tiles = gm * gn;
    // one CTA per SM: split K so tiles x splits fills the SMs (K chunks of >= 64)
    int splits = std::max(1, std::min(ctx->num_sms / tiles, n / 64));
    int kchunk = (n + splits - 1) / splits;
    kchunk = (kchunk + BK - 1) / BK * BK;
    splits = (n + kchunk - 1) / kchunk;
    const int grid = std::max(tiles * splits, std::min(ctx->num_sms, max_blocks));
    if (tiles * splits > max_blocks) return -1;  // caller falls back to per-step launches
    DevBuf<double> part(ctx, size_t(splits) * n * k);
    DevBuf<unsigned> bar(ctx, 2);
    ATK_CUDA(cudaMemsetAsync(bar.get(), 0, 2 * sizeof(unsigned), ctx->stream));
    ChebArgs p{S, n, k, deg, {y[0], y[1], y[2], y[3]}, part.get(), bar.get(), gm, gn, splits, kchunk, a1, b1, a, b, c};
    void* args[] = {&p};
    ATK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(cheb_filter_kernel), dim3(unsigned(grid)), dim3(NT),
                                         args, SMEM_BYTES, ctx->stream));
    ATK_LAUNCHED(ctx);
    return cheb_final_buffer(deg);
}

}  // namespace atk
