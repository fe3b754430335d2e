// contract_simt.cu — general-shape matricization-free contractions.
//
// fp64 storage runs on the fp64 tensor cores (DMMA m8n8k4, dmma.cuh); fp32
// storage shapes the tcgen05 kernels do not cover (P not in {1} u 32N, tiny I,
// R > 128) run on CUDA cores with fp64 accumulation.  Option "simt" forces
// this file for every shape.
//
// Index contract (kernels.hpp:34-118, tensor.hpp:175-187): X viewed as
// (P, I, O), element (p, i, o) at p + P*i + P*I*o.  No unfolding is ever
// materialised: the K index of every contraction is the (p, o) pair walked in
// place by the tile loaders.
#include <algorithm>
#include <type_traits>

#include "atk_internal.cuh"
#include "dmma.cuh"

namespace atk {
namespace {

// (p, o) of the linear index base + off, given (p0, o0) of base: one 32-bit
// division at most (off < 2^31) instead of a 64-bit div/mod per element.
__device__ __forceinline__ void split_po(uint64_t p0, uint64_t o0, uint32_t off, uint64_t P, uint64_t& p,
                                         uint64_t& o) {
    if (P == 1) {  // mode 0: k is the outer index itself
        p = 0;
        o = o0 + off;
        return;
    }
    p = p0 + off;
    o = o0;
    if (p >= P) {
        if (P <= 0xffffffffull && p <= 0xffffffffull) {
            const uint32_t q = uint32_t(p) / uint32_t(P);
            o += q;
            p -= uint64_t(q) * P;
        } else {
            o += p / P;
            p %= P;
        }
    }
}

// LD = 68 = 4 (mod 16): conflict-free DMMA fragment loads (dmma.cuh)
constexpr int TM = 64, TN = 64, KT = 16, NT = 256, LD = TM + 4;
constexpr int WM = 2, FM = 4, FN = 2;  // 8 warps: 2 x 4, each 32 x 16

// Z(I x R) partial over k in [k0, k1) of sum_k X(k, i) Y(k, r), k = (p, o).
template <class T>
__global__ void __launch_bounds__(NT) ttt_tile_kernel(const T* __restrict__ x, const T* __restrict__ y, uint64_t P,
                                                      uint64_t I, uint64_t R, uint64_t K, uint64_t kchunk, bool sym,
                                                      double* __restrict__ part) {
    const int tm = blockIdx.x, tn = blockIdx.y;
    if (sym && tn < tm) return;
    __shared__ double As[KT][LD];
    __shared__ double Bs[KT][LD];
    const uint64_t i0 = uint64_t(tm) * TM, r0 = uint64_t(tn) * TN;
    const uint64_t kb = uint64_t(blockIdx.z) * kchunk;
    const uint64_t ke = min(K, kb + kchunk);
    const int tid = threadIdx.x;
    const int ty = tid / 16, tx = tid % 16;
    double acc[4][4] = {};
    dmma::Acc<FM, FN> dacc;
    dmma::zero(dacc);
    uint64_t tp0 = kb % P, to0 = kb / P;  // (p, o) of the tile's first k, advanced per tile
    for (uint64_t k0 = kb; k0 < ke; k0 += KT) {
        for (int e = tid; e < KT * TM; e += NT) {
            int kk, ii;
            if (P == 1) { ii = e % TM; kk = e / TM; } else { kk = e % KT; ii = e / KT; }
            const uint64_t k = k0 + kk, i = i0 + ii;
            double v = 0.0;
            if (k < ke && i < I) {
                uint64_t p, o;
                split_po(tp0, to0, uint32_t(kk), P, p, o);
                v = double(x[p + P * i + P * I * o]);
            }
            As[kk][ii] = v;
        }
        for (int e = tid; e < KT * TN; e += NT) {
            int kk, rr;
            if (P == 1) { rr = e % TN; kk = e / TN; } else { kk = e % KT; rr = e / KT; }
            const uint64_t k = k0 + kk, r = r0 + rr;
            double v = 0.0;
            if (k < ke && r < R) {
                uint64_t p, o;
                split_po(tp0, to0, uint32_t(kk), P, p, o);
                v = double(y[p + P * r + P * R * o]);
            }
            Bs[kk][rr] = v;
        }
        split_po(tp0, to0, KT, P, tp0, to0);
        __syncthreads();
        if constexpr (std::is_same_v<T, double>) {
            dmma::tile_step<LD, LD, WM, FM, FN>(dacc, &As[0][0], &Bs[0][0], KT);
        } else {
#pragma unroll
            for (int kk = 0; kk < KT; ++kk) {
                double a[4], b[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) a[u] = As[kk][ty + 16 * u];
#pragma unroll
                for (int v = 0; v < 4; ++v) b[v] = Bs[kk][tx + 16 * v];
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
            }
        }
        __syncthreads();
    }
    double* out = part + uint64_t(blockIdx.z) * I * R;
    if constexpr (std::is_same_v<T, double>) {
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
            for (int j = 0; j < FN; ++j)
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const uint64_t ii = i0 + dmma::row_of<WM, FM>(i), rr = r0 + dmma::col_of<WM, FN>(j, t);
                    if (ii < I && rr < R) out[ii + I * rr] = dacc.v[i][j][t];
                }
    } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const uint64_t i = i0 + ty + 16 * u, r = r0 + tx + 16 * v;
                if (i < I && r < R) out[i + I * r] = acc[u][v];
            }
    }
}

// Z = sum_z part[z] in fixed order; for Gram mirror the computed upper
// triangle (i <= r) onto the lower one => exactly symmetric (kernels.hpp:127-138).
__global__ void reduce_partials(const double* __restrict__ part, int nsplit, uint64_t I, uint64_t R, bool sym,
                                double* __restrict__ z) {
    const uint64_t n = I * R;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = e % I, r = e / I;
        uint64_t src = e;
        if (sym && i > r) src = r + I * i;
        double s = 0.0;
        for (int k = 0; k < nsplit; ++k) s += part[uint64_t(k) * n + src];
        z[e] = s;
    }
}

// The same with many splits and few elements (skinny Grams: I x R small, J
// huge): one warp per element, lanes stride the splits, fixed shuffle tree
// (deterministic: the summation order depends only on nsplit).
__global__ void reduce_partials_wide(const double* __restrict__ part, int nsplit, uint64_t I, uint64_t R, bool sym,
                                     double* __restrict__ z) {
    const uint64_t n = I * R;
    const uint64_t e = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (e >= n) return;  // warp-uniform
    const uint64_t i = e % I, r = e / I;
    const uint64_t src = (sym && i > r) ? r + I * i : e;
    double s = 0.0;
    for (int k = lane; k < nsplit; k += 32) s += part[uint64_t(k) * n + src];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) z[e] = s;
}

// Y(m, r) = sum_i X(m, i) U(r, i), m = (p, o).
template <class T>
__global__ void __launch_bounds__(NT) ttm_tile_kernel(const T* __restrict__ x, const double* __restrict__ u, uint64_t P,
                                                      uint64_t I, uint64_t O, uint64_t R, T* __restrict__ y) {
    __shared__ double As[KT][LD];
    __shared__ double Bs[KT][LD];
    const uint64_t M = P * O;
    const uint64_t m0 = uint64_t(blockIdx.x) * TM, r0 = uint64_t(blockIdx.y) * TN;
    const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
    double acc[4][4] = {};
    dmma::Acc<FM, FN> dacc;
    dmma::zero(dacc);
    const uint64_t mp0 = m0 % P, mo0 = m0 / P;  // (p, o) of the tile's first row
    for (uint64_t k0 = 0; k0 < I; k0 += KT) {
        for (int e = tid; e < KT * TM; e += NT) {
            int kk, mm;
            if (P == 1) { kk = e % KT; mm = e / KT; } else { mm = e % TM; kk = e / TM; }
            const uint64_t i = k0 + kk, m = m0 + mm;
            double v = 0.0;
            if (i < I && m < M) {
                uint64_t p, o;
                split_po(mp0, mo0, uint32_t(mm), P, p, o);
                v = double(x[p + P * i + P * I * o]);
            }
            As[kk][mm] = v;
        }
        for (int e = tid; e < KT * TN; e += NT) {
            const int rr = e % TN, kk = e / TN;
            const uint64_t i = k0 + kk, r = r0 + rr;
            Bs[kk][rr] = (i < I && r < R) ? u[r + R * i] : 0.0;
        }
        __syncthreads();
        if constexpr (std::is_same_v<T, double>) {
            dmma::tile_step<LD, LD, WM, FM, FN>(dacc, &As[0][0], &Bs[0][0], KT);
        } else {
#pragma unroll
            for (int kk = 0; kk < KT; ++kk) {
                double a[4], b[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) a[q] = As[kk][ty + 16 * q];
#pragma unroll
                for (int v = 0; v < 4; ++v) b[v] = Bs[kk][tx + 16 * v];
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[q][v] = fma(a[q], b[v], acc[q][v]);
            }
        }
        __syncthreads();
    }
    if constexpr (std::is_same_v<T, double>) {
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
            for (int j = 0; j < FN; ++j)
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const int mm = dmma::row_of<WM, FM>(i);
                    const uint64_t m = m0 + mm, r = r0 + dmma::col_of<WM, FN>(j, t);
                    if (m < M && r < R) {
                        uint64_t p, o;
                        split_po(mp0, mo0, uint32_t(mm), P, p, o);
                        y[p + P * r + P * R * o] = dacc.v[i][j][t];
                    }
                }
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const uint64_t m = m0 + ty + 16 * q, r = r0 + tx + 16 * v;
                if (m < M && r < R) {
                    uint64_t p, o;
                    split_po(mp0, mo0, uint32_t(ty + 16 * q), P, p, o);
                    y[p + P * r + P * R * o] = T(acc[q][v]);
                }
            }
    }
}

// fp64 TTM with the DMMA tile narrowed to R: TN_ = 16 / 32 columns (8 warps
// stacked along M), so R = 16 (C3) no longer pays for 64 DMMA columns.
template <int TN_, int WM_, int FM_, int FN_>
__global__ void __launch_bounds__(NT) ttm_f64_kernel(const double* __restrict__ x, const double* __restrict__ u,
                                                     uint64_t P, uint64_t I, uint64_t O, uint64_t R,
                                                     double* __restrict__ y) {
    constexpr int LDB_ = TN_ + 4;  // = 4 (mod 16)
    __shared__ double As[KT][LD];
    __shared__ double Bs[KT][LDB_];
    const uint64_t M = P * O;
    const uint64_t m0 = uint64_t(blockIdx.x) * TM, r0 = uint64_t(blockIdx.y) * TN_;
    const int tid = threadIdx.x;
    dmma::Acc<FM_, FN_> dacc;
    dmma::zero(dacc);
    const uint64_t mp0 = m0 % P, mo0 = m0 / P;
    for (uint64_t k0 = 0; k0 < I; k0 += KT) {
        for (int e = tid; e < KT * TM; e += NT) {
            int kk, mm;
            if (P == 1) { kk = e % KT; mm = e / KT; } else { mm = e % TM; kk = e / TM; }
            const uint64_t i = k0 + kk, m = m0 + mm;
            double v = 0.0;
            if (i < I && m < M) {
                uint64_t p, o;
                split_po(mp0, mo0, uint32_t(mm), P, p, o);
                v = x[p + P * i + P * I * o];
            }
            As[kk][mm] = v;
        }
        for (int e = tid; e < KT * TN_; e += NT) {
            const int rr = e % TN_, kk = e / TN_;
            const uint64_t i = k0 + kk, r = r0 + rr;
            Bs[kk][rr] = (i < I && r < R) ? u[r + R * i] : 0.0;
        }
        __syncthreads();
        dmma::tile_step<LD, LDB_, WM_, FM_, FN_>(dacc, &As[0][0], &Bs[0][0], KT);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < FM_; ++i)
#pragma unroll
        for (int j = 0; j < FN_; ++j)
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int mm = dmma::row_of<WM_, FM_>(i);
                const uint64_t m = m0 + mm, r = r0 + dmma::col_of<WM_, FN_>(j, t);
                if (m < M && r < R) {
                    uint64_t p, o;
                    split_po(mp0, mo0, uint32_t(mm), P, p, o);
                    y[p + P * r + P * R * o] = dacc.v[i][j][t];
                }
            }
}

// Small-R TTM, one output row m = (p, o) per thread: y(p, :, o) = U x(p, :, o).
// The I-vector of a row is read once (threads with consecutive p share 32-B
// sectors), U (R x I, fp64) sits in shared memory, the R accumulators in
// registers (fp64).  For the HBM-bound shapes the tile kernels waste on
// (R <= 32, e.g. C4 mode 1: P = 8, I = 48, R = 8).
template <class T, int RMAX>
__global__ void __launch_bounds__(256) ttm_rows_kernel(const T* __restrict__ x, const double* __restrict__ u,
                                                       uint64_t P, uint64_t I, uint64_t O, int R, T* __restrict__ y) {
    extern __shared__ double us[];  // [i][r], R x I
    for (int e = threadIdx.x; e < int(I) * R; e += blockDim.x) {
        const int r = e % R, i = e / R;
        us[e] = u[r + size_t(R) * i];
    }
    __syncthreads();
    const uint64_t m = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (m >= P * O) return;
    const uint64_t pp = m % P, o = m / P;  // one division per thread (row), not per element
    const T* xr = x + pp + P * I * o;
    double acc[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) acc[r] = 0.0;
    for (uint64_t i = 0; i < I; ++i) {
        const double v = double(xr[P * i]);
        const double* ui = us + i * R;
#pragma unroll
        for (int r = 0; r < RMAX; ++r)
            if (r < R) acc[r] = fma(ui[r], v, acc[r]);
    }
    T* yr = y + pp + P * uint64_t(R) * o;
#pragma unroll
    for (int r = 0; r < RMAX; ++r)
        if (r < R) yr[P * uint64_t(r)] = T(acc[r]);
}

}  // namespace

void ttt_simt(atk_ctx* ctx, const void* x, const void* y, atk_dtype dt, Split s, uint64_t R, double* z_dev, bool sym) {
    const uint64_t K = s.P * s.O;
    const uint64_t gm = (s.I + TM - 1) / TM, gn = (R + TN - 1) / TN;
    const uint64_t tiles = sym ? gm * (gm + 1) / 2 : gm * gn;
    uint64_t splits = std::max<uint64_t>(1, (uint64_t(ctx->num_sms) * 4) / std::max<uint64_t>(1, tiles));
    splits = std::min<uint64_t>(splits, std::max<uint64_t>(1, K / (KT * 16)));
    splits = std::min<uint64_t>(splits, 4096);
    uint64_t kchunk = (K + splits - 1) / splits;
    kchunk = (kchunk + KT - 1) / KT * KT;
    splits = (K + kchunk - 1) / kchunk;
    if (splits == 0) splits = 1;
    if (K == 0) {
        ATK_CUDA(cudaMemsetAsync(z_dev, 0, s.I * R * sizeof(double), ctx->stream));
        return;
    }
    DevBuf<double> part(ctx, splits * s.I * R);
    dim3 grid{unsigned(gm), unsigned(gn), unsigned(splits)};
    if (dt == ATK_F32)
        ttt_tile_kernel<float><<<grid, NT, 0, ctx->stream>>>((const float*)x, (const float*)y, s.P, s.I, R, K, kchunk,
                                                             sym, part.get());
    else
        ttt_tile_kernel<double><<<grid, NT, 0, ctx->stream>>>((const double*)x, (const double*)y, s.P, s.I, R, K,
                                                              kchunk, sym, part.get());
    ATK_LAUNCHED(ctx);
    const uint64_t n = s.I * R;
    if (splits >= 64 && n <= (uint64_t(1) << 22)) {
        reduce_partials_wide<<<unsigned((n + 7) / 8), 256, 0, ctx->stream>>>(part.get(), int(splits), s.I, R, sym,
                                                                            z_dev);
    } else {
        const int g = int(std::min<uint64_t>((n + 255) / 256, uint64_t(ctx->num_sms) * 8));
        reduce_partials<<<g, 256, 0, ctx->stream>>>(part.get(), int(splits), s.I, R, sym, z_dev);
    }
    ATK_LAUNCHED(ctx);
}

void ttm_simt(atk_ctx* ctx, const void* x, atk_dtype dt, Split s, const double* u_dev, uint64_t R, void* y) {
    const uint64_t M = s.P * s.O;
    // fp64 first / last mode: the unfolding is a plain column-major matrix, so the pipelined
    // DMMA GEMM applies (mode 0 writes Y = U X as (X^T U^T)^T; the last mode Y = X U^T directly)
    if (dt == ATK_F64 && !ctx->force_simt && (s.P == 1 || s.O == 1) && R <= 64 && s.I < (1u << 30) &&
        M < (1ull << 31)) {
        const double* xd = static_cast<const double*>(x);
        if (s.P == 1)
            dgemm_ttm(ctx, true, true, int(s.O), int(R), int(s.I), xd, int(s.I), u_dev, int(R), (double*)y, int(R),
                      true);
        else
            dgemm_ttm(ctx, false, true, int(s.P), int(R), int(s.I), xd, int(s.P), u_dev, int(R), (double*)y,
                      int(s.P), false);
        return;
    }
    if (R <= 32 && s.I * R <= 6144 && s.P > 1 && M >= uint64_t(ctx->num_sms) * 256) {
        const unsigned blocks = unsigned((M + 255) / 256);
        const size_t smem = size_t(s.I) * R * sizeof(double);
        if (dt == ATK_F32) {
            if (R <= 8) ttm_rows_kernel<float, 8><<<blocks, 256, smem, ctx->stream>>>((const float*)x, u_dev, s.P, s.I, s.O, int(R), (float*)y);
            else if (R <= 16) ttm_rows_kernel<float, 16><<<blocks, 256, smem, ctx->stream>>>((const float*)x, u_dev, s.P, s.I, s.O, int(R), (float*)y);
            else ttm_rows_kernel<float, 32><<<blocks, 256, smem, ctx->stream>>>((const float*)x, u_dev, s.P, s.I, s.O, int(R), (float*)y);
        } else {
            if (R <= 8) ttm_rows_kernel<double, 8><<<blocks, 256, smem, ctx->stream>>>((const double*)x, u_dev, s.P, s.I, s.O, int(R), (double*)y);
            else if (R <= 16) ttm_rows_kernel<double, 16><<<blocks, 256, smem, ctx->stream>>>((const double*)x, u_dev, s.P, s.I, s.O, int(R), (double*)y);
            else ttm_rows_kernel<double, 32><<<blocks, 256, smem, ctx->stream>>>((const double*)x, u_dev, s.P, s.I, s.O, int(R), (double*)y);
        }
        ATK_LAUNCHED(ctx);
        return;
    }
    dim3 grid{unsigned((M + TM - 1) / TM), unsigned((R + TN - 1) / TN)};
    if (dt == ATK_F32)
        ttm_tile_kernel<float><<<grid, NT, 0, ctx->stream>>>((const float*)x, u_dev, s.P, s.I, s.O, R, (float*)y);
    else
        if (R <= 16) {  // 8 warps x (8 rows x 16 cols): no DMMA columns wasted on R
            const dim3 g{grid.x, unsigned((R + 15) / 16)};
            ttm_f64_kernel<16, 8, 1, 2><<<g, NT, 0, ctx->stream>>>((const double*)x, u_dev, s.P, s.I, s.O, R,
                                                                   (double*)y);
        } else if (R <= 32) {
            const dim3 g{grid.x, unsigned((R + 31) / 32)};
            ttm_f64_kernel<32, 4, 2, 2><<<g, NT, 0, ctx->stream>>>((const double*)x, u_dev, s.P, s.I, s.O, R,
                                                                   (double*)y);
        } else {
            ttm_tile_kernel<double><<<grid, NT, 0, ctx->stream>>>((const double*)x, u_dev, s.P, s.I, s.O, R,
                                                                  (double*)y);
        }
    ATK_LAUNCHED(ctx);
}

}  // namespace atk
