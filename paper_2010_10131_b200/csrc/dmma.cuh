// dmma.cuh — fp64 tensor-core (DMMA, mma.sync m8n8k4 f64) warp microkernel.
//
// A CTA tile is split over its warps as WARPS_M along M x (nwarps / WARPS_M)
// along N; each warp owns FM x FN fragments of 8 x 8.  Operands come from
// shared memory laid out k-major: As[k][m], Bs[k][n] with leading dimensions
// LDA / LDB.  Bank-conflict-free fragment loads need LD = 4 (mod 16): the 16
// lanes of a half-warp read k-rows r = lane & 3 at columns c = lane >> 2, i.e.
// doubles r * LD + c, distinct mod 16 exactly when LD = 4 (mod 16).
// Used by the fp64 contractions (contract_simt.cu) and the fp64 GEMM of the
// eigensolver (dgemm.cu).  fp64 has no tcgen05 kind; DMMA is sm_100's fp64
// tensor path.
#pragma once

namespace atk {
namespace dmma {

template <int FM, int FN>
struct Acc {
    double v[FM][FN][2];  // [m-frag][n-frag][pair]
};

template <int FM, int FN>
__device__ __forceinline__ void zero(Acc<FM, FN>& a) {
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) a.v[i][j][0] = a.v[i][j][1] = 0.0;
}

__device__ __forceinline__ void mma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// acc += As[0:kk_count, warp's M block]^T x Bs[0:kk_count, warp's N block]
template <int LDA, int LDB, int WARPS_M, int FM, int FN>
__device__ __forceinline__ void tile_step(Acc<FM, FN>& acc, const double* As, const double* Bs, int kk_count) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp % WARPS_M, wn = warp / WARPS_M;
    const int r = lane & 3, c = lane >> 2;
    const double* ap = As + r * LDA + wm * FM * 8 + c;
    const double* bp = Bs + r * LDB + wn * FN * 8 + c;
#pragma unroll 2
    for (int kk = 0; kk < kk_count; kk += 4) {
        double a[FM], b[FN];
#pragma unroll
        for (int i = 0; i < FM; ++i) a[i] = ap[kk * LDA + i * 8];
#pragma unroll
        for (int j = 0; j < FN; ++j) b[j] = bp[kk * LDB + j * 8];
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
            for (int j = 0; j < FN; ++j) mma_8x8x4(acc.v[i][j][0], acc.v[i][j][1], a[i], b[j]);
    }
}

// Tile coordinates of accumulator element v[i][j][t].
template <int WARPS_M, int FM>
__device__ __forceinline__ int row_of(int i) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    return (warp % WARPS_M) * FM * 8 + i * 8 + (lane >> 2);
}
template <int WARPS_M, int FN>
__device__ __forceinline__ int col_of(int j, int t) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    return (warp / WARPS_M) * FN * 8 + j * 8 + 2 * (lane & 3) + t;
}

}  // namespace dmma
}  // namespace atk
