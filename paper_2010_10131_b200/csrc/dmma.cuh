// dmma.cuh — fp64 tensor-core (DMMA, mma.sync m8n8k4 f64) microkernel for a
// 64 x 64 output tile computed by 8 warps (2 along M x 4 along N; each warp a
// 32 x 16 block = 4 x 2 fragments of 8 x 8).  Operands come from shared memory
// laid out k-major: As[k][m], Bs[k][n] with leading dimensions LDA / LDB.
// Used by the fp64 contractions (contract_simt.cu) and the fp64 GEMM
// (dgemm.cu).  fp64 has no tcgen05 kind; DMMA is the sm_100 fp64 tensor path.
#pragma once

namespace atk {
namespace dmma {

struct Acc {
    double v[4][2][2];  // [m-frag][n-frag][pair]
};

__device__ __forceinline__ void zero(Acc& a) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) a.v[i][j][0] = a.v[i][j][1] = 0.0;
}

__device__ __forceinline__ void mma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// acc += As[k0:k0+kk, wm*32 .. +32]^T-fragments x Bs[k0:k0+kk, wn*16 .. +16]
template <int LDA, int LDB>
__device__ __forceinline__ void tile_step(Acc& acc, const double* As, const double* Bs, int kk_count) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp & 1, wn = warp >> 1;
    const int r = lane & 3, c = lane >> 2;
    for (int kk = 0; kk < kk_count; kk += 4) {
        double a[4], b[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[(kk + r) * LDA + wm * 32 + i * 8 + c];
#pragma unroll
        for (int j = 0; j < 2; ++j) b[j] = Bs[(kk + r) * LDB + wn * 16 + j * 8 + c];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) mma_8x8x4(acc.v[i][j][0], acc.v[i][j][1], a[i], b[j]);
    }
}

// Output coordinates of accumulator element (i, j, t) within the 64 x 64 tile.
__device__ __forceinline__ int row_of(int i) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    return (warp & 1) * 32 + i * 8 + (lane >> 2);
}
__device__ __forceinline__ int col_of(int j, int t) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    return (warp >> 1) * 16 + j * 8 + 2 * (lane & 3) + t;
}

}  // namespace dmma
}  // namespace atk
