// dgemm.cu — fp64 GEMM for the eigensolver / ALS small dense algebra.
//
// C(m x n) = alpha op(A) op(B) + beta C, column-major.  128x64 block tile,
// 8-deep K slices, 256 threads each owning an 8x4 register tile (DFMA), and a
// deterministic split-K (fixed-order fp64 partial sums) so that the skinny
// shapes of Chebyshev filtering (2048 x 96 x 2048) still fill all 148 SMs.
#include <algorithm>

#include "atk_internal.cuh"

namespace atk {
namespace {

constexpr int BM = 128, BN = 64, BK = 8, NT = 256;

__global__ void __launch_bounds__(NT) dgemm_tile(bool ta, bool tb, int m, int n, int k, int kchunk,
                                                 const double* __restrict__ a, int lda,
                                                 const double* __restrict__ b, int ldb,
                                                 double* __restrict__ out, size_t out_split_stride,
                                                 int ldo, double alpha, double beta, bool direct) {
    __shared__ __align__(16) double As[2][BK][BM];
    __shared__ __align__(16) double Bs[2][BK][BN];
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const int kb = blockIdx.z * kchunk, ke = min(k, kb + kchunk);
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    double acc[8][4] = {};

    auto load = [&](int buf, int k0) {
#pragma unroll
        for (int e = tid; e < BK * BM; e += NT) {
            int kk, mm;
            if (!ta) { mm = e % BM; kk = e / BM; } else { kk = e % BK; mm = e / BK; }
            const int gm = m0 + mm, gk = k0 + kk;
            As[buf][kk][mm] = (gm < m && gk < ke) ? (ta ? a[gk + size_t(lda) * gm] : a[gm + size_t(lda) * gk]) : 0.0;
        }
#pragma unroll
        for (int e = tid; e < BK * BN; e += NT) {
            int kk, nn;
            if (tb) { nn = e % BN; kk = e / BN; } else { kk = e % BK; nn = e / BK; }
            const int gn = n0 + nn, gk = k0 + kk;
            Bs[buf][kk][nn] = (gn < n && gk < ke) ? (tb ? b[gn + size_t(ldb) * gk] : b[gk + size_t(ldb) * gn]) : 0.0;
        }
    };

    int buf = 0;
    if (kb < ke) load(0, kb);
    __syncthreads();
    for (int k0 = kb; k0 < ke; k0 += BK) {
        if (k0 + BK < ke) load(buf ^ 1, k0 + BK);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            const double2* ap = reinterpret_cast<const double2*>(&As[buf][kk][ty * 8]);
            const double2* bp = reinterpret_cast<const double2*>(&Bs[buf][kk][tx * 4]);
            double av[8], bv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double2 t = ap[u];
                av[2 * u] = t.x;
                av[2 * u + 1] = t.y;
            }
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const double2 t = bp[v];
                bv[2 * v] = t.x;
                bv[2 * v + 1] = t.y;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
        }
        __syncthreads();
        buf ^= 1;
    }
    double* o = out + size_t(blockIdx.z) * out_split_stride;
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int gm = m0 + ty * 8 + u, gn = n0 + tx * 4 + v;
            if (gm < m && gn < n) {
                double* cp = o + gm + size_t(ldo) * gn;
                if (direct) *cp = alpha * acc[u][v] + (beta == 0.0 ? 0.0 : beta * *cp);
                else *cp = acc[u][v];
            }
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

void dgemm(atk_ctx* ctx, bool ta, bool tb, int m, int n, int k, double alpha, const double* a, int lda,
           const double* b, int ldb, double beta, double* c, int ldc) {
    if (m <= 0 || n <= 0) return;
    const int gm = (m + BM - 1) / BM, gn = (n + BN - 1) / BN;
    const int tiles = gm * gn;
    int splits = 1;
    if (tiles < 2 * ctx->num_sms && k >= 512)
        splits = std::min(std::max(1, (2 * ctx->num_sms + tiles - 1) / tiles), std::max(1, k / 256));
    int kchunk = (k + splits - 1) / splits;
    kchunk = (kchunk + BK - 1) / BK * BK;
    splits = std::max(1, (k + kchunk - 1) / std::max(1, kchunk));
    if (k <= 0) {
        kchunk = 0;
        splits = 1;
    }
    if (splits == 1) {
        dim3 grid{unsigned(gm), unsigned(gn), 1u};
        dgemm_tile<<<grid, NT, 0, ctx->stream>>>(ta, tb, m, n, std::max(k, 0), std::max(kchunk, BK), a, lda, b, ldb, c,
                                                 0, ldc, alpha, beta, true);
        ATK_LAUNCHED(ctx);
        return;
    }
    DevBuf<double> part(ctx, size_t(splits) * m * n);
    dim3 grid{unsigned(gm), unsigned(gn), unsigned(splits)};
    dgemm_tile<<<grid, NT, 0, ctx->stream>>>(ta, tb, m, n, k, kchunk, a, lda, b, ldb, part.get(), size_t(m) * n, m,
                                             1.0, 0.0, false);
    ATK_LAUNCHED(ctx);
    const size_t mn = size_t(m) * n;
    dgemm_splitk_reduce<<<unsigned(std::min<size_t>((mn + 255) / 256, size_t(ctx->num_sms) * 8)), 256, 0,
                          ctx->stream>>>(part.get(), splits, m, n, alpha, beta, c, ldc);
    ATK_LAUNCHED(ctx);
}

}  // namespace atk
