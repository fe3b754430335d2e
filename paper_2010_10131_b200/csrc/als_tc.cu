// als_tc.cu — one ALS iteration's contractions in ONE pass over Y (mode 0, fp32).
//
// als_iterate (solvers.hpp:88-118) contracts the big tensor twice per
// iteration: W = Y x_n L^T (ttm), rfac = W x_n (L^T L)^{-1} (ttm), then
// YR = Y_(n) rfac_(n)^T and GR = rfac rfac^T (ttt).  Both passes are HBM
// bound (C2: 2 x 4.3 GB per iteration).  rfac = M Y_(n) with M = (L^T L)^{-1}
// L^T (R x I), so every 128-column tile of Y_(n) can produce its rfac tile and
// consume it immediately:
//
//   phase 1  rfac_t^T (128 j x R) = Y_t^T . M^T       tcgen05 kind::tf32, TMEM,
//            A = Y_t K-major (box 32 i x 128 j), B = M^T K-major (the TTM layout)
//   convert  4 warps read rfac_t from TMEM, round to tf32 (RN) and write it to
//            shared memory as a K-major SW128 operand (32 x 128 j, rows >= R
//            zero); rfac_t is also stored to HBM (the caller keeps the last one)
//   phase 2  YR_i (128 i x R) += Y_t(i-tile) . rfac_t^T   A = Y_t MN-major
//            (boxes 32 i x 32 j, SWIZZLE_128B_ATOM_32B: a re-read that hits L2)
//
// and GR = rfac rfac^T = M Y_(0) Y_(0)^T M^T = M YR follows from YR with an
// R x R x I GEMM (no third phase).  Y crosses HBM once per iteration.
// Phase 2 of a tile follows its phase 1 directly (newest i-tiles first) so the
// re-read hits L2 (rfac stays double-buffered in TMEM so phase 1 of the next
// tile never waits for the conversion).  Each CTA owns a contiguous range of tiles; its YR accumulators
// (fp32 chains <= 16K terms) are drained once into fp64 partials and summed
// across CTAs in a fixed order (deterministic).
// Roles: warp 0 TMA, warp 1 MMA (one elected thread), warps 2-5 convert/drain.
#include <algorithm>
#include <vector>

#include "atk_driver.cuh"
#include "tc_common.cuh"

namespace atk {
namespace {

constexpr int JT = 128, BK = 32, THREADS = 192, NB = 32, RB_ROWS = NB;
constexpr uint32_t P1_A = BK * JT * 4, P1_B = BK * NB * 4;  // 16 KB + 4 KB
constexpr uint32_t STAGE = 16384 + 4096;                     // both phases fit one stage
constexpr uint32_t RB_CHUNK = RB_ROWS * 128, RB_BYTES = 4 * RB_CHUNK;  // 4 K-chunks of 32 j

struct AlsParams {
    int I, R, ntiles_i;   // rows, rank, I / 128
    uint64_t J;           // columns of Y_(0)
    int tiles;            // ceil(J / 128)
    int stages;
    int head;             // phase-1 K-blocks of tile t+1 issued before phase 2 of t (< 0: no overlap)
    float* rfac;          // R x J output (the iteration whose rfac is kept) or null
    double* acc_yr;       // [cta][I][NB]
};

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ float tf32_rn(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// The stage order both the TMA warp and the MMA thread follow.  Default
// (head < 0): P1(t), P2(t) strictly in turn.  head >= 0 (option als_head)
// interleaves tile t's phase 2 (the L2 re-read) with tile t+1's phase 1 (the
// HBM stream), `head` phase-1 K-blocks of t+1 first, so the MMA pipe has work
// while rfac_t is converted; measured slower on C2 (1.63 vs 1.31 ms per
// iteration on one box), so it stays off.
template <class F1, class F2>
__device__ __forceinline__ void als_schedule(int t0, int t1, int nkb1, int n2, int head, F1&& p1, F2&& p2) {
    if (t0 >= t1) return;
    if (head < 0) {  // P1(t), P2(t) strictly in turn
        for (int t = t0; t < t1; ++t) {
            for (int kb = 0; kb < nkb1; ++kb) p1(t, kb);
            for (int q = 0; q < n2; ++q) p2(t, q);
        }
        return;
    }
    for (int kb = 0; kb < nkb1; ++kb) p1(t0, kb);
    for (int t = t0; t < t1; ++t) {
        const bool nxt = t + 1 < t1;
        const int h = nxt ? min(head, nkb1) : 0, rem = nxt ? nkb1 - h : 0;
        int done = 0;
        for (; done < h; ++done) p1(t + 1, done);
        for (int q = 0; q < n2; ++q) {
            p2(t, q);
            const int target = h + int(int64_t(q + 1) * rem / n2);
            for (; done < target; ++done) p1(t + 1, done);
        }
    }
}

__global__ void __launch_bounds__(THREADS, 1)
    als_pass_kernel(const __grid_constant__ CUtensorMap tma_yk, const __grid_constant__ CUtensorMap tma_ym,
                    const __grid_constant__ CUtensorMap tma_f, const AlsParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages;
    uint8_t* rb = smem + size_t(S) * STAGE;  // rfac tile operand (1024-aligned: S * 20 KB + ...)
    uint64_t* full = reinterpret_cast<uint64_t*>(rb + RB_BYTES);
    uint64_t* empty = full + S;
    uint64_t* rf_full = empty + S;   // [2] MMA -> convert (phase 1 done)
    uint64_t* rf_empty = rf_full + 2;  // [2] convert -> MMA (TMEM buffer read)
    uint64_t* rb_full = rf_empty + 2;  // convert -> MMA (smem tile written)
    uint64_t* rb_empty = rb_full + 1;  // MMA -> convert (phases 2/3 done with the tile)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rb_empty + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // this CTA's contiguous tile range
    const int t0 = int(int64_t(p.tiles) * blockIdx.x / gridDim.x);
    const int t1 = int(int64_t(p.tiles) * (blockIdx.x + 1) / gridDim.x);
    const int nkb1 = p.I / BK;               // phase-1 K-blocks per tile

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < S; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&rf_full[b], 1);
            tc::mbar_init(&rf_empty[b], 4);
        }
        tc::mbar_init(rb_full, 4);
        tc::mbar_init(rb_empty, 1);
        tc::fence_barrier_init();
        tc::tma_prefetch(&tma_yk);
        tc::tma_prefetch(&tma_ym);
        tc::tma_prefetch(&tma_f);
    }
    // rows >= R of the rfac operand stay zero for the whole kernel
    for (int e = threadIdx.x; e < int(RB_BYTES / 16); e += THREADS)
        reinterpret_cast<uint4*>(rb)[e] = make_uint4(0, 0, 0, 0);
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    fence_proxy_async();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // TMEM columns: rf[2] at 0 / NB, YR tiles at 2 NB + it NB
    const uint32_t col_yr = 2 * NB;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint64_t keep = tc::policy_evict_last(), drop = tc::policy_evict_first();
            auto next = [&]() {
                if (++stage == S) { stage = 0; phase ^= 1; }
            };
            auto load_p1 = [&](int t, int kb) {
                tc::mbar_wait(&empty[stage], phase ^ 1);
                tc::mbar_arrive_expect_tx(&full[stage], P1_A + P1_B);
                uint8_t* a = smem + size_t(stage) * STAGE;
                tc::tma_load_2d_hint(a, &tma_yk, &full[stage], kb * BK, t * JT, keep);  // re-read in phase 2
                tc::tma_load_2d(a + P1_A, &tma_f, &full[stage], kb * BK, 0);
                next();
            };
            auto load_p2 = [&](int t, int q) {
                // i-tiles newest-first: phase 1 streamed i upwards, so the last rows are the
                // likeliest to still be in L2
                const int it = p.ntiles_i - 1 - q / (JT / BK), c = q % (JT / BK);
                tc::mbar_wait(&empty[stage], phase ^ 1);
                tc::mbar_arrive_expect_tx(&full[stage], 16384);
                uint8_t* a = smem + size_t(stage) * STAGE;
#pragma unroll
                for (int qq = 0; qq < 4; ++qq)
                    tc::tma_load_2d_hint(a + qq * 4096, &tma_ym, &full[stage], it * 128 + qq * 32, t * JT + c * BK,
                                         drop);  // last use of the tile
                next();
            };
            als_schedule(t0, t1, nkb1, p.ntiles_i * (JT / BK), p.head, load_p1, load_p2);
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t id_p1 = tc::idesc_tf32(128, NB, false, false);
            const uint32_t id_p2 = tc::idesc_tf32(128, NB, true, false);
            int stage = 0;
            uint32_t phase = 0, rbe_phase = 0;
            uint32_t rfe_phase[2] = {0, 0};
            bool yr_started = false;
            auto next = [&]() {
                if (++stage == S) { stage = 0; phase ^= 1; }
            };
            auto issue_p1 = [&](int t, int kb) {
                const int buf = (t - t0) & 1;
                const uint32_t d = tmem + uint32_t(buf * NB);
                if (kb == 0) {
                    // the TMEM buffer must have been read by the conversion of tile t - 2
                    if (t - t0 >= 2) {
                        tc::mbar_wait(&rf_empty[buf], rfe_phase[buf]);
                        rfe_phase[buf] ^= 1;
                    }
                    tc::tc_fence_after();
                }
                tc::mbar_wait(&full[stage], phase);
                tc::tc_fence_after();
                const uint32_t a_base = tc::smem_u32(smem + size_t(stage) * STAGE);
                const uint32_t b_base = a_base + P1_A;
#pragma unroll
                for (int k = 0; k < BK / 8; ++k)
                    tc::mma_tf32(d, tc::smem_desc(a_base + k * 32, 16, 1024, 2),
                                 tc::smem_desc(b_base + k * 32, 16, 1024, 2), id_p1, (kb > 0 || k > 0) ? 1u : 0u);
                tc::mma_commit(&empty[stage]);
                next();
                if (kb == nkb1 - 1) tc::mma_commit(&rf_full[buf]);
            };
            const int n2 = p.ntiles_i * (JT / BK);
            auto issue_p2 = [&](int t, int q) {
                (void)t;
                if (q == 0) {
                    tc::mbar_wait(rb_full, rbe_phase);  // the tile's rfac operand is in smem
                    rbe_phase ^= 1;
                    tc::tc_fence_after();
                }
                const int it = p.ntiles_i - 1 - q / (JT / BK), c = q % (JT / BK);
                const uint32_t rb_base = tc::smem_u32(rb);
                tc::mbar_wait(&full[stage], phase);
                tc::tc_fence_after();
                const uint32_t a_base = tc::smem_u32(smem + size_t(stage) * STAGE);
#pragma unroll
                for (int k = 0; k < BK / 8; ++k)
                    tc::mma_tf32(tmem + col_yr + uint32_t(it * NB), tc::smem_desc(a_base + k * 1024, 4096, 512, 1),
                                 tc::smem_desc(rb_base + c * RB_CHUNK + k * 32, 16, 1024, 2), id_p2,
                                 (yr_started || c > 0 || k > 0) ? 1u : 0u);
                tc::mma_commit(&empty[stage]);
                next();
                if (q == n2 - 1) {
                    yr_started = true;
                    tc::mma_commit(rb_empty);
                }
            };
            als_schedule(t0, t1, nkb1, n2, p.head, issue_p1, issue_p2);
        }
        __syncwarp();
    } else {
        const int q = warp & 3;
        const int row = q * 32 + lane;  // j within the tile (TMEM lane quadrant q)
        uint32_t rff_phase[2] = {0, 0}, rbe_phase = 0;
        for (int t = t0; t < t1; ++t) {
            const int buf = (t - t0) & 1;
            tc::mbar_wait(&rf_full[buf], rff_phase[buf]);
            rff_phase[buf] ^= 1;
            tc::tc_fence_after();
            uint32_t r[32];
            tc::tmem_ld_32x32b_x32(tmem + (uint32_t(q * 32) << 16) + uint32_t(buf * NB), r);
            tc::tmem_ld_wait();
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&rf_empty[buf]);  // TMEM buffer free for tile t + 2
            // the previous tile's phase 2 must be done with the smem operand
            if (t > t0) {
                tc::mbar_wait(rb_empty, rbe_phase);
                rbe_phase ^= 1;
            }
            // K-major SW128 operand: chunk c = row / 32, row r, 16-B granule g ^ (r & 7)
            const int c = row >> 5, e = row & 31, g = e >> 2, w = e & 3;
            uint8_t* chunk = rb + size_t(c) * RB_CHUNK;
#pragma unroll
            for (int rr = 0; rr < NB; ++rr) {
                const float v = rr < p.R ? tf32_rn(__uint_as_float(r[rr])) : 0.0f;
                *reinterpret_cast<float*>(chunk + rr * 128 + ((g ^ (rr & 7)) << 4) + (w << 2)) = v;
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(rb_full);
            // off the critical path: rfac_t to HBM (last iteration only)
            const uint64_t j = uint64_t(t) * JT + row;
            if (p.rfac && j < p.J) {
                float* dst = p.rfac + uint64_t(p.R) * j;
                if ((p.R & 3) == 0) {
                    for (int c4 = 0; c4 < p.R; c4 += 4)
                        *reinterpret_cast<float4*>(dst + c4) =
                            make_float4(__uint_as_float(r[c4]), __uint_as_float(r[c4 + 1]),
                                        __uint_as_float(r[c4 + 2]), __uint_as_float(r[c4 + 3]));
                } else {
                    for (int c = 0; c < p.R; ++c) dst[c] = __uint_as_float(r[c]);
                }
            }
        }
        // drain: wait for the last phases 2/3, then YR and GR -> fp64 partials
        if (t1 > t0) {
            tc::mbar_wait(rb_empty, rbe_phase);
            tc::tc_fence_after();
        }
        double* yr = p.acc_yr + size_t(blockIdx.x) * p.I * NB;
        for (int it = 0; it < p.ntiles_i; ++it) {
            uint32_t r[32];
            tc::tmem_ld_32x32b_x32(tmem + (uint32_t(q * 32) << 16) + col_yr + uint32_t(it * NB), r);
            tc::tmem_ld_wait();
            double* dst = yr + size_t(it * 128 + row) * NB;
#pragma unroll
            for (int c = 0; c < NB; ++c) dst[c] = (t1 > t0) ? double(__uint_as_float(r[c])) : 0.0;
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem, 512);
    }
}

// YR (I x R) = sum of the per-CTA partials [cta][I][NB]: one 128-thread block
// per row i, lane = r (a warp reads one contiguous 256-byte row per CTA), warp g
// sums CTAs g, g+4, ... in order (8 loads in flight), then the 4 warp partials in
// order (deterministic).  Element-per-thread loops were 148-deep chains of
// uncoalesced L2 reads (30 us per call at C2's I = 1024).
__global__ void __launch_bounds__(128) als_reduce_rows(const double* __restrict__ acc_yr, int ncta, int I, int R,
                                                       double* __restrict__ yr) {
    __shared__ double part[4][NB];
    const int i = blockIdx.x, lane = threadIdx.x & 31, g = threadIdx.x >> 5;
    double v = 0.0;
    int c = g;
    for (; c + 28 < ncta; c += 32) {
        double t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) t[u] = acc_yr[(size_t(c + 4 * u) * I + i) * NB + lane];
#pragma unroll
        for (int u = 0; u < 8; ++u) v += t[u];
    }
    for (; c < ncta; c += 4) v += acc_yr[(size_t(c) * I + i) * NB + lane];
    part[g][lane] = v;
    __syncthreads();
    if (g == 0 && lane < R) yr[i + size_t(I) * lane] = ((part[0][lane] + part[1][lane]) + part[2][lane]) + part[3][lane];
}

// F[i + I r] = M(r, i) (fp32), rows r >= R zero: the K-major B operand of phase 1
__global__ void m_to_f32(const double* __restrict__ m, int R, int I, float* __restrict__ f) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= NB * I) return;
    const int i = e % I, r = e / I;
    f[e] = r < R ? float(m[r + size_t(R) * i]) : 0.0f;
}

}  // namespace

bool als_fused_supported(atk_ctx* ctx, const atk_tensor* y, int mode, uint64_t R) {
    static_assert(NB == 32 && JT == 128, "als_fused_shape_ok (atk_driver.cuh) mirrors NB / JT");
    if (!ctx->als_fused || ctx->force_simt || y->dtype != ATK_F32 || mode != 0) return false;
    const Split s = loop_split(y->dims, y->order, mode);
    return s.P == 1 && als_fused_shape_ok(s.I, R, s.O, ctx->num_sms);
}

// One ALS iteration's contractions on mode 0: M (R x I, fp64 device) = (L^T L)^{-1} L^T;
// YR = Y_(0) rfac^T, GR = rfac rfac^T with rfac = M Y_(0); rfac_out (R x J fp32) optional.
void als_fused_pass(atk_ctx* ctx, const atk_tensor* y, const double* m_dev, uint64_t R, double* yr_dev,
                    double* gr_dev, atk_tensor* rfac_out) {
    const Split s = loop_split(y->dims, y->order, 0);
    const int I = int(s.I);
    const uint64_t J = s.O;
    DevBuf<float> f(ctx, size_t(NB) * I);
    m_to_f32<<<unsigned((NB * I + 255) / 256), 256, 0, ctx->stream>>>(m_dev, int(R), I, f.get());
    ATK_LAUNCHED(ctx);
    const CUtensorMapDataType dt = ctx->tma_tf32 ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    CUtensorMap tyk{}, tym{}, tf{};
    {
        const uint64_t dims[2] = {uint64_t(I), J};
        const uint64_t str[1] = {uint64_t(I) * 4};
        const uint32_t bk[2] = {BK, JT}, bm[2] = {32, BK};
        if (encode_tensor_map(&tyk, dt, 2, y->data, dims, str, bk, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS ||
            encode_tensor_map(&tym, dt, 2, y->data, dims, str, bm, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) != CUDA_SUCCESS)
            fail(ATK_CUDA_ERROR, "als: tensor map encoding failed");
        const uint64_t fd[2] = {uint64_t(I), uint64_t(NB)};
        const uint64_t fs[1] = {uint64_t(I) * 4};
        const uint32_t fb[2] = {BK, NB};
        if (encode_tensor_map(&tf, dt, 2, f.get(), fd, fs, fb, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
            fail(ATK_CUDA_ERROR, "als: factor tensor map encoding failed");
    }
    AlsParams p{};
    p.I = I;
    p.R = int(R);
    p.ntiles_i = I / 128;
    p.J = J;
    p.tiles = int((J + JT - 1) / JT);
    p.stages = 10;
    p.head = ctx->als_head;
    const int grid = std::min(ctx->num_sms, p.tiles);
    DevBuf<double> ayr(ctx, size_t(grid) * I * NB);
    p.rfac = rfac_out ? static_cast<float*>(rfac_out->data) : nullptr;
    p.acc_yr = ayr.get();
    const size_t smem = size_t(p.stages) * STAGE + RB_BYTES + 1024 + 256;
    static bool attr = false;
    if (!attr) {
        ATK_CUDA(cudaFuncSetAttribute(als_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr = true;
    }
    als_pass_kernel<<<grid, THREADS, smem, ctx->stream>>>(tyk, tym, tf, p);
    ATK_LAUNCHED(ctx);
    als_reduce_rows<<<unsigned(I), 128, 0, ctx->stream>>>(ayr.get(), grid, I, int(R), yr_dev);
    ATK_LAUNCHED(ctx);
    // GR = rfac rfac^T = M (Y_(0) rfac^T) = M YR, exactly symmetrised
    dgemm(ctx, false, false, int(R), int(R), I, 1.0, m_dev, int(R), yr_dev, I, 0.0, gr_dev, int(R));
    symmetrize(ctx, gr_dev, int(R));
}

}  // namespace atk
