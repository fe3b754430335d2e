// ttm_tc.cu — matricization-free TTM Y = X x_n U on the 5th-gen tensor cores.
//
// kernels::ttm (kernels.hpp:88-118) for fp32 storage.  The factor F = U^T
// (I x R, fp32, i contiguous) is the K-major B operand; the A operand comes
// straight from the tensor through TMA (TFLOAT32 => round-to-nearest tf32):
//   mode 0 (P == 1): D(j, r) = sum_i X(i, j) F(i, r): A = X^T is K-major
//                    (2-D map {I, J}, box 32 i x 128 j, SWIZZLE_128B);
//                    D row j is the contiguous R-vector Y(:, j) of the output.
//   P % 32 == 0    : D((p,o), r) = sum_i X(p, i, o) F(i, r): A is MN-major
//                    (3-D map {P, I, O}, 32x32x1 boxes, 128B/32B-atom swizzle);
//                    covers the middle modes and the last mode (O == 1).
// Each CTA owns 256-row M tiles (two M=128 UMMAs sharing the F stage), the
// accumulators are double-buffered in TMEM so the store epilogue of tile t
// overlaps the MMAs of tile t+1.  Persistent grid, warp-specialised:
// warp 0 TMA, warp 1 MMA, warps 2-5 epilogue.  HBM-bound by design
// (arithmetic intensity R/2 flop/B for fp32).
#include <algorithm>
#include <cstdlib>

#include "atk_driver.cuh"
#include "tc_common.cuh"

namespace atk {
namespace {

constexpr int MT = 256, BK = 32, THREADS = 192;

struct TtmParams {
    uint64_t M;       // rows of D (J for mode 0, P*O otherwise)
    uint64_t P;       // inner size (MN-major layout)
    int R, NB;        // rank and padded N (multiple of 32)
    int nkb;          // K-blocks (ceil(I / 32))
    int ks;           // K pieces per M tile (split-K when the tiles alone underfill the GPU)
    int box4;         // MN-major A: one 4-D TMA box per stage ({32 p, 32 i, p-blocks, o}) instead of 8
    int pb, ob;       // 4-D box: 32-row p blocks and o slabs per 256-row tile
    int stages;
    int split;        // 1: the factor is staged as tf32 hi + lo parts and each K step issues two MMAs
    uint32_t stage_bytes, a_bytes, b_bytes;
    float* y;         // the output, or ks partial outputs (piece q at y + q M R) when ks > 1
};

template <bool KMAJOR_A>
__global__ void __launch_bounds__(THREADS, 1)
    ttm_tf32_kernel(const __grid_constant__ CUtensorMap tma_x, const __grid_constant__ CUtensorMap tma_f,
                    const TtmParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * p.stage_bytes);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t ntiles = (p.M + MT - 1) / MT;
    const uint32_t tcols = uint32_t(4 * p.NB) <= 32 ? 32 : (uint32_t(4 * p.NB) <= 64 ? 64 : (uint32_t(4 * p.NB) <= 128 ? 128 : (uint32_t(4 * p.NB) <= 256 ? 256 : 512)));

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < S; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&tfull[b], 1);
            tc::mbar_init(&tempty[b], 4);
        }
        tc::fence_barrier_init();
        tc::tma_prefetch(&tma_x);
        tc::tma_prefetch(&tma_f);
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, tcols);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint64_t pblk = p.P / 32;
            for (uint64_t it = blockIdx.x; it < ntiles * p.ks; it += gridDim.x) {
                const uint64_t t = it / p.ks;
                const int q = int(it % p.ks);
                const uint64_t m0 = t * MT;
                for (int kb = p.nkb * q / p.ks; kb < p.nkb * (q + 1) / p.ks; ++kb) {
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    tc::mbar_arrive_expect_tx(&full[stage], p.stage_bytes);
                    uint8_t* a = smem + size_t(stage) * p.stage_bytes;
                    uint8_t* b = a + p.a_bytes;
                    const int k0 = kb * BK;
                    if (KMAJOR_A) {
                        tc::tma_load_2d(a, &tma_x, &full[stage], k0, int(m0));
                        tc::tma_load_2d(a + 16384, &tma_x, &full[stage], k0, int(m0 + 128));
                    } else if (p.box4) {
                        // {32 p_lo, 32 i, pb p_hi, ob o}: lands as the 8 MN-major 4 KB groups in order
                        tc::tma_load_4d(a, &tma_x, &full[stage], 0, k0, int((m0 % p.P) / 32), int(m0 / p.P));
                    } else {
#pragma unroll
                        for (int g = 0; g < MT / 32; ++g) {
                            const uint64_t blk = m0 / 32 + g;
                            tc::tma_load_3d(a + g * 4096, &tma_x, &full[stage], int((blk % pblk) * 32), k0,
                                            int(blk / pblk));
                        }
                    }
                    if (p.split) tc::tma_load_3d(b, &tma_f, &full[stage], k0, 0, 0);  // hi, then lo
                    else tc::tma_load_2d(b, &tma_f, &full[stage], k0, 0);
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = tc::idesc_tf32(128, p.NB, !KMAJOR_A, false);
            int stage = 0, abuf = 0;
            uint32_t phase = 0, aphase = 0;
            for (uint64_t it = blockIdx.x; it < ntiles * p.ks; it += gridDim.x) {
                const int q = int(it % p.ks);
                const int kb0 = p.nkb * q / p.ks;
                tc::mbar_wait(&tempty[abuf], aphase ^ 1);
                tc::tc_fence_after();
                const uint32_t d0 = tmem_base + uint32_t(abuf * 2 * p.NB);
                for (int kb = kb0; kb < p.nkb * (q + 1) / p.ks; ++kb) {
                    tc::mbar_wait(&full[stage], phase);
                    tc::tc_fence_after();
                    const uint32_t a_base = tc::smem_u32(smem + size_t(stage) * p.stage_bytes);
                    const uint32_t b_base = a_base + p.a_bytes;
#pragma unroll
                    for (int k = 0; k < BK / 8; ++k) {
                        const uint64_t bd = tc::smem_desc(b_base + k * 32, 16, 1024, 2);
                        const uint64_t bdl = tc::smem_desc(b_base + p.b_bytes + k * 32, 16, 1024, 2);
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            uint64_t ad;
                            if (KMAJOR_A) ad = tc::smem_desc(a_base + h * 16384 + k * 32, 16, 1024, 2);
                            else ad = tc::smem_desc(a_base + h * 16384 + k * 1024, 4096, 512, 1);
                            tc::mma_tf32(d0 + uint32_t(h * p.NB), ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
                            if (p.split) tc::mma_tf32(d0 + uint32_t(h * p.NB), ad, bdl, idesc, 1u);  // X F_lo
                        }
                    }
                    tc::mma_commit(&empty[stage]);
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
                tc::mma_commit(&tfull[abuf]);
                if (++abuf == 2) { abuf = 0; aphase ^= 1; }
            }
        }
        __syncwarp();
    } else {
        const int q = warp & 3;
        int abuf = 0;
        uint32_t aphase = 0;
        for (uint64_t it = blockIdx.x; it < ntiles * p.ks; it += gridDim.x) {
            const uint64_t t = it / p.ks;
            float* const yq = p.y + uint64_t(it % p.ks) * p.M * uint64_t(p.R);
            tc::mbar_wait(&tfull[abuf], aphase);
            tc::tc_fence_after();
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const uint64_t m = t * MT + h * 128 + q * 32 + lane;
                const bool ok = m < p.M;
#pragma unroll 1
                for (int c = 0; c < p.NB; c += 32) {
                    uint32_t r[32];
                    tc::tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) + uint32_t(abuf * 2 * p.NB + h * p.NB + c), r);
                    tc::tmem_ld_wait();
                    if (!ok) continue;
                    const int nc = min(32, p.R - c);
                    if (KMAJOR_A) {
                        float* dst = yq + m * uint64_t(p.R) + c;
                        if (nc == 32 && (p.R % 4) == 0) {
#pragma unroll
                            for (int j = 0; j < 32; j += 4)
                                *reinterpret_cast<float4*>(dst + j) =
                                    make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
                        } else {
                            for (int j = 0; j < nc; ++j) dst[j] = __uint_as_float(r[j]);
                        }
                    } else {
                        const uint64_t pp = m % p.P, o = m / p.P;
                        float* dst = yq + pp + p.P * (uint64_t(c) + uint64_t(p.R) * o);
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (j < nc) dst[uint64_t(j) * p.P] = __uint_as_float(r[j]);
                    }
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[abuf]);
            if (++abuf == 2) { abuf = 0; aphase ^= 1; }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, tcols);
    }
}

// y = the ks split-K partials summed in a fixed order (fp32, as the accumulators)
__global__ void ttm_reduce(const float* __restrict__ part, uint64_t n, int ks, float* __restrict__ y) {
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += uint64_t(gridDim.x) * blockDim.x) {
        float v = part[e];
        for (int q = 1; q < ks; ++q) v += part[uint64_t(q) * n + e];
        y[e] = v;
    }
}

// F (I x R, fp32) = U^T from U (R x I, fp64).  split: F_hi = tf32_rn(U^T) at f,
// F_lo = fp32(U^T - F_hi) at f + I R (rounded to tf32 again by the TMA): the
// factor enters the MMAs to ~2^-22 instead of 2^-12 (its rounding is one
// coherent perturbation of every output column, unlike the data's)
__device__ __forceinline__ float tf32_rn(float x) {
    uint32_t b = __float_as_uint(x);
    b += 0xfffu + ((b >> 13) & 1u);  // round to nearest even on the 13 dropped bits
    return __uint_as_float(b & 0xffffe000u);
}
__global__ void factor_to_f32(const double* __restrict__ u, int R, int I, float* __restrict__ f, int split) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= R * I) return;
    const int i = e % I, r = e / I;
    const double v = u[r + size_t(R) * i];
    if (!split) {
        f[i + size_t(I) * r] = float(v);
        return;
    }
    const float hi = tf32_rn(float(v));
    f[i + size_t(I) * r] = hi;
    f[size_t(I) * R + i + size_t(I) * r] = float(v - double(hi));
}

}  // namespace

bool tc_ttm_supported(atk_ctx* ctx, const atk_tensor* x, uint64_t R, int mode) {
    (void)ctx;
    if (x->dtype != ATK_F32 || R < 1 || R > 128) return false;  // 2 bufs x 2 halves x NB <= 512 TMEM cols
    const Split s = loop_split(x->dims, x->order, mode);
    if (s.I < 32 || s.I % 4 != 0 || s.I >= (1u << 30)) return false;
    if (s.P == 1) return s.O < (1ull << 31);
    return s.P % 32 == 0 && s.P * s.I < (1ull << 40) && s.O < (1ull << 31);
}

void tc_ttm(atk_ctx* ctx, const atk_tensor* x, const double* u_dev, uint64_t R, int mode, atk_tensor* y) {
    const Split s = loop_split(x->dims, x->order, mode);
    const bool kmajor = s.P == 1;
    const int NB = int((R + 31) / 32 * 32);
    const int I = int(s.I);
    const int split = ctx->ttm_split && ctx->tma_tf32 ? 1 : 0;
    DevBuf<float> f(ctx, size_t(I) * R * (split ? 2 : 1));
    factor_to_f32<<<unsigned((R * I + 255) / 256), 256, 0, ctx->stream>>>(u_dev, int(R), I, f.get(), split);
    ATK_LAUNCHED(ctx);
    const CUtensorMapDataType dt = ctx->tma_tf32 ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    CUtensorMap tx{}, tf{};
    {
        const uint64_t dims[3] = {s.I, R, 2};
        const uint64_t str[2] = {s.I * 4, s.I * R * 4};
        const uint32_t box[3] = {BK, uint32_t(NB), 2};
        if (encode_tensor_map(&tf, dt, split ? 3 : 2, f.get(), dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B) !=
            CUDA_SUCCESS)
            fail(ATK_CUDA_ERROR, "ttm: factor tensor map encoding failed");
    }
    TtmParams p{};
    p.split = split;
    if (kmajor) {
        const uint64_t dims[2] = {s.I, s.O};
        const uint64_t str[1] = {s.I * 4};
        const uint32_t box[2] = {BK, 128};
        if (encode_tensor_map(&tx, dt, 2, x->data, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
            fail(ATK_CUDA_ERROR, "ttm: tensor map (mode 0) encoding failed");
        p.M = s.O;
        p.P = 1;
    } else {
        // one 4-D box per stage when a 256-row tile is whole p blocks of whole o slabs
        // (P | 256) or whole p blocks of one o slab (256 | P): map {32 p_lo, I, P/32 p_hi, O}
        const bool box4 = !std::getenv("ATK_TTM_BOX3") && ((MT % s.P == 0) || (s.P % MT == 0));
        if (box4) {
            const uint64_t dims[4] = {32, s.I, s.P / 32, s.O};
            const uint64_t str[3] = {s.P * 4, 32 * 4, s.P * s.I * 4};
            p.pb = int(std::min<uint64_t>(s.P / 32, MT / 32));
            p.ob = int(MT / 32 / p.pb);
            const uint32_t box[4] = {32, BK, uint32_t(p.pb), uint32_t(p.ob)};
            if (encode_tensor_map(&tx, dt, 4, x->data, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) !=
                CUDA_SUCCESS)
                fail(ATK_CUDA_ERROR, "ttm: tensor map (MN-major, 4-D) encoding failed");
            p.box4 = 1;
        } else {
            const uint64_t dims[3] = {s.P, s.I, s.O};
            const uint64_t str[2] = {s.P * 4, s.P * s.I * 4};
            const uint32_t box[3] = {32, BK, 1};
            if (encode_tensor_map(&tx, dt, 3, x->data, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) !=
                CUDA_SUCCESS)
                fail(ATK_CUDA_ERROR, "ttm: tensor map (MN-major) encoding failed");
        }
        p.M = s.P * s.O;
        p.P = s.P;
    }
    p.R = int(R);
    p.NB = NB;
    p.nkb = (I + BK - 1) / BK;
    p.a_bytes = MT * BK * 4;
    p.b_bytes = uint32_t(NB) * BK * 4;
    p.stage_bytes = p.a_bytes + p.b_bytes * (split ? 2 : 1);
    p.stages = std::max(2, std::min(8, int((200 * 1024) / p.stage_bytes)));
    p.y = static_cast<float*>(y->data);
    const size_t smem = size_t(p.stages) * p.stage_bytes + 1024 + 256;
    auto kern = kmajor ? ttm_tf32_kernel<true> : ttm_tf32_kernel<false>;
    ATK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const uint64_t ntiles = (p.M + MT - 1) / MT;
    // split-K over I when the M tiles alone leave most SMs idle (C5's last
    // mode: 16 tiles of 4096 x 64 over K = 2048); pieces of >= 8 K-blocks
    p.ks = 1;
    if (ntiles * 2 <= uint64_t(ctx->num_sms) && !std::getenv("ATK_TTM_NOSPLIT"))
        p.ks = int(std::max<uint64_t>(1, std::min<uint64_t>(uint64_t(ctx->num_sms) / ntiles, uint64_t(p.nkb / 8))));
    DevBuf<float> part(ctx, p.ks > 1 ? size_t(p.ks) * p.M * R : 0);
    if (p.ks > 1) p.y = part.get();
    const int grid = int(std::min<uint64_t>(ntiles * p.ks, uint64_t(ctx->num_sms)));
    kern<<<grid, THREADS, smem, ctx->stream>>>(tx, tf, p);
    ATK_LAUNCHED(ctx);
    if (p.ks > 1) {
        const uint64_t n = p.M * R;
        ttm_reduce<<<unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(ctx->num_sms) * 8)), 256, 0,
                     ctx->stream>>>(part.get(), n, p.ks, static_cast<float*>(y->data));
        ATK_LAUNCHED(ctx);
    }
}

}  // namespace atk
