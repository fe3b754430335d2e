// ttt_tc.cu — the ALS contraction YR = Y_(n) rfac_(n)^T on the tensor cores.
//
// kernels::ttt_mode (kernels.hpp:122-124) as used by als_iterate
// (solvers.hpp:107): Z (I x R) = sum_k X(k, i) Y(k, r), k = (p, o), with
// X the big work tensor (fp32) and Y = rfac (same dims but R along mode n).
// tcgen05.mma kind::tf32, M = 128 rows of I per tile, N = R padded to 32
// (R <= 128), split-K over J so the HBM-bound stream of X fills every SM;
// TMA (TFLOAT32, round-to-nearest) stages both operands straight from the
// tensors: MN-major for mode 0, the permuted K-major 3-D map otherwise.
// fp32 accumulation in TMEM is drained every `chunk` K-blocks into per-unit
// fp64 partial tiles; a fixed-order reduction sums the splits.
#include <algorithm>
#include <vector>

#include "atk_driver.cuh"
#include "tc_common.cuh"

namespace atk {
namespace {

constexpr int BM = 128, BK = 32, THREADS = 192;

struct TttParams {
    const int4* units;  // {tile_m, 0, kb_begin, kb_end}
    int num_units;
    int chunk_kb;
    int kmajor;
    int nkb_p;
    int nb;             // padded N (multiple of 32, <= 128)
    int stages;
    uint32_t a_bytes, stage_bytes;
    double* acc;        // [unit][nb][BM]
};

__global__ void __launch_bounds__(THREADS, 1)
    ttt_tf32_kernel(const __grid_constant__ CUtensorMap tma_x, const __grid_constant__ CUtensorMap tma_y,
                    const TttParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(S) * p.stage_bytes);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tcols = (2 * p.nb <= 64) ? 64 : (2 * p.nb <= 128 ? 128 : 256);

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
        tc::tma_prefetch(&tma_y);
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
            for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
                const int4 un = p.units[u];
                for (int kb = un.z; kb < un.w; ++kb) {
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    tc::mbar_arrive_expect_tx(&full[stage], p.stage_bytes);
                    uint8_t* a = smem + size_t(stage) * p.stage_bytes;
                    uint8_t* b = a + p.a_bytes;
                    if (!p.kmajor) {
                        const int k0 = kb * BK;
                        for (int q = 0; q < BM / 32; ++q)
                            tc::tma_load_2d(a + q * 4096, &tma_x, &full[stage], un.x * BM + q * 32, k0);
                        for (int q = 0; q < p.nb / 32; ++q) tc::tma_load_2d(b + q * 4096, &tma_y, &full[stage], q * 32, k0);
                    } else {
                        const int p0 = (kb % p.nkb_p) * BK, o0 = kb / p.nkb_p;
                        tc::tma_load_3d(a, &tma_x, &full[stage], p0, o0, un.x * BM);
                        tc::tma_load_3d(b, &tma_y, &full[stage], p0, o0, 0);
                    }
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = tc::idesc_tf32(BM, p.nb, !p.kmajor, !p.kmajor);
            int stage = 0, abuf = 0;
            uint32_t phase = 0, aphase = 0;
            for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
                const int4 un = p.units[u];
                for (int c0 = un.z; c0 < un.w; c0 += p.chunk_kb) {
                    const int c1 = min(un.w, c0 + p.chunk_kb);
                    tc::mbar_wait(&tempty[abuf], aphase ^ 1);
                    tc::tc_fence_after();
                    const uint32_t d = tmem_base + uint32_t(abuf * p.nb);
                    for (int kb = c0; kb < c1; ++kb) {
                        tc::mbar_wait(&full[stage], phase);
                        tc::tc_fence_after();
                        const uint32_t a_base = tc::smem_u32(smem + size_t(stage) * p.stage_bytes);
                        const uint32_t b_base = a_base + p.a_bytes;
#pragma unroll
                        for (int k = 0; k < BK / 8; ++k) {
                            uint64_t ad, bd;
                            if (!p.kmajor) {
                                ad = tc::smem_desc(a_base + k * 1024, 4096, 512, 1);
                                bd = tc::smem_desc(b_base + k * 1024, 4096, 512, 1);
                            } else {
                                ad = tc::smem_desc_sw128(a_base + k * 32, 16, 1024);
                                bd = tc::smem_desc_sw128(b_base + k * 32, 16, 1024);
                            }
                            tc::mma_tf32(d, ad, bd, idesc, (kb > c0 || k > 0) ? 1u : 0u);
                        }
                        tc::mma_commit(&empty[stage]);
                        if (++stage == S) { stage = 0; phase ^= 1; }
                    }
                    tc::mma_commit(&tfull[abuf]);
                    if (++abuf == 2) { abuf = 0; aphase ^= 1; }
                }
            }
        }
        __syncwarp();
    } else {
        const int q = warp & 3;
        const int row = q * 32 + lane;
        int abuf = 0;
        uint32_t aphase = 0;
        for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
            const int4 un = p.units[u];
            double* tile = p.acc + size_t(u) * BM * p.nb;
            for (int c0 = un.z; c0 < un.w; c0 += p.chunk_kb) {
                tc::mbar_wait(&tfull[abuf], aphase);
                tc::tc_fence_after();
                const bool first = (c0 == un.z);
#pragma unroll 1
                for (int cc = 0; cc < p.nb / 32; ++cc) {
                    uint32_t r[32];
                    tc::tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) + uint32_t(abuf * p.nb + cc * 32), r);
                    tc::tmem_ld_wait();
                    double* dst = tile + size_t(cc * 32) * BM + row;
                    if (first) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) dst[size_t(j) * BM] = double(__uint_as_float(r[j]));
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j) dst[size_t(j) * BM] += double(__uint_as_float(r[j]));
                    }
                }
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&tempty[abuf]);
                if (++abuf == 2) { abuf = 0; aphase ^= 1; }
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, tcols);
    }
}

// Z(i, r) = sum_s acc[tile(i) * splits + s](i % BM, r)
__global__ void ttt_reduce(const double* __restrict__ acc, int splits, int nb, int I, int R, double* __restrict__ z) {
    const size_t n = size_t(I) * R;
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += size_t(gridDim.x) * blockDim.x) {
        const int i = int(e % I), r = int(e / I);
        const int u0 = (i / BM) * splits;
        const size_t off = size_t(r) * BM + (i % BM);
        double v = 0.0;
        for (int k = 0; k < splits; ++k) v += acc[size_t(u0 + k) * BM * nb + off];
        z[e] = v;
    }
}

}  // namespace

bool tc_ttt_ns_supported(atk_ctx* ctx, const atk_tensor* x, const atk_tensor* y, int mode) {
    if (ctx->force_simt || x->dtype != ATK_F32 || y->dtype != ATK_F32) return false;
    const Split s = loop_split(x->dims, x->order, mode);
    const uint64_t R = y->dims[mode];
    if (s.I < 128 || R < 1 || R > 128) return false;
    if (s.P == 1) return s.I % 4 == 0 && R % 4 == 0 && s.O < (1ull << 31) / BK;
    return s.P >= 32 && s.P % 4 == 0 && s.P * s.I < (1ull << 40) && s.O < (1ull << 31);
}

void tc_ttt_ns(atk_ctx* ctx, const atk_tensor* x, const atk_tensor* y, int mode, double* z_dev) {
    const Split s = loop_split(x->dims, x->order, mode);
    const int I = int(s.I), R = int(y->dims[mode]);
    const int nb = (R + 31) / 32 * 32;
    const bool kmajor = s.P != 1;
    const CUtensorMapDataType dt = ctx->tma_tf32 ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    CUtensorMap tx{}, ty{};
    uint64_t nkb;
    int nkb_p = 1;
    if (!kmajor) {
        const uint64_t dx[2] = {s.I, s.O}, sx[1] = {s.I * 4};
        const uint64_t dy[2] = {uint64_t(R), s.O}, sy[1] = {uint64_t(R) * 4};
        const uint32_t box[2] = {32, BK};
        if (encode_tensor_map(&tx, dt, 2, x->data, dx, sx, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) != CUDA_SUCCESS ||
            encode_tensor_map(&ty, dt, 2, y->data, dy, sy, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) != CUDA_SUCCESS)
            fail(ATK_CUDA_ERROR, "ttt: tensor map (mode 0) encoding failed");
        nkb = (s.O + BK - 1) / BK;
    } else {
        nkb_p = int((s.P + BK - 1) / BK);
        const uint64_t dx[3] = {s.P, s.O, s.I}, sx[2] = {s.P * s.I * 4, s.P * 4};
        const uint64_t dy[3] = {s.P, s.O, uint64_t(R)}, sy[2] = {s.P * uint64_t(R) * 4, s.P * 4};
        const uint32_t bx[3] = {BK, 1, BM}, by[3] = {BK, 1, uint32_t(nb)};
        if (encode_tensor_map(&tx, dt, 3, x->data, dx, sx, bx, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS ||
            encode_tensor_map(&ty, dt, 3, y->data, dy, sy, by, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
            fail(ATK_CUDA_ERROR, "ttt: tensor map (K-major) encoding failed");
        nkb = uint64_t(nkb_p) * s.O;
    }
    const int ntm = (I + BM - 1) / BM;
    // floor: units <= CTAs.  Rounding up left a few CTAs with two units, i.e. a
    // second wave (measured 1.18 ms instead of ~0.7 at C2 mode 1, 152 units / 148 SMs)
    int splits = std::max(1, ctx->num_sms / ntm);
    splits = int(std::min<uint64_t>(uint64_t(splits), std::max<uint64_t>(1, nkb / 8)));
    std::vector<int4> units;
    for (int t = 0; t < ntm; ++t)
        for (int sp = 0; sp < splits; ++sp) {
            const int kb0 = int(nkb * sp / splits), kb1 = int(nkb * (sp + 1) / splits);
            units.push_back(make_int4(t, 0, kb0, std::max(kb0 + 1, kb1)));
        }
    DevBuf<int4> du(ctx, units.size());
    DevBuf<double> acc(ctx, units.size() * size_t(BM) * nb);
    ATK_CUDA(cudaMemcpyAsync(du.get(), units.data(), units.size() * sizeof(int4), cudaMemcpyHostToDevice, ctx->stream));
    TttParams prm{};
    prm.units = du.get();
    prm.num_units = int(units.size());
    prm.chunk_kb = ctx->gram_chunk_kb > 0 ? ctx->gram_chunk_kb : 512;
    prm.kmajor = kmajor ? 1 : 0;
    prm.nkb_p = nkb_p;
    prm.nb = nb;
    prm.a_bytes = BM * BK * 4;
    prm.stage_bytes = prm.a_bytes + uint32_t(nb) * BK * 4;
    prm.stages = std::max(2, std::min(8, int((200 * 1024) / prm.stage_bytes)));
    prm.acc = acc.get();
    const size_t smem = size_t(prm.stages) * prm.stage_bytes + 1024 + 256;
    ATK_CUDA(cudaFuncSetAttribute(ttt_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const int grid = std::min<int>(int(units.size()), ctx->num_sms);
    ttt_tf32_kernel<<<grid, THREADS, smem, ctx->stream>>>(tx, ty, prm);
    ATK_LAUNCHED(ctx);
    const size_t n = size_t(I) * R;
    ttt_reduce<<<unsigned(std::min<size_t>((n + 255) / 256, size_t(ctx->num_sms) * 8)), 256, 0, ctx->stream>>>(
        acc.get(), splits, nb, I, R, z_dev);
    ATK_LAUNCHED(ctx);
}

}  // namespace atk
