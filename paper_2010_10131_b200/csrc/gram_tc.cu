// gram_tc.cu — matricization-free mode-n Gram on the 5th-gen tensor cores.
//
// S = X_(n) X_(n)^T (kernels.hpp:127-138) for fp32 storage, computed as
// tcgen05.mma kind::tf32 with fp32 accumulators in TMEM, operands staged by
// TMA straight from the strided tensor (no unfolding):
//   mode 0 (P == 1)   X is I x J column-major: both operands MN-major
//                     (2-D tensor map {I, J}, 32x32 boxes, SWIZZLE_128B);
//   P >= 32, P%4 == 0 X viewed as (p, o, i) through a permuted 3-D tensor map
//                     {P, O, I} with strides {P*I, P}: a box of 32 p lands as
//                     one 128-byte K-major row per i (SWIZZLE_128B).
// Work = upper-triangle 128x256 tiles x split-K ranges, persistent CTAs.
// Warp roles (192 threads): warp 0 TMA producer, warp 1 TMEM alloc + MMA
// issuer (one elected lane), warps 2-5 epilogue.  The accumulator is
// double-buffered in TMEM (2 x 256 columns) and drained every `chunk`
// K-blocks into a per-unit fp64 tile in global memory (bounded fp32 chains,
// SURVEY H3); a final kernel sums the split-K partials in a fixed order and
// mirrors the upper triangle => deterministic and exactly symmetric.
#include <algorithm>
#include <vector>

#include "atk_driver.cuh"
#include "tc_common.cuh"

namespace atk {
namespace {

constexpr int BM = 128, BN = 256, BK = 32;
constexpr uint32_t A_BYTES = BM * BK * 4, B_BYTES = BN * BK * 4;
constexpr int THREADS = 192;
// Ring geometry.  Small mode (I <= 128, mode 0 or the P in {4, 8, 16} panels: C4's 48-wide modes,
// the R x R Grams): the
// single diagonal tile's A and B are the same rows, so ONE operand tile (ceil(I / 32) TMA boxes
// of 4 KB) is staged per K-block and read as both A and B (N = I rounded up to 32): 12 stages
// of 16 KB keep ~3x more bytes in flight than the general 4 x 48 KB ring, whose stages were
// mostly zero fill at I = 48 (C4 mode 0 at 26 % of HBM).
template <bool SMALL>
struct Ring {
    static constexpr int STAGES = SMALL ? 12 : 4;
    static constexpr uint32_t STAGE_BYTES = SMALL ? A_BYTES : A_BYTES + B_BYTES;
    static constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES + 1024 + 256;
};

struct GramParams {
    const int4* units;  // {tile_m, tile_n, kb_begin, kb_end}
    int num_units;
    int chunk_kb;       // K-blocks accumulated in TMEM before an fp64 drain
    int kmajor;         // 0: MN-major mode-0 map, 1: permuted 3-D K-major map
    int nkb_p;          // K-major: K-blocks per o (= ceil(P / 32))
    int panel;          // 1: P in {4, 8, 16}: unswizzled K-major 16-byte panels (4-D map {4, I, P/4, O})
    int opb;            // panel mode: o values per K-block (32 / P)
    double* acc;        // [unit][BN][BM] fp64 partial tiles
    uint32_t* progress; // [gridDim.x] K-blocks issued per CTA (drift limiter), or null
    int slack_kb;       // allowed lead over the slowest CTA, in K-blocks
    int small_boxes;    // small mode: 32-row TMA boxes per K-block (ceil(I / 32))
    int small_n;        // small mode: MMA N (I rounded up to whole 32-element MN-major atoms)
};

template <bool SMALL>
__global__ void __launch_bounds__(THREADS, 1)
    gram_tf32_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                     const GramParams p) {
    constexpr int STAGES = Ring<SMALL>::STAGES;
    constexpr uint32_t STAGE_BYTES = Ring<SMALL>::STAGE_BYTES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&tfull[b], 1);
            tc::mbar_init(&tempty[b], 4);
        }
        tc::fence_barrier_init();
        tc::tma_prefetch(&tma_a);
        tc::tma_prefetch(&tma_b);
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        // Drift limiter: every CTA publishes how many K-blocks it has issued;
        // a CTA more than `slack` blocks ahead of the slowest one waits.  All
        // CTAs then stream through X in near lockstep, so each K-block is read
        // from HBM once and served to the other tiles from L2 (measured 4.2x
        // HBM re-reads without it, profiles/r1).
        if (lane == 0) {
        uint32_t issued = 0;
        const uint32_t slack = uint32_t(p.slack_kb);
        int stage = 0;
        uint32_t phase = 0;
        for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
            const int4 un = p.units[u];
            for (int kb = un.z; kb < un.w; ++kb) {
                if (p.progress && (issued & 15u) == 0) {
                    p.progress[blockIdx.x] = issued;
                    uint32_t spins = 0;
                    for (;;) {
                        uint32_t mn = 0xffffffffu;
                        for (int j = 0; j < int(gridDim.x); ++j) mn = min(mn, ((volatile uint32_t*)p.progress)[j]);
                        if (mn + slack >= issued || ++spins > 200000) break;
                        __nanosleep(256);
                    }
                }
                ++issued;
                {
                    // half units: only the right 128 columns of the 256-wide tile are
                    // on/above the diagonal -> load and multiply just those
                    const int tm = un.x & 0xffff, half = un.x >> 16;
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* a = smem + stage * STAGE_BYTES;
                    uint8_t* b = a + A_BYTES;
                    if (SMALL) {  // one operand tile
                        if (!p.kmajor) {  // MN-major: rows 0 .. 32 boxes - 1
                            tc::mbar_arrive_expect_tx(&full[stage], uint32_t(p.small_boxes) * 4096u);
                            for (int q = 0; q < p.small_boxes; ++q)
                                tc::tma_load_2d(a + q * 4096, &tma_a, &full[stage], q * 32, kb * BK);
                        } else {  // 16-B panels: one 4-D box of BM rows (zero fill past I)
                            tc::mbar_arrive_expect_tx(&full[stage], A_BYTES);
                            tc::tma_load_4d(a, &tma_a, &full[stage], 0, 0, 0, kb * p.opb);
                        }
                    } else {
                    tc::mbar_arrive_expect_tx(&full[stage], half ? A_BYTES + B_BYTES / 2 : A_BYTES + B_BYTES);
                    if (!p.kmajor) {
                        const int k0 = kb * BK;
#pragma unroll
                        for (int q = 0; q < BM / 32; ++q)
                            tc::tma_load_2d(a + q * 4096, &tma_a, &full[stage], tm * BM + q * 32, k0);
                        const int q0 = half == 1 ? BN / 64 : 0, q1 = half == 2 ? BN / 64 : BN / 32;
                        for (int q = q0; q < q1; ++q)
                            tc::tma_load_2d(b + (q - q0) * 4096, &tma_a, &full[stage], un.y * BN + q * 32, k0);
                    } else {
                        if (p.panel) {  // K-block = 32/P whole o slabs: panels [o][p_hi][row][4 p]
                            const int o0 = kb * p.opb;
                            tc::tma_load_4d(a, &tma_a, &full[stage], 0, tm * BM, 0, o0);
                            if (half)
                                tc::tma_load_4d(b, &tma_a, &full[stage], 0, un.y * BN + (half == 1 ? BN / 2 : 0), 0, o0);
                            else
                                tc::tma_load_4d(b, &tma_b, &full[stage], 0, un.y * BN, 0, o0);
                        } else {
                            const int p0 = (kb % p.nkb_p) * BK, o0 = kb / p.nkb_p;
                            tc::tma_load_3d(a, &tma_a, &full[stage], p0, o0, tm * BM);
                            if (half) tc::tma_load_3d(b, &tma_a, &full[stage], p0, o0, un.y * BN + (half == 1 ? BN / 2 : 0));
                            else tc::tma_load_3d(b, &tma_b, &full[stage], p0, o0, un.y * BN);
                        }
                    }
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
        if (p.progress) p.progress[blockIdx.x] = 0xffffffffu;  // never hold others back
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc_full = SMALL ? tc::idesc_tf32(BM, p.small_n, !p.kmajor, !p.kmajor)
                                              : tc::idesc_tf32(BM, BN, !p.kmajor, !p.kmajor);
            const uint32_t idesc_half = SMALL ? idesc_full : tc::idesc_tf32(BM, BN / 2, !p.kmajor, !p.kmajor);
            int stage = 0, abuf = 0;
            uint32_t phase = 0, aphase = 0;
            for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
                const int4 un = p.units[u];
                const uint32_t idesc = (un.x >> 16) ? idesc_half : idesc_full;
                const uint32_t bpanel = (un.x >> 16) ? BM * 16 : BN * 16;  // panel mode: B rows x 16 B
                for (int c0 = un.z; c0 < un.w; c0 += p.chunk_kb) {
                    const int c1 = min(un.w, c0 + p.chunk_kb);
                    tc::mbar_wait(&tempty[abuf], aphase ^ 1);
                    tc::tc_fence_after();
                    const uint32_t d = tmem_base + uint32_t(abuf * BN);
                    for (int kb = c0; kb < c1; ++kb) {
                        tc::mbar_wait(&full[stage], phase);
                        tc::tc_fence_after();
                        const uint32_t a_base = tc::smem_u32(smem + stage * STAGE_BYTES);
                        const uint32_t b_base = a_base + A_BYTES;
#pragma unroll
                        for (int k = 0; k < BK / 8; ++k) {
                            uint64_t ad, bd;
                            if (SMALL) {  // A and B: the same staged rows
                                ad = !p.kmajor ? tc::smem_desc(a_base + k * 1024, 4096, 512, 1)
                                               : tc::smem_desc(a_base + k * 2 * (BM * 16), BM * 16, 128, 0);
                                bd = ad;
                            } else if (!p.kmajor) {
                                // MN-major tf32: 128B/32B-atom swizzle, 4-row K groups (SBO 512 B),
                                // 32-element MN blocks one TMA box apart (LBO 4 KB)
                                ad = tc::smem_desc(a_base + k * 1024, 4096, 512, 1);
                                bd = tc::smem_desc(b_base + k * 1024, 4096, 512, 1);
                            } else if (p.panel) {
                                // no swizzle, K-major: 8-row x 16-B core matrices, K-adjacent
                                // ones a panel apart (LBO), M/N-adjacent ones 128 B apart (SBO)
                                ad = tc::smem_desc(a_base + k * 2 * (BM * 16), BM * 16, 128, 0);
                                bd = tc::smem_desc(b_base + k * 2 * bpanel, bpanel, 128, 0);
                            } else {
                                ad = tc::smem_desc_sw128(a_base + k * 32, 16, 1024);
                                bd = tc::smem_desc_sw128(b_base + k * 32, 16, 1024);
                            }
                            tc::mma_tf32(d, ad, bd, idesc, (kb > c0 || k > 0) ? 1u : 0u);
                        }
                        tc::mma_commit(&empty[stage]);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    tc::mma_commit(&tfull[abuf]);
                    if (++abuf == 2) { abuf = 0; aphase ^= 1; }
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ epilogue: TMEM -> fp64 tile
        const int q = warp & 3;
        const int row = q * 32 + lane;
        int abuf = 0;
        uint32_t aphase = 0;
        for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
            const int4 un = p.units[u];
            double* tile = p.acc + size_t(u) * BM * BN;
            for (int c0 = un.z; c0 < un.w; c0 += p.chunk_kb) {
                tc::mbar_wait(&tfull[abuf], aphase);
                tc::tc_fence_after();
                const bool first = (c0 == un.z);
                // half units: mode 1 fills columns 128..255, mode 2 columns 0..127
                const int cc0 = SMALL ? 0 : ((un.x >> 16) == 1 ? BN / 64 : 0);
                const int cc1 = SMALL ? (p.small_n + 31) / 32 : ((un.x >> 16) == 2 ? BN / 64 : BN / 32);
#pragma unroll 1
                for (int cc = cc0; cc < cc1; ++cc) {
                    uint32_t r[32];
                    tc::tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) +
                                               uint32_t(abuf * BN + (cc - cc0) * 32), r);
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
        tc::tmem_dealloc(tmem_base, 512);
    }
}

// S(i, j) = S(j, i) = sum_s acc[unit(tile(i, j), s)](i, j) for i <= j.
__global__ void gram_reduce(const double* __restrict__ acc, const int* __restrict__ tile_unit,
                            int splits, int ntn, int I, double* __restrict__ s) {
    const size_t n = size_t(I) * I;
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += size_t(gridDim.x) * blockDim.x) {
        const int i = int(e % I), j = int(e / I);
        if (i > j) continue;
        const int tm = i / BM, tn = j / BN;
        const int u0 = tile_unit[tm * ntn + tn];
        const size_t off = size_t(j % BN) * BM + (i % BM);
        double v = 0.0;
        for (int k = 0; k < splits; ++k) v += acc[size_t(u0 + k) * BM * BN + off];
        s[size_t(i) + size_t(I) * j] = v;
        s[size_t(j) + size_t(I) * i] = v;
    }
}

// Small Grams (I <= 256, many split partials: C4's 48 x 5.3M): 32 lanes per
// element, lane t sums splits t, t+32, ... in order, then a fixed xor tree.  The
// one-thread-per-element loop was a chain of ~150 L2 round trips (34 us at I = 48).
__global__ void gram_reduce_lanes(const double* __restrict__ acc, const int* __restrict__ tile_unit, int splits,
                                  int ntn, int I, double* __restrict__ s) {
    const size_t gid = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t e = gid >> 5;
    const int t = int(gid & 31);
    const size_t n = size_t(I) * I;
    const int i = e < n ? int(e % I) : 0, j = e < n ? int(e / I) : 0;
    const bool live = e < n && i <= j;
    double v = 0.0;
    if (live) {
        const int u0 = tile_unit[(i / BM) * ntn + (j / BN)];
        const size_t off = size_t(j % BN) * BM + (i % BM);
        for (int k = t; k < splits; k += 32) v += acc[size_t(u0 + k) * BM * BN + off];
    }
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (live && t == 0) {
        s[size_t(i) + size_t(I) * j] = v;
        s[size_t(j) + size_t(I) * i] = v;
    }
}

}  // namespace

CUresult encode_tensor_map(CUtensorMap* map, CUtensorMapDataType dt, uint32_t rank, void* base,
                           const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box,
                           CUtensorMapSwizzle swz) {
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p)
            fail(ATK_CUDA_ERROR, "cuTensorMapEncodeTiled entry point unavailable");
        fn = reinterpret_cast<Fn>(p);
    }
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    return fn(map, dt, rank, base, reinterpret_cast<const cuuint64_t*>(dims),
              reinterpret_cast<const cuuint64_t*>(strides_bytes), reinterpret_cast<const cuuint32_t*>(box), estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

static bool gram_tc_layout_ok(const atk_tensor* x, int mode) {
    if (x->dtype != ATK_F32) return false;
    const Split s = loop_split(x->dims, x->order, mode);
    // small I (ALS R x R Grams, C4's 48-wide modes): still tensor cores, on a
    // half-width 128 x 128 tile (the SIMT path ran C4 mode 1 at 4.4 ms vs 0.16 HBM)
    if (s.I < 8) return false;
    if (s.P == 1) return s.I % 4 == 0 && s.O < (1ull << 31) / BK;
    const bool panel = s.P == 4 || s.P == 8 || s.P == 16;  // unswizzled 16-B panels, 32/P o per K-block
    return (s.P >= 32 || panel) && s.P % 4 == 0 && s.P * s.I < (1ull << 40) && s.O < (1ull << 31);
}

bool tc_gram_supported(atk_ctx* ctx, const atk_tensor* x, int mode) {
    (void)ctx;
    return gram_tc_layout_ok(x, mode);
}

void tc_gram(atk_ctx* ctx, const atk_tensor* x, int mode, double* s_dev) {
    const Split s = loop_split(x->dims, x->order, mode);
    const int I = int(s.I);
    const bool kmajor = s.P != 1;
    CUtensorMap ta{}, tb{};
    const CUtensorMapDataType dt = ctx->tma_tf32 ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    uint64_t nkb;
    int nkb_p = 1, panel = 0, opb = 1;
    if (!kmajor) {
        const uint64_t K = s.O;
        const uint64_t dims[2] = {s.I, K};
        const uint64_t str[1] = {s.I * 4};
        const uint32_t box[2] = {32, BK};
        if (encode_tensor_map(&ta, dt, 2, x->data, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) !=
            CUDA_SUCCESS)
            fail(ATK_CUDA_ERROR, "gram: tensor map (mode 0) encoding failed");
        tb = ta;
        nkb = (K + BK - 1) / BK;
    } else if (s.P < 32) {
        // 4-D map {4 p_lo, I, P/4 p_hi, O}: box {4, rows, P/4, 32/P} lands as 8 panels of
        // rows x 16 B, i.e. unswizzled K-major core matrices (8 rows x 16 B) for tcgen05
        panel = 1;
        opb = int(BK / s.P);
        const uint64_t dims[4] = {4, s.I, s.P / 4, s.O};
        const uint64_t str[3] = {s.P * 4, 16, s.P * s.I * 4};
        const uint32_t boxa[4] = {4, BM, uint32_t(s.P / 4), uint32_t(opb)};
        const uint32_t boxb[4] = {4, BN, uint32_t(s.P / 4), uint32_t(opb)};
        if (encode_tensor_map(&ta, dt, 4, x->data, dims, str, boxa, CU_TENSOR_MAP_SWIZZLE_NONE) != CUDA_SUCCESS ||
            encode_tensor_map(&tb, dt, 4, x->data, dims, str, boxb, CU_TENSOR_MAP_SWIZZLE_NONE) != CUDA_SUCCESS)
            fail(ATK_CUDA_ERROR, "gram: tensor map (panel) encoding failed");
        nkb = (s.O + opb - 1) / opb;
    } else {
        nkb_p = int((s.P + BK - 1) / BK);
        const uint64_t dims[3] = {s.P, s.O, s.I};
        const uint64_t str[2] = {s.P * s.I * 4, s.P * 4};
        const uint32_t boxa[3] = {BK, 1, BM};
        const uint32_t boxb[3] = {BK, 1, BN};
        if (encode_tensor_map(&ta, dt, 3, x->data, dims, str, boxa, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS ||
            encode_tensor_map(&tb, dt, 3, x->data, dims, str, boxb, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
            fail(ATK_CUDA_ERROR, "gram: tensor map (K-major) encoding failed");
        nkb = uint64_t(nkb_p) * s.O;
    }
    // upper-triangle tiles: (tm, tn) is needed iff tm*BM <= tn*BN + BN - 1
    const int ntm = (I + BM - 1) / BM, ntn = (I + BN - 1) / BN;
    std::vector<int> tiles_m, tiles_n;
    for (int tn = 0; tn < ntn; ++tn)
        for (int tm = 0; tm < ntm; ++tm)
            if (tm * BM <= tn * BN + BN - 1) {
                tiles_m.push_back(tm);
                tiles_n.push_back(tn);
            }
    const int ntiles = int(tiles_m.size());
    int splits = std::max(1, ctx->num_sms / ntiles);  // floor: units <= CTAs (one wave)
    splits = int(std::min<uint64_t>(uint64_t(splits), std::max<uint64_t>(1, nkb / 8)));
    const int chunk_kb = ctx->gram_chunk_kb > 0 ? ctx->gram_chunk_kb : 512;  // 16K-element fp32 chains
    std::vector<int4> units;
    std::vector<int> tile_unit(size_t(ntm) * ntn, 0);
    for (int t = 0; t < ntiles; ++t) {
        tile_unit[size_t(tiles_m[t]) * ntn + tiles_n[t]] = int(units.size());
        for (int sp = 0; sp < splits; ++sp) {
            const int kb0 = int(nkb * sp / splits), kb1 = int(nkb * (sp + 1) / splits);
            // half-width units (N = 128): mode 1 when the left 128 columns lie entirely
            // below the diagonal, mode 2 when the right 128 columns lie beyond I
            const int half = (tiles_m[t] * BM >= tiles_n[t] * BN + BN / 2) ? 1
                             : (I <= tiles_n[t] * BN + BN / 2)              ? 2
                                                                            : 0;
            units.push_back(make_int4(tiles_m[t] | (half << 16), tiles_n[t], kb0, std::max(kb0 + 1, kb1)));
        }
    }
    // guard: a split may be empty only when nkb < splits (excluded above)
    DevBuf<int4> du(ctx, units.size());
    DevBuf<int> dtu(ctx, tile_unit.size());
    DevBuf<double> acc(ctx, units.size() * size_t(BM) * BN);
    ATK_CUDA(cudaMemcpyAsync(du.get(), units.data(), units.size() * sizeof(int4), cudaMemcpyHostToDevice, ctx->stream));
    ATK_CUDA(cudaMemcpyAsync(dtu.get(), tile_unit.data(), tile_unit.size() * sizeof(int), cudaMemcpyHostToDevice,
                             ctx->stream));
    const int grid = std::min<int>(int(units.size()), ctx->num_sms);
    DevBuf<uint32_t> progress(ctx, size_t(grid));
    ATK_CUDA(cudaMemsetAsync(progress.get(), 0, size_t(grid) * sizeof(uint32_t), ctx->stream));
    // L2 window per in-flight K-block: I rows x 32 fp32 x (#split streams); keep the
    // lockstep window well inside the 126 MB L2.
    const double kb_bytes = double(I) * BK * 4.0 * splits;
    const int slack = int(std::max(8.0, std::min(256.0, 32e6 / kb_bytes)));
    const bool small = (!kmajor || panel) && I <= 128 && ntiles == 1 && !ctx->gram_lockstep && ctx->gram_small;
    GramParams prm{du.get(), int(units.size()), chunk_kb, kmajor ? 1 : 0, nkb_p, panel, opb, acc.get(),
                   ctx->gram_lockstep ? progress.get() : nullptr, slack, (I + 31) / 32, (I + 31) / 32 * 32};
    static bool attr = false;
    if (!attr) {
        ATK_CUDA(cudaFuncSetAttribute(gram_tf32_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(Ring<false>::SMEM)));
        ATK_CUDA(cudaFuncSetAttribute(gram_tf32_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(Ring<true>::SMEM)));
        attr = true;
    }
    if (small)
        gram_tf32_kernel<true><<<grid, THREADS, Ring<true>::SMEM, ctx->stream>>>(ta, tb, prm);
    else
        gram_tf32_kernel<false><<<grid, THREADS, Ring<false>::SMEM, ctx->stream>>>(ta, tb, prm);
    ATK_LAUNCHED(ctx);
    const size_t n = size_t(I) * I;
    if (I <= 256 && splits >= 8)
        gram_reduce_lanes<<<unsigned((n * 32 + 255) / 256), 256, 0, ctx->stream>>>(acc.get(), dtu.get(), splits, ntn,
                                                                                  I, s_dev);
    else
        gram_reduce<<<unsigned(std::min<size_t>((n + 255) / 256, size_t(ctx->num_sms) * 8)), 256, 0, ctx->stream>>>(
            acc.get(), dtu.get(), splits, ntn, I, s_dev);
    ATK_LAUNCHED(ctx);
}

}  // namespace atk
