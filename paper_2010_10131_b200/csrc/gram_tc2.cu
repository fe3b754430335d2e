// gram_tc2.cu — the mode-n Gram on CTA PAIRS (tcgen05 cta_group::2).
//
// Same contraction as gram_tc.cu (kernels.hpp:127-138, fp32 storage,
// kind::tf32, TMA TFLOAT32 round-to-nearest, no unfolding) but each 256x256
// output tile is computed by a 2-CTA cluster: CTA c stages rows
// [128c, 128c+128) of the A slab and columns [128c, 128c+128) of the B slab,
// the leader CTA issues one M=256 x N=256 x K=8 UMMA per K-step that reads
// both CTAs' shared memory, and each CTA holds its 128 accumulator rows in its
// own TMEM.  Per SM that halves the operand bytes staged per flop relative to
// the 1-CTA 128x256 tile (32 KB instead of 48 KB per 32-deep K step), which
// moves the kernel off the shared-memory-bandwidth ceiling (TMA writes + UMMA
// reads ~ 192 B/clk/SM > 128 B/clk/SM for 1-CTA tiles).
//
// K is cut into several launches (option "gram_launch_kb": K-blocks per unit
// per launch, default 1024) that accumulate into the same fp32 partial tiles:
// every launch boundary re-aligns the pairs, so their K fronts cannot drift
// apart and each K-block of X is fetched from HBM ~once and served to the
// other tiles from L2.  Measured at I = 2048 (profiles/gram_probe.cu): one
// launch over J = 4M 515-519 TF/s (2.5x HBM re-reads, profiles/r1), launches
// of J = 256K 608 TF/s.  An in-kernel epoch drift bound (leaders wait on a
// global counter) measured slower (40 ms vs 34-38 ms).
//
// Pipeline per CTA: warp 0 = TMA producer (both CTAs; the leader arms the
// leader's full barrier with the bytes of BOTH CTAs, the peer's TMA completes
// on it through the cluster window), warp 1 = TMEM alloc + (leader only) MMA
// issuer, warps 2-5 = epilogue (TMEM -> fp64 partial tile, then a remote
// arrive on the leader's tmem-empty barrier).  Commits are multicast to both
// CTAs' barriers.
#include <algorithm>
#include <vector>

#include "atk_driver.cuh"
#include "tc_common.cuh"

namespace atk {
namespace {

constexpr int TM2 = 256, TN2 = 256, HALF = 128, BK = 32, THREADS = 192;
constexpr uint32_t A_BYTES = HALF * BK * 4, B_BYTES = HALF * BK * 4;
// narrow unit: one 256 x 256 tile, 6 stages of A + B halves (32 KB);
// wide unit: two tiles of one tile row sharing A, 4 stages of A + B0 + B1 (48 KB)
template <bool WIDE>
struct Cfg {
    static constexpr int STAGES = WIDE ? 4 : 6;
    static constexpr uint32_t STAGE_BYTES = A_BYTES + (WIDE ? 2 : 1) * B_BYTES;
    static constexpr size_t SMEM = STAGES * STAGE_BYTES + 1024 + 256;
    static constexpr int NBUF = WIDE ? 1 : 2;  // accumulator buffers in TMEM (2 x 256 columns either way)
};

struct Gram2Params {
    const int4* units;  // {tile_m, tile_n0 | tile_n1 << 16 (0xffff: none), kb_begin, kb_end} in 256-tiles
    int num_units;      // units are dealt to clusters round-robin
    int chunk_kb;
    int kmajor;
    int nkb_p;
    float* acc;         // [slot][TN2][TM2] fp32 partial tiles; unit u owns slots 2u (, 2u + 1)
    int accumulate;     // 1: add into acc (a later K-launch of the same Gram)
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// TMA whose completion is counted on the LEADER CTA's barrier (peer bit cleared).
__device__ __forceinline__ void tma2_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
    const uint32_t b = tc::smem_u32(bar) & 0xFEFFFFFFu;
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(tc::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(b), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void tma2_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                                             int c2) {
    const uint32_t b = tc::smem_u32(bar) & 0xFEFFFFFFu;
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(tc::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(b), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

__device__ __forceinline__ void mma2_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void mma2_commit_mc(uint64_t* bar) {
    const uint16_t mask = 0x3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            tc::smem_u32(bar)),
        "h"(mask)
        : "memory");
}

template <bool WIDE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    gram_tf32_2cta_kernel(const __grid_constant__ CUtensorMap tma_x, const Gram2Params p) {
    constexpr int STAGES2 = Cfg<WIDE>::STAGES;
    constexpr uint32_t STAGE_BYTES = Cfg<WIDE>::STAGE_BYTES;
    constexpr int NBUF = Cfg<WIDE>::NBUF;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES2 * STAGE_BYTES);
    uint64_t* empty = full + STAGES2;
    uint64_t* tfull = empty + STAGES2;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = cluster_rank();
    const bool leader = crank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES2; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&tfull[b], 1);
            tc::mbar_init(&tempty[b], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is the live one)
        }
        tc::fence_barrier_init();
        tc::tma_prefetch(&tma_x);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                     "r"(512u)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc::tc_fence_before();
    cluster_sync();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int u = pair; u < p.num_units; u += npairs) {
                const int4 un = p.units[u];
                const int tn0 = un.y & 0xffff, tn1 = un.y >> 16;
                const bool two = WIDE && tn1 != 0xffff;
                const int arow = un.x * TM2 + int(crank) * HALF, brow = tn0 * TN2 + int(crank) * HALF;
                const int brow1 = two ? tn1 * TN2 + int(crank) * HALF : 0;
                const uint32_t bytes = 2 * (A_BYTES + (two ? 2 : 1) * B_BYTES);  // both CTAs of the pair
                for (int kb = un.z; kb < un.w; ++kb) {
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) tc::mbar_arrive_expect_tx(&full[stage], bytes);
                    uint8_t* a = smem + stage * STAGE_BYTES;
                    uint8_t* b = a + A_BYTES;
                    uint8_t* b1 = b + B_BYTES;
                    if (!p.kmajor) {
                        const int k0 = kb * BK;
#pragma unroll
                        for (int q = 0; q < HALF / 32; ++q) tma2_load_2d(a + q * 4096, &tma_x, &full[stage], arow + q * 32, k0);
#pragma unroll
                        for (int q = 0; q < HALF / 32; ++q) tma2_load_2d(b + q * 4096, &tma_x, &full[stage], brow + q * 32, k0);
                        if (two) {
#pragma unroll
                            for (int q = 0; q < HALF / 32; ++q)
                                tma2_load_2d(b1 + q * 4096, &tma_x, &full[stage], brow1 + q * 32, k0);
                        }
                    } else {
                        const int p0 = (kb % p.nkb_p) * BK, o0 = kb / p.nkb_p;
                        tma2_load_3d(a, &tma_x, &full[stage], p0, o0, arow);
                        tma2_load_3d(b, &tma_x, &full[stage], p0, o0, brow);
                        if (two) tma2_load_3d(b1, &tma_x, &full[stage], p0, o0, brow1);
                    }
                    if (++stage == STAGES2) { stage = 0; phase ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (leader && lane == 0) {
            const uint32_t idesc = tc::idesc_tf32(TM2, TN2, !p.kmajor, !p.kmajor);
            int stage = 0, abuf = 0;
            uint32_t phase = 0, aphase = 0;
            for (int u = pair; u < p.num_units; u += npairs) {
                const int4 un = p.units[u];
                const bool two = WIDE && (un.y >> 16) != 0xffff;
                for (int c0 = un.z; c0 < un.w; c0 += p.chunk_kb) {
                    const int c1 = min(un.w, c0 + p.chunk_kb);
                    tc::mbar_wait(&tempty[abuf], aphase ^ 1);
                    tc::tc_fence_after();
                    const uint32_t d = tmem_base + uint32_t(abuf * TN2);  // WIDE: tile 0 at 0, tile 1 at 256
                    for (int kb = c0; kb < c1; ++kb) {
                        tc::mbar_wait(&full[stage], phase);
                        tc::tc_fence_after();
                        const uint32_t a_base = tc::smem_u32(smem + stage * STAGE_BYTES);
                        const uint32_t b_base = a_base + A_BYTES;
#pragma unroll
                        for (int k = 0; k < BK / 8; ++k) {
                            uint64_t ad, bd, bd1 = 0;
                            if (!p.kmajor) {
                                ad = tc::smem_desc(a_base + k * 1024, 4096, 512, 1);
                                bd = tc::smem_desc(b_base + k * 1024, 4096, 512, 1);
                                if (two) bd1 = tc::smem_desc(b_base + B_BYTES + k * 1024, 4096, 512, 1);
                            } else {
                                ad = tc::smem_desc_sw128(a_base + k * 32, 16, 1024);
                                bd = tc::smem_desc_sw128(b_base + k * 32, 16, 1024);
                                if (two) bd1 = tc::smem_desc_sw128(b_base + B_BYTES + k * 32, 16, 1024);
                            }
                            const uint32_t acc = (kb > c0 || k > 0) ? 1u : 0u;
                            mma2_tf32(d, ad, bd, idesc, acc);
                            if (two) mma2_tf32(d + uint32_t(TN2), ad, bd1, idesc, acc);  // A reused from smem
                        }
                        mma2_commit_mc(&empty[stage]);
                        if (++stage == STAGES2) { stage = 0; phase ^= 1; }
                    }
                    mma2_commit_mc(&tfull[abuf]);
                    if (++abuf == NBUF) { abuf = 0; aphase ^= 1; }
                }
            }
        }
        __syncwarp();
    } else {
        const int q = warp & 3;
        const int row = int(crank) * HALF + q * 32 + lane;  // row within the 256-row tile
        const uint32_t tempty_leader0 = mapa_shared(tc::smem_u32(&tempty[0]), 0);
        const uint32_t tempty_leader1 = mapa_shared(tc::smem_u32(&tempty[1]), 0);
        int abuf = 0;
        uint32_t aphase = 0;
        for (int u = pair; u < p.num_units; u += npairs) {
            const int4 un = p.units[u];
            const int ntile = (WIDE && (un.y >> 16) != 0xffff) ? 2 : 1;
            float* tile = p.acc + size_t(2 * u) * TM2 * TN2;
            for (int c0 = un.z; c0 < un.w; c0 += p.chunk_kb) {
                tc::mbar_wait(&tfull[abuf], aphase);
                tc::tc_fence_after();
                const bool first = !p.accumulate && (c0 == un.z);
#pragma unroll 1
                for (int cc = 0; cc < ntile * (TN2 / 32); ++cc) {  // WIDE: tile 1's columns follow tile 0's
                    uint32_t r[32];
                    tc::tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) + uint32_t(abuf * TN2 + cc * 32), r);
                    tc::tmem_ld_wait();
                    float* dst = tile + size_t(cc * 32) * TM2 + row;  // slot 2u + cc / 8 continues contiguously
                    if (first) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) dst[size_t(j) * TM2] = __uint_as_float(r[j]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j) dst[size_t(j) * TM2] += __uint_as_float(r[j]);
                    }
                }
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(abuf ? tempty_leader1 : tempty_leader0);
                if (++abuf == NBUF) { abuf = 0; aphase ^= 1; }
            }
        }
    }
    tc::tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc::tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512u) : "memory");
    }
}

// S = fixed-order sum of the split partials, mirrored: one 32 x 32 block
// (bi <= bj) per CTA iteration, the mirror written through a shared-memory
// transpose so both stores are coalesced (the direct mirror store was a
// 2048-stride scatter: 33 us per C5 Gram).  Tile (ti, tj), ti <= tj, is the sum
// of slots tslots[(ti nt + tj) smax + k] (k < count, -1 terminated); a tile
// computed transposed (as (tj, ti), to keep every tile row's count even for the
// wide units) is read transposed.
__global__ void __launch_bounds__(256) gram2_reduce(const float* __restrict__ acc, const int* __restrict__ tslots,
                                                    const int* __restrict__ ttrans, int smax, int nt, int I,
                                                    double* __restrict__ s) {
    __shared__ double tb[32][33];
    const int nb = (I + 31) / 32, nblk = nb * (nb + 1) / 2;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
        int bj = int((sqrtf(8.0f * float(b) + 1.0f) - 1.0f) * 0.5f);  // b = bj (bj + 1) / 2 + bi
        while ((bj + 1) * (bj + 2) / 2 <= b) ++bj;
        while (bj * (bj + 1) / 2 > b) --bj;
        const int bi = b - bj * (bj + 1) / 2;
        for (int r = ty; r < 32; r += 8) {
            const int i = 32 * bi + tx, j = 32 * bj + r;  // column j, row i (i fastest)
            double v = 0.0;
            if (i < I && j < I && i <= j) {
                const int t = (i / TM2) * nt + (j / TN2);
                const int* sl = tslots + size_t(t) * smax;
                const size_t off = ttrans[t] ? size_t(i % TM2) * TM2 + (j % TN2) : size_t(j % TN2) * TM2 + (i % TM2);
                for (int k = 0; k < smax && sl[k] >= 0; ++k) v += double(acc[size_t(sl[k]) * TM2 * TN2 + off]);
                s[size_t(i) + size_t(I) * j] = v;
            }
            tb[r][tx] = v;  // tb[j - 32 bj][i - 32 bi]
        }
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {
            const int j = 32 * bj + tx, i = 32 * bi + r;  // mirror: S(j, i) = S(i, j), j fastest
            if (i < I && j < I && i < j) s[size_t(j) + size_t(I) * i] = tb[tx][r];
        }
        __syncthreads();
    }
}

}  // namespace

bool tc_gram2_supported(atk_ctx* ctx, const atk_tensor* x, int mode) {
    if (!ctx->gram_2cta || x->dtype != ATK_F32) return false;
    const Split s = loop_split(x->dims, x->order, mode);
    if (s.I < 512) return false;  // small Grams: the 1-CTA kernel wastes less on the diagonal
    if (s.P == 1) return s.I % 4 == 0 && s.O < (1ull << 31) / BK;
    return s.P >= 32 && s.P % 4 == 0 && s.P * s.I < (1ull << 40) && s.O < (1ull << 31);
}

void tc_gram2(atk_ctx* ctx, const atk_tensor* x, int mode, double* s_dev) {
    const Split s = loop_split(x->dims, x->order, mode);
    const int I = int(s.I);
    const bool kmajor = s.P != 1;
    CUtensorMap tm{};
    const CUtensorMapDataType dt = ctx->tma_tf32 ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    uint64_t nkb;
    int nkb_p = 1;
    if (!kmajor) {
        const uint64_t dims[2] = {s.I, s.O};
        const uint64_t str[1] = {s.I * 4};
        const uint32_t box[2] = {32, BK};
        if (encode_tensor_map(&tm, dt, 2, x->data, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) != CUDA_SUCCESS)
            fail(ATK_CUDA_ERROR, "gram2: tensor map (mode 0) encoding failed");
        nkb = (s.O + BK - 1) / BK;
    } else {
        nkb_p = int((s.P + BK - 1) / BK);
        const uint64_t dims[3] = {s.P, s.O, s.I};
        const uint64_t str[2] = {s.P * s.I * 4, s.P * 4};
        const uint32_t box[3] = {BK, 1, HALF};
        if (encode_tensor_map(&tm, dt, 3, x->data, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
            fail(ATK_CUDA_ERROR, "gram2: tensor map (K-major) encoding failed");
        nkb = uint64_t(nkb_p) * s.O;
    }
    const int nt = (I + TM2 - 1) / TM2;
    const bool wide = ctx->gram_wide != 0;
    // tile rows: the upper triangle (ti <= tj).  Wide units pair two tiles of one
    // row (A staged once, two N = 256 MMAs); a row with an odd count hands one
    // tile (a, b) to another odd row b as its transpose (b, a), so (for an even
    // tile count) every unit is wide.
    std::vector<std::vector<int>> row_tiles(nt);
    std::vector<int> trans(size_t(nt) * nt, 0);
    for (int ti = 0; ti < nt; ++ti)
        for (int tj = ti; tj < nt; ++tj) row_tiles[ti].push_back(tj);
    if (wide) {
        int pend = -1;
        for (int ti = 0; ti < nt; ++ti) {
            if (row_tiles[ti].size() % 2 == 0) continue;
            if (pend < 0) {
                pend = ti;
            } else {  // move tile (pend, ti) to row ti as (ti, pend)
                auto& rp = row_tiles[pend];
                rp.erase(std::find(rp.begin(), rp.end(), ti));
                row_tiles[ti].push_back(pend);
                trans[size_t(pend) * nt + ti] = 1;
                pend = -1;
            }
        }
    }
    struct WUnit {
        int tm, tn0, tn1;
    };
    std::vector<WUnit> wu;
    for (int ti = 0; ti < nt; ++ti) {
        const auto& rt = row_tiles[ti];
        for (size_t q = 0; q < rt.size(); q += wide ? 2 : 1)
            wu.push_back({ti, rt[q], (wide && q + 1 < rt.size()) ? rt[q + 1] : 0xffff});
    }
    const int nwu = int(wu.size());
    if (wide) {
        static bool attr_w = false;
        if (!attr_w) {
            ATK_CUDA(cudaFuncSetAttribute(gram_tf32_2cta_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(Cfg<true>::SMEM)));
            attr_w = true;
        }
    } else {
        static bool attr_n = false;
        if (!attr_n) {
            ATK_CUDA(cudaFuncSetAttribute(gram_tf32_2cta_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(Cfg<false>::SMEM)));
            attr_n = true;
        }
    }
    // CTA pairs that are co-resident (GPCs with an odd SM count leave SMs unused)
    static int pairs_resident[2] = {0, 0};
    int& pr = pairs_resident[wide ? 1 : 0];
    if (!pr) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2 * (ctx->num_sms / 2), 1, 1);
        cfg.blockDim = dim3(THREADS, 1, 1);
        cfg.dynamicSmemBytes = wide ? Cfg<true>::SMEM : Cfg<false>::SMEM;
        cudaLaunchAttribute at{};
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = 2;
        at.val.clusterDim.y = 1;
        at.val.clusterDim.z = 1;
        cfg.attrs = &at;
        cfg.numAttrs = 1;
        int nc = 0;
        const cudaError_t e = wide ? cudaOccupancyMaxActiveClusters(&nc, gram_tf32_2cta_kernel<true>, &cfg)
                                   : cudaOccupancyMaxActiveClusters(&nc, gram_tf32_2cta_kernel<false>, &cfg);
        if (e != cudaSuccess || nc <= 0) {
            cudaGetLastError();
            nc = ctx->num_sms / 2;
        }
        pr = std::min(nc, ctx->num_sms / 2);
    }
    const int pairs_avail = pr;
    // split-K: every unit into the same number of K pieces, as many as keep one wave
    int splits = std::max(1, pairs_avail / nwu);
    splits = int(std::min<uint64_t>(uint64_t(splits), std::max<uint64_t>(1, nkb / 8)));
    const int chunk_kb = ctx->gram_chunk_kb > 0 ? ctx->gram_chunk_kb : 512;
    std::vector<int4> units;
    const int smax = splits;
    std::vector<int> tslots(size_t(nt) * nt * smax, -1);
    for (int w = 0; w < nwu; ++w) {
        for (int sp = 0; sp < splits; ++sp) {
            const int kb0 = int(nkb * sp / splits), kb1 = int(nkb * (sp + 1) / splits);
            const int u = int(units.size());
            units.push_back(make_int4(wu[w].tm, wu[w].tn0 | (wu[w].tn1 << 16), kb0, std::max(kb0 + 1, kb1)));
            for (int t = 0; t < (wu[w].tn1 != 0xffff ? 2 : 1); ++t) {
                const int tn = t ? wu[w].tn1 : wu[w].tn0;
                const int a = std::min(wu[w].tm, tn), b = std::max(wu[w].tm, tn);  // upper-triangle tile id
                tslots[(size_t(a) * nt + b) * smax + sp] = 2 * u + t;
            }
        }
    }
    DevBuf<int4> du(ctx, units.size());
    DevBuf<int> dts(ctx, tslots.size()), dtr(ctx, trans.size());
    DevBuf<float> acc(ctx, units.size() * 2 * size_t(TM2) * TN2);
    ATK_CUDA(cudaMemcpyAsync(du.get(), units.data(), units.size() * sizeof(int4), cudaMemcpyHostToDevice, ctx->stream));
    ATK_CUDA(cudaMemcpyAsync(dts.get(), tslots.data(), tslots.size() * sizeof(int), cudaMemcpyHostToDevice,
                             ctx->stream));
    ATK_CUDA(cudaMemcpyAsync(dtr.get(), trans.data(), trans.size() * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    const int npairs = std::min<int>(int(units.size()), pairs_avail);
    Gram2Params prm{du.get(), int(units.size()), chunk_kb, kmajor ? 1 : 0, nkb_p, acc.get(), 0};
    // K-launches: unit u's K range [kb0, kb1) is walked in slices of launch_kb
    // K-blocks, one launch per slice index (all units advance together)
    int launch_kb = ctx->gram_launch_kb > 0 ? ctx->gram_launch_kb : (1 << 30);
    if (wide && ctx->gram_launch_kb > 0) launch_kb = std::max(1, launch_kb / 2);  // same bytes per launch
    int max_len = 0;
    for (const int4& u : units) max_len = std::max(max_len, u.w - u.z);
    const int nlaunch = (max_len + launch_kb - 1) / launch_kb;
    DevBuf<int4> dlu(ctx, nlaunch > 1 ? units.size() * size_t(nlaunch) : 0);
    if (nlaunch > 1) {
        std::vector<int4> all;
        all.reserve(units.size() * size_t(nlaunch));
        for (int L = 0; L < nlaunch; ++L)
            for (const int4& u : units) {
                const int a = std::min(u.w, u.z + L * launch_kb), b = std::min(u.w, a + launch_kb);
                all.push_back(make_int4(u.x, u.y, a, b));
            }
        ATK_CUDA(cudaMemcpyAsync(dlu.get(), all.data(), all.size() * sizeof(int4), cudaMemcpyHostToDevice,
                                 ctx->stream));
    }
    for (int L = 0; L < nlaunch; ++L) {
        if (nlaunch > 1) {
            prm.units = dlu.get() + size_t(L) * units.size();
            prm.accumulate = L > 0 ? 1 : 0;
        }
        if (wide)
            gram_tf32_2cta_kernel<true><<<2 * npairs, THREADS, Cfg<true>::SMEM, ctx->stream>>>(tm, prm);
        else
            gram_tf32_2cta_kernel<false><<<2 * npairs, THREADS, Cfg<false>::SMEM, ctx->stream>>>(tm, prm);
        ATK_LAUNCHED(ctx);
    }
    const int nb32 = (I + 31) / 32;
    gram2_reduce<<<unsigned(std::min(nb32 * (nb32 + 1) / 2, ctx->num_sms * 8)), 256, 0, ctx->stream>>>(
        acc.get(), dts.get(), dtr.get(), smax, nt, I, s_dev);
    ATK_LAUNCHED(ctx);
}

}  // namespace atk
