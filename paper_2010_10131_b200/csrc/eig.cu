// eig.cu — linalg::sym_eig_top_r (linalg.hpp:101-123) on the device, fp64.
//
// The reference computes ALL eigenpairs with Eigen's SelfAdjointEigenSolver
// and keeps the top r.  On the device (eig_method -1):
//   n <= 200 : the tridiagonal solver (tridiag.cu); one-sided Jacobi
//              (jacobi.cu) as eig_method 0 for n <= 112;
//   n  > 200 : Chebyshev-filtered subspace iteration (ChFSI) on a block of
//              k = r + max(16, r/4) vectors:
//                bounds  : lo = 0 for PSD input; otherwise one m = 40 Lanczos
//                          run on a cluster (S resident in 16 CTAs' shared
//                          memory when it fits) + bisection / inverse
//                          iteration on its tridiagonal;
//                filter  : T_d on [lo, cut] (scaled recurrence, fp64 DMMA,
//                          one cooperative launch per pass, dgemm.cu), on
//                          the unconverged Ritz vectors with S deflated by
//                          the locked (converged) pairs;
//                orthonormalisation : shifted CholeskyQR3 (GEMMs + one-CTA
//                          Cholesky); SVQB if a pivot still fails;
//                Rayleigh-Ritz : tridiagonal solver on V^T S V;
//              until every wanted Ritz pair has relative residual
//              ||S v - theta v|| <= tol * max|theta| (tol 1e-12 for fp64
//              data, 1e-9 for tf32-computed Grams).
// Both paths finish with descending order + fix_signs (linalg.hpp:34-50) so
// factors compare entry-wise with the reference on gapped spectra.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "atk_internal.cuh"

namespace atk {
namespace {

inline unsigned nblk(size_t n) { return unsigned(std::min<size_t>((n + 255) / 256, 4096)); }

// ------------------------------------------------------------------ grid barrier
__device__ __forceinline__ void grid_sync(unsigned* count, unsigned* gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* vg = gen;
        const unsigned g = *vg;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*vg == g) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ double block_sum3(double& a, double& b, double& c, double* sh) {
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (l == 0) {
        sh[w] = a;
        sh[32 + w] = b;
        sh[64 + w] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double x = 0, y = 0, z = 0;
        for (int i = 0; i < nw; ++i) {
            x += sh[i];
            y += sh[32 + i];
            z += sh[64 + i];
        }
        sh[96] = x;
        sh[97] = y;
        sh[98] = z;
    }
    __syncthreads();
    a = sh[96];
    b = sh[97];
    c = sh[98];
    return a;
}

// The same m-step Lanczos on ONE 8-CTA cluster: hardware cluster barriers
// (~0.2 us) instead of a 148-CTA software grid barrier (~25 us measured), an
// fp32 copy of S (bounds only; halves the L2 traffic) and q staged in smem.
constexpr int kLzCluster = 8, kLzThreads = 512;

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(kLzCluster, 1, 1) __launch_bounds__(kLzThreads)
    lanczos_cluster(const float* __restrict__ S, int n, int m, double* __restrict__ q, double* __restrict__ qprev,
                    double* __restrict__ w, double* __restrict__ part, double* __restrict__ alpha,
                    double* __restrict__ beta) {
    extern __shared__ double qs[];  // n doubles
    __shared__ double sh[100];
    const int G = kLzCluster, cb = blockIdx.x;
    const int r0 = int(int64_t(cb) * n / G), r1 = int(int64_t(cb + 1) * n / G);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    double bprev = 0.0;
    for (int j = 0; j < m; ++j) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) qs[i] = q[i];
        __syncthreads();
        // four rows per warp at a time, 4 column chunks each: 16 independent
        // 16-byte L2 loads in flight per lane
        int rbase = r0 + warp * 4;
        if ((n & 3) == 0)
            for (; rbase + 3 < r1; rbase += nw * 4) {
                const float* c0p = S + size_t(n) * rbase;
                double acc[4] = {0, 0, 0, 0};
                for (int c = lane * 4; c < n; c += 4 * 128) {
                    float4 v[4][4];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int rr = 0; rr < 4; ++rr)
                            v[rr][u] = (c + u * 128 < n) ? *reinterpret_cast<const float4*>(c0p + size_t(n) * rr + c + u * 128)
                                                         : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int cc = c + u * 128;
                        if (cc >= n) break;
                        const double q0 = qs[cc], q1 = qs[cc + 1], q2 = qs[cc + 2], q3 = qs[cc + 3];
#pragma unroll
                        for (int rr = 0; rr < 4; ++rr)
                            acc[rr] += double(v[rr][u].x) * q0 + double(v[rr][u].y) * q1 + double(v[rr][u].z) * q2 +
                                       double(v[rr][u].w) * q3;
                    }
                }
#pragma unroll
                for (int rr = 0; rr < 4; ++rr) {
                    double t = acc[rr];
                    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
                    if (lane == 0) w[rbase + rr] = t;
                }
            }
        // leftover rows (and n % 4 != 0): one row per warp
        for (int r = ((n & 3) == 0 ? rbase : r0 + warp); r < r1; r += ((n & 3) == 0 ? 1 : nw)) {
            if ((n & 3) == 0 && r >= rbase + 4) break;
            const float* col = S + size_t(n) * r;  // S symmetric: row r == column r
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int c = lane * 4;
            if ((n & 3) == 0) {
                // 8 independent 16-byte loads in flight per lane (one chain of L2
                // round trips per row measured 80 us per Lanczos step)
                for (; c + 7 * 128 < n; c += 8 * 128) {
                    float4 v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = *reinterpret_cast<const float4*>(col + c + u * 128);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int cc = c + u * 128;
                        s0 = fma(double(v[u].x), qs[cc], s0);
                        s1 = fma(double(v[u].y), qs[cc + 1], s1);
                        s2 = fma(double(v[u].z), qs[cc + 2], s2);
                        s3 = fma(double(v[u].w), qs[cc + 3], s3);
                    }
                }
                for (; c < n; c += 128) {
                    const float4 v = *reinterpret_cast<const float4*>(col + c);
                    s0 = fma(double(v.x), qs[c], s0);
                    s1 = fma(double(v.y), qs[c + 1], s1);
                    s2 = fma(double(v.z), qs[c + 2], s2);
                    s3 = fma(double(v.w), qs[c + 3], s3);
                }
            } else {
                for (c = lane; c < n; c += 32) s0 = fma(double(col[c]), qs[c], s0);
            }
            double t = (s0 + s1) + (s2 + s3);
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (lane == 0) w[r] = t;
        }
        __syncthreads();
        double ww = 0, wq = 0, wp = 0;
        for (int r = r0 + int(threadIdx.x); r < r1; r += blockDim.x) {
            ww += w[r] * w[r];
            wq += w[r] * qs[r];
            wp += w[r] * qprev[r];
        }
        block_sum3(ww, wq, wp, sh);
        if (threadIdx.x == 0) {
            part[3 * cb] = ww;
            part[3 * cb + 1] = wq;
            part[3 * cb + 2] = wp;
        }
        cluster_sync_all();
        double tw = 0, tq = 0, tp = 0;
        for (int i = 0; i < G; ++i) {  // fixed order => identical on every CTA
            tw += part[3 * i];
            tq += part[3 * i + 1];
            tp += part[3 * i + 2];
        }
        const double a = tq;
        const double bb = tw - 2.0 * a * tq - 2.0 * bprev * tp + a * a + bprev * bprev;
        const double b = bb > 0 ? sqrt(bb) : 0.0;
        const double inv = b > 0 ? 1.0 / b : 0.0;
        for (int r = r0 + int(threadIdx.x); r < r1; r += blockDim.x) {
            const double nv = (w[r] - a * qs[r] - bprev * qprev[r]) * inv;
            qprev[r] = qs[r];
            q[r] = nv;
        }
        if (cb == 0 && threadIdx.x == 0) {
            alpha[j] = a;
            beta[j] = b;
        }
        bprev = b;
        cluster_sync_all();
    }
}

// The same m-step Lanczos with S RESIDENT in the shared memory of one
// 16-CTA cluster (n <= ~1250): the lower triangle as 32 x 32 fp32 tiles
// (padded to 32 x 33: conflict-free by rows and by columns), tile t of the
// row-major order (I, J <= I) on CTA t / per.  Per step a warp forms, for
// each of its tiles, the row part T q_J (-> y_I) and the column part T^T q_I
// (-> y_J) from smem only; the owner of each row block B (the CTA holding
// tile (B, B)) then sums the nb partials that land on B through DSMEM in a
// fixed order (bit-reproducible).  The previous kernel re-read S from L2
// every step (~11.5 us per step at n = 1024 on 8 SMs).
constexpr int kLtCluster = 16, kLtThreads = 1024, kLtLd = 33;

__device__ __forceinline__ uint32_t lt_mapa(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                 : "=r"(r)
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))), "r"(rank));
    return r;
}
__device__ __forceinline__ float lt_ld_remote(uint32_t addr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}

__device__ __forceinline__ double lt_ld_remote_d(uint32_t addr) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
}

__device__ __forceinline__ void lt_tile_of(int t, int& I, int& J) {  // t = I (I + 1) / 2 + J
    int i = int((sqrtf(8.0f * float(t) + 1.0f) - 1.0f) * 0.5f);
    while ((i + 1) * (i + 2) / 2 <= t) ++i;
    while (i * (i + 1) / 2 > t) --i;
    I = i;
    J = t - i * (i + 1) / 2;
}

__global__ void __launch_bounds__(kLtThreads) lanczos_tiles(const double* __restrict__ S, int n, int m, int per,
                                                            double* __restrict__ q, double* __restrict__ alpha,
                                                            double* __restrict__ beta) {
    extern __shared__ __align__(16) float lsm[];
    const int nb = (n + 31) / 32, ntiles = nb * (nb + 1) / 2;
    const int cb = int(blockIdx.x);  // rank in the cluster (grid = one cluster)
    const int t0 = cb * per, t1 = min(ntiles, t0 + per);
    float* tiles = lsm;                       // per x 32 x 33
    float* rowp = tiles + size_t(per) * 32 * kLtLd;  // per x 32: T q_J of each tile
    float* colp = rowp + per * 32;            // per x 32: T^T q_I
    float* qf = colp + per * 32;              // nb x 32, fp32 copy of q
    __shared__ double sh[100];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    // stage this CTA's tiles: S column-major, lanes down a column (coalesced)
    for (int t = t0 + warp; t < t1; t += nw) {
        int I, J;
        lt_tile_of(t, I, J);
        float* T = tiles + size_t(t - t0) * 32 * kLtLd;
        const int r = 32 * I + lane;
        for (int c0 = 0; c0 < 32; c0 += 16) {  // 16 loads in flight per lane
            double v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int cc = 32 * J + c0 + u;
                v[u] = (r < n && cc < n) ? S[r + size_t(n) * cc] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) T[lane * kLtLd + c0 + u] = float(v[u]);
        }
    }
    __shared__ double cpart[3];  // this CTA's {w.w, w.q, w.qprev}, read by the cluster
    __shared__ double tot[3];
    // row blocks owned here: B with tile (B, B) in [t0, t1); warp w <-> the w-th
    int bfirst = nb, bcount = 0;
    for (int B = 0; B < nb; ++B) {
        const int td = B * (B + 1) / 2 + B;
        if (td >= t0 && td < t1) {
            bfirst = min(bfirst, B);
            ++bcount;
        }
    }
    const int myB = warp < bcount ? bfirst + warp : -1;
    const int row = myB >= 0 ? 32 * myB + lane : n;
    double qi = row < n ? q[row] : 0.0, qpi = 0.0, bprev = 0.0;
    for (int j = 0; j < m; ++j) {
        // L2 reads (__ldcg): q and part are rewritten by the other CTAs every step
        for (int i = threadIdx.x; i < nb * 32; i += blockDim.x) qf[i] = i < n ? float(__ldcg(q + i)) : 0.0f;
        __syncthreads();
        for (int t = t0 + warp; t < t1; t += nw) {
            int I, J;
            lt_tile_of(t, I, J);
            const float* T = tiles + size_t(t - t0) * 32 * kLtLd;
            const float* qJ = qf + 32 * J;
            const float* qI = qf + 32 * I;
            float rs0 = 0.f, rs1 = 0.f, cs0 = 0.f, cs1 = 0.f;
#pragma unroll
            for (int c = 0; c < 32; c += 2) {
                rs0 = fmaf(T[lane * kLtLd + c], qJ[c], rs0);
                rs1 = fmaf(T[lane * kLtLd + c + 1], qJ[c + 1], rs1);
            }
            if (I != J) {
#pragma unroll
                for (int r = 0; r < 32; r += 2) {
                    cs0 = fmaf(T[r * kLtLd + lane], qI[r], cs0);
                    cs1 = fmaf(T[(r + 1) * kLtLd + lane], qI[r + 1], cs1);
                }
            }
            rowp[(t - t0) * 32 + lane] = rs0 + rs1;
            colp[(t - t0) * 32 + lane] = cs0 + cs1;
        }
        cluster_sync_all();  // every CTA's partials are final
        double w = 0.0;
        if (myB >= 0) {
            // y_B = sum_{J <= B} rowp(B, J) + sum_{I > B} colp(I, B): nb DSMEM
            // loads, all in flight, summed in a fixed order
            const int base = myB * (myB + 1) / 2;
            for (int s0 = 0; s0 < nb; s0 += 16) {
                float v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int s = s0 + u;  // s <= B: rowp(B, s); s > B: colp(s, B)
                    const int t = s <= myB ? base + s : s * (s + 1) / 2 + myB;
                    const float* src = (s <= myB ? rowp : colp) + (t % per) * 32 + lane;
                    v[u] = s < nb ? lt_ld_remote(lt_mapa(src, t / per)) : 0.0f;
                }
#pragma unroll
                for (int u = 0; u < 16; ++u) w += double(v[u]);
            }
        }
        double ww = w * w, wq = w * qi, wp = w * qpi;
        block_sum3(ww, wq, wp, sh);
        if (threadIdx.x == 0) {
            cpart[0] = ww;
            cpart[1] = wq;
            cpart[2] = wp;
        }
        cluster_sync_all();
        // the 16 CTA triples over DSMEM, one per lane, summed in rank order
        if (warp == 0) {
            double x0 = 0, x1 = 0, x2 = 0;
            if (lane < kLtCluster) {
                x0 = lt_ld_remote_d(lt_mapa(&cpart[0], lane));
                x1 = lt_ld_remote_d(lt_mapa(&cpart[1], lane));
                x2 = lt_ld_remote_d(lt_mapa(&cpart[2], lane));
            }
            double tw = 0, tq = 0, tp = 0;
            for (int i = 0; i < kLtCluster; ++i) {
                tw += __shfl_sync(0xffffffffu, x0, i);
                tq += __shfl_sync(0xffffffffu, x1, i);
                tp += __shfl_sync(0xffffffffu, x2, i);
            }
            if (lane == 0) {
                tot[0] = tw;
                tot[1] = tq;
                tot[2] = tp;
            }
        }
        __syncthreads();
        const double tw = tot[0], tq = tot[1], tp = tot[2];
        const double a = tq;
        const double bb = tw - 2.0 * a * tq - 2.0 * bprev * tp + a * a + bprev * bprev;
        const double b = bb > 0 ? sqrt(bb) : 0.0;
        const double inv = b > 0 ? 1.0 / b : 0.0;
        if (row < n) {
            const double nv = (w - a * qi - bprev * qpi) * inv;
            qpi = qi;
            qi = nv;
            q[row] = nv;
        }
        if (cb == 0 && threadIdx.x == 0) {
            alpha[j] = a;
            beta[j] = b;
        }
        bprev = b;
        cluster_sync_all();
    }
}

// smem bytes of lanczos_tiles for n, or 0 when the triangle does not fit
inline size_t lanczos_tiles_smem(int n, int& per) {
    const int nb = (n + 31) / 32, ntiles = nb * (nb + 1) / 2;
    per = (ntiles + kLtCluster - 1) / kLtCluster;
    const size_t bytes = (size_t(per) * 32 * kLtLd + 2 * size_t(per) * 32 + size_t(nb) * 32) * sizeof(float);
    return bytes <= 220 * 1024 ? bytes : 0;
}

__global__ void to_f32(const double* __restrict__ a, size_t n, float* __restrict__ b) {
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += size_t(gridDim.x) * blockDim.x)
        b[e] = float(a[e]);
}

__global__ void fill_normalish(double* __restrict__ v, size_t n, uint64_t seed) {
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += size_t(gridDim.x) * blockDim.x) {
        uint64_t x = (e + 1) * 0x9e3779b97f4a7c15ULL ^ seed;
        x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
        x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
        x ^= x >> 31;
        v[e] = double(int64_t(x >> 11) - (int64_t(1) << 52)) * (1.0 / 4503599627370496.0);
    }
}

__global__ void scale_vec(double* v, int n, const double* nrm2) {
    const double s = *nrm2 > 0 ? 1.0 / sqrt(*nrm2) : 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] *= s;
}

__global__ void dot_self(const double* v, int n, double* out) {
    __shared__ double sh[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += v[i] * v[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int i = 0; i < int(blockDim.x >> 5); ++i) t += sh[i];
        *out = t;
    }
}

// ynew = g1 * y + g2 * yprev  (elementwise; dgemm then adds a * S y)
__global__ void cheb_combine(double* __restrict__ ynew, const double* __restrict__ y,
                             const double* __restrict__ yprev, size_t n, double g1, double g2) {
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += size_t(gridDim.x) * blockDim.x)
        ynew[e] = g1 * y[e] + (yprev ? g2 * yprev[e] : 0.0);
}

// res[j] = || W(:, j) - theta_j V(:, j) ||, j < r   (one CTA per column, a
// fixed-order block sum; one warp per column was a 64-deep chain of L2
// round trips at n = 2048)
__global__ void __launch_bounds__(256) ritz_residual(const double* __restrict__ w, const double* __restrict__ v,
                                                     const double* __restrict__ theta, int n, int r,
                                                     double* __restrict__ res) {
    __shared__ double sh[8];
    const int col = blockIdx.x;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const double th = theta[col];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double d = w[i + size_t(n) * col] - th * v[i + size_t(n) * col];
        s = fma(d, d, s);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) sh[wp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < int(blockDim.x >> 5); ++q) t += sh[q];
        res[col] = sqrt(t);
    }
}

// SVQB step 1: d_i = 1/sqrt(G_ii); G <- D G D.
__global__ void svqb_scale(double* g, int k, double* d) {
    __shared__ double sd[128];
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        const double gi = g[i + size_t(k) * i];
        sd[i] = gi > 0 ? 1.0 / sqrt(gi) : 0.0;
        d[i] = sd[i];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) g[e] *= sd[e % k] * sd[e / k];
}

// SVQB step 2: M = D Z Theta^{-1/2}, eigenvalues clamped at tau * theta_max.
__global__ void svqb_form(const double* d, const double* z, const double* th, int k, double tau, double* mm) {
    const double tmax = th[0];
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int i = e % k, j = e / k;
        const double t = fmax(th[j], tau * tmax);
        mm[e] = t > 0 ? d[i] * z[e] / sqrt(t) : 0.0;
    }
}

struct Bounds {
    double lo, hi;
};

struct Ws {
    DevBuf<double> G, Z, th, d, M, tmp;
    DevBuf<int> sweeps;
    DevBuf<int> info;  // 3 Cholesky status words
};

// G += s I with s = 11 (m k + k (k+1)) u ||Y||_F^2  (shifted CholeskyQR, Fukaya et al.)
__global__ void add_shift(double* g, int k, int m) {
    __shared__ double tr;
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < k; ++i) t += g[i + size_t(k) * i];
        tr = t;
    }
    __syncthreads();
    const double s = 11.0 * (double(m) * k + double(k) * (k + 1)) * 1.1102230246251565e-16 * tr;
    for (int i = threadIdx.x; i < k; i += blockDim.x) g[i + size_t(k) * i] += s;
}

// X = L^{-T} (upper triangular) from the lower Cholesky factor L; one thread per column.
__global__ void chol_inv_t(const double* __restrict__ l, int k, double* __restrict__ x) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= k) return;
    double* xc = x + size_t(k) * j;
    for (int i = k - 1; i >= 0; --i) {
        if (i > j) {
            xc[i] = 0.0;
            continue;
        }
        double s = (i == j) ? 1.0 : 0.0;
        for (int t = i + 1; t <= j; ++t) s -= l[t + size_t(k) * i] * xc[t];
        xc[i] = s / l[i + size_t(k) * i];
    }
}

// Orthonormal basis of span(Y) into V (n x k): SVQB twice.
void svqb(atk_ctx* ctx, const double* Y, int n, int k, double* V, Ws& ws) {
    const double* src = Y;
    for (int pass = 0; pass < 2; ++pass) {
        double* dst = (pass == 0) ? V : ws.tmp.get();
        dgemm(ctx, true, false, k, k, n, 1.0, src, n, src, n, 0.0, ws.G.get(), k);
        svqb_scale<<<1, 256, 0, ctx->stream>>>(ws.G.get(), k, ws.d.get());
        ATK_LAUNCHED(ctx);
        jacobi_eig(ctx, ws.G.get(), k, k, ws.th.get(), ws.Z.get(), k, ws.sweeps.get(), true);
        svqb_form<<<1, 256, 0, ctx->stream>>>(ws.d.get(), ws.Z.get(), ws.th.get(), k, 1e-13, ws.M.get());
        ATK_LAUNCHED(ctx);
        dgemm(ctx, false, false, n, k, k, 1.0, src, n, ws.M.get(), k, 0.0, dst, n);
        src = dst;
    }
    ATK_CUDA(cudaMemcpyAsync(V, ws.tmp.get(), size_t(n) * k * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
}

// Shifted CholeskyQR3 (three GEMM-based passes, the first with a diagonal
// shift so a moderately ill-conditioned Y cannot break it down; Fukaya et al.).
// Returns false if a Cholesky pivot still failed (V is then unusable).
// cholqr3_async enqueues the passes and leaves the pivot status of each in
// ws.info[0..2] for the caller's next synchronisation (ChFSI reads it with its
// residuals: no host round trip of its own).
void cholqr3_async(atk_ctx* ctx, const double* Y, int n, int k, double* V, Ws& ws) {
    const double* src = Y;
    double* bufs[2] = {V, ws.tmp.get()};
    for (int pass = 0; pass < 3; ++pass) {
        double* dst = bufs[pass & 1];
        dgemm(ctx, true, false, k, k, n, 1.0, src, n, src, n, 0.0, ws.G.get(), k);
        if (pass == 0) {
            add_shift<<<1, 128, 0, ctx->stream>>>(ws.G.get(), k, n);
            ATK_LAUNCHED(ctx);
        } else if (std::getenv("ATK_TRACE_QR")) {  // orthogonality defect entering this pass
            std::vector<double> g(size_t(k) * k);
            ATK_CUDA(cudaStreamSynchronize(ctx->stream));
            ATK_CUDA(cudaMemcpy(g.data(), ws.G.get(), g.size() * sizeof(double), cudaMemcpyDeviceToHost));
            double mx = 0.0;
            for (int c = 0; c < k; ++c)
                for (int r = 0; r < k; ++r) mx = std::max(mx, std::fabs(g[r + size_t(k) * c] - (r == c ? 1.0 : 0.0)));
            std::fprintf(stderr, "[atk cholqr n=%d k=%d] pass %d: max|G - I| = %.3e\n", n, k, pass, mx);
        }
        // the third pass is the identity when the second already left the block
        // orthonormal to ~1e-16 (C2's filtered blocks, measured); then X = I and
        // the apply below is an exact copy
        cholesky_inv_t(ctx, ws.G.get(), k, ws.M.get(), ws.info.get() + pass, pass == 2 ? 1e-14 : 0.0);
        dgemm(ctx, false, false, n, k, k, 1.0, src, n, ws.M.get(), k, 0.0, dst, n);
        src = dst;
    }
    // result of pass 2 is in bufs[0] == V
}

bool cholqr3(atk_ctx* ctx, const double* Y, int n, int k, double* V, Ws& ws) {
    cholqr3_async(ctx, Y, n, k, V, ws);
    int h[3] = {0, 0, 0};
    ATK_CUDA(cudaMemcpyAsync(h, ws.info.get(), 3 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ATK_CUDA(cudaStreamSynchronize(ctx->stream));
    return !(h[0] || h[1] || h[2]);
}

// Orthonormal basis of span(Y) into V: shifted CholeskyQR3, SVQB if a
// Cholesky pivot still fails.
void orthonormalize(atk_ctx* ctx, const double* Y, int n, int k, double* V, Ws& ws) {
    if (!cholqr3(ctx, Y, n, k, V, ws)) svqb(ctx, Y, n, k, V, ws);
}

// S re-read from L2 each step (any n whose q fits in smem): the fp32 copy of S
// and the 8-CTA cluster kernel above.
void lanczos_l2(atk_ctx* ctx, const double* S, int n, int m, double* q, double* qp, double* w, double* part,
                double* al, double* be) {
    cudaStream_t st = ctx->stream;
    DevBuf<float> s32(ctx, size_t(n) * n);
    to_f32<<<nblk(size_t(n) * n), 256, 0, st>>>(S, size_t(n) * n, s32.get());
    ATK_LAUNCHED(ctx);
    const size_t smem = size_t(n) * sizeof(double);
    static bool attr = false;
    if (!attr) {
        ATK_CUDA(cudaFuncSetAttribute(lanczos_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    if (smem > 200 * 1024) fail(ATK_UNSUPPORTED, "lanczos: n too large for the staged vector");
    lanczos_cluster<<<kLzCluster, kLzThreads, smem, st>>>(s32.get(), n, m, q, qp, w, part, al, be);
    ATK_LAUNCHED(ctx);
}

Bounds lanczos_bounds(atk_ctx* ctx, const double* S, int n, bool psd) {
    cudaStream_t st = ctx->stream;
    const int m = std::min(n, 40);
    DevBuf<double> q(ctx, n), qp(ctx, n), w(ctx, n), part(ctx, 3 * kLzCluster), al(ctx, m),
        be(ctx, m), tv(ctx, m), tz(ctx, 2 * size_t(m)), nrm(ctx, 1);
    ATK_CUDA(cudaMemsetAsync(qp.get(), 0, n * sizeof(double), st));
    fill_normalish<<<nblk(n), 256, 0, st>>>(q.get(), n, 0x5eed1234ULL);
    ATK_LAUNCHED(ctx);
    dot_self<<<1, 256, 0, st>>>(q.get(), n, nrm.get());
    ATK_LAUNCHED(ctx);
    scale_vec<<<nblk(n), 256, 0, st>>>(q.get(), n, nrm.get());
    ATK_LAUNCHED(ctx);
    int per = 0;
    const size_t tsmem = lanczos_tiles_smem(n, per);
    static int tiles_ok = -1;  // 16-CTA clusters with this smem schedulable?
    if (tsmem && tiles_ok < 0) {
        tiles_ok = 0;
        if (cudaFuncSetAttribute(lanczos_tiles, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
            cudaFuncSetAttribute(lanczos_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024) ==
                cudaSuccess) {
            cudaLaunchConfig_t cfg{};
            cudaLaunchAttribute at{};
            at.id = cudaLaunchAttributeClusterDimension;
            at.val.clusterDim.x = kLtCluster;
            at.val.clusterDim.y = at.val.clusterDim.z = 1;
            cfg.gridDim = dim3(kLtCluster);
            cfg.blockDim = dim3(kLtThreads);
            cfg.dynamicSmemBytes = 220 * 1024;
            cfg.attrs = &at;
            cfg.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, lanczos_tiles, &cfg) == cudaSuccess && nclusters > 0)
                tiles_ok = 1;
        }
        cudaGetLastError();  // clear a refused attribute / query
    }
    if (tsmem && tiles_ok == 1 && ctx->lanczos_tiles) {
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute at{};
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = kLtCluster;
        at.val.clusterDim.y = at.val.clusterDim.z = 1;
        cfg.gridDim = dim3(kLtCluster);
        cfg.blockDim = dim3(kLtThreads);
        cfg.dynamicSmemBytes = tsmem;
        cfg.stream = st;
        cfg.attrs = &at;
        cfg.numAttrs = 1;
        ATK_CUDA(cudaLaunchKernelEx(&cfg, lanczos_tiles, static_cast<const double*>(S), n, m, per, q.get(), al.get(),
                                    be.get()));
        ATK_LAUNCHED(ctx);
    } else {
        lanczos_l2(ctx, S, n, m, q.get(), qp.get(), w.get(), part.get(), al.get(), be.get());
    }
    // T is tridiagonal already: bisection + inverse iteration on (alpha, beta)
    // directly (the dense Jacobi on T took ~0.3 ms)
    tridiag_extreme_eig(ctx, al.get(), be.get(), m, tv.get(), tz.get());
    std::vector<double> hv(m), hb(m), zlast(2);
    ATK_CUDA(cudaMemcpyAsync(hv.data(), tv.get(), m * sizeof(double), cudaMemcpyDeviceToHost, st));
    ATK_CUDA(cudaMemcpyAsync(hb.data(), be.get(), m * sizeof(double), cudaMemcpyDeviceToHost, st));
    // last components of the extreme Ritz vectors (columns 0: top, 1: bottom)
    ATK_CUDA(cudaMemcpy2DAsync(zlast.data(), sizeof(double), tz.get() + (m - 1), size_t(m) * sizeof(double),
                               sizeof(double), 2, cudaMemcpyDeviceToHost, st));
    ATK_CUDA(cudaStreamSynchronize(st));
    const double bm = std::fabs(hb[m - 1]);
    Bounds b{hv[m - 1] - bm * std::fabs(zlast[1]) - 1e-12 * std::fabs(hv[0]), hv[0] + bm * std::fabs(zlast[0])};
    if (psd) b.lo = std::max(b.lo, 0.0);
    return b;
}

// Rayleigh-Ritz on the orthonormal block V (n x k): W = S V, T = V^T W,
// theta = all k Ritz values (descending), Z = the top nv Ritz vectors of T
// (nv = r, or k when converged pairs are being locked);
// Vk = V Z (n x nv), Wr = W Z (n x r, for the residuals).
void rayleigh_ritz(atk_ctx* ctx, const double* S, int n, int k, int r, int nv, const double* V, double* W,
                   double* T, double* Z, double* theta, double* Vk, double* Wr, int* sweeps, bool psd) {
    dgemm(ctx, false, false, n, k, n, 1.0, S, n, V, n, 0.0, W, n);
    dgemm(ctx, true, false, k, k, n, 1.0, V, n, W, n, 0.0, T, k);
    if (ctx->eig_method == 0)
        jacobi_eig(ctx, T, k, k, theta, Z, k, sweeps, psd);  // V^T S V is PSD when S is; all k vectors
    else
        tridiag_eig(ctx, T, k, k, nv, theta, Z, k, k);
    dgemm(ctx, false, false, n, nv, k, 1.0, V, n, Z, k, 0.0, Vk, n);
    dgemm(ctx, false, false, n, r, k, 1.0, W, n, Z, k, 0.0, Wr, n);
}

// M(:, j) = (theta_j - sigma) L(:, j), j < nc: the deflation term of S - L diag(theta - sigma) L^T
__global__ void scale_cols_shift(const double* __restrict__ l, const double* __restrict__ theta, double sigma,
                                 int n, int nc, double* __restrict__ m) {
    const size_t tot = size_t(n) * nc;
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += size_t(gridDim.x) * blockDim.x)
        m[e] = (theta[e / n] - sigma) * l[e];
}

}  // namespace

// ------------------------------------------------------------------ scaling
// Eigen's SelfAdjointEigenSolver (linalg.hpp:108) divides the matrix by max|a_ij| before it
// tridiagonalises, so squares of huge or tiny entries (Householder norms, Sturm counts, S^2
// products) neither overflow nor underflow.  Here S is scaled in place by a power of two (exact)
// only when max|S| lies outside [2^-200, 2^200], so ordinary inputs are untouched bit for bit;
// fac[0] = the factor the eigenvalues are multiplied back by (1 when untouched).
namespace {
constexpr int kScT = 256;
__global__ void __launch_bounds__(kScT) eig_maxabs_kernel(const double* __restrict__ s, int n, int diag_only,
                                                          double* __restrict__ fac) {
    __shared__ double red[kScT / 32];
    double m = 0.0;
    const size_t tot = diag_only ? size_t(n) : size_t(n) * n;
    for (size_t e = threadIdx.x; e < tot; e += kScT)
        m = fmax(m, fabs(diag_only ? s[e + size_t(n) * e] : s[e]));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kScT / 32; ++w) m = fmax(m, red[w]);
        const bool safe = !(m > 0.0) || (m >= 0x1p-200 && m <= 0x1p200) || isinf(m) || isnan(m);
        const int ex = safe ? 0 : ilogb(m);
        fac[0] = ldexp(1.0, ex);   // eigenvalues x fac
        fac[1] = ldexp(1.0, -ex);  // S x fac[1]
    }
}
__global__ void eig_scale_kernel(double* __restrict__ s, size_t tot, const double* __restrict__ fac) {
    const double f = fac[1];
    if (f == 1.0) return;  // uniform: the common case writes nothing
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += size_t(gridDim.x) * blockDim.x)
        s[e] *= f;
}
__global__ void eig_unscale_kernel(double* __restrict__ v, int count, const double* __restrict__ fac) {
    const double f = fac[0];
    if (f == 1.0) return;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < count; e += gridDim.x * blockDim.x) v[e] *= f;
}
}  // namespace

void eig_scale(atk_ctx* ctx, double* s, int n, bool psd, double* fac_dev) {
    // a PSD matrix's largest |entry| sits on its diagonal: n reads instead of n^2
    eig_maxabs_kernel<<<1, kScT, 0, ctx->stream>>>(s, n, psd ? 1 : 0, fac_dev);
    ATK_LAUNCHED(ctx);
    const size_t tot = size_t(n) * n;
    eig_scale_kernel<<<unsigned(std::max<size_t>(1, std::min<size_t>((tot + 255) / 256, size_t(ctx->num_sms) * 8))),
                       256, 0, ctx->stream>>>(s, tot, fac_dev);
    ATK_LAUNCHED(ctx);
}

void eig_unscale_values(atk_ctx* ctx, double* values, int count, const double* fac_dev) {
    if (count <= 0) return;
    eig_unscale_kernel<<<unsigned((count + 255) / 256), 256, 0, ctx->stream>>>(values, count, fac_dev);
    ATK_LAUNCHED(ctx);
}

namespace {
EigInfo sym_eig_top_r_impl(atk_ctx* ctx, const double* s_dev, int n, int r, double* values_dev, double* vectors_dev,
                           bool psd, double tol, bool exact_sym);
}

// The inputs are the engine's own device buffers (a mode's Gram, the API's copy of the host
// matrix): scaled in place when their range demands it (eig_scale).
EigInfo sym_eig_top_r(atk_ctx* ctx, const double* s_dev, int n, int r, double* values_dev, double* vectors_dev,
                      bool psd, double tol, bool exact_sym) {
    DevBuf<double> fac(ctx, 2);
    eig_scale(ctx, const_cast<double*>(s_dev), n, psd, fac.get());
    EigInfo info = sym_eig_top_r_impl(ctx, s_dev, n, r, values_dev, vectors_dev, psd, tol, exact_sym);
    eig_unscale_values(ctx, values_dev, r, fac.get());
    return info;
}

namespace {
EigInfo sym_eig_top_r_impl(atk_ctx* ctx, const double* s_dev, int n, int r, double* values_dev, double* vectors_dev,
                           bool psd, double tol, bool exact_sym) {
    EigInfo info;
    cudaStream_t st = ctx->stream;
    if (n <= kTridiagMax && (ctx->eig_method == -1 || ctx->eig_method >= 2)) {
        tridiag_eig(ctx, s_dev, n, n, r, values_dev, vectors_dev, n);
        fix_signs(ctx, vectors_dev, n, r, n);
        if (std::getenv("ATK_TRACE")) std::fprintf(stderr, "[atk eig n=%d r=%d] tridiagonal\n", n, r);
        info.method = 2;
        return info;
    }
    // exact dense path above 200 (trd_big.cu): on request, or when the ChFSI block
    // cannot hold r + a guard band (r > kJacobiMax)
    auto dense_big = [&](const char* why) {
        dense_eig_big(ctx, s_dev, n, n, r, values_dev, vectors_dev, n, exact_sym);
        fix_signs(ctx, vectors_dev, n, r, n);
        if (std::getenv("ATK_TRACE")) std::fprintf(stderr, "[atk eig n=%d r=%d] dense tridiagonal (%s)\n", n, r, why);
        info.method = 3;
        return info;
    };
    if (n <= kBigEigMax && (ctx->eig_method == 3 || ctx->eig_method == 2)) return dense_big("requested");
    if (n <= kBigEigMax && ctx->eig_method != 1 && std::min(n, r + std::max(16, r / 4)) > kJacobiMax &&
        !(n <= kJacobiMax || (psd && n <= kJacobiPsdMax)))
        return dense_big("r too large for the ChFSI block");
    const bool dense = (n <= kJacobiMax || (psd && n <= kJacobiPsdMax)) && ctx->eig_method != 1;
    if (dense) {
        DevBuf<double> vals(ctx, n), vecs(ctx, size_t(n) * n);
        DevBuf<int> sweeps(ctx, 1);
        jacobi_eig(ctx, s_dev, n, n, vals.get(), vecs.get(), n, sweeps.get(), psd);
        int sw = 0;
        ATK_CUDA(cudaMemcpyAsync(&sw, sweeps.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
        ATK_CUDA(cudaStreamSynchronize(st));
        if (std::getenv("ATK_TRACE")) std::fprintf(stderr, "[atk eig n=%d r=%d] dense jacobi sweeps %d\n", n, r, sw);
        if (sw >= 40) fail(ATK_NO_CONVERGENCE, "symmetric eigendecomposition failed (Jacobi sweeps)");
        if (sw >= 0) {
            ATK_CUDA(cudaMemcpyAsync(values_dev, vals.get(), r * sizeof(double), cudaMemcpyDeviceToDevice, st));
            ATK_CUDA(cudaMemcpyAsync(vectors_dev, vecs.get(), size_t(n) * r * sizeof(double),
                                     cudaMemcpyDeviceToDevice, st));
            fix_signs(ctx, vectors_dev, n, r, n);
            info.method = 0;
            info.iterations = sw;
            return info;
        }
        // sw < 0: the large (U-only) dense variant found the input not numerically
        // PSD; ChFSI below handles it
    }

    // ---------------- ChFSI
    if (tol <= 0) tol = ctx->chfsi_tol;
    // block size: r + max(16, r / 4) (the Rayleigh-Ritz Jacobi costs ~k^2; the
    // S^2 Omega start makes a thin guard band enough on gapped spectra)
    int k = std::min(n, r + std::max(16, r / 4));
    if (ctx->chfsi_k > 0) k = std::min(n, std::max(r, ctx->chfsi_k));  // option "chfsi_k"
    // the block's CholeskyQR / SVQB kernels hold k x k in one CTA's shared memory
    k = std::min(k, kJacobiMax);
    if (k < r) fail(ATK_UNSUPPORTED, "sym_eig_top_r: r > 112 with n > 200 is not supported");
    const size_t nn = size_t(n) * n, nk = size_t(n) * k, kk = size_t(k) * k;
    const size_t nr = size_t(n) * r;
    // an exactly symmetric input (the engine's Grams are mirrored) is used in
    // place; anything else is copied and symmetrised first (linalg.hpp:104)
    // the block buffers come from the context's persistent scratch: no allocation or free
    // sits between the converged check and the caller's next launch
    auto rb = [](size_t count, size_t sz) { return ScratchScope::round(count * sz); };
    ScratchScope scr(ctx, 7 * rb(nk, 8) + rb(nr, 8) + 5 * rb(kk, 8) + 4 * rb(k, 8) + 3 * rb(3, 4));
    // the per-pass check reads theta (k), the residuals (r of k) and the CholeskyQR status words
    // (3 ints) in ONE device-to-host copy: they sit back to back in `chk`
    DevBuf<double> chk(scr, 2 * size_t(k) + 2);
    DevBuf<double> Sbuf(ctx, exact_sym ? 0 : nn), V(scr, nk), W(scr, nk), Ya(scr, nk), Yb(scr, nk), Yc(scr, nk),
        T(scr, kk), Z(scr, kk), theta(ctx, chk.get(), k), res(ctx, chk.get() + k, k), Vr(scr, nk), Wr(scr, nr);
    DevBuf<double> Sd(ctx, 0), Dm(ctx, 0);  // deflated copy of S, deflation term (allocated on first lock)
    Ws ws{DevBuf<double>(scr, kk), DevBuf<double>(scr, kk), DevBuf<double>(scr, k), DevBuf<double>(scr, k),
          DevBuf<double>(scr, kk), DevBuf<double>(scr, nk), DevBuf<int>(scr, 1),
          DevBuf<int>(ctx, reinterpret_cast<int*>(chk.get() + 2 * size_t(k)), 3)};
    DevBuf<int> sweeps(scr, 1);
    static const bool trace = std::getenv("ATK_TRACE") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    // ATK_TRACE=events: CUDA events instead of synchronising at every mark
    // (the launch / host-sync gaps stay in), printed when the solve ends
    static const bool trace_ev = trace && std::string(std::getenv("ATK_TRACE")) == "events";
    struct Ev {
        cudaEvent_t e;
        const char* what;
        std::chrono::steady_clock::time_point host;
    };
    std::vector<Ev> evs;
    auto mark = [&](const char* what, int a = -1, double v = 0.0) {
        if (!trace) return;
        if (trace_ev) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            cudaEventRecord(e, st);
            evs.push_back({e, what, std::chrono::steady_clock::now()});
            return;
        }
        cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[atk eig n=%d r=%d k=%d] %-10s %8.3f ms  %d %.3e\n", n, r, k, what,
                     std::chrono::duration<double, std::milli>(now - t_last).count(), a, v);
        t_last = now;
    };
    auto trace_sweeps = [&](const int* d) {  // Jacobi sweeps of the last RR (trace only)
        int h = -1;
        if (trace && !trace_ev) cudaMemcpy(&h, d, sizeof(int), cudaMemcpyDeviceToHost);
        return h;
    };
    mark("begin");
    if (!exact_sym) {
        ATK_CUDA(cudaMemcpyAsync(Sbuf.get(), s_dev, nn * sizeof(double), cudaMemcpyDeviceToDevice, st));
        symmetrize(ctx, Sbuf.get(), n);
    }
    const double* Sp = exact_sym ? s_dev : Sbuf.get();
    mark("prep");
    // start: two power steps on a random block (S^2 Omega: on gapped spectra this
    // alone resolves the wanted subspace), orthonormalise, Rayleigh-Ritz
    fill_normalish<<<nblk(nk), 256, 0, st>>>(Yb.get(), nk, 0xc0ffee11ULL);
    ATK_LAUNCHED(ctx);
    dgemm(ctx, false, false, n, k, n, 1.0, Sp, n, Yb.get(), n, 0.0, Ya.get(), n);
    dgemm(ctx, false, false, n, k, n, 1.0, Sp, n, Ya.get(), n, 0.0, Yb.get(), n);
    // CholeskyQR3 without a host round trip: its status is read with the
    // residuals below, and a failed pass is redone by SVQB from the same input
    struct {
        const double* src;
        double* dst;
        int ka;
    } qr_job{Yb.get(), V.get(), k};
    cholqr3_async(ctx, Yb.get(), n, k, V.get(), ws);
    mark("qr0");
    // Ritz vectors formed: the top r; all k once locking has started (the
    // active block is then Vk(:, nc:k)).  Forming all k from the start cost
    // C5 0.85 ms per step: its 16 guard-band Ritz values are noise, one tight
    // cluster for inverse iteration, and C5 never filters.
    int nv = r;
    rayleigh_ritz(ctx, Sp, n, k, r, nv, V.get(), W.get(), T.get(), Z.get(), theta.get(), Vr.get(), Wr.get(),
                  sweeps.get(), psd);
    mark("rr0", trace_sweeps(sweeps.get()));

    const int max_outer = 100;
    std::vector<double> hth(k), hres(r);
    // spectrum bounds for the filter: for a PSD matrix with a clear gap between the
    // wanted and the block-edge Ritz values, lo = 0 already gives a strong filter;
    // otherwise (flat spectra) a Lanczos run tightens lo (computed lazily, once)
    Bounds b{psd ? 0.0 : 0.0, 0.0};
    bool have_bounds = false;
    double scale = 0.0;
    int it = 0;
    double worst = 0.0, prev_worst = 0.0;
    for (;; ++it) {
        ritz_residual<<<r, 256, 0, st>>>(Wr.get(), Vr.get(), theta.get(), n, r, res.get());
        ATK_LAUNCHED(ctx);
        // the result as if this check passes, enqueued before the host waits on it (a later pass
        // overwrites it): the GPU forms the output while the host reads the residuals
        auto emit = [&] {
            ATK_CUDA(cudaMemcpyAsync(values_dev, theta.get(), r * sizeof(double), cudaMemcpyDeviceToDevice, st));
            ATK_CUDA(cudaMemcpyAsync(vectors_dev, Vr.get(), nr * sizeof(double), cudaMemcpyDeviceToDevice, st));
            fix_signs(ctx, vectors_dev, n, r, n);
        };
        int qinfo[3] = {0, 0, 0};
        // one host round trip through the context's page-locked staging (pageable destinations made
        // each copy a synchronous staged transfer: ~40 us of gaps per check)
        {
            const size_t chk_bytes = (2 * size_t(k) + 2) * sizeof(double);
            auto* pin = static_cast<uint8_t*>(pinned_host(ctx, chk_bytes));
            double* pth = reinterpret_cast<double*>(pin);
            double* pres = pth + k;
            int* pq = reinterpret_cast<int*>(pth + 2 * size_t(k));
            ATK_CUDA(cudaMemcpyAsync(pin, chk.get(), chk_bytes, cudaMemcpyDeviceToHost, st));
            cudaEvent_t& got = ctx->ev[7];
            if (!got) ATK_CUDA(cudaEventCreateWithFlags(&got, cudaEventDisableTiming));
            ATK_CUDA(cudaEventRecord(got, st));
            emit();
            ATK_CUDA(cudaEventSynchronize(got));
            std::copy(pth, pth + k, hth.begin());
            std::copy(pres, pres + r, hres.begin());
            std::copy(pq, pq + 3, qinfo);
        }
        if (qr_job.src && (qinfo[0] || qinfo[1] || qinfo[2])) {  // CholeskyQR broke down: SVQB, same Rayleigh-Ritz
            svqb(ctx, qr_job.src, n, qr_job.ka, qr_job.dst, ws);
            qr_job.src = nullptr;
            rayleigh_ritz(ctx, Sp, n, k, r, nv, V.get(), W.get(), T.get(), Z.get(), theta.get(), Vr.get(), Wr.get(),
                          sweeps.get(), psd);
            --it;
            continue;
        }
        qr_job.src = nullptr;
        scale = std::max(scale, std::fabs(hth[0]));
        worst = 0.0;
        for (int j = 0; j < r; ++j) worst = std::max(worst, hres[j]);
        if (!(scale > 0.0) || worst <= tol * scale || it >= max_outer) break;
        // hand-over to the exact dense solver (flat spectra; bounded time on any input).
        // Measured convergence: the residual reduction of the last pass predicts the passes still
        // needed; hand over as soon as they would cost more than the dense solver.  Costs (r2,
        // n = 2048, k = 80): a degree-64 pass ~5.9 ms, the dense solver ~22 ms (10 ms at n = 1024).
        // C2's flat modes gain >= 1e3 per pass and stay.
        const bool auto_dense = ctx->eig_dense_passes >= 0 && n <= kBigEigMax && ctx->eig_method == -1;
        double left = -1.0;  // predicted passes still needed (unknown before the first filter pass)
        if (auto_dense && it >= 1 && prev_worst > 0.0 && n > kTridiagMax) {
            const double rate = prev_worst / std::max(worst, 1e-300);
            const double need = std::log(std::max(1.0, worst / (tol * scale)));
            left = rate > 1.0 ? need / std::log(rate) : 1e9;
            const double t_step = 4.0 + 2.0 * double(n) * n * k / 9e12 * 1e6;  // us
            const double t_pass = 64.0 * t_step * 1e-3 + 0.9;                  // ms
            const double fn = double(n) / 2048.0;
            const double t_dense = 6.0 + 16.0 * fn * fn;  // ms
            if (trace)
                std::fprintf(stderr, "[atk eig n=%d] pass rate %.3g, %.1f passes left (%.1f ms) vs dense %.1f ms\n",
                             n, rate, left, left * t_pass, t_dense);
            // 1.3x: the rate of a locking ChFSI grows pass by pass (C5u mode 2: 43 -> 8450), so a
            // constant-rate prediction overestimates what is left
            if (left * t_pass > 1.3 * t_dense) {
                mark("to-dense", it, worst / scale);
                return dense_big("predicted ChFSI passes");
            }
        }
        // pass budget: after eig_dense_passes passes, unless the measured rate promises
        // convergence within about two more passes (C5u mode 1 reached 1e-8 after three passes,
        // one short of 1e-10: the budget used to force the 22 ms dense solve there); always
        // after twice the budget
        if (auto_dense && it >= ctx->eig_dense_passes &&
            (left < 0.0 || left > 2.5 || it >= 2 * std::max(1, ctx->eig_dense_passes))) {
            mark("to-dense", it, worst / scale);
            return dense_big("ChFSI pass budget");
        }
        prev_worst = worst;
        if (!have_bounds) {
            if (trace)
                std::fprintf(stderr, "[atk eig n=%d r=%d k=%d] theta_1 %.6e theta_r %.6e theta_k %.6e\n", n, r, k,
                             hth[0], hth[r - 1], hth[k - 1]);
            // PSD: lo = 0.  (The m = 40 Lanczos bound, lowest Ritz value minus its
            // residual, came out below 0 on every flat Gram spectrum measured, C2
            // included, i.e. it only cost 0.7 ms per mode.)  Indefinite: Lanczos.
            if (psd && hth[k - 1] >= 0.0) {
                b = Bounds{0.0, hth[0]};
            } else {
                b = lanczos_bounds(ctx, Sp, n, psd);
                mark("lanczos", 0, b.lo);
                if (trace) std::fprintf(stderr, "[atk eig n=%d] bounds lo %.9e hi %.9e\n", n, b.lo, b.hi);
            }
            have_bounds = true;
        }
        // locking: the leading nc Ritz pairs that already meet tol are kept as
        // they are, and the filter runs on the k - nc others with S deflated,
        // S' = S - L diag(theta_L - c) L^T, which moves the locked eigenvalues
        // to the centre of the damped interval.  Without it a dominant top
        // eigenvalue (a non-centred Gram's mean direction, 1e3 x the rest)
        // forces the dynamic-range cap below down to degree 2.
        int nc = 0;
        if (ctx->chfsi_lock) {
            while (nc < r - 1 && hres[nc] <= tol * scale) ++nc;
            if (nc > 0 && nv < k) {  // no guard-band vectors yet: lock from the next pass on
                nc = 0;
                nv = k;
            }
        }
        // Chebyshev filter on the unwanted interval [lo, cut]
        const double cut = hth[k - 1];
        const double lo = std::min(b.lo, cut - 1e-12 * scale);
        double e = 0.5 * (cut - lo), c = 0.5 * (cut + lo);
        if (!(e > 0.0)) e = 1e-12 * scale;
        const double top = nc > 0 ? hth[nc] : std::max(b.hi, hth[0]);  // top of the filtered spectrum
        const double smax = std::max(1.0, (top - c) / e);
        const double g = 1.0 / (2.0 * smax + 1.0);  // per-step rescale, keeps the recurrence linear
        // degree: damp [lo, cut] relative to the wanted end by at most ~1e10 per
        // pass (T_d(x) ~ e^{d acosh x} / 2), 1..64: on flat spectra a pass costs
        // d skinny GEMMs plus a CholeskyQR + Rayleigh-Ritz, so fewer, stronger
        // passes win (measured C2 mode 2, n = 1024: cap 16 -> 9 passes).  A stronger pass leaves the
        // block's unwanted columns numerically parallel to the wanted ones (their
        // O(eps) wanted-direction residue is amplified past 1/eps) and CholeskyQR
        // breaks down; on wide gaps this means a single S V power step.
        const double ac = std::acosh(std::max(1.0 + 1e-12, (hth[r - 1] - c) / e));
        int degree = std::max(1, std::min(64, int(23.0 / std::max(ac, 1e-3))));
        // dynamic range inside the wanted set: the top Ritz direction grows
        // T_d(x_1) / T_d(x_r) times faster than the lowest wanted one; past ~1e9
        // (~1 / sqrt(eps)) the lowest wanted directions come out of the
        // orthonormalisation with relative errors ~eps x that ratio and the
        // residual stalls (seen on a n = 128, r = 64 indefinite block)
        const double atop = std::acosh(std::max(1.0 + 1e-12, (top - c) / e));
        if (atop - ac > 1e-12) degree = std::max(1, std::min(degree, int(20.7 / (atop - ac))));  // ln 1e9
        // Y1 = g (S V - c V) / e ; Y_{j+1} = g (2/e)(S Y_j - c Y_j) - g^2 Y_{j-1}
        const double* Sf = Sp;      // the filter's matrix
        double* X = V.get();        // the filtered block (n x ka)
        int ka = k;
        if (nc > 0) {
            if (!Sd.get()) {
                Sd = DevBuf<double>(ctx, nn);
                Dm = DevBuf<double>(ctx, nr);
            }
            ATK_CUDA(cudaMemcpyAsync(Sd.get(), Sp, nn * sizeof(double), cudaMemcpyDeviceToDevice, st));
            scale_cols_shift<<<nblk(size_t(n) * nc), 256, 0, st>>>(Vr.get(), theta.get(), c, n, nc, Dm.get());
            ATK_LAUNCHED(ctx);
            dgemm(ctx, false, true, n, n, nc, -1.0, Dm.get(), n, Vr.get(), n, 1.0, Sd.get(), n);
            Sf = Sd.get();
            X = Vr.get() + size_t(n) * nc;  // Ritz vectors nc..k-1
            ka = k - nc;
        }
        const size_t nka = size_t(n) * ka;
        double* ycur = nullptr;
        double* const ys[4] = {X, Ya.get(), Yb.get(), Yc.get()};
        const int fused = ctx->cheb_fused
                              ? cheb_filter(ctx, Sf, n, ka, degree, ys, g / e, -g * c / e, 2.0 * g / e,
                                            -2.0 * g * c / e, -g * g)
                              : -1;
        if (fused >= 0) {
            ycur = ys[fused];
        } else {  // per-step launches (option cheb_fused = 0, or no co-resident grid)
            double* yprev = X;
            ycur = Ya.get();
            double* ynext = Yb.get();
            cheb_combine<<<nblk(nka), 256, 0, st>>>(ycur, X, nullptr, nka, -g * c / e, 0.0);
            ATK_LAUNCHED(ctx);
            dgemm(ctx, false, false, n, ka, n, g / e, Sf, n, X, n, 1.0, ycur, n);
            for (int j = 1; j < degree; ++j) {
                cheb_combine<<<nblk(nka), 256, 0, st>>>(ynext, ycur, yprev, nka, -2.0 * g * c / e, -g * g);
                ATK_LAUNCHED(ctx);
                dgemm(ctx, false, false, n, ka, n, 2.0 * g / e, Sf, n, ycur, n, 1.0, ynext, n);
                double* spare = (yprev == X) ? Yc.get() : yprev;
                yprev = ycur;
                ycur = ynext;
                ynext = spare;
            }
        }
        mark("filter", degree, worst / scale);
        if (nc > 0) {
            // V = [L, orth((I - L L^T) Y)]: project the locked directions out twice
            double* P = ws.M.get();  // nc x ka <= k x k
            for (int pass = 0; pass < 2; ++pass) {
                dgemm(ctx, true, false, nc, ka, n, 1.0, Vr.get(), n, ycur, n, 0.0, P, nc);
                dgemm(ctx, false, false, n, ka, nc, -1.0, Vr.get(), n, P, nc, 1.0, ycur, n);
            }
            qr_job = {ycur, V.get() + size_t(n) * nc, ka};
            cholqr3_async(ctx, ycur, n, ka, V.get() + size_t(n) * nc, ws);
            ATK_CUDA(cudaMemcpyAsync(V.get(), Vr.get(), size_t(n) * nc * sizeof(double), cudaMemcpyDeviceToDevice,
                                     st));
        } else {
            qr_job = {ycur, V.get(), k};
            cholqr3_async(ctx, ycur, n, k, V.get(), ws);
        }
        mark("qr", nc);
        rayleigh_ritz(ctx, Sp, n, k, r, nv, V.get(), W.get(), T.get(), Z.get(), theta.get(), Vr.get(), Wr.get(),
                      sweeps.get(), psd);
        mark("rr", trace_sweeps(sweeps.get()));
    }
    mark("done", it, worst / scale);
    if (trace_ev && !evs.empty()) {
        cudaEventSynchronize(evs.back().e);
        for (size_t q = 1; q < evs.size(); ++q) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, evs[q - 1].e, evs[q].e);
            std::fprintf(stderr, "[atk eig n=%d r=%d k=%d] gpu %-10s %8.3f ms  (host enqueue %.3f ms)\n", n, r, k,
                         evs[q].what, ms,
                         std::chrono::duration<double, std::milli>(evs[q].host - evs[q - 1].host).count());
        }
        for (auto& x : evs) cudaEventDestroy(x.e);
    }
    // values / vectors: already enqueued by the last check (emit above)
    info.method = 1;
    info.iterations = it;
    info.residual = scale > 0 ? worst / scale : 0.0;
    if (it >= max_outer && worst > 1e3 * tol * scale)
        fail(ATK_NO_CONVERGENCE, "symmetric eigendecomposition failed (ChFSI did not converge)");
    return info;
}
}  // namespace

bool orthonormal_basis_cholqr(atk_ctx* ctx, const double* a, int m, int n, double* q) {
    if (n > kJacobiMax || m < n) return false;
    const size_t mn = size_t(m) * n, nn = size_t(n) * n;
    Ws ws{DevBuf<double>(ctx, nn), DevBuf<double>(ctx, nn), DevBuf<double>(ctx, n), DevBuf<double>(ctx, n),
          DevBuf<double>(ctx, nn), DevBuf<double>(ctx, mn), DevBuf<int>(ctx, 1), DevBuf<int>(ctx, 3)};
    return cholqr3(ctx, a, m, n, q, ws);
}

}  // namespace atk
