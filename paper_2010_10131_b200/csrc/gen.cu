// gen.cu — input generation and streaming reductions (HBM-bound helpers).
//
//  fill_uniform : counter-hash uniform [-1,1) on a 2^-23 grid, bit-identical
//                 to the oracle's or_hash_uniform (oracle/atk_oracle.cpp).
//  norm2_sq     : frobenius_norm (tensor.hpp:158-168) with fp64 accumulation,
//                 deterministic two-pass block reduction.
#include "atk_internal.cuh"

namespace atk {
namespace {

__device__ __forceinline__ uint64_t hash64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

__device__ __forceinline__ float hash_uniform(uint64_t hseed, uint64_t idx) {
    const uint64_t h = hash64(idx ^ hseed);
    const int32_t k = int32_t(h >> 40) - (1 << 23);
    return float(k) * (1.0f / 8388608.0f);
}

template <class T>
__global__ void fill_uniform_kernel(T* __restrict__ x, uint64_t n, uint64_t hseed, uint64_t off) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * 4;
    for (uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (i + k < n) x[i + k] = T(hash_uniform(hseed, off + i + k));
    }
}

constexpr int kRedBlocks = 592;  // 4 x 148 SMs, fixed => deterministic order
constexpr int kRedThreads = 512;

template <class T>
__device__ __forceinline__ double sq(T v) {
    const double d = double(v);
    return d * d;
}

__device__ double block_sum(double v) {
    __shared__ double sh[32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    double t = 0;
    if (w == 0) {
        t = (l < int(blockDim.x >> 5)) ? sh[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    __syncthreads();
    return t;
}

template <class T>
__global__ void norm2_partial(const T* __restrict__ x, uint64_t n, double* __restrict__ part) {
    double acc = 0.0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        acc += sq(x[i]);
    const double s = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

template <class T>
__global__ void diff2_partial(const T* __restrict__ x, const T* __restrict__ y, uint64_t n,
                              double* __restrict__ part) {
    double acc = 0.0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double d = double(x[i]) - double(y[i]);
        acc += d * d;
    }
    const double s = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void final_sum(const double* __restrict__ part, int n, double* __restrict__ out) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += part[i];
    const double s = block_sum(acc);
    if (threadIdx.x == 0) *out = s;
}

template <class T>
__global__ void axpy_kernel(T* __restrict__ x, const T* __restrict__ y, uint64_t n, double a) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        x[i] = T(double(x[i]) + a * double(y[i]));
}

template <class D, class S>
__global__ void convert_kernel(D* __restrict__ d, const S* __restrict__ s, uint64_t n) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        d[i] = D(s[i]);
}

uint64_t host_hash64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

int grid_for(atk_ctx* ctx, uint64_t n, int threads, int per_thread) {
    const uint64_t want = (n + uint64_t(threads) * per_thread - 1) / (uint64_t(threads) * per_thread);
    const uint64_t cap = uint64_t(ctx->num_sms) * 16;
    return int(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

void fill_uniform(atk_ctx* ctx, atk_tensor* t, uint64_t seed, uint64_t offset) {
    const uint64_t n = t->numel();
    const uint64_t hs = host_hash64(seed);
    const int g = grid_for(ctx, n, 256, 4);
    if (t->dtype == ATK_F32)
        fill_uniform_kernel<float><<<g, 256, 0, ctx->stream>>>((float*)t->data, n, hs, offset);
    else
        fill_uniform_kernel<double><<<g, 256, 0, ctx->stream>>>((double*)t->data, n, hs, offset);
    ATK_LAUNCHED(ctx);
}

double norm2_sq(atk_ctx* ctx, const void* x, atk_dtype dt, uint64_t n) {
    DevBuf<double> part(ctx, kRedBlocks + 1);
    if (dt == ATK_F32)
        norm2_partial<float><<<kRedBlocks, kRedThreads, 0, ctx->stream>>>((const float*)x, n, part.get());
    else
        norm2_partial<double><<<kRedBlocks, kRedThreads, 0, ctx->stream>>>((const double*)x, n, part.get());
    ATK_LAUNCHED(ctx);
    final_sum<<<1, 1024, 0, ctx->stream>>>(part.get(), kRedBlocks, part.get() + kRedBlocks);
    ATK_LAUNCHED(ctx);
    double out = 0;
    ATK_CUDA(cudaMemcpyAsync(&out, part.get() + kRedBlocks, sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    ATK_CUDA(cudaStreamSynchronize(ctx->stream));
    return out;
}

double diff_norm2_sq(atk_ctx* ctx, const void* x, const void* y, atk_dtype dt, uint64_t n) {
    DevBuf<double> part(ctx, kRedBlocks + 1);
    if (dt == ATK_F32)
        diff2_partial<float><<<kRedBlocks, kRedThreads, 0, ctx->stream>>>((const float*)x, (const float*)y, n, part.get());
    else
        diff2_partial<double><<<kRedBlocks, kRedThreads, 0, ctx->stream>>>((const double*)x, (const double*)y, n, part.get());
    ATK_LAUNCHED(ctx);
    final_sum<<<1, 1024, 0, ctx->stream>>>(part.get(), kRedBlocks, part.get() + kRedBlocks);
    ATK_LAUNCHED(ctx);
    double out = 0;
    ATK_CUDA(cudaMemcpyAsync(&out, part.get() + kRedBlocks, sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    ATK_CUDA(cudaStreamSynchronize(ctx->stream));
    return out;
}

void axpy(atk_ctx* ctx, void* x, const void* y, atk_dtype dt, uint64_t n, double alpha) {
    const int g = grid_for(ctx, n, 256, 1);
    if (dt == ATK_F32)
        axpy_kernel<float><<<g, 256, 0, ctx->stream>>>((float*)x, (const float*)y, n, alpha);
    else
        axpy_kernel<double><<<g, 256, 0, ctx->stream>>>((double*)x, (const double*)y, n, alpha);
    ATK_LAUNCHED(ctx);
}

void convert(atk_ctx* ctx, void* dst, atk_dtype ddt, const void* src, atk_dtype sdt, uint64_t n) {
    const int g = grid_for(ctx, n, 256, 1);
    if (ddt == ATK_F32 && sdt == ATK_F64)
        convert_kernel<float, double><<<g, 256, 0, ctx->stream>>>((float*)dst, (const double*)src, n);
    else if (ddt == ATK_F64 && sdt == ATK_F32)
        convert_kernel<double, float><<<g, 256, 0, ctx->stream>>>((double*)dst, (const float*)src, n);
    else {
        ATK_CUDA(cudaMemcpyAsync(dst, src, n * (ddt == ATK_F32 ? 4 : 8), cudaMemcpyDeviceToDevice,
                                 ctx->stream));
        return;
    }
    ATK_LAUNCHED(ctx);
}

}  // namespace atk
