// barrier_probe.cu — cycles per grid barrier, one 512-thread CTA per SM (probe, not product)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_probe barrier_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) bar_kernel(unsigned* cnt, unsigned* flags, double* data, int iters,
                                                    long long* out) {
    extern __shared__ double sm[];
    const int G = gridDim.x, c = blockIdx.x, t = threadIdx.x;
    const long long t0 = clock64();
    for (int k = 0; k < iters; ++k) {
        if (t == 0) data[c] = k;  // a store that must be ordered before the arrival
        __syncthreads();
        if (t == 0) {
            if (MODE == 0) {  // red.release + poll the counter
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
                while (ld_acq(cnt) < unsigned(G) * unsigned(k + 1)) {
                }
            } else if (MODE == 1) {  // same + nanosleep backoff
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
                while (ld_acq(cnt) < unsigned(G) * unsigned(k + 1)) __nanosleep(40);
            } else if (MODE == 2) {  // atom + generation flag on another line
                unsigned old;
                asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
                if (old == unsigned(G) * unsigned(k + 1) - 1) {
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(cnt + 64), "r"(unsigned(k + 1)) : "memory");
                } else {
                    while (ld_acq(cnt + 64) < unsigned(k + 1)) {
                    }
                }
            }
        }
        if (MODE == 3) {  // per-CTA epoch flags, warp 0 polls all of them
            if (t == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + c), "r"(unsigned(k + 1)) : "memory");
            if (t < 32) {
                for (;;) {
                    bool ok = true;
                    for (int q = t; q < G; q += 32) ok &= ld_acq(flags + q) >= unsigned(k + 1);
                    if (__all_sync(0xffffffffu, ok)) break;
                }
            }
        }
        if (MODE == 4) {  // per-CTA epoch flags, polled by 5 warps (one line each)
            if (t == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + c), "r"(unsigned(k + 1)) : "memory");
            if (t < 32 * ((G + 31) / 32)) {
                const int q = t;
                if (q < G)
                    while (ld_acq(flags + q) < unsigned(k + 1)) {
                    }
            }
        }
        __syncthreads();
    }
    if (t == 0 && c == 0) *out = clock64() - t0;
}

// cluster barrier (hardware) inside one cluster of size CS
__global__ void __launch_bounds__(512, 1) cbar_kernel(int iters, long long* out) {
    const long long t0 = clock64();
    for (int k = 0; k < iters; ++k) {
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = clock64() - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *cnt, *flags;
    double* data;
    long long* out;
    cudaMalloc(&cnt, 4096);
    cudaMalloc(&flags, 4096);
    cudaMalloc(&data, 8 * 4096);
    cudaMalloc(&out, 8);
    const int iters = 4000;
    void (*ks[5])(unsigned*, unsigned*, double*, int, long long*) = {bar_kernel<0>, bar_kernel<1>, bar_kernel<2>,
                                                                     bar_kernel<3>, bar_kernel<4>};
    const char* names[5] = {"red+poll counter", "red+poll+nanosleep40", "atom+gen flag", "epoch flags, warp0 polls",
                            "epoch flags, 1 thread per flag"};
    for (int m = 0; m < 5; ++m) {
        cudaFuncSetAttribute(ks[m], cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(cnt, 0, 4096);
            cudaMemset(flags, 0, 4096);
            int it = iters;
            void* args[] = {&cnt, &flags, &data, &it, &out};
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            cudaError_t e = cudaLaunchCooperativeKernel((void*)ks[m], dim3(sms), dim3(512), args, 200 * 1024, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            long long h;
            cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            if (rep) printf("%-32s %s: %.0f cycles, %.3f us per barrier (G=%d)\n", names[m], cudaGetErrorString(e),
                            h / double(iters), ms * 1e3 / iters, sms);
        }
    }
    // red+poll at smaller grids
    for (int g : {8, 16, 32, 74, 96}) {
        cudaMemset(cnt, 0, 4096);
        int it = iters;
        void* args[] = {&cnt, &flags, &data, &it, &out};
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchCooperativeKernel((void*)ks[0], dim3(g), dim3(512), args, 200 * 1024, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        long long h;
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        printf("red+poll G=%-3d %s: %.0f cycles, %.3f us per barrier\n", g, cudaGetErrorString(e), h / double(iters),
               ms * 1e3 / iters);
    }
    cudaFuncSetAttribute(cbar_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(cbar_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int cs : {2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = 200 * 1024;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int it = iters;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchKernelEx(&cfg, cbar_kernel, it, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        long long h;
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        printf("cluster barrier CS=%-2d %s: %.0f cycles, %.3f us per barrier\n", cs, cudaGetErrorString(e),
               h / double(iters), ms * 1e3 / iters);
    }
    return 0;
}
