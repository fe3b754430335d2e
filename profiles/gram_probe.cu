// gram_probe.cu — device-timed repeated mode-0 Grams at different input sizes:
// is the C5 Gram bound by HBM/L2 traffic or by the tensor pipe at the power
// cap?  (profiling aid, not part of the library; build: profiles/gram_probe.sh)
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "atk_driver.cuh"

int main() {
    atk_ctx* ctx = nullptr;
    if (atk_ctx_create(0, &ctx) != ATK_OK) return 1;
    // C5 mode-0 shape, the K-launch size and the fp32 chain length (drain interval) swept
    struct Case { uint64_t I, J; int reps; int launch_kb; int chunk_kb; };
    const Case cases[] = {{2048, 1ull << 22, 3, 4096, 512},  {2048, 1ull << 22, 3, 4096, 1024},
                          {2048, 1ull << 22, 3, 4096, 2048}, {2048, 1ull << 22, 3, 2048, 512},
                          {2048, 1ull << 22, 3, 8192, 512},  {2048, 1ull << 22, 3, 4096, 256},
                          {2048, 1ull << 22, 3, 4096, 512}};
    for (const Case& c : cases) {
        atk_ctx_set_option(ctx, "gram_launch_kb", c.launch_kb);
        atk_ctx_set_option(ctx, "gram_chunk_kb", c.chunk_kb);
        atk_tensor* x = nullptr;
        const uint64_t dims[2] = {c.I, c.J};
        if (atk_tensor_create(ctx, ATK_F32, 2, dims, &x) != ATK_OK) return 2;
        atk_fill_uniform(ctx, x, 3, 0);
        double* s = nullptr;
        cudaMalloc(&s, c.I * c.I * sizeof(double));
        atk::contract_ttt(ctx, x, x, 0, s, true);  // warm
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaStreamSynchronize(ctx->stream);
        cudaEventRecord(a, ctx->stream);
        for (int r = 0; r < c.reps; ++r) atk::contract_ttt(ctx, x, x, 0, s, true);
        cudaEventRecord(b, ctx->stream);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double per = ms / c.reps;
        std::printf("I=%llu J=%llu (%.2f GB) launch_kb=%d chunk_kb=%d: %.3f ms/Gram -> %.1f TF/s\n",
                    (unsigned long long)c.I, (unsigned long long)c.J, c.I * c.J * 4 / 1e9, c.launch_kb, c.chunk_kb, per,
                    double(c.I) * c.I * c.J / per / 1e9);
        std::fflush(stdout);
        cudaFree(s);
        atk_tensor_free(x);
    }
    return 0;
}
