// contract_tc.cu — dispatch of the tensor-core contraction paths.
#include "atk_driver.cuh"

namespace atk {

bool tc_gram_supported(atk_ctx* ctx, const atk_tensor* x, int mode);
void tc_gram(atk_ctx* ctx, const atk_tensor* x, int mode, double* s_dev);
bool tc_gram2_supported(atk_ctx* ctx, const atk_tensor* x, int mode);
void tc_gram2(atk_ctx* ctx, const atk_tensor* x, int mode, double* s_dev);
bool tc_ttt_ns_supported(atk_ctx* ctx, const atk_tensor* x, const atk_tensor* y, int mode);
void tc_ttt_ns(atk_ctx* ctx, const atk_tensor* x, const atk_tensor* y, int mode, double* z_dev);

bool tc_ttt_supported(atk_ctx* ctx, const atk_tensor* x, const atk_tensor* y, int mode, bool sym) {
    if (sym && x == y) return tc_gram2_supported(ctx, x, mode) || tc_gram_supported(ctx, x, mode);
    return tc_ttt_ns_supported(ctx, x, y, mode);
}

void tc_ttt(atk_ctx* ctx, const atk_tensor* x, const atk_tensor* y, int mode, double* z_dev, bool sym) {
    if (sym && x == y) {
        if (tc_gram2_supported(ctx, x, mode)) tc_gram2(ctx, x, mode, z_dev);  // CTA-pair 256x256 tiles
        else tc_gram(ctx, x, mode, z_dev);                                     // 1-CTA 128x256 tiles
        return;
    }
    tc_ttt_ns(ctx, x, y, mode, z_dev);  // ALS: Y_(n) rfac_(n)^T
}

}  // namespace atk
