// contract_tc.cu — dispatch of the tensor-core contraction paths.
#include "atk_driver.cuh"

namespace atk {

bool tc_gram_supported(atk_ctx* ctx, const atk_tensor* x, int mode);
void tc_gram(atk_ctx* ctx, const atk_tensor* x, int mode, double* s_dev);

bool tc_ttt_supported(atk_ctx* ctx, const atk_tensor* x, const atk_tensor* y, int mode, bool sym) {
    return sym && x == y && tc_gram_supported(ctx, x, mode);
}

void tc_ttt(atk_ctx* ctx, const atk_tensor* x, const atk_tensor* y, int mode, double* z_dev, bool sym) {
    if (!(sym && x == y)) fail(ATK_UNSUPPORTED, "tensor-core ttt: only the Gram is wired");
    tc_gram(ctx, x, mode, z_dev);
}

}  // namespace atk
