// contract_tc.cu — tensor-core contraction paths (placeholder: filled in by
// the tcgen05 / DMMA kernels).
#include "atk_driver.cuh"

namespace atk {
bool tc_ttt_supported(atk_ctx*, const atk_tensor*, const atk_tensor*, int, bool) { return false; }
void tc_ttt(atk_ctx*, const atk_tensor*, const atk_tensor*, int, double*, bool) {
    fail(ATK_UNSUPPORTED, "tensor-core ttt not built");
}
bool tc_ttm_supported(atk_ctx*, const atk_tensor*, uint64_t, int) { return false; }
void tc_ttm(atk_ctx*, const atk_tensor*, const double*, uint64_t, int, atk_tensor*) {
    fail(ATK_UNSUPPORTED, "tensor-core ttm not built");
}
}  // namespace atk
