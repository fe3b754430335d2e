// Host-side checks of the C++ drop-in (include/atucker_b200.hpp) that need no
// GPU: built twice by tests/test_cpp_types.py — against the reference's own
// Eigen-free headers (/root/reference/proj/include: atucker::DenseTensor,
// atucker::NotSPD, atucker::SolverKind, atucker::selector::predict) and
// standalone (-DATUCKER_B200_STANDALONE) — and run on the CPU.  Prints PASS
// lines, exits non-zero on failure.
#include <cstdio>
#include <type_traits>

#include "atucker_b200.hpp"

#define REQUIRE(c)                                                  \
    do {                                                            \
        if (!(c)) {                                                 \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            return 1;                                               \
        }                                                           \
    } while (0)

namespace ab = atucker_b200;

// A strategy with exactly the reference's decide signature (sthosvd.hpp:64-65),
// parameterised on the params type the drop-in hands over.
struct RefSignatureStrategy {
    ab::SolverKind decide(std::size_t mode, std::size_t, std::size_t, std::size_t,
                          const ab::CostModelParams& params) const {
        return (mode == 1 || params.num_iters == 7) ? ab::SolverKind::Als : ab::SolverKind::Eig;
    }
};

template <class E>
static bool maps_to(atk_status s) {
    try {
        ab::check(s);
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
#if ATUCKER_B200_REFERENCE_TYPES
    // the reference's own types cross the drop-in unchanged (errors.hpp, tensor.hpp, solver_kind.hpp)
    static_assert(std::is_same_v<ab::DenseTensor, atucker::DenseTensor>);
    static_assert(std::is_same_v<ab::DenseMatrix, atucker::DenseMatrix>);
    static_assert(std::is_same_v<ab::SolverKind, atucker::SolverKind>);
    static_assert(std::is_same_v<ab::CostModelParams, atucker::selector::CostModelParams>);
    REQUIRE(maps_to<atucker::NotSPD>(ATK_NOT_SPD));
    REQUIRE(maps_to<atucker::RankExceedsDim>(ATK_RANK_EXCEEDS_DIM));
    REQUIRE(maps_to<atucker::NoConvergence>(ATK_NO_CONVERGENCE));
    REQUIRE(maps_to<atucker::Error>(ATK_CUDA_ERROR));
    std::printf("PASS reference types\n");
#else
    static_assert(!std::is_same_v<ab::Error, std::runtime_error>);
    std::printf("PASS standalone types\n");
#endif
    // status -> exception, 1:1 with errors.hpp:9-25
    REQUIRE(maps_to<ab::ModeOutOfRange>(ATK_MODE_OUT_OF_RANGE));
    REQUIRE(maps_to<ab::ShapeMismatch>(ATK_SHAPE_MISMATCH));
    REQUIRE(maps_to<ab::NotSquare>(ATK_NOT_SQUARE));
    REQUIRE(maps_to<ab::RankTooLarge>(ATK_RANK_TOO_LARGE));
    REQUIRE(maps_to<ab::RankDeficient>(ATK_RANK_DEFICIENT));
    REQUIRE(maps_to<ab::ZeroNormInput>(ATK_ZERO_NORM_INPUT));
    REQUIRE(maps_to<ab::EmptyDataset>(ATK_EMPTY_DATASET));
    REQUIRE(maps_to<ab::FeatureVersionMismatch>(ATK_FEATURE_VERSION));
    REQUIRE(maps_to<ab::SchemaMismatch>(ATK_SCHEMA_MISMATCH));
    REQUIRE(maps_to<ab::IoFailure>(ATK_IO_FAILURE));
    REQUIRE(maps_to<ab::DeviceError>(ATK_OOM));
    std::printf("PASS status mapping\n");

    // the selector hook trampoline forwards the caller's CostModelParams
    RefSignatureStrategy rs;
    ab::detail::HookBox<RefSignatureStrategy> box{&rs, ab::CostModelParams{5}};
    REQUIRE(ab::detail::HookBox<RefSignatureStrategy>::call(&box, 0, 10, 2, 30) == 0);
    REQUIRE(ab::detail::HookBox<RefSignatureStrategy>::call(&box, 1, 10, 2, 30) == 1);
    box.params.num_iters = 7;
    REQUIRE(ab::detail::HookBox<RefSignatureStrategy>::call(&box, 0, 10, 2, 30) == 1);
    std::printf("PASS reference-signature strategy\n");

    // cost model honours num_iters (selector.hpp:36-58): (64, 8, 1e4) is EIG at
    // 5 ALS iterations and ALS at 2
    auto cm = ab::Strategy::cost_model();
    REQUIRE(cm.decide(0, 64, 8, 10000, ab::CostModelParams{5}) == ab::SolverKind::Eig);
    REQUIRE(cm.decide(0, 64, 8, 10000, ab::CostModelParams{2}) == ab::SolverKind::Als);
#if ATUCKER_B200_REFERENCE_TYPES
    for (int it : {1, 2, 5, 9})
        for (double i : {32.0, 64.0, 128.0, 512.0})
            for (double r : {4.0, 8.0, 16.0})
                for (double j : {1e3, 1e4, 1e6})
                    REQUIRE(cm.decide(0, std::size_t(i), std::size_t(r), std::size_t(j), ab::CostModelParams{it}) ==
                            atucker::selector::heuristic_choice(i, r, j, atucker::selector::CostModelParams{it}));
#endif
    std::printf("PASS cost model params\n");

    // Adaptive: the trained tree's descent (selector.hpp:88-104).  Root: I_n <= 100
    // -> EIG leaf, else R_n^2/I_n (feature 6) <= 0.5 -> ALS leaf, else EIG leaf.
    ab::DecisionTreeModel m;
    m.nodes.resize(5);
    m.nodes[0].feature_index = 0, m.nodes[0].threshold = 100.0, m.nodes[0].left = 1, m.nodes[0].right = 2;
    m.nodes[1].leaf = true, m.nodes[1].label = 0;
    m.nodes[2].feature_index = 6, m.nodes[2].threshold = 0.5, m.nodes[2].left = 3, m.nodes[2].right = 4;
    m.nodes[3].leaf = true, m.nodes[3].label = 1;
    m.nodes[4].leaf = true, m.nodes[4].label = 0;
    m.root = 0;
    auto ad = ab::Strategy::adaptive(m);
    REQUIRE(ad.decide(0, 64, 8, 1000, {}) == ab::SolverKind::Eig);
    REQUIRE(ad.decide(0, 1024, 16, 1000, {}) == ab::SolverKind::Als);   // 256/1024 <= 0.5
    REQUIRE(ad.decide(0, 1024, 32, 1000, {}) == ab::SolverKind::Eig);   // 1024/1024 > 0.5
    ab::DecisionTreeModel bad = m;
    bad.feature_order_version = 2;
    bool thrown = false;
    try {
        ab::Strategy::adaptive(bad).decide(0, 64, 8, 1000, {});
    } catch (const ab::FeatureVersionMismatch&) {
        thrown = true;
    }
    REQUIRE(thrown);
    std::printf("PASS adaptive strategy\n");

    // containers follow tensor.hpp's contract
    thrown = false;
    try {
        ab::DenseMatrix(2, 2, std::vector<double>(3, 0.0));
    } catch (const ab::ShapeMismatch&) {
        thrown = true;
    }
    REQUIRE(thrown);
    ab::DenseTensor t({2, 3}, {1, 2, 3, 4, 5, 6});
    REQUIRE(t.order() == 2 && t.dim(1) == 3 && t.values()[5] == 6.0);
    std::printf("PASS containers\n");
    return 0;
}
