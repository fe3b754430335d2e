// C++ drop-in check: the reference's calling convention (atucker::sthosvd et al.)
// through include/atucker_b200.hpp + libatk_cuda.so.  Built and run by
// tests/test_gpu_cpp.py on the GPU box; prints PASS lines, exits non-zero on failure.
#include <cmath>
#include <cstdio>
#include <random>

#include "atucker_b200.hpp"

using namespace atucker_b200;

static DenseTensor random_signed(std::vector<std::size_t> dims, std::uint64_t seed) {
    DenseTensor x(std::move(dims));
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> g(0.0, 1.0);
    for (std::size_t i = 0; i < x.size(); ++i) x.data()[i] = g(rng);
    return x;
}

#define REQUIRE(c)                                                  \
    do {                                                            \
        if (!(c)) {                                                 \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            return 1;                                               \
        }                                                           \
    } while (0)

int main(int argc, char** argv) {
    // full ranks give an exact decomposition (test_sthosvd.cpp:54-58)
    DenseTensor x = random_signed({8, 7, 6}, 5);
    SthosvdResult res = sthosvd(x, {8, 7, 6}, Strategy::fixed_eig());
    REQUIRE(relative_error(x, res.decomposition) <= 1e-12);
    std::printf("PASS full-rank exact\n");

    // manual strategy recorded in the reports (test_sthosvd.cpp:110-131)
    DenseTensor y = random_signed({9, 8, 7}, 13);
    res = sthosvd(y, {3, 4, 5}, Strategy::manual({SolverKind::Eig, SolverKind::Als, SolverKind::Eig}));
    REQUIRE(res.reports.size() == 3);
    REQUIRE(res.reports[1].solver_used == SolverKind::Als);
    REQUIRE(res.decomposition.core.dims() == std::vector<std::size_t>({3, 4, 5}));
    std::printf("PASS manual strategy\n");

    // gram closed form (test_kernels.cpp:97-101)
    DenseTensor ones({2, 3, 4}, std::vector<double>(24, 1.0));
    DenseMatrix g = kernels::gram(ones, 1);
    for (std::size_t i = 0; i < g.size(); ++i) REQUIRE(g.data()[i] == 8.0);
    std::printf("PASS gram ones\n");

    // error taxonomy crosses the ABI (test_sthosvd.cpp:190-205, test_linalg.cpp:212-217)
    bool thrown = false;
    try {
        sthosvd(y, {3, 4}, Strategy::fixed_eig());
    } catch (const RankExceedsDim&) {
        thrown = true;
    }
    REQUIRE(thrown);
    thrown = false;
    try {
        DenseMatrix neg(2, 2);
        neg(0, 0) = 1.0;
        neg(1, 1) = -1.0;
        linalg::spd_solve(neg, DenseMatrix(2, 1, {2.0, 8.0}));
    } catch (const NotSPD&) {
        thrown = true;
    }
    REQUIRE(thrown);
    thrown = false;
    try {
        DenseTensor thin = random_signed({9, 2, 2}, 37);
        sthosvd(thin, {5, 1, 1}, Strategy::fixed_svd());
    } catch (const Error& e) {
        thrown = std::string(e.what()).find("mode 1") != std::string::npos;
    }
    REQUIRE(thrown);
    std::printf("PASS error taxonomy\n");

    // tensor_io.hpp: the reference-written golden round-trips byte-identically
    // on the host; the engine streams it into HBM unchanged
    if (argc > 1) {
        const std::string golden = std::string(argv[1]) + "/ref_normal_4x3x5_seed7.dten";
        DenseTensor g = read_dten(golden);
        REQUIRE(g.dims() == std::vector<std::size_t>({4, 3, 5}));
        const std::string out = std::string(argv[2]) + "/cpp_roundtrip.dten";
        write_dten(out, g);
        auto slurp = [](const std::string& p) {
            std::vector<char> b;
            FILE* f = std::fopen(p.c_str(), "rb");
            for (int c; (c = std::fgetc(f)) != EOF;) b.push_back(char(c));
            std::fclose(f);
            return b;
        };
        REQUIRE(slurp(out) == slurp(golden));
        atk_tensor* d = read_dten_device(golden, ATK_F64);
        std::vector<double> back(g.size());
        check(atk_tensor_to_host(Engine::instance().ctx(), d, back.data()));
        atk_tensor_free(d);
        for (std::size_t i = 0; i < back.size(); ++i) REQUIRE(back[i] == g.data()[i]);
        thrown = false;
        try {
            read_dten(std::string(argv[2]) + "/missing.dten");
        } catch (const IoFailure&) {
            thrown = true;
        }
        REQUIRE(thrown);
        std::printf("PASS dten io\n");
    }
    return 0;
}
