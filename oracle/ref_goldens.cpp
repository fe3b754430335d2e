// ref_goldens.cpp — golden-vector generator built FROM THE REFERENCE'S OWN
// Eigen-free headers (compiled in place under /root/reference/proj/include by
// oracle/Makefile target `ref`; output binary lives in oracle/_ref/, never
// committed).  Test infrastructure only: it pins the oracle's restatement of
// mix_seed / random_tensor / the ALS initial-guess stream / the cost model to
// the reference itself.  Output: JSON on stdout -> tests/golden/ref_goldens.json
// (regenerate with `make -C oracle goldens`).
#include <cstdio>
#include <random>
#include <vector>

#include "atucker/selector.hpp"
#include "atucker/tensor.hpp"

using namespace atucker;

static void dump(const char* key, const std::vector<double>& v, bool last = false) {
    std::printf("  \"%s\": [", key);
    for (size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? ", " : "", v[i]);
    std::printf("]%s\n", last ? "" : ",");
}

int main() {
    std::printf("{\n");
    std::printf("  \"mix_seed\": [[0, 0, \"%llu\"], [5, 1, \"%llu\"], [2024, 0, \"%llu\"], [7, 3, \"%llu\"]],\n",
                (unsigned long long)detail::mix_seed(0, 0), (unsigned long long)detail::mix_seed(5, 1),
                (unsigned long long)detail::mix_seed(2024, 0), (unsigned long long)detail::mix_seed(7, 3));
    {
        DenseTensor u = random_tensor({3, 3}, 42, Distribution::Uniform01);
        dump("uniform_3x3_seed42", u.values());
    }
    {
        DenseTensor g = random_tensor({3, 4, 5}, 42, Distribution::StandardNormal);
        dump("normal_3x4x5_seed42", g.values());
        std::printf("  \"normal_3x4x5_seed42_norm\": %.17g,\n", frobenius_norm(g));
    }
    {
        DenseTensor c1 = random_tensor({200, 200, 200}, 1, Distribution::StandardNormal);
        std::vector<double> head(c1.values().begin(), c1.values().begin() + 8);
        std::vector<double> tail(c1.values().end() - 4, c1.values().end());
        dump("c1_head", head);
        dump("c1_tail", tail);
        std::printf("  \"c1_norm\": %.17g,\n", frobenius_norm(c1));
    }
    {
        // ALS initial guess stream (solvers.hpp:125-128) for seed 0 / mode 0 and seed 3 / mode 2.
        std::vector<double> a, b;
        std::mt19937_64 r0(detail::mix_seed(0, 0));
        std::normal_distribution<double> g0(0.0, 1.0);
        for (int i = 0; i < 16; ++i) a.push_back(g0(r0));
        std::mt19937_64 r1(detail::mix_seed(3, 2));
        std::normal_distribution<double> g1(0.0, 1.0);
        for (int i = 0; i < 16; ++i) b.push_back(g1(r1));
        dump("als_l0_seed0_mode0", a);
        dump("als_l0_seed3_mode2", b);
    }
    {
        std::vector<double> ce, ca;
        const double cases[][3] = {{10, 2, 100}, {200, 20, 40000}, {1024, 32, 1048576}, {2048, 64, 4194304}, {48, 8, 5308416}};
        for (auto& c : cases) {
            ce.push_back(selector::cost_eig(c[0], c[1], c[2]));
            ca.push_back(selector::cost_als(c[0], c[1], c[2]));
        }
        dump("cost_eig", ce);
        dump("cost_als", ca, true);
    }
    std::printf("}\n");
    return 0;
}
