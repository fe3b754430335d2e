// atucker_b200.hpp — C++ drop-in for the reference hot path (namespace
// atucker, /root/reference/proj/include/atucker/{sthosvd,solvers,kernels,
// linalg}.hpp) implemented over the C ABI of atk.h / libatk_cuda.so.
//
// Signatures mirror the reference:
//   sthosvd(x, ranks, strategy, opts)            sthosvd.hpp:126-127
//   eig_mode_solver / als_mode_solver / svd_mode_solver   solvers.hpp:64,122,142
//   kernels::gram / ttm / ttt_mode               kernels.hpp:88,122,127
//   linalg::sym_eig_top_r / thin_qr / spd_solve  linalg.hpp:101,126,169
//   reconstruct / relative_error                 sthosvd.hpp:197,212
// Containers are the reference's layout (column-major doubles).  `Strategy`
// is any type with the reference's `decide(mode, i, r, j, params)` member
// (so atucker::Strategy itself plugs in unchanged) or the local Strategy.
// Errors come back as the reference's exception hierarchy (errors.hpp:9-25) —
// the reference's own types when its headers are on the include path (see
// below) — with sthosvd's "mode n: " prefix preserved (sthosvd.hpp:177-183).
#pragma once

#include <cstdint>
#include <cstdio>
#include <array>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "atk.h"

// Reference types.  When the reference's Eigen-free headers are on the include
// path (atucker/{errors,solver_kind,tensor,selector}.hpp), the drop-in uses
// them directly: atucker::DenseTensor / DenseMatrix go in and come out,
// failures throw atucker::NotSPD and friends, SolverKind is
// atucker::SolverKind and the Adaptive strategy runs the reference's own
// selector::predict.  Without them (the GPU box, a standalone build) the
// same names are declared here with the reference's layout and semantics.
// Define ATUCKER_B200_STANDALONE to force the local declarations.
#if !defined(ATUCKER_B200_STANDALONE) && __has_include("atucker/tensor.hpp") && \
    __has_include("atucker/selector.hpp")
#define ATUCKER_B200_REFERENCE_TYPES 1
#include "atucker/errors.hpp"
#include "atucker/selector.hpp"
#include "atucker/solver_kind.hpp"
#include "atucker/tensor.hpp"

namespace atucker_b200 {
using atucker::DenseMatrix;
using atucker::DenseTensor;
using atucker::EmptyDataset;
using atucker::Error;
using atucker::FeatureVersionMismatch;
using atucker::IoFailure;
using atucker::ModeOutOfRange;
using atucker::NoConvergence;
using atucker::NotSPD;
using atucker::NotSquare;
using atucker::RankDeficient;
using atucker::RankExceedsDim;
using atucker::RankTooLarge;
using atucker::SchemaMismatch;
using atucker::ShapeMismatch;
using atucker::SolverKind;
using atucker::ZeroNormInput;
using atucker::selector::CostModelParams;
using atucker::selector::DecisionTreeModel;
using atucker::selector::extract_features;
using atucker::selector::FeatureVector;
using atucker::selector::predict;
struct DeviceError : Error { using Error::Error; };  // CUDA / NCCL / OOM (no CPU fallback)
}  // namespace atucker_b200
#else
#define ATUCKER_B200_REFERENCE_TYPES 0
namespace atucker_b200 {

// ---------------------------------------------------------------- errors.hpp:9-25
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct ModeOutOfRange : Error { using Error::Error; };
struct ShapeMismatch : Error { using Error::Error; };
struct RankExceedsDim : Error { using Error::Error; };
struct NotSquare : Error { using Error::Error; };
struct RankTooLarge : Error { using Error::Error; };
struct NoConvergence : Error { using Error::Error; };
struct RankDeficient : Error { using Error::Error; };
struct NotSPD : Error { using Error::Error; };
struct ZeroNormInput : Error { using Error::Error; };
struct EmptyDataset : Error { using Error::Error; };
struct FeatureVersionMismatch : Error { using Error::Error; };
struct SchemaMismatch : Error { using Error::Error; };
struct IoFailure : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };  // CUDA / NCCL / OOM (no CPU fallback)

// ---------------------------------------------------------------- tensor.hpp:44-156
struct DenseMatrix {
    DenseMatrix() = default;
    DenseMatrix(std::size_t r, std::size_t c) : rows_(r), cols_(c), data_(r * c, 0.0) {}
    DenseMatrix(std::size_t r, std::size_t c, std::vector<double> d) : rows_(r), cols_(c), data_(std::move(d)) {
        if (data_.size() != r * c) throw ShapeMismatch("matrix data length does not match rows*cols");
    }
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    std::size_t size() const { return data_.size(); }
    double operator()(std::size_t i, std::size_t j) const { return data_[i + rows_ * j]; }
    double& operator()(std::size_t i, std::size_t j) { return data_[i + rows_ * j]; }
    const double* data() const { return data_.data(); }
    double* data() { return data_.data(); }
    const std::vector<double>& values() const { return data_; }

private:
    std::size_t rows_ = 0, cols_ = 0;
    std::vector<double> data_;
};

struct DenseTensor {
    DenseTensor() = default;
    explicit DenseTensor(std::vector<std::size_t> dims) : dims_(std::move(dims)) {
        if (dims_.empty()) throw ShapeMismatch("tensor order must be at least 1");
        std::size_t n = 1;
        for (auto d : dims_) {
            if (d == 0) throw ShapeMismatch("tensor dimensions must be positive");
            n *= d;
        }
        data_.assign(n, 0.0);
    }
    DenseTensor(std::vector<std::size_t> dims, std::vector<double> d) : dims_(std::move(dims)), data_(std::move(d)) {
        std::size_t n = 1;
        for (auto x : dims_) n *= x;
        if (dims_.empty() || n == 0) throw ShapeMismatch("tensor dimensions must be positive");
        if (data_.size() != n) throw ShapeMismatch("tensor data length does not match the product of dims");
    }
    std::size_t order() const { return dims_.size(); }
    const std::vector<std::size_t>& dims() const { return dims_; }
    std::size_t dim(std::size_t m) const { return dims_.at(m); }
    std::size_t size() const { return data_.size(); }
    const double* data() const { return data_.data(); }
    double* data() { return data_.data(); }
    const std::vector<double>& values() const { return data_; }

private:
    std::vector<std::size_t> dims_;
    std::vector<double> data_;
};

enum class SolverKind { Eig = 0, Als = 1, Svd = 2 };  // solver_kind.hpp:11

struct CostModelParams { int num_iters = 5; };  // selector.hpp:31-33

// selector.hpp:19-29, 60-104: the ten shape features and the trained tree's
// deterministic root-to-leaf descent (the tree payload comes from the
// reference's trainer / selector_io; this side only evaluates it).
constexpr int kFeatureOrderVersion = 1;
using FeatureVector = std::array<double, 10>;
inline FeatureVector extract_features(double i, double r, double j) {
    return {i, r, j, i * i, r * r, i * r, r * r / i, r * r / j, i / j, r / j};
}
struct DecisionTreeModel {
    struct Node {
        bool leaf = false;
        int feature_index = -1;
        double threshold = 0.0;
        int left = -1, right = -1, label = 0;
        std::array<long long, 2> class_counts{0, 0};
    };
    std::vector<Node> nodes;
    int root = -1;
    int feature_order_version = kFeatureOrderVersion;
};
inline SolverKind predict(const DecisionTreeModel& m, const FeatureVector& f) {
    if (m.feature_order_version != kFeatureOrderVersion)
        throw FeatureVersionMismatch("model was trained with feature order version " +
                                     std::to_string(m.feature_order_version));
    if (m.root < 0 || m.root >= int(m.nodes.size())) throw SchemaMismatch("decision tree has no valid root");
    int id = m.root;
    for (std::size_t steps = 0; steps <= m.nodes.size(); ++steps) {
        const auto& nd = m.nodes[std::size_t(id)];
        if (nd.leaf) return nd.label == 0 ? SolverKind::Eig : SolverKind::Als;
        id = f[std::size_t(nd.feature_index)] <= nd.threshold ? nd.left : nd.right;
        if (id < 0 || id >= int(m.nodes.size())) throw SchemaMismatch("decision tree child id out of range");
    }
    throw SchemaMismatch("decision tree descent did not reach a leaf");
}
}  // namespace atucker_b200
#endif

namespace atucker_b200 {

inline void check(atk_status s) {
    if (s == ATK_OK) return;
    const std::string m = atk_last_error();
    switch (s) {
        case ATK_MODE_OUT_OF_RANGE: throw ModeOutOfRange(m);
        case ATK_SHAPE_MISMATCH: throw ShapeMismatch(m);
        case ATK_RANK_EXCEEDS_DIM: throw RankExceedsDim(m);
        case ATK_NOT_SQUARE: throw NotSquare(m);
        case ATK_RANK_TOO_LARGE: throw RankTooLarge(m);
        case ATK_NO_CONVERGENCE: throw NoConvergence(m);
        case ATK_RANK_DEFICIENT: throw RankDeficient(m);
        case ATK_NOT_SPD: throw NotSPD(m);
        case ATK_ZERO_NORM_INPUT: throw ZeroNormInput(m);
        case ATK_EMPTY_DATASET: throw EmptyDataset(m);
        case ATK_FEATURE_VERSION: throw FeatureVersionMismatch(m);
        case ATK_SCHEMA_MISMATCH: throw SchemaMismatch(m);
        case ATK_IO_FAILURE: throw IoFailure(m);
        case ATK_CUDA_ERROR: case ATK_NCCL_ERROR: case ATK_OOM: throw DeviceError(m);
        default: throw Error(m);
    }
}

struct AlsOptions {  // solvers.hpp:18-22
    int num_iters = 5;
    double rel_tol = 0.0;
    std::uint64_t seed = 0;
};

// Local Strategy (sthosvd.hpp:39-107): the trained tree (Adaptive), the flop
// cost model, a fixed choice, a manual list, the B200 roofline model, or any
// callable hook.  `decide` forwards the caller's CostModelParams (sthosvd
// passes {opts.num_iters}, as sthosvd.hpp:160 does).
class Strategy {
public:
    using Hook = std::function<SolverKind(std::size_t, std::size_t, std::size_t, std::size_t, const CostModelParams&)>;
    static Strategy adaptive(DecisionTreeModel model) {
        return Strategy([m = std::move(model)](std::size_t, std::size_t i, std::size_t r, std::size_t j,
                                               const CostModelParams&) {
            return predict(m, extract_features(double(i), double(r), double(j)));
        });
    }
    static Strategy fixed_eig() { return Strategy([](auto...) { return SolverKind::Eig; }); }
    static Strategy fixed_als() { return Strategy([](auto...) { return SolverKind::Als; }); }
    static Strategy fixed_svd() { return Strategy([](auto...) { return SolverKind::Svd; }); }
    static Strategy cost_model() {  // selector.hpp:52-58, ties go to EIG
        return Strategy([](std::size_t, std::size_t i, std::size_t r, std::size_t j, const CostModelParams& p) {
            return atk_cost_eig(double(i), double(r), double(j)) <=
                           atk_cost_als(double(i), double(r), double(j), p.num_iters)
                       ? SolverKind::Eig : SolverKind::Als;
        });
    }
    // B200 roofline model (atk_roofline_selector): stage time = max(flops / peak,
    // bytes / HBM bandwidth) + measured fixed costs; SURVEY §8(f) row 2.
    static Strategy roofline(atk_dtype dtype = ATK_F32, int num_iters = 5) {
        atk_roofline_params p;
        atk_roofline_params_default(&p, int(dtype), num_iters);
        return Strategy([p](std::size_t mode, std::size_t i, std::size_t r, std::size_t j, const CostModelParams&) {
            auto q = p;
            return atk_roofline_selector(&q, int(mode), i, r, j) == ATK_SOLVER_EIG ? SolverKind::Eig
                                                                                    : SolverKind::Als;
        });
    }
    static Strategy manual(std::vector<SolverKind> c) {
        for (auto k : c) if (k == SolverKind::Svd) throw Error("manual strategies choose between eig and als");
        return Strategy([c](std::size_t mode, std::size_t, std::size_t, std::size_t, const CostModelParams&) {
            return c.at(mode);
        }, c.size());
    }
    explicit Strategy(Hook h, std::size_t manual_len = 0) : hook_(std::move(h)), manual_len_(manual_len) {}
    SolverKind decide(std::size_t mode, std::size_t i, std::size_t r, std::size_t j,
                      const CostModelParams& params) const {
        return hook_(mode, i, r, j, params);
    }
    std::size_t manual_len() const { return manual_len_; }

private:
    Hook hook_;
    std::size_t manual_len_;
};

struct ModeReport {  // sthosvd.hpp:25-34 (+ device per-stage times)
    std::size_t mode = 0;
    SolverKind solver_used = SolverKind::Eig;
    double selector_decision_time = 0.0, solver_time = 0.0;
    double predicted_cost_eig = 0.0, predicted_cost_als = 0.0;
    std::vector<std::size_t> dims_before, dims_after;
    atk_stage_times times{};
};

struct TuckerDecomposition {  // sthosvd.hpp:18-22
    DenseTensor core;
    std::vector<DenseMatrix> factors;
    std::vector<std::size_t> original_dims;
};

struct SthosvdResult {  // sthosvd.hpp:109-112
    TuckerDecomposition decomposition;
    std::vector<ModeReport> reports;
};

// ---------------------------------------------------------------- engine context
class Engine {
public:
    static Engine& instance(int device = 0) {
        static Engine e(device);
        return e;
    }
    atk_ctx* ctx() const { return ctx_; }
    ~Engine() { if (ctx_) atk_ctx_destroy(ctx_); }

private:
    explicit Engine(int device) { check(atk_ctx_create(device, &ctx_)); }
    atk_ctx* ctx_ = nullptr;
};

namespace detail {
struct Dev {  // RAII device tensor
    atk_tensor* t = nullptr;
    Dev() = default;
    explicit Dev(const DenseTensor& x) {
        std::vector<uint64_t> d(x.dims().begin(), x.dims().end());
        check(atk_tensor_from_host(Engine::instance().ctx(), ATK_F64, int(d.size()), d.data(), x.data(), &t));
    }
    ~Dev() { if (t) atk_tensor_free(t); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    DenseTensor host() const {
        atk_dtype dt;
        int order;
        uint64_t dims[ATK_MAX_ORDER];
        check(atk_tensor_info(t, &dt, &order, dims, nullptr));
        DenseTensor out(std::vector<std::size_t>(dims, dims + order));
        check(atk_tensor_to_host(Engine::instance().ctx(), t, out.data()));
        return out;
    }
};

template <class S>
struct HookBox {
    const S* s;
    CostModelParams params;
    static int call(void* user, int mode, uint64_t i, uint64_t r, uint64_t j) {
        auto* b = static_cast<HookBox*>(user);
        try {
            return static_cast<int>(b->s->decide(std::size_t(mode), std::size_t(i), std::size_t(r), std::size_t(j), b->params));
        } catch (...) {
            return -1;
        }
    }
};
}  // namespace detail

// ---------------------------------------------------------------- kernels.hpp
namespace kernels {
inline DenseMatrix gram(const DenseTensor& x, std::size_t mode) {
    detail::Dev d(x);
    if (mode >= x.order()) throw ModeOutOfRange("mode " + std::to_string(mode) + " out of range");
    DenseMatrix s(x.dim(mode), x.dim(mode));
    check(atk_gram(Engine::instance().ctx(), d.t, int(mode), s.data()));
    return s;
}
inline DenseTensor ttm(const DenseTensor& x, const DenseMatrix& u, std::size_t mode) {
    detail::Dev d(x);
    detail::Dev y;
    check(atk_ttm(Engine::instance().ctx(), d.t, u.data(), u.rows(), u.cols(), int(mode), &y.t));
    return y.host();
}
inline DenseMatrix ttt_mode(const DenseTensor& x, const DenseTensor& y, std::size_t mode) {
    detail::Dev a(x), b(y);
    if (mode >= x.order() || mode >= y.order()) throw ModeOutOfRange("mode out of range");
    DenseMatrix z(x.dim(mode), y.dim(mode));
    check(atk_ttt(Engine::instance().ctx(), a.t, b.t, int(mode), z.data()));
    return z;
}
}  // namespace kernels

// ---------------------------------------------------------------- linalg.hpp
namespace linalg {
struct EigPair { std::vector<double> values; DenseMatrix vectors; };
struct QrPair { DenseMatrix q, r; };
inline EigPair sym_eig_top_r(const DenseMatrix& s, std::size_t r) {
    if (s.rows() != s.cols()) throw NotSquare("sym_eig_top_r expects a square matrix");
    EigPair p{std::vector<double>(r), DenseMatrix(s.rows(), r)};
    check(atk_sym_eig_top_r(Engine::instance().ctx(), s.data(), s.rows(), r, p.values.data(), p.vectors.data()));
    return p;
}
inline QrPair thin_qr(const DenseMatrix& a) {
    QrPair p{DenseMatrix(a.rows(), a.cols()), DenseMatrix(a.cols(), a.cols())};
    check(atk_thin_qr(Engine::instance().ctx(), a.data(), a.rows(), a.cols(), p.q.data(), p.r.data()));
    return p;
}
inline DenseMatrix spd_solve(const DenseMatrix& a, const DenseMatrix& b) {
    if (a.rows() != a.cols()) throw NotSquare("spd_solve expects a square matrix");
    DenseMatrix x(b.rows(), b.cols());
    check(atk_spd_solve(Engine::instance().ctx(), a.data(), a.rows(), b.data(), b.cols(), x.data()));
    return x;
}
}  // namespace linalg

// ---------------------------------------------------------------- solvers.hpp
struct ModeResult {  // solvers.hpp:26-31
    DenseMatrix factor;
    DenseTensor shrunk;
    int iterations_run = 0;
    SolverKind solver_used = SolverKind::Eig;
};

inline ModeResult eig_mode_solver(const DenseTensor& y, std::size_t mode, std::size_t r) {
    detail::Dev d(y), s;
    if (mode >= y.order()) throw ModeOutOfRange("mode out of range");
    ModeResult out{DenseMatrix(y.dim(mode), r), {}, 0, SolverKind::Eig};
    check(atk_eig_mode(Engine::instance().ctx(), d.t, int(mode), r, out.factor.data(), &s.t, nullptr));
    out.shrunk = s.host();
    return out;
}

inline ModeResult als_mode_solver(const DenseTensor& y, std::size_t mode, std::size_t r, const AlsOptions& opts = {}) {
    detail::Dev d(y), s;
    if (mode >= y.order()) throw ModeOutOfRange("mode out of range");
    ModeResult out{DenseMatrix(y.dim(mode), r), {}, 0, SolverKind::Als};
    atk_als_opts o{opts.num_iters, opts.rel_tol, opts.seed};
    check(atk_als_mode(Engine::instance().ctx(), d.t, int(mode), r, &o, nullptr, out.factor.data(), &s.t,
                       &out.iterations_run, nullptr));
    out.shrunk = s.host();
    return out;
}

inline ModeResult svd_mode_solver(const DenseTensor& y, std::size_t mode, std::size_t r) {
    detail::Dev d(y), s;
    if (mode >= y.order()) throw ModeOutOfRange("mode out of range");
    ModeResult out{DenseMatrix(y.dim(mode), r), {}, 0, SolverKind::Svd};
    check(atk_svd_mode(Engine::instance().ctx(), d.t, int(mode), r, out.factor.data(), &s.t, nullptr));
    out.shrunk = s.host();
    return out;
}

// ---------------------------------------------------------------- sthosvd.hpp
template <class StrategyT>
SthosvdResult sthosvd(const DenseTensor& x, const std::vector<std::size_t>& ranks, const StrategyT& strategy,
                      const AlsOptions& opts = {}) {
    const std::size_t order = x.order();
    if (ranks.size() != order)
        throw RankExceedsDim("expected " + std::to_string(order) + " truncations, got " + std::to_string(ranks.size()));
    if constexpr (std::is_same_v<StrategyT, Strategy>) {
        if (strategy.manual_len() && strategy.manual_len() != order)
            throw Error("manual strategy must choose a solver for each of the " + std::to_string(order) + " modes");
    }
    detail::Dev d(x), core;
    detail::HookBox<StrategyT> box{&strategy, CostModelParams{opts.num_iters}};
    std::vector<uint64_t> rk(ranks.begin(), ranks.end());
    std::size_t ftotal = 0;
    for (std::size_t n = 0; n < order; ++n) ftotal += x.dim(n) * ranks[n];
    std::vector<double> factors(ftotal);
    std::vector<atk_mode_report> reps(order);
    atk_als_opts o{opts.num_iters, opts.rel_tol, opts.seed};
    check(atk_sthosvd(Engine::instance().ctx(), d.t, rk.data(), &detail::HookBox<StrategyT>::call, &box, &o, &core.t,
                      factors.data(), reps.data()));
    SthosvdResult res;
    res.decomposition.core = core.host();
    res.decomposition.original_dims = x.dims();
    std::size_t off = 0;
    for (std::size_t n = 0; n < order; ++n) {
        std::vector<double> f(factors.begin() + off, factors.begin() + off + x.dim(n) * ranks[n]);
        off += x.dim(n) * ranks[n];
        res.decomposition.factors.emplace_back(x.dim(n), ranks[n], std::move(f));
        ModeReport r;
        r.mode = n;
        r.solver_used = static_cast<SolverKind>(reps[n].solver_used);
        r.selector_decision_time = reps[n].selector_decision_time;
        r.solver_time = reps[n].solver_time;
        r.predicted_cost_eig = reps[n].predicted_cost_eig;
        r.predicted_cost_als = reps[n].predicted_cost_als;
        r.dims_before.assign(reps[n].dims_before, reps[n].dims_before + order);
        r.dims_after.assign(reps[n].dims_after, reps[n].dims_after + order);
        r.times = reps[n].times;
        res.reports.push_back(std::move(r));
    }
    return res;
}

inline double relative_error(const DenseTensor& x, const TuckerDecomposition& t) {
    detail::Dev d(x), c(t.core);
    std::vector<double> flat;
    for (const auto& f : t.factors) flat.insert(flat.end(), f.data(), f.data() + f.size());
    double out = 0.0;
    check(atk_relative_error(Engine::instance().ctx(), d.t, c.t, flat.data(), &out));
    return out;
}

inline DenseTensor reconstruct(const TuckerDecomposition& t) {
    detail::Dev c(t.core), y;
    std::vector<double> flat;
    for (const auto& f : t.factors) flat.insert(flat.end(), f.data(), f.data() + f.size());
    std::vector<uint64_t> od(t.original_dims.begin(), t.original_dims.end());
    check(atk_reconstruct(Engine::instance().ctx(), c.t, flat.data(), od.data(), &y.t));
    return y.host();
}

// ---------------------------------------------------------------- tensor_io.hpp:15-99
// Host containers: the reference's format, written and read on the host
// (header-only, byte-identical to the reference's writer).  Large tensors:
// read_dten_device streams the file straight into HBM through the engine
// (atk_tensor_read_dten: double-buffered pinned chunks, fp32 narrowing on the
// device) and hands back an engine handle for atk_sthosvd.
inline void write_dten(const std::string& path, const std::vector<std::size_t>& dims, const double* data) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw IoFailure("cannot open " + path + " for writing");
    const std::uint32_t version = 1, order = static_cast<std::uint32_t>(dims.size());
    std::vector<std::uint64_t> d64(dims.begin(), dims.end());
    std::size_t n = 1;
    for (auto d : dims) n *= d;
    bool ok = std::fwrite("DTEN", 1, 4, f) == 4 && std::fwrite(&version, 4, 1, f) == 1 &&
              std::fwrite(&order, 4, 1, f) == 1 && std::fwrite(d64.data(), 8, d64.size(), f) == d64.size() &&
              std::fwrite(data, 8, n, f) == n;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw IoFailure("failed writing " + path);
}
inline void write_dten(const std::string& path, const DenseTensor& x) { write_dten(path, x.dims(), x.data()); }
inline void write_dten(const std::string& path, const DenseMatrix& m) {
    write_dten(path, {m.rows(), m.cols()}, m.data());
}

inline DenseTensor read_dten(const std::string& path) {
    int order = 0;
    std::uint64_t dims[ATK_MAX_ORDER] = {};
    check(atk_dten_info(path.c_str(), &order, dims));  // the engine's header validation
    std::vector<std::size_t> d(dims, dims + order);
    DenseTensor t(d);
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw IoFailure("cannot open " + path);
    std::fseek(f, long(12 + 8 * order), SEEK_SET);
    const std::size_t got = std::fread(t.data(), 8, t.size(), f);
    std::fclose(f);
    if (got != t.size())
        throw IoFailure(path + ": truncated payload, expected " + std::to_string(t.size() * 8) +
                        " bytes but read " + std::to_string(got * 8));
    return t;
}
inline DenseMatrix read_dten_matrix(const std::string& path) {
    DenseTensor t = read_dten(path);
    if (t.order() != 2) throw IoFailure(path + ": expected an order-2 .dten");
    return DenseMatrix(t.dim(0), t.dim(1), std::vector<double>(t.data(), t.data() + t.size()));
}
// Engine handle (caller frees with atk_tensor_free).
inline atk_tensor* read_dten_device(const std::string& path, atk_dtype dtype = ATK_F32) {
    atk_tensor* t = nullptr;
    check(atk_tensor_read_dten(Engine::instance().ctx(), path.c_str(), dtype, &t));
    return t;
}

}  // namespace atucker_b200
