// atk_oracle.cpp — CPU restatement of the a-Tucker st-HOSVD hot path.
//
// TEST INFRASTRUCTURE ONLY.  This library is the *checker*: tests/, the
// `smoke()` entry and bench.py's `cpu_baseline` / `--impl reference` legs may
// load it; the product path (paper_2010_10131_b200/, libatk_cuda.so) never
// does.  It restates the reference algorithm (reference: /root/reference/proj,
// header-only C++20 + Eigen 3, which is NOT buildable here: Eigen/vendor/Catch2
// absent) with the arithmetic delegated to LAPACK/BLAS (scipy's bundled
// OpenBLAS, loaded with dlopen; path passed by the caller).
//
// Every function cites the reference file:line it follows.  Layout contract
// (tensor.hpp:99-156): column-major, element (i_1..i_N) at
// i_1 + I_1*i_2 + I_1*I_2*i_3 + ...; matrices column-major (i + rows*j).
//
// Parity is pinned by tests/test_oracle_*.py against (a) golden vectors
// produced by the reference's own Eigen-free headers compiled here
// (oracle/ref_goldens.cpp -> oracle/_ref/, tests/golden/ref_goldens.json) and
// (b) the reference's closed-form KATs / properties (tests/*.cpp restated).

#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- errors
// errors.hpp:9-25 — status codes mirror include/atk.h (atk_status).
enum Status {
    OK = 0,
    E_ERROR = 1,
    E_MODE_OUT_OF_RANGE = 2,
    E_SHAPE_MISMATCH = 3,
    E_RANK_EXCEEDS_DIM = 4,
    E_NOT_SQUARE = 5,
    E_RANK_TOO_LARGE = 6,
    E_NO_CONVERGENCE = 7,
    E_RANK_DEFICIENT = 8,
    E_NOT_SPD = 9,
    E_ZERO_NORM_INPUT = 10,
    E_INVALID_ARGUMENT = 23,
};

struct Err : std::runtime_error {
    int code;
    Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

thread_local std::string g_last_error;

// ---------------------------------------------------------------- BLAS
using dgemm_t = void (*)(const char*, const char*, const int*, const int*, const int*,
                         const double*, const double*, const int*, const double*, const int*,
                         const double*, double*, const int*, size_t, size_t);
using dsyevd_t = void (*)(const char*, const char*, const int*, double*, const int*, double*,
                          double*, const int*, int*, const int*, int*, size_t, size_t);
using dgeqrf_t = void (*)(const int*, const int*, double*, const int*, double*, double*,
                          const int*, int*);
using dorgqr_t = void (*)(const int*, const int*, const int*, double*, const int*, const double*,
                          double*, const int*, int*);
using dpotrf_t = void (*)(const char*, const int*, double*, const int*, int*, size_t);
using dpotrs_t = void (*)(const char*, const int*, const int*, const double*, const int*,
                          double*, const int*, int*, size_t);
using dgesdd_t = void (*)(const char*, const int*, const int*, double*, const int*, double*,
                          double*, const int*, double*, const int*, double*, const int*, int*,
                          int*, size_t);
using setthreads_t = void (*)(int);

struct Blas {
    void* h = nullptr;
    dgemm_t dgemm = nullptr;
    dsyevd_t dsyevd = nullptr;
    dgeqrf_t dgeqrf = nullptr;
    dorgqr_t dorgqr = nullptr;
    dpotrf_t dpotrf = nullptr;
    dpotrs_t dpotrs = nullptr;
    dgesdd_t dgesdd = nullptr;
    setthreads_t set_threads = nullptr;
} g_blas;

static void* sym(void* h, const char* name) {
    void* p = dlsym(h, name);
    if (!p) throw Err(E_ERROR, std::string("oracle: missing BLAS symbol ") + name);
    return p;
}

static void need_blas() {
    if (!g_blas.h) throw Err(E_ERROR, "oracle: or_init(blas_path) not called");
}

// ---------------------------------------------------------------- counters
// instrumentation.hpp:13-34: one record per logical GEMM with its flop charge.
std::atomic<long long> g_calls{0}, g_flops{0};
inline void record_gemm(long long charge) {
    g_calls.fetch_add(1, std::memory_order_relaxed);
    g_flops.fetch_add(charge, std::memory_order_relaxed);
}

// Per-stage wall timers (seconds) accumulated by the solvers; bench.py reads
// them for the CPU baseline's per-stage split.
double g_t_gram = 0, g_t_eig = 0, g_t_ttm = 0, g_t_als = 0;
using clk = std::chrono::steady_clock;
inline double since(clk::time_point t0) {
    return std::chrono::duration<double>(clk::now() - t0).count();
}

// ---------------------------------------------------------------- types
struct Tensor {
    std::vector<uint64_t> dims;
    std::vector<double> v;
    uint64_t size() const { return v.size(); }
    uint64_t dim(size_t m) const { return dims.at(m); }
    size_t order() const { return dims.size(); }
};

struct Matrix {
    uint64_t rows = 0, cols = 0;
    std::vector<double> v;
    Matrix() = default;
    Matrix(uint64_t r, uint64_t c) : rows(r), cols(c), v(r * c, 0.0) {}
    double& operator()(uint64_t i, uint64_t j) { return v[i + rows * j]; }
    double operator()(uint64_t i, uint64_t j) const { return v[i + rows * j]; }
    static Matrix identity(uint64_t n) {
        Matrix m(n, n);
        for (uint64_t i = 0; i < n; ++i) m(i, i) = 1.0;
        return m;
    }
};

static uint64_t prod(const std::vector<uint64_t>& d) {
    uint64_t p = 1;
    for (auto x : d) p *= x;
    return p;
}

// tensor.hpp:26-31
static void validate_dims(const std::vector<uint64_t>& dims) {
    if (dims.empty()) throw Err(E_SHAPE_MISMATCH, "tensor order must be at least 1");
    for (auto d : dims)
        if (d == 0) throw Err(E_SHAPE_MISMATCH, "tensor dimensions must be positive");
}

// tensor.hpp:33-39 (splitmix64 finalizer)
uint64_t mix_seed(uint64_t seed, uint64_t salt) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// tensor.hpp:175-187
struct Split {
    uint64_t inner = 1, axis = 1, outer = 1;
};
static Split loop_split(const std::vector<uint64_t>& dims, size_t mode) {
    Split s;
    for (size_t m = 0; m < mode; ++m) s.inner *= dims[m];
    s.axis = dims[mode];
    for (size_t m = mode + 1; m < dims.size(); ++m) s.outer *= dims[m];
    return s;
}

// tensor.hpp:189-193
static void check_mode(size_t order, size_t mode) {
    if (mode >= order)
        throw Err(E_MODE_OUT_OF_RANGE, "mode " + std::to_string(mode) + " out of range for order " +
                                           std::to_string(order));
}

// tensor.hpp:158-168
double frob(const double* x, uint64_t n) {
    double s = 0.0;
    for (uint64_t i = 0; i < n; ++i) s += x[i] * x[i];
    return std::sqrt(s);
}

// ---------------------------------------------------------------- GEMM
// C(m x n) = op(A) * op(B) (+ beta C), column-major, plain dgemm.
static void gemm_raw(bool ta, bool tb, uint64_t m, uint64_t n, uint64_t k, const double* a,
                     uint64_t lda, const double* b, uint64_t ldb, double* c, uint64_t ldc,
                     double beta = 0.0) {
    need_blas();
    if (m == 0 || n == 0) return;
    const double one = 1.0;
    if (k == 0) {
        for (uint64_t j = 0; j < n; ++j)
            for (uint64_t i = 0; i < m; ++i) c[i + ldc * j] *= beta;
        return;
    }
    const uint64_t kmax = 0x7fffffffULL;
    // K can exceed int range at the big configs: chunk it (beta=1 after the first).
    uint64_t k0 = 0;
    double bcur = beta;
    while (k0 < k) {
        const uint64_t kc = std::min(kmax, k - k0);
        int im = int(m), in = int(n), ik = int(kc), ilda = int(lda), ildb = int(ldb), ildc = int(ldc);
        const double* ap = ta ? a + k0 : a + k0 * lda;
        const double* bp = tb ? b + k0 * ldb : b + k0;
        g_blas.dgemm(ta ? "T" : "N", tb ? "T" : "N", &im, &in, &ik, &one, ap, &ilda, bp, &ildb,
                     &bcur, c, &ildc, 1, 1);
        bcur = 1.0;
        k0 += kc;
    }
}

// linalg.hpp:75-97
Matrix gemm(const Matrix& a, const Matrix& b, bool ta = false, bool tb = false) {
    const uint64_t m = ta ? a.cols : a.rows;
    const uint64_t k = ta ? a.rows : a.cols;
    const uint64_t kb = tb ? b.cols : b.rows;
    const uint64_t n = tb ? b.rows : b.cols;
    if (k != kb) throw Err(E_SHAPE_MISMATCH, "gemm inner dimensions disagree");
    Matrix c(m, n);
    gemm_raw(ta, tb, m, n, k, a.v.data(), std::max<uint64_t>(1, a.rows), b.v.data(),
             std::max<uint64_t>(1, b.rows), c.v.data(), std::max<uint64_t>(1, m));
    record_gemm(2LL * (long long)m * (long long)n * (long long)k);
    return c;
}

// ---------------------------------------------------------------- kernels.hpp
// kernels.hpp:34-80 — Z = X_(n) Y_(n)^T in the three loop regimes; middle
// modes accumulate per-slab GEMMs in long double (kernels.hpp:59-78).
static Matrix ttt_impl(const Tensor& x, const Tensor& y, size_t mode, bool half_flops) {
    check_mode(x.order(), mode);
    check_mode(y.order(), mode);
    if (x.order() != y.order()) throw Err(E_SHAPE_MISMATCH, "ttt_mode operands differ in order");
    for (size_t m = 0; m < x.order(); ++m)
        if (m != mode && x.dim(m) != y.dim(m))
            throw Err(E_SHAPE_MISMATCH,
                      "ttt_mode operands disagree on dimension " + std::to_string(m));
    const Split sx = loop_split(x.dims, mode);
    const uint64_t rows = sx.axis, cols = y.dim(mode);
    const long long scale = half_flops ? 1 : 2;
    Matrix z(rows, cols);
    if (mode == 0) {
        const uint64_t j = sx.inner * sx.outer;
        gemm_raw(false, true, rows, cols, j, x.v.data(), rows, y.v.data(), cols, z.v.data(), rows);
        record_gemm(scale * (long long)(rows * cols) * (long long)j);
    } else if (mode + 1 == x.order()) {
        const uint64_t p = sx.inner;
        gemm_raw(true, false, rows, cols, p, x.v.data(), p, y.v.data(), p, z.v.data(), rows);
        record_gemm(scale * (long long)(rows * cols) * (long long)p);
    } else {
        const uint64_t p = sx.inner;
        std::vector<long double> acc(rows * cols, 0.0L);
        std::vector<double> tmp(rows * cols);
        for (uint64_t o = 0; o < sx.outer; ++o) {
            gemm_raw(true, false, rows, cols, p, x.v.data() + o * p * rows, p,
                     y.v.data() + o * p * cols, p, tmp.data(), rows);
            for (size_t i = 0; i < acc.size(); ++i) acc[i] += tmp[i];
            record_gemm(scale * (long long)(rows * cols) * (long long)p);
        }
        for (size_t i = 0; i < acc.size(); ++i) z.v[i] = double(acc[i]);
    }
    return z;
}

// kernels.hpp:88-118 — Y = X x_n U, U is R x I_n.
Tensor ttm(const Tensor& x, const Matrix& u, size_t mode) {
    check_mode(x.order(), mode);
    if (u.cols != x.dim(mode))
        throw Err(E_SHAPE_MISMATCH, "ttm matrix has " + std::to_string(u.cols) +
                                        " columns but mode has dimension " +
                                        std::to_string(x.dim(mode)));
    const Split s = loop_split(x.dims, mode);
    const uint64_t r = u.rows;
    Tensor out;
    out.dims = x.dims;
    out.dims[mode] = r;
    out.v.assign(prod(out.dims), 0.0);
    const auto t0 = clk::now();
    if (mode == 0) {
        const uint64_t j = s.inner * s.outer;
        gemm_raw(false, false, r, j, s.axis, u.v.data(), r, x.v.data(), s.axis, out.v.data(), r);
        record_gemm(2LL * (long long)(r * j) * (long long)s.axis);
    } else if (mode + 1 == x.order()) {
        const uint64_t p = s.inner;
        gemm_raw(false, true, p, r, s.axis, x.v.data(), p, u.v.data(), r, out.v.data(), p);
        record_gemm(2LL * (long long)(r * p) * (long long)s.axis);
    } else {
        const uint64_t p = s.inner;
        for (uint64_t o = 0; o < s.outer; ++o) {
            gemm_raw(false, true, p, r, s.axis, x.v.data() + o * p * s.axis, p, u.v.data(), r,
                     out.v.data() + o * p * r, p);
            record_gemm(2LL * (long long)(r * p) * (long long)s.axis);
        }
    }
    g_t_ttm += since(t0);
    return out;
}

// kernels.hpp:122-124
Matrix ttt_mode(const Tensor& x, const Tensor& y, size_t mode) {
    return ttt_impl(x, y, mode, false);
}

// kernels.hpp:127-138 — symmetrized self-TTT, charged I^2 J.
Matrix gram(const Tensor& x, size_t mode) {
    const auto t0 = clk::now();
    Matrix z = ttt_impl(x, x, mode, true);
    const uint64_t n = z.rows;
    for (uint64_t j = 0; j < n; ++j)
        for (uint64_t i = j + 1; i < n; ++i) {
            const double v = 0.5 * (z(i, j) + z(j, i));
            z(i, j) = v;
            z(j, i) = v;
        }
    g_t_gram += since(t0);
    return z;
}

// tensor.hpp:201-241 — explicit unfolding (SVD solver / test oracle only).
Matrix matricize(const Tensor& x, size_t mode) {
    check_mode(x.order(), mode);
    const Split s = loop_split(x.dims, mode);
    Matrix m(s.axis, s.inner * s.outer);
    for (uint64_t o = 0; o < s.outer; ++o)
        for (uint64_t a = 0; a < s.axis; ++a) {
            const double* slab = x.v.data() + (o * s.axis + a) * s.inner;
            for (uint64_t p = 0; p < s.inner; ++p) m.v[a + s.axis * (o * s.inner + p)] = slab[p];
        }
    return m;
}

Tensor tensorize(const Matrix& m, std::vector<uint64_t> dims, size_t mode) {
    validate_dims(dims);
    check_mode(dims.size(), mode);
    const Split s = loop_split(dims, mode);
    if (m.rows != s.axis || m.cols != s.inner * s.outer)
        throw Err(E_SHAPE_MISMATCH, "matrix shape does not match the requested folding");
    Tensor x;
    x.dims = dims;
    x.v.assign(prod(dims), 0.0);
    for (uint64_t o = 0; o < s.outer; ++o)
        for (uint64_t a = 0; a < s.axis; ++a) {
            double* slab = x.v.data() + (o * s.axis + a) * s.inner;
            for (uint64_t p = 0; p < s.inner; ++p) slab[p] = m.v[a + s.axis * (o * s.inner + p)];
        }
    return x;
}

// ---------------------------------------------------------------- linalg.hpp
// linalg.hpp:34-50 — flip each column so its largest-|v| entry (first on ties)
// is positive; `coupled` (rows of V^T for the SVD) flips with it.
static void fix_signs(Matrix& v, Matrix* coupled_rows = nullptr) {
    for (uint64_t j = 0; j < v.cols; ++j) {
        uint64_t best = 0;
        double mag = 0.0;
        for (uint64_t i = 0; i < v.rows; ++i) {
            const double a = std::fabs(v(i, j));
            if (a > mag) {
                mag = a;
                best = i;
            }
        }
        if (v(best, j) < 0.0) {
            for (uint64_t i = 0; i < v.rows; ++i) v(i, j) = -v(i, j);
            if (coupled_rows)
                for (uint64_t c = 0; c < coupled_rows->cols; ++c)
                    (*coupled_rows)(j, c) = -(*coupled_rows)(j, c);
        }
    }
}

struct EigPair {
    std::vector<double> values;
    Matrix vectors;
};

// linalg.hpp:101-123 — symmetrize, all eigenpairs, keep top r descending, fix signs.
EigPair sym_eig_top_r(const Matrix& s, uint64_t r) {
    if (s.rows != s.cols) throw Err(E_NOT_SQUARE, "sym_eig_top_r expects a square matrix");
    const uint64_t n = s.rows;
    if (r < 1 || r > n)
        throw Err(E_RANK_TOO_LARGE, "requested " + std::to_string(r) + " eigenpairs of a " +
                                        std::to_string(n) + "x" + std::to_string(n) + " matrix");
    need_blas();
    const auto t0 = clk::now();
    std::vector<double> a(n * n);
    for (uint64_t j = 0; j < n; ++j)
        for (uint64_t i = 0; i < n; ++i) a[i + n * j] = 0.5 * (s(i, j) + s(j, i));
    std::vector<double> w(n);
    int in = int(n), lda = int(n), info = 0, lwork = -1, liwork = -1, iwq = 0;
    double wq = 0;
    g_blas.dsyevd("V", "L", &in, a.data(), &lda, w.data(), &wq, &lwork, &iwq, &liwork, &info, 1, 1);
    lwork = int(wq) + 1;
    liwork = iwq + 1;
    std::vector<double> work(lwork);
    std::vector<int> iwork(liwork);
    g_blas.dsyevd("V", "L", &in, a.data(), &lda, w.data(), work.data(), &lwork, iwork.data(),
                  &liwork, &info, 1, 1);
    if (info != 0) throw Err(E_NO_CONVERGENCE, "symmetric eigendecomposition failed");
    EigPair out;
    out.values.resize(r);
    out.vectors = Matrix(n, r);
    for (uint64_t j = 0; j < r; ++j) {
        const uint64_t src = n - 1 - j;  // LAPACK returns ascending
        out.values[j] = w[src];
        std::memcpy(&out.vectors.v[n * j], &a[n * src], n * sizeof(double));
    }
    fix_signs(out.vectors);
    g_t_eig += since(t0);
    return out;
}

struct QrPair {
    Matrix q, r;
};

// linalg.hpp:126-149 — Householder thin QR, diag(R) >= 0, RankDeficient floor.
QrPair thin_qr(const Matrix& a) {
    if (a.rows < a.cols) throw Err(E_SHAPE_MISMATCH, "thin_qr expects rows >= cols");
    need_blas();
    const uint64_t m = a.rows, n = a.cols;
    std::vector<double> f = a.v;
    std::vector<double> tau(std::max<uint64_t>(1, n));
    int im = int(m), in = int(n), lda = int(std::max<uint64_t>(1, m)), info = 0, lwork = -1;
    double wq = 0;
    g_blas.dgeqrf(&im, &in, f.data(), &lda, tau.data(), &wq, &lwork, &info);
    lwork = std::max(1, int(wq));
    std::vector<double> work(lwork);
    g_blas.dgeqrf(&im, &in, f.data(), &lda, tau.data(), work.data(), &lwork, &info);
    QrPair out;
    out.r = Matrix(n, n);
    for (uint64_t j = 0; j < n; ++j)
        for (uint64_t i = 0; i <= j; ++i) out.r(i, j) = f[i + m * j];
    lwork = -1;
    g_blas.dorgqr(&im, &in, &in, f.data(), &lda, tau.data(), &wq, &lwork, &info);
    lwork = std::max(1, int(wq));
    work.assign(lwork, 0.0);
    g_blas.dorgqr(&im, &in, &in, f.data(), &lda, tau.data(), work.data(), &lwork, &info);
    out.q = Matrix(m, n);
    out.q.v.assign(f.begin(), f.begin() + m * n);
    for (uint64_t k = 0; k < n; ++k) {
        if (out.r(k, k) < 0.0) {
            for (uint64_t c = 0; c < n; ++c) out.r(k, c) = -out.r(k, c);
            for (uint64_t i = 0; i < m; ++i) out.q(i, k) = -out.q(i, k);
        }
    }
    const double floor = 1e-12 * frob(a.v.data(), a.v.size());
    for (uint64_t k = 0; k < n; ++k)
        if (std::fabs(out.r(k, k)) < floor)
            throw Err(E_RANK_DEFICIENT, "QR diagonal " + std::to_string(k) + " below tolerance");
    return out;
}

struct SvdResult {
    Matrix u;
    std::vector<double> sigma;
    Matrix vt;
};

// linalg.hpp:153-166 — thin SVD, sigma descending, sign rule on U (V coupled).
SvdResult thin_svd(const Matrix& a) {
    if (a.v.empty()) throw Err(E_SHAPE_MISMATCH, "thin_svd expects a nonempty matrix");
    need_blas();
    const uint64_t m = a.rows, n = a.cols, k = std::min(m, n);
    std::vector<double> f = a.v;
    SvdResult out;
    out.u = Matrix(m, k);
    out.vt = Matrix(k, n);
    out.sigma.assign(k, 0.0);
    int im = int(m), in = int(n), lda = int(m), ldu = int(m), ldvt = int(k), info = 0, lwork = -1;
    std::vector<int> iwork(8 * k);
    double wq = 0;
    g_blas.dgesdd("S", &im, &in, f.data(), &lda, out.sigma.data(), out.u.v.data(), &ldu,
                  out.vt.v.data(), &ldvt, &wq, &lwork, iwork.data(), &info, 1);
    lwork = int(wq) + 1;
    std::vector<double> work(lwork);
    g_blas.dgesdd("S", &im, &in, f.data(), &lda, out.sigma.data(), out.u.v.data(), &ldu,
                  out.vt.v.data(), &ldvt, work.data(), &lwork, iwork.data(), &info, 1);
    if (info != 0) throw Err(E_NO_CONVERGENCE, "singular value decomposition failed");
    fix_signs(out.u, &out.vt);
    return out;
}

// linalg.hpp:169-177 — Cholesky solve, NotSPD on a non-positive pivot.
Matrix spd_solve(const Matrix& a, const Matrix& b) {
    if (a.rows != a.cols) throw Err(E_NOT_SQUARE, "spd_solve expects a square matrix");
    if (a.rows != b.rows) throw Err(E_SHAPE_MISMATCH, "spd_solve right-hand side has wrong row count");
    need_blas();
    std::vector<double> l = a.v;
    int in = int(a.rows), lda = int(std::max<uint64_t>(1, a.rows)), info = 0;
    g_blas.dpotrf("L", &in, l.data(), &lda, &info, 1);
    if (info != 0) throw Err(E_NOT_SPD, "Cholesky factorization hit a non-positive pivot");
    Matrix x = b;
    int nrhs = int(b.cols), ldb = lda;
    g_blas.dpotrs("L", &in, &nrhs, l.data(), &lda, x.v.data(), &ldb, &info, 1);
    return x;
}

// ---------------------------------------------------------------- solvers.hpp
struct AlsOptions {
    int num_iters = 5;
    double rel_tol = 0.0;
    uint64_t seed = 0;
};

struct ModeResult {
    Matrix factor;
    Tensor shrunk;
    int iterations_run = 0;
    int solver_used = 0;
};

// solvers.hpp:35-41
static void check_truncation(const Tensor& y, size_t mode, uint64_t r) {
    check_mode(y.order(), mode);
    if (r < 1 || r > y.dim(mode))
        throw Err(E_RANK_EXCEEDS_DIM, "truncation " + std::to_string(r) + " invalid for mode " +
                                          std::to_string(mode) + " of dimension " +
                                          std::to_string(y.dim(mode)));
}

static Matrix transposed(const Matrix& m) {
    Matrix t(m.cols, m.rows);
    for (uint64_t j = 0; j < m.cols; ++j)
        for (uint64_t i = 0; i < m.rows; ++i) t(j, i) = m(i, j);
    return t;
}

// solvers.hpp:50-58
static double rel_change(const Matrix& next, const Matrix& prev) {
    double diff = 0, base = 0;
    for (size_t i = 0; i < prev.v.size(); ++i) {
        const double d = next.v[i] - prev.v[i];
        diff += d * d;
        base += prev.v[i] * prev.v[i];
    }
    return base > 0.0 ? std::sqrt(diff / base) : 0.0;
}

// solvers.hpp:64-73
ModeResult eig_mode_solver(const Tensor& y, size_t mode, uint64_t r) {
    check_truncation(y, mode, r);
    const Matrix s = gram(y, mode);
    EigPair e = sym_eig_top_r(s, r);
    ModeResult out;
    out.shrunk = ttm(y, transposed(e.vectors), mode);
    out.factor = std::move(e.vectors);
    out.solver_used = 0;
    return out;
}

struct AlsIterateResult {
    Matrix l;
    Tensor rfac;
    int iterations_run = 0;
};

// solvers.hpp:88-118 — update order: W=ttm(Y,L^T); rfac=ttm(W,(L^T L)^-1);
// YR=ttt(Y,rfac); GR=ttt(rfac,rfac); L=YR GR^-1; early stop on rel_change.
AlsIterateResult als_iterate(const Tensor& y, size_t mode, Matrix l0, const AlsOptions& opts,
                             std::vector<double>* l_history = nullptr) {
    check_mode(y.order(), mode);
    if (l0.rows != y.dim(mode))
        throw Err(E_SHAPE_MISMATCH, "initial guess has " + std::to_string(l0.rows) +
                                        " rows but mode has dimension " +
                                        std::to_string(y.dim(mode)));
    if (opts.num_iters < 1) throw Err(E_ERROR, "num_iters must be at least 1");
    const auto t0 = clk::now();
    const uint64_t r = l0.cols;
    const Matrix eye = Matrix::identity(r);
    AlsIterateResult out;
    out.l = std::move(l0);
    for (int k = 0; k < opts.num_iters; ++k) {
        Tensor w = ttm(y, transposed(out.l), mode);
        Matrix gl = gemm(out.l, out.l, true, false);
        out.rfac = ttm(w, spd_solve(gl, eye), mode);
        Matrix yr = ttt_mode(y, out.rfac, mode);
        Matrix gr = ttt_mode(out.rfac, out.rfac, mode);
        Matrix next = gemm(yr, spd_solve(gr, eye));
        out.iterations_run = k + 1;
        const double change = rel_change(next, out.l);
        out.l = std::move(next);
        if (l_history) l_history->insert(l_history->end(), out.l.v.begin(), out.l.v.end());
        if (opts.rel_tol > 0.0 && change <= opts.rel_tol) break;
    }
    g_t_als += since(t0);
    return out;
}

// solvers.hpp:122-138 — L0 ~ N(0,1) from mt19937_64(mix_seed(seed, mode)).
Matrix als_initial_guess(uint64_t rows, uint64_t r, uint64_t seed, uint64_t mode) {
    Matrix l0(rows, r);
    std::mt19937_64 rng(mix_seed(seed, mode));
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (auto& v : l0.v) v = gauss(rng);
    return l0;
}

ModeResult als_mode_solver(const Tensor& y, size_t mode, uint64_t r, const AlsOptions& opts) {
    check_truncation(y, mode, r);
    Matrix l0 = als_initial_guess(y.dim(mode), r, opts.seed, mode);
    AlsIterateResult it = als_iterate(y, mode, std::move(l0), opts);
    const auto t0 = clk::now();
    QrPair qr = thin_qr(it.l);
    ModeResult out;
    out.shrunk = ttm(it.rfac, qr.r, mode);
    out.factor = std::move(qr.q);
    out.iterations_run = it.iterations_run;
    out.solver_used = 1;
    g_t_als += since(t0);
    return out;
}

// solvers.hpp:142-162 — explicit-unfolding truncated SVD (accuracy oracle).
ModeResult svd_mode_solver(const Tensor& y, size_t mode, uint64_t r) {
    check_truncation(y, mode, r);
    const Matrix m = matricize(y, mode);
    if (r > std::min(m.rows, m.cols))
        throw Err(E_RANK_TOO_LARGE, "truncation exceeds the rank bound of the unfolding");
    SvdResult svd = thin_svd(m);
    ModeResult out;
    out.factor = Matrix(m.rows, r);
    for (uint64_t j = 0; j < r; ++j)
        for (uint64_t i = 0; i < m.rows; ++i) out.factor(i, j) = svd.u(i, j);
    Matrix b(r, m.cols);
    for (uint64_t jc = 0; jc < m.cols; ++jc)
        for (uint64_t i = 0; i < r; ++i) b(i, jc) = svd.sigma[i] * svd.vt(i, jc);
    std::vector<uint64_t> dims = y.dims;
    dims[mode] = r;
    out.shrunk = tensorize(b, dims, mode);
    out.solver_used = 2;
    return out;
}

// ---------------------------------------------------------------- selector.hpp
// selector.hpp:36-58 (cost model used by Strategy::cost_model)
double f_eig(double i) { return 9.0 * i * i * i; }
double f_qr(double i, double r) { return 2.0 * i * r * r - (2.0 / 3.0) * r * r * r; }
double f_inv(double r) { return 2.0 * r * r * r; }
double cost_eig(double i, double r, double j) { return i * i * j + 2.0 * i * r * j + f_eig(i); }
double cost_als(double i, double r, double j, int num_iters) {
    const double per_iter = 2.0 * i * j * r + 2.0 * j * r * r + 2.0 * i * j * r + 2.0 * j * r * r +
                            4.0 * i * r * r + 2.0 * f_inv(r);
    return per_iter * num_iters + 2.0 * j * r * r + f_qr(i, r);
}

// ---------------------------------------------------------------- sthosvd.hpp
typedef int (*selector_fn)(void* user, int mode, uint64_t i, uint64_t r, uint64_t j);

struct Report {
    int solver_used;
    double decide_s, solve_s, cost_eig, cost_als;
};

// sthosvd.hpp:126-194 — ascending mode loop over the shrinking work tensor.
void sthosvd(const Tensor& x, const std::vector<uint64_t>& ranks, selector_fn decide, void* user,
             const AlsOptions& opts, Tensor& core, std::vector<Matrix>& factors,
             std::vector<Report>& reports) {
    const size_t order = x.order();
    if (ranks.size() != order)
        throw Err(E_RANK_EXCEEDS_DIM, "expected " + std::to_string(order) + " truncations, got " +
                                          std::to_string(ranks.size()));
    for (size_t n = 0; n < order; ++n)
        if (ranks[n] < 1 || ranks[n] > x.dim(n))
            throw Err(E_RANK_EXCEEDS_DIM, "truncation " + std::to_string(ranks[n]) +
                                              " invalid for mode " + std::to_string(n) +
                                              " of dimension " + std::to_string(x.dim(n)));
    factors.assign(order, Matrix());
    reports.clear();
    Tensor work = x;
    for (size_t n = 0; n < order; ++n) {
        const uint64_t i = work.dim(n), r = ranks[n];
        uint64_t j = 1;
        for (size_t m = 0; m < order; ++m)
            if (m != n) j *= work.dim(m);
        Report rep{};
        rep.cost_eig = cost_eig(double(i), double(r), double(j));
        rep.cost_als = cost_als(double(i), double(r), double(j), opts.num_iters);
        auto td = clk::now();
        int choice = decide ? decide(user, int(n), i, r, j) : 0;
        rep.decide_s = since(td);
        if (choice < 0) throw Err(E_INVALID_ARGUMENT, "selector callback failed");
        auto ts = clk::now();
        ModeResult mr;
        try {
            switch (choice) {
                case 0: mr = eig_mode_solver(work, n, r); break;
                case 1: mr = als_mode_solver(work, n, r, opts); break;
                case 2: mr = svd_mode_solver(work, n, r); break;
                default: throw Err(E_INVALID_ARGUMENT, "unknown solver kind");
            }
        } catch (const Err& e) {
            // sthosvd.hpp:177-183: NotSPD / NoConvergence keep their type, the rest become Error.
            const int code = (e.code == E_NOT_SPD || e.code == E_NO_CONVERGENCE) ? e.code : E_ERROR;
            throw Err(code, "mode " + std::to_string(n + 1) + ": " + e.what());
        }
        rep.solve_s = since(ts);
        rep.solver_used = mr.solver_used;
        factors[n] = std::move(mr.factor);
        work = std::move(mr.shrunk);
        reports.push_back(rep);
    }
    core = std::move(work);
}

// sthosvd.hpp:197-209
Tensor reconstruct(const Tensor& core, const std::vector<Matrix>& factors,
                   const std::vector<uint64_t>& original_dims) {
    const size_t order = core.order();
    if (factors.size() != order || original_dims.size() != order)
        throw Err(E_SHAPE_MISMATCH, "decomposition has inconsistent order");
    Tensor y = core;
    for (size_t n = 0; n < order; ++n) {
        if (factors[n].rows != original_dims[n] || factors[n].cols != y.dim(n))
            throw Err(E_SHAPE_MISMATCH, "factor " + std::to_string(n + 1) +
                                            " does not match the core and original dims");
        y = ttm(y, factors[n], n);
    }
    return y;
}

// sthosvd.hpp:212-223
double relative_error(const Tensor& x, const Tensor& core, const std::vector<Matrix>& factors) {
    const double nx = frob(x.v.data(), x.v.size());
    if (nx == 0.0) throw Err(E_ZERO_NORM_INPUT, "relative error is undefined for a zero tensor");
    Tensor xh = reconstruct(core, factors, x.dims);
    if (xh.dims != x.dims) throw Err(E_SHAPE_MISMATCH, "reconstruction shape differs from input");
    double s = 0.0;
    for (uint64_t i = 0; i < x.size(); ++i) {
        const double d = xh.v[i] - x.v[i];
        s += d * d;
    }
    return std::sqrt(s) / nx;
}

// tensor.hpp:246-258 — sequential mt19937_64 fill.
void random_tensor(uint64_t n, uint64_t seed, int dist, double* out) {
    std::mt19937_64 rng(seed);
    if (dist == 0) {
        std::uniform_real_distribution<double> u(0.0, 1.0);
        for (uint64_t i = 0; i < n; ++i) out[i] = u(rng);
    } else {
        std::normal_distribution<double> g(0.0, 1.0);
        for (uint64_t i = 0; i < n; ++i) out[i] = g(rng);
    }
}

// generators.hpp:17-35
Tensor synth_lowrank(const std::vector<uint64_t>& dims, const std::vector<uint64_t>& ranks,
                     uint64_t seed) {
    if (dims.size() != ranks.size())
        throw Err(E_SHAPE_MISMATCH, "synth_lowrank dims and ranks differ in length");
    for (size_t n = 0; n < dims.size(); ++n)
        if (ranks[n] < 1 || ranks[n] > dims[n])
            throw Err(E_RANK_EXCEEDS_DIM, "rank " + std::to_string(ranks[n]) +
                                              " invalid for dimension " + std::to_string(dims[n]) +
                                              " at mode " + std::to_string(n));
    Tensor x;
    x.dims = ranks;
    x.v.resize(prod(ranks));
    random_tensor(x.v.size(), mix_seed(seed, 0), 1, x.v.data());
    for (size_t n = 0; n < dims.size(); ++n) {
        Matrix g(dims[n], ranks[n]);
        std::mt19937_64 rng(mix_seed(seed, n + 1));
        std::normal_distribution<double> gauss(0.0, 1.0);
        for (auto& v : g.v) v = gauss(rng);
        x = ttm(x, thin_qr(g).q, n);
    }
    return x;
}

// Counter-hash uniform [-1, 1) on a 2^-23 grid (exactly representable in
// fp32): the generator the CUDA engine implements bit-identically on device
// (paper_2010_10131_b200/csrc/atk_gen.cu) for the big fp32 configs.
inline uint64_t hash64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
inline float hash_uniform(uint64_t seed, uint64_t idx) {
    const uint64_t h = hash64(idx ^ hash64(seed));
    const int32_t k = int32_t(h >> 40) - (1 << 23);  // [-2^23, 2^23)
    return float(k) * (1.0f / 8388608.0f);
}

// ---------------------------------------------------------------- C helpers
static Tensor make_tensor(const double* x, const uint64_t* dims, int nd) {
    Tensor t;
    t.dims.assign(dims, dims + nd);
    validate_dims(t.dims);
    t.v.assign(x, x + prod(t.dims));
    return t;
}

static Matrix make_matrix(const double* a, uint64_t rows, uint64_t cols) {
    Matrix m(rows, cols);
    if (rows != 0 && cols != 0) std::memcpy(m.v.data(), a, rows * cols * sizeof(double));
    return m;
}

template <class F>
static int guard(F&& f) {
    try {
        f();
        return OK;
    } catch (const Err& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return E_ERROR;
    }
}

}  // namespace orc

using namespace orc;

extern "C" {

const char* or_last_error(void) { return g_last_error.c_str(); }

int or_init(const char* blas_path) {
    return guard([&] {
        if (g_blas.h) return;
        void* h = dlopen(blas_path, RTLD_NOW | RTLD_LOCAL);
        if (!h) throw Err(E_ERROR, std::string("oracle: dlopen failed: ") + dlerror());
        g_blas.dgemm = (dgemm_t)sym(h, "scipy_dgemm_");
        g_blas.dsyevd = (dsyevd_t)sym(h, "scipy_dsyevd_");
        g_blas.dgeqrf = (dgeqrf_t)sym(h, "scipy_dgeqrf_");
        g_blas.dorgqr = (dorgqr_t)sym(h, "scipy_dorgqr_");
        g_blas.dpotrf = (dpotrf_t)sym(h, "scipy_dpotrf_");
        g_blas.dpotrs = (dpotrs_t)sym(h, "scipy_dpotrs_");
        g_blas.dgesdd = (dgesdd_t)sym(h, "scipy_dgesdd_");
        g_blas.set_threads = (setthreads_t)sym(h, "scipy_openblas_set_num_threads");
        g_blas.h = h;
        g_blas.set_threads(1);  // reference build is single-threaded (README.md:95-96)
    });
}

void or_set_threads(int n) {
    if (g_blas.set_threads) g_blas.set_threads(n < 1 ? 1 : n);
}

uint64_t or_mix_seed(uint64_t seed, uint64_t salt) { return mix_seed(seed, salt); }

void or_reset_counters(void) {
    g_calls = 0;
    g_flops = 0;
    g_t_gram = g_t_eig = g_t_ttm = g_t_als = 0;
}
long long or_gemm_calls(void) { return g_calls.load(); }
long long or_gemm_flops(void) { return g_flops.load(); }
void or_stage_times(double* out4) {
    out4[0] = g_t_gram;
    out4[1] = g_t_eig;
    out4[2] = g_t_ttm;
    out4[3] = g_t_als;
}

double or_cost_eig(double i, double r, double j) { return cost_eig(i, r, j); }
double or_cost_als(double i, double r, double j, int iters) { return cost_als(i, r, j, iters); }

int or_random_tensor(const uint64_t* dims, int nd, uint64_t seed, int dist, double* out) {
    return guard([&] {
        std::vector<uint64_t> d(dims, dims + nd);
        validate_dims(d);
        random_tensor(prod(d), seed, dist, out);
    });
}

void or_hash_uniform(uint64_t seed, uint64_t start, uint64_t n, float* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = hash_uniform(seed, start + i);
}

int or_als_initial_guess(uint64_t rows, uint64_t r, uint64_t seed, uint64_t mode, double* out) {
    return guard([&] {
        Matrix l0 = als_initial_guess(rows, r, seed, mode);
        std::memcpy(out, l0.v.data(), l0.v.size() * sizeof(double));
    });
}

double or_frobenius_norm(const double* x, uint64_t n) { return frob(x, n); }

int or_gram(const double* x, const uint64_t* dims, int nd, int mode, double* out) {
    return guard([&] {
        Tensor t = make_tensor(x, dims, nd);
        check_mode(t.order(), size_t(mode));
        Matrix g = gram(t, size_t(mode));
        std::memcpy(out, g.v.data(), g.v.size() * sizeof(double));
    });
}

int or_ttt(const double* x, const uint64_t* xdims, const double* y, const uint64_t* ydims, int nd,
           int mode, double* out) {
    return guard([&] {
        Tensor a = make_tensor(x, xdims, nd), b = make_tensor(y, ydims, nd);
        Matrix z = ttt_mode(a, b, size_t(mode));
        std::memcpy(out, z.v.data(), z.v.size() * sizeof(double));
    });
}

int or_ttm(const double* x, const uint64_t* dims, int nd, const double* u, uint64_t urows,
           uint64_t ucols, int mode, double* out) {
    return guard([&] {
        Tensor t = make_tensor(x, dims, nd);
        Tensor y = ttm(t, make_matrix(u, urows, ucols), size_t(mode));
        std::memcpy(out, y.v.data(), y.v.size() * sizeof(double));
    });
}

int or_matricize(const double* x, const uint64_t* dims, int nd, int mode, double* out) {
    return guard([&] {
        Tensor t = make_tensor(x, dims, nd);
        Matrix m = matricize(t, size_t(mode));
        std::memcpy(out, m.v.data(), m.v.size() * sizeof(double));
    });
}

int or_sym_eig_top_r(const double* s, uint64_t rows, uint64_t cols, uint64_t r, double* values,
                     double* vectors) {
    return guard([&] {
        EigPair e = sym_eig_top_r(make_matrix(s, rows, cols), r);
        std::memcpy(values, e.values.data(), r * sizeof(double));
        std::memcpy(vectors, e.vectors.v.data(), e.vectors.v.size() * sizeof(double));
    });
}

int or_thin_qr(const double* a, uint64_t rows, uint64_t cols, double* q, double* r) {
    return guard([&] {
        QrPair p = thin_qr(make_matrix(a, rows, cols));
        std::memcpy(q, p.q.v.data(), p.q.v.size() * sizeof(double));
        std::memcpy(r, p.r.v.data(), p.r.v.size() * sizeof(double));
    });
}

int or_thin_svd(const double* a, uint64_t rows, uint64_t cols, double* u, double* sigma,
                double* vt) {
    return guard([&] {
        SvdResult s = thin_svd(make_matrix(a, rows, cols));
        std::memcpy(u, s.u.v.data(), s.u.v.size() * sizeof(double));
        std::memcpy(sigma, s.sigma.data(), s.sigma.size() * sizeof(double));
        std::memcpy(vt, s.vt.v.data(), s.vt.v.size() * sizeof(double));
    });
}

int or_spd_solve(const double* a, uint64_t n, const double* b, uint64_t nrhs, double* x) {
    return guard([&] {
        Matrix s = spd_solve(make_matrix(a, n, n), make_matrix(b, n, nrhs));
        std::memcpy(x, s.v.data(), s.v.size() * sizeof(double));
    });
}

int or_gemm(const double* a, uint64_t ar, uint64_t ac, const double* b, uint64_t br, uint64_t bc,
            int ta, int tb, double* c) {
    return guard([&] {
        Matrix m = gemm(make_matrix(a, ar, ac), make_matrix(b, br, bc), ta != 0, tb != 0);
        std::memcpy(c, m.v.data(), m.v.size() * sizeof(double));
    });
}

static void out_mode(const ModeResult& m, double* factor, double* shrunk, int* iters) {
    std::memcpy(factor, m.factor.v.data(), m.factor.v.size() * sizeof(double));
    std::memcpy(shrunk, m.shrunk.v.data(), m.shrunk.v.size() * sizeof(double));
    if (iters) *iters = m.iterations_run;
}

int or_eig_mode(const double* y, const uint64_t* dims, int nd, int mode, uint64_t r,
                double* factor, double* shrunk) {
    return guard([&] {
        Tensor t = make_tensor(y, dims, nd);
        out_mode(eig_mode_solver(t, size_t(mode), r), factor, shrunk, nullptr);
    });
}

int or_svd_mode(const double* y, const uint64_t* dims, int nd, int mode, uint64_t r,
                double* factor, double* shrunk) {
    return guard([&] {
        Tensor t = make_tensor(y, dims, nd);
        out_mode(svd_mode_solver(t, size_t(mode), r), factor, shrunk, nullptr);
    });
}

int or_als_mode(const double* y, const uint64_t* dims, int nd, int mode, uint64_t r, int iters,
                double rel_tol, uint64_t seed, double* factor, double* shrunk, int* iters_run) {
    return guard([&] {
        Tensor t = make_tensor(y, dims, nd);
        AlsOptions o{iters, rel_tol, seed};
        out_mode(als_mode_solver(t, size_t(mode), r, o), factor, shrunk, iters_run);
    });
}

// L history: iters_max * (I*R) doubles (the L after each completed iteration).
int or_als_iterate(const double* y, const uint64_t* dims, int nd, int mode, const double* l0,
                   uint64_t r, int iters, double rel_tol, double* l_out, double* rfac_out,
                   int* iters_run, double* l_history) {
    return guard([&] {
        Tensor t = make_tensor(y, dims, nd);
        check_mode(t.order(), size_t(mode));
        AlsOptions o{iters, rel_tol, 0};
        std::vector<double> hist;
        AlsIterateResult res =
            als_iterate(t, size_t(mode), make_matrix(l0, t.dim(size_t(mode)), r), o,
                        l_history ? &hist : nullptr);
        std::memcpy(l_out, res.l.v.data(), res.l.v.size() * sizeof(double));
        std::memcpy(rfac_out, res.rfac.v.data(), res.rfac.v.size() * sizeof(double));
        *iters_run = res.iterations_run;
        if (l_history) std::memcpy(l_history, hist.data(), hist.size() * sizeof(double));
    });
}

// factors_out: concatenation of I_n x R_n column-major blocks in mode order.
// reports_out: order x 5 doubles {solver, decide_s, solve_s, cost_eig, cost_als}.
int or_sthosvd(const double* x, const uint64_t* dims, int nd, const uint64_t* ranks,
               selector_fn decide, void* user, int iters, double rel_tol, uint64_t seed,
               double* core_out, double* factors_out, double* reports_out) {
    return guard([&] {
        Tensor t = make_tensor(x, dims, nd);
        std::vector<uint64_t> rk(ranks, ranks + nd);
        AlsOptions o{iters, rel_tol, seed};
        Tensor core;
        std::vector<Matrix> factors;
        std::vector<Report> reps;
        sthosvd(t, rk, decide, user, o, core, factors, reps);
        std::memcpy(core_out, core.v.data(), core.v.size() * sizeof(double));
        size_t off = 0;
        for (auto& f : factors) {
            std::memcpy(factors_out + off, f.v.data(), f.v.size() * sizeof(double));
            off += f.v.size();
        }
        if (reports_out)
            for (size_t n = 0; n < reps.size(); ++n) {
                reports_out[5 * n + 0] = reps[n].solver_used;
                reports_out[5 * n + 1] = reps[n].decide_s;
                reports_out[5 * n + 2] = reps[n].solve_s;
                reports_out[5 * n + 3] = reps[n].cost_eig;
                reports_out[5 * n + 4] = reps[n].cost_als;
            }
    });
}

// Memory-lean st-HOSVD of an fp32 tensor (BASELINE C5: 34 GB fp32 would be
// 69 GB as fp64, plus the reference's `work = x` copy).  Same arithmetic as
// sthosvd() with an EIG first mode: the mode-0 Gram X_(0) X_(0)^T
// (kernels.hpp:49-53) and TTM U^T X (kernels.hpp:99-102) are accumulated over
// column chunks converted to fp64 on the fly (dgemm with beta = 1), then the
// remaining modes run on the (small) shrunk fp64 tensor through sthosvd().
int or_sthosvd_f32_eig0(const float* x, const uint64_t* dims, int nd, const uint64_t* ranks,
                        selector_fn decide, void* user, int iters, double rel_tol, uint64_t seed,
                        double* core_out, double* factors_out, int threads) {
    return guard([&] {
        need_blas();
        if (nd < 2) throw Err(E_SHAPE_MISMATCH, "or_sthosvd_f32_eig0 needs order >= 2");
        if (threads > 0) g_blas.set_threads(threads);
        const uint64_t I = dims[0], r0 = ranks[0];
        uint64_t J = 1;
        for (int m = 1; m < nd; ++m) J *= dims[m];
        if (r0 < 1 || r0 > I) throw Err(E_RANK_EXCEEDS_DIM, "truncation invalid for mode 0");
        const uint64_t CH = std::max<uint64_t>(1, (uint64_t(1) << 27) / I);  // ~1 GB fp64 per chunk
        std::vector<double> buf(I * std::min(CH, J));
        // fp32 -> fp64 chunk conversion on the same host threads as the BLAS
        // (an artifact of streaming an fp32 input; the reference holds fp64)
        const int nth = threads > 0 ? threads : 1;
        auto widen = [&](uint64_t j0, uint64_t nc) {
            const uint64_t tot = I * nc;
            std::vector<std::thread> pool;
            for (int t = 0; t < nth; ++t)
                pool.emplace_back([&, t] {
                    const uint64_t a = tot * t / nth, b = tot * (t + 1) / nth;
                    for (uint64_t e = a; e < b; ++e) buf[e] = double(x[I * j0 + e]);
                });
            for (auto& th : pool) th.join();
        };
        auto t_gram = clk::now();
        Matrix s(I, I);
        for (uint64_t j0 = 0; j0 < J; j0 += CH) {
            const uint64_t nc = std::min(CH, J - j0);
            widen(j0, nc);
            gemm_raw(false, true, I, I, nc, buf.data(), I, buf.data(), I, s.v.data(), I, j0 ? 1.0 : 0.0);
        }
        record_gemm((long long)(I * I) * (long long)J);
        for (uint64_t j = 0; j < I; ++j)
            for (uint64_t i = j + 1; i < I; ++i) {
                const double v = 0.5 * (s(i, j) + s(j, i));
                s(i, j) = v;
                s(j, i) = v;
            }
        g_t_gram += since(t_gram);
        EigPair e = sym_eig_top_r(s, r0);  // times itself
        auto t_ttm = clk::now();
        Tensor work;
        work.dims.assign(dims, dims + nd);
        work.dims[0] = r0;
        work.v.assign(r0 * J, 0.0);
        for (uint64_t j0 = 0; j0 < J; j0 += CH) {
            const uint64_t nc = std::min(CH, J - j0);
            widen(j0, nc);
            // Y(:, j0:j0+nc) = U^T X(:, j0:j0+nc)
            gemm_raw(true, false, r0, nc, I, e.vectors.v.data(), I, buf.data(), I, work.v.data() + r0 * j0, r0);
        }
        record_gemm(2LL * (long long)(r0 * J) * (long long)I);
        g_t_ttm += since(t_ttm);
        // remaining modes: the reference loop on the shrunk tensor (mode 0 already done)
        std::vector<uint64_t> rk(ranks, ranks + nd);
        std::vector<Matrix> factors(nd);
        factors[0] = std::move(e.vectors);
        AlsOptions o{iters, rel_tol, seed};
        for (int n = 1; n < nd; ++n) {
            const uint64_t i = work.dim(n), r = rk[n];
            uint64_t j = 1;
            for (int m = 0; m < nd; ++m)
                if (m != n) j *= work.dim(m);
            const int choice = decide ? decide(user, n, i, r, j) : 0;
            ModeResult mr = choice == 1 ? als_mode_solver(work, n, r, o)
                            : choice == 2 ? svd_mode_solver(work, n, r) : eig_mode_solver(work, n, r);
            factors[n] = std::move(mr.factor);
            work = std::move(mr.shrunk);
        }
        std::memcpy(core_out, work.v.data(), work.v.size() * sizeof(double));
        size_t off = 0;
        for (auto& f : factors) {
            std::memcpy(factors_out + off, f.v.data(), f.v.size() * sizeof(double));
            off += f.v.size();
        }
    });
}

// ||X||^2 of an fp32 tensor in fp64 (for the projection identity at full size).
double or_norm2_f32(const float* x, uint64_t n) {
    double s = 0.0;
    for (uint64_t i = 0; i < n; ++i) s += double(x[i]) * double(x[i]);
    return s;
}

static std::vector<Matrix> unpack_factors(const double* factors, const uint64_t* odims,
                                          const uint64_t* ranks, int nd) {
    std::vector<Matrix> f;
    size_t off = 0;
    for (int n = 0; n < nd; ++n) {
        f.push_back(make_matrix(factors + off, odims[n], ranks[n]));
        off += odims[n] * ranks[n];
    }
    return f;
}

int or_reconstruct(const double* core, const uint64_t* ranks, int nd, const double* factors,
                   const uint64_t* odims, double* out) {
    return guard([&] {
        Tensor c = make_tensor(core, ranks, nd);
        std::vector<uint64_t> od(odims, odims + nd);
        Tensor y = reconstruct(c, unpack_factors(factors, odims, ranks, nd), od);
        std::memcpy(out, y.v.data(), y.v.size() * sizeof(double));
    });
}

int or_relative_error(const double* x, const uint64_t* dims, int nd, const double* core,
                      const uint64_t* ranks, const double* factors, double* out) {
    return guard([&] {
        Tensor t = make_tensor(x, dims, nd);
        Tensor c = make_tensor(core, ranks, nd);
        *out = relative_error(t, c, unpack_factors(factors, dims, ranks, nd));
    });
}

int or_synth_lowrank(const uint64_t* dims, const uint64_t* ranks, int nd, uint64_t seed,
                     double* out) {
    return guard([&] {
        Tensor x = synth_lowrank(std::vector<uint64_t>(dims, dims + nd),
                                 std::vector<uint64_t>(ranks, ranks + nd), seed);
        std::memcpy(out, x.v.data(), x.v.size() * sizeof(double));
    });
}

}  // extern "C"
