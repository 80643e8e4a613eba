// Drop-in C++ API tests: the reference's own test style (proj/tests/*.cpp) run against
// include/sketchcp/*.hpp backed by the B200 library. Exit code 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <functional>
#include <string>
#include <vector>

#include "sketchcp/contraction.hpp"
#include "sketchcp/decompose.hpp"
#include "sketchcp/fft.hpp"
#include "sketchcp/hashing.hpp"
#include "sketchcp/lda.hpp"
#include "sketchcp/metrics.hpp"
#include "sketchcp/sketch.hpp"

using namespace sketchcp;

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                                   \
    do {                                                                           \
        if (c) {                                                                   \
            ++g_pass;                                                              \
        } else {                                                                   \
            ++g_fail;                                                              \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);               \
        }                                                                          \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                                   \
    do {                                                                           \
        bool thrown_ = false;                                                      \
        try {                                                                      \
            expr;                                                                  \
        } catch (const T&) {                                                       \
            thrown_ = true;                                                        \
        } catch (...) {                                                            \
        }                                                                          \
        CHECK(thrown_);                                                            \
    } while (0)

static std::vector<std::pair<const char*, std::function<void()>>>& registry() {
    static std::vector<std::pair<const char*, std::function<void()>>> r;
    return r;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { registry().emplace_back(n, std::move(f)); }
};
#define TEST_CASE(name, fn) static void fn(); static Reg reg_##fn(name, fn); static void fn()

static double max_abs_diff(const cvec& a, const cvec& b) {
    double m = 0;
    for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
    return m;
}
static DenseTensor3 random_symmetric(int n, std::uint64_t seed) {
    Rng rng(seed);
    DenseTensor3 T(n);
    for (int i = 0; i < n; ++i)
        for (int j = i; j < n; ++j)
            for (int k = j; k < n; ++k) {
                const double v = rng.gaussian();
                const int p[6][3] = {{i, j, k}, {i, k, j}, {j, i, k}, {j, k, i}, {k, i, j}, {k, j, i}};
                for (auto& q : p) T.at(q[0], q[1], q[2]) = v;
            }
    return T;
}
static DenseTensor3 rank1(const Eigen::VectorXd& u, double a) {
    const int n = static_cast<int>(u.size());
    DenseTensor3 T(n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < n; ++k) T.at(i, j, k) = a * u[i] * u[j] * u[k];
    return T;
}

TEST_CASE("compat Eigen: column-to-column assignment copies coefficients", test_column_assign) {
    Eigen::MatrixXd A(3, 2), B(3, 2);
    for (int i = 0; i < 3; ++i) {
        A(i, 0) = i + 1;
        A(i, 1) = 10 * (i + 1);
    }
    B.col(1) = A.col(0);  // both non-const views: must copy, not rebind
    for (int i = 0; i < 3; ++i) CHECK(B(i, 1) == i + 1 && B(i, 0) == 0.0);
    const Eigen::MatrixXd& Ac = A;
    B.col(0) = Ac.col(1);
    for (int i = 0; i < 3; ++i) CHECK(B(i, 0) == 10 * (i + 1));
}

TEST_CASE("hash KATs (test_hashing.cpp:47-56,142-146)", hash_kats) {
    PolyHash c = PolyHash::from_coefficients({5}, 4);
    for (std::uint64_t i = 0; i < 100; ++i) CHECK(c.eval(i) == 1);
    PolyHash id = PolyHash::from_coefficients({0, 1}, 8);
    for (std::uint64_t i = 0; i < 4096; ++i) CHECK(id.eval(i) == i % 8);
    PolyHash id10 = PolyHash::from_coefficients({0, 1}, 10);
    CHECK(symmetric_bucket(id10, 1, 2, 3) == 6);
    CHECK(symmetric_bucket(id10, 4, 4, 4) == 2);
    PolyHash h = PolyHash::from_seed(6, 1024, 42);  // corrected frozen KAT
    const std::uint32_t kat[10] = {726, 169, 929, 615, 29, 671, 183, 93, 240, 366};
    for (int i = 0; i < 10; ++i) CHECK(h.eval(i) == kat[i]);
    CHECK_THROWS_AS(PolyHash::from_seed(9, 8, 0), std::invalid_argument);
}

TEST_CASE("fft on the device (test_fft.cpp:37-90)", fft_tests) {
    Rng rng(7);
    for (std::size_t b : {2u, 16u, 64u, 1024u, 16384u}) {
        cvec x(b);
        for (auto& z : x) z = {rng.gaussian(), rng.gaussian()};
        cvec y = x;
        fft::forward_inplace(y);
        fft::inverse_inplace(y);
        CHECK(max_abs_diff(x, y) < 1e-12);
    }
    cvec x = {{1, 0}, {2, 0}, {3, 0}, {4, 0}}, y = {{1, 0}, {0, 0}, {0, 0}, {1, 0}};
    cvec z = fft::circular_convolve(x, y);
    CHECK(std::abs(z[0] - std::complex<double>(3, 0)) < 1e-12 && std::abs(z[3] - std::complex<double>(5, 0)) < 1e-12);
    cvec bad(12, {1.0, 0.0});
    CHECK_THROWS_AS(fft::forward_inplace(bad), std::invalid_argument);
    cvec c(16, {1.0, 0.0});
    const auto before = fft::transform_count();
    fft::forward_inplace(c);
    fft::inverse_inplace(c);
    CHECK(fft::transform_count() == before + 2);
}

TEST_CASE("sym set: single-entry recovery and rank-1 identities (SPEC.md:275-295)", sym_identities) {
    const int n = 6;
    DenseTensor3 T(n);
    const int p[6][3] = {{1, 2, 3}, {1, 3, 2}, {2, 1, 3}, {2, 3, 1}, {3, 1, 2}, {3, 2, 1}};
    for (auto& q : p) T.at(q[0], q[1], q[2]) = 6.0;
    SymTensorSketchSet s(n, 64, 5, 9);
    s.accumulate_dense(T);
    CHECK(s.version() == 1);
    CHECK(std::abs(s.recover_entry(1, 2, 3) - 6.0) < 1e-12);
    Eigen::VectorXd u(n);
    Rng rng(3);
    for (int i = 0; i < n; ++i) u[i] = rng.gaussian();
    SymTensorSketchSet a(n, 32, 4, 77), d(n, 32, 4, 77);
    a.add_scaled_rank1(u, 2.5);
    d.accumulate_dense(rank1(u, 2.5), true);
    for (int m = 0; m < 4; ++m) CHECK(max_abs_diff(a.replicate(m).data, d.replicate(m).data) < 1e-9);
    SymTensorSketchSet r = s;  // copy semantics
    r.add_scaled_rank1(u, 1.5);
    r.add_scaled_rank1(u, -1.5);
    for (int m = 0; m < 5; ++m) CHECK(max_abs_diff(r.replicate(m).data, s.replicate(m).data) < 1e-12);
    CHECK_THROWS_AS(s.accumulate_dense(DenseTensor3(n + 1)), std::invalid_argument);
    DenseTensor3 A = random_symmetric(n, 5);
    A.at(0, 1, 2) += 1.0;
    CHECK_THROWS_AS(s.accumulate_dense(A), std::invalid_argument);
}

TEST_CASE("contractions: collision-free rank-1 and mutable_replicate coherence", sym_contractions) {
    const int n = 4;
    DenseTensor3 T(n);
    T.at(0, 0, 0) = 1.0;
    SymTensorSketchSet s(n, 4096, 5, 2);
    s.accumulate_dense(T, true);
    SymContractionWorkspace ws(s);
    Eigen::VectorXd e0 = Eigen::VectorXd::Unit(n, 0);
    Eigen::VectorXd iv = ws.Ivv(e0);
    CHECK(std::abs(iv[0] - 1.0) < 1e-12 && std::abs(iv[1]) < 1e-12);
    CHECK(std::abs(ws.vvv(e0) - 1.0) < 1e-12);
    const cvec f0 = ws.cached_transform(1);
    for (auto& z : s.mutable_replicate(1).data) z *= 2.0;  // host edit, version bump
    CHECK(s.version() == 2);
    const cvec f1 = ws.cached_transform(1);
    double worst = 0;
    for (std::size_t t = 0; t < f0.size(); ++t) worst = std::max(worst, std::abs(f1[t] - 2.0 * f0[t]));
    CHECK(worst < 1e-12);
}

TEST_CASE("robust_tpm_fast noiseless 2 v^3 (SPEC.md:400,407)", rtpm_noiseless) {
    const int n = 8;
    Rng rng(6);
    Eigen::VectorXd v = rng.unit_sphere(n);
    SymTensorSketchSet s(n, 4096, 10, 5);
    s.accumulate_dense(rank1(v, 2.0), true);
    PowerConfig cfg;
    cfg.k = 1;
    cfg.L = 5;
    cfg.T_iters = 10;
    cfg.seed = 1;
    CpDecomposition D = robust_tpm_fast(s, cfg);
    CHECK(std::abs(D.lambda[0] - 2.0) < 2e-2);
    CHECK(std::min((D.A.col(0) - v).norm(), (Eigen::VectorXd(D.A.col(0)) + v).norm()) < 0.05);
    auto match = greedy_match(D.A, D.A);
    CHECK(match.size() == 1 && wrong_vector_count(match) == 0);
    PowerConfig bad = cfg;
    bad.k = n + 1;
    CHECK_THROWS_AS(robust_tpm_fast(s, bad), std::invalid_argument);
    SymTensorSketchSet z(n, 64, 3, 1);
    CHECK_THROWS_AS(robust_tpm_fast(z, cfg), DegenerateIterationError);
}

TEST_CASE("asym set: rank-1 FFT = dense, Ibc(u,u) == Ivv(u) (SPEC.md:237,344)", asym_tests) {
    const int n = 4;
    Rng rng(9);
    Eigen::VectorXd u = rng.gaussian_vector(n), v = rng.gaussian_vector(n), w = rng.gaussian_vector(n);
    AsymTensorSketchSet s(n, 8, 3, 21), d(n, 8, 3, 21);
    DenseTensor3 T(n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < n; ++k) T.at(i, j, k) = u[i] * v[j] * w[k];
    d.accumulate_dense(T);
    for (int m = 0; m < 3; ++m) CHECK(max_abs_diff(s.rank1_sketch(m, u, v, w), d.replicate(m).data) < 1e-10);
    AsymContractionWorkspace ws(d);
    const Eigen::VectorXd a = ws.Ibc(u, u), b = ws.Ivv(u);
    bool same = true;
    for (int i = 0; i < n; ++i) same = same && a[i] == b[i];
    CHECK(same);
    CHECK_THROWS_AS(ws.mode_contraction(3, u, u), std::invalid_argument);
    FactoredTensor F;
    F.n = n;
    F.add(0.5, u, v, w);
    AsymTensorSketchSet f(n, 8, 3, 21);
    f.accumulate_factored(F);
    for (int m = 0; m < 3; ++m) {
        cvec half = d.replicate(m).data;
        for (auto& z : half) z *= 0.5;
        CHECK(max_abs_diff(f.replicate(m).data, half) < 1e-10);
    }
}

TEST_CASE("save/load round trip and peek (sketch.cpp:264-449)", save_load) {
    const auto dir = std::filesystem::temp_directory_path();
    const std::string p = (dir / "skc_dropin_sym.skt").string();
    SymTensorSketchSet s(5, 128, 3, 4);
    s.accumulate_dense(random_symmetric(5, 1), true);
    s.save(p);
    CHECK(peek_sketch_mode(p) == SketchMode::kSym);
    SymTensorSketchSet t = SymTensorSketchSet::load(p);
    for (int m = 0; m < 3; ++m) CHECK(max_abs_diff(t.replicate(m).data, s.replicate(m).data) == 0.0);
    CHECK(t.replicate(2).bucket1 == s.replicate(2).bucket1);
    CHECK_THROWS_AS(AsymTensorSketchSet::load(p), FormatError);
    std::filesystem::remove(p);
}

TEST_CASE("sketch_whitened_m3 stream statistics (lda.cpp:145-226)", lda_stats) {
    Corpus c;
    c.V = 6;
    Rng rng(2);
    for (int d = 0; d < 30; ++d) {
        Document doc;
        const int len = 1 + static_cast<int>(rng.uniform_below(6));
        for (int w = 0; w < c.V && doc.total < len; ++w)
            if (rng.uniform() < 0.5) {
                doc.word.push_back(w);
                doc.count.push_back(1);
                doc.total += 1;
            }
        c.docs.push_back(doc);
    }
    WhiteningMap wm;
    wm.W = Eigen::MatrixXd(c.V, 3);
    for (int i = 0; i < c.V; ++i)
        for (int a = 0; a < 3; ++a) wm.W(i, a) = rng.gaussian();
    SymTensorSketchSet s(3, 64, 2, 8);
    long long used = 0, skipped = 0;
    for (const auto& d : c.docs) (d.total >= 3 ? used : skipped)++;
    StreamStats st = sketch_whitened_m3(c, wm, 1.0, s);
    CHECK(st.used == used && st.skipped == skipped);
    CHECK(s.version() == 2);
    SymTensorSketchSet wrong(4, 64, 2, 8);
    CHECK_THROWS_AS(sketch_whitened_m3(c, wm, 1.0, wrong), std::invalid_argument);
}

TEST_CASE("lda moments, whitening, recovery", lda_whitening_pipeline) {
    // lda.cpp:88-320 through the reference-named API: dense M2 + whiten equals the
    // corpus (implicit-M2) whitening; recover_params yields column-stochastic topics.
    Rng rng(77);
    Corpus c;
    c.V = 40;
    for (int d = 0; d < 400; ++d) {
        Document doc;
        const int topic = d % 3;
        for (int t = 0; t < 20; ++t) {
            int w = (rng.uniform() < 0.8) ? topic * 10 + static_cast<int>(rng.uniform_below(10))
                                          : static_cast<int>(rng.uniform_below(40));
            auto it = std::find(doc.word.begin(), doc.word.end(), w);
            if (it == doc.word.end()) {
                doc.word.push_back(w);
                doc.count.push_back(1);
            } else {
                ++doc.count[it - doc.word.begin()];
            }
            doc.total += 1;
        }
        c.docs.push_back(doc);
    }
    const Eigen::VectorXd m1 = compute_m1(c);
    CHECK(std::abs(m1.sum() - 1.0) < 1e-12);
    const Eigen::MatrixXd m2 = compute_m2(c, 1.0);
    const WhiteningMap a = whiten(m2, 3), b = whiten_corpus(c, 1.0, 3);
    for (int i = 0; i < 3; ++i) CHECK(std::abs(a.singular_values[i] - b.singular_values[i]) < 1e-9 * a.singular_values[i]);
    // W' M2 W = I
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int u = 0; u < c.V; ++u)
                for (int v = 0; v < c.V; ++v) s += b.W(u, i) * m2(u, v) * b.W(v, j);
            CHECK(std::abs(s - (i == j ? 1.0 : 0.0)) < 1e-8);
        }
    CHECK_THROWS_AS(whiten(m2, 41), std::invalid_argument);
    CpDecomposition D = CpDecomposition::symmetric_of(Eigen::VectorXd::Constant(3, 1.5), Eigen::MatrixXd::Identity(3, 3));
    const LdaModel m = recover_params(D, b, 1.0);
    for (int i = 0; i < 3; ++i) {
        double s = 0.0;
        for (int w = 0; w < c.V; ++w) {
            CHECK(m.Phi(w, i) >= 0.0);
            s += m.Phi(w, i);
        }
        CHECK(std::abs(s - 1.0) < 1e-12);
    }
    long long floored = -1;
    const double ll = heldout_likelihood(m, c, &floored);
    CHECK(std::isfinite(ll) && ll < 0.0 && floored >= 0);
    const Eigen::VectorXd y = project_to_simplex(Eigen::VectorXd{0.5, 0.5, 0.5});
    CHECK(std::abs(y[0] - 1.0 / 3.0) < 1e-15);
}

TEST_CASE("fast ALS on the asymmetric set (decompose.cpp:117-205)", als_fast_case) {
    const int n = 16, k = 2;
    Rng rng(5);
    std::vector<double> a(n * k), b(n * k), c(n * k);
    for (auto* f : {&a, &b, &c})
        for (int r = 0; r < k; ++r) {
            auto u = rng.unit_sphere(n);
            for (int i = 0; i < n; ++i) (*f)[r * n + i] = u[i];
        }
    DenseTensor3 T(n);
    const double lam[2] = {3.0, 1.0};
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            for (int q = 0; q < n; ++q) {
                double v = 0.0;
                for (int r = 0; r < k; ++r) v += lam[r] * a[r * n + i] * b[r * n + j] * c[r * n + q];
                T.at(i, j, q) = v;
            }
    AsymTensorSketchSet s(n, 4096, 20, 3);
    s.accumulate_dense(T);
    AlsConfig cfg;
    cfg.k = k;
    cfg.max_iters = 200;
    cfg.tol = 1e-9;
    cfg.seed = 2;
    const CpDecomposition d = als_fast(s, cfg);
    CHECK(d.rank() == k);
    double best0 = 0.0;
    for (int r = 0; r < k; ++r) {
        double dot = 0.0;
        for (int i = 0; i < n; ++i) dot += d.A(i, r) * a[i];
        best0 = std::max(best0, std::abs(dot));
    }
    CHECK(best0 > 0.99);
    AlsConfig bad = cfg;
    bad.k = n + 1;
    CHECK_THROWS_AS(als_fast(s, bad), std::invalid_argument);
    Eigen::MatrixXd G = Eigen::MatrixXd::Identity(3, 3);
    for (int i = 0; i < 3; ++i) G(i, i) = 2.0;
    const Eigen::MatrixXd P = pinv_spectral(G);
    CHECK(std::abs(P(1, 1) - 0.5) < 1e-15 && std::abs(P(0, 1)) < 1e-15);
}

int main() {
    for (auto& [name, fn] : registry()) {
        try {
            fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::printf("FAIL %s: unexpected exception: %s\n", name, e.what());
        }
    }
    std::printf("%d checks passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
