// Drop-in implementation of the reference C++ API (include/sketchcp/*.hpp) over the
// B200 C-ABI (include/sketchcp_b200.h). Host-side pieces that must stay bit-exact
// (seeds, mt19937_64 stream, polynomial hashes) run here; every sketch, contraction
// and decomposition runs in libsketchcp_b200.so on the GPU.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>

#include "sketchcp/common.hpp"
#include "sketchcp/contraction.hpp"
#include "sketchcp/decompose.hpp"
#include "sketchcp/fft.hpp"
#include "sketchcp/hashing.hpp"
#include "sketchcp/lda.hpp"
#include "sketchcp/metrics.hpp"
#include "sketchcp/rng.hpp"
#include "sketchcp/sketch.hpp"
#include "sketchcp/tensor.hpp"
#include "sketchcp_b200.h"

namespace sketchcp {

namespace {

[[noreturn]] void rethrow(int st) {
    const std::string msg = skc_last_error();
    switch (st) {
        case SKC_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case SKC_DEGENERATE: throw DegenerateIterationError(msg);
        case SKC_NUMERICAL_ERROR: throw NumericalError(msg);
        case SKC_FORMAT_ERROR: throw FormatError(msg);
        case SKC_OUT_OF_MEMORY: throw std::bad_alloc();
        default: throw std::runtime_error(msg);  // CUDA: there is no CPU fallback
    }
}
inline void check(int st) {
    if (st != SKC_OK) rethrow(st);
}

skc_context* context() {
    static std::once_flag once;
    static skc_context* ctx = nullptr;
    std::call_once(once, [] { check(skc_context_create(0, &ctx)); });
    return ctx;
}

double* dptr(cvec& v) { return reinterpret_cast<double*>(v.data()); }

}  // namespace

// ---- common.hpp / tensor.cpp:16-24 ---------------------------------------------------
double median_inplace(std::vector<double>& v) {
    if (v.empty()) throw std::invalid_argument("median of empty set");
    const std::size_t mid = v.size() / 2;
    std::nth_element(v.begin(), v.begin() + static_cast<long>(mid), v.end());
    const double upper = v[mid];
    if (v.size() & 1u) return upper;
    const double lower = *std::max_element(v.begin(), v.begin() + static_cast<long>(mid));
    return 0.5 * (lower + upper);
}

// ---- rng.hpp -------------------------------------------------------------------------
std::uint64_t Rng::uniform_below(std::uint64_t bound) {
    if (bound <= 1) return 0;
    const unsigned bits = 64 - static_cast<unsigned>(__builtin_clzll(bound - 1));
    const std::uint64_t mask = bits >= 64 ? ~std::uint64_t{0} : ((std::uint64_t{1} << bits) - 1);
    for (;;) {
        const std::uint64_t x = eng_() & mask;
        if (x < bound) return x;
    }
}
double Rng::gaussian() {
    if (have_spare_) {
        have_spare_ = false;
        return spare_;
    }
    const double u1 = uniform_open();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    spare_ = r * std::sin(a);
    have_spare_ = true;
    return r * std::cos(a);
}
Eigen::VectorXd Rng::gaussian_vector(int n) {
    Eigen::VectorXd v(n);
    for (int i = 0; i < n; ++i) v[i] = gaussian();
    return v;
}
Eigen::VectorXd Rng::unit_sphere(int n) {
    for (;;) {
        Eigen::VectorXd v = gaussian_vector(n);
        const double nrm = v.norm();
        if (nrm > 1e-12) return v / nrm;
    }
}
double Rng::gamma(double shape) {
    if (shape < 1.0) {
        const double u = uniform_open();
        return gamma(shape + 1.0) * std::pow(u, 1.0 / shape);
    }
    const double d = shape - 1.0 / 3.0, c = 1.0 / std::sqrt(9.0 * d);
    for (;;) {
        const double x = gaussian();
        double v = 1.0 + c * x;
        if (v <= 0.0) continue;
        v = v * v * v;
        const double u = uniform_open();
        if (std::log(u) < 0.5 * x * x + d - d * v + d * std::log(v)) return d * v;
    }
}
Eigen::VectorXd Rng::dirichlet(const Eigen::VectorXd& alpha) {
    Eigen::VectorXd g(alpha.size());
    for (Eigen::Index i = 0; i < alpha.size(); ++i) g[i] = gamma(alpha[i]);
    const double s = g.sum();
    if (s <= 0.0) return Eigen::VectorXd::Constant(alpha.size(), 1.0 / static_cast<double>(alpha.size()));
    return g / s;
}

// ---- hashing.hpp ---------------------------------------------------------------------
PolyHash PolyHash::from_seed(int independence, std::uint32_t b, std::uint64_t seed) {
    if (independence < 1 || independence > 8) throw std::invalid_argument("PolyHash: independence must be in [1, 8]");
    if (b < 2) throw std::invalid_argument("PolyHash: need at least 2 buckets");
    Rng rng(seed);
    std::vector<std::uint64_t> c(static_cast<std::size_t>(independence));
    for (auto& x : c) x = rng.uniform_below(kHashPrime);
    return from_coefficients(std::move(c), b);
}
PolyHash PolyHash::from_coefficients(std::vector<std::uint64_t> coeffs, std::uint32_t b) {
    if (coeffs.empty()) throw std::invalid_argument("PolyHash: no coefficients");
    if (b < 2) throw std::invalid_argument("PolyHash: need at least 2 buckets");
    for (auto x : coeffs)
        if (x >= kHashPrime) throw std::invalid_argument("PolyHash: coefficient out of range");
    PolyHash h;
    h.coeffs_ = std::move(coeffs);
    h.b_ = b;
    return h;
}
SignGenerator::SignGenerator(SignMode mode, std::uint64_t seed, int independence)
    : mode_(mode), backing_(PolyHash::from_seed(independence, mode == SignMode::kRademacher ? 2 : 4, seed)) {}
SignGenerator SignGenerator::from_backing(SignMode mode, PolyHash backing) {
    if (backing.buckets() != (mode == SignMode::kRademacher ? 2u : 4u))
        throw std::invalid_argument("SignGenerator: backing hash bucket count must equal the sign modulus");
    SignGenerator s;
    s.mode_ = mode;
    s.backing_ = std::move(backing);
    return s;
}

// ---- fft.hpp (device) ----------------------------------------------------------------
namespace fft {
void forward_inplace(cvec& x) { check(skc_fft(dptr(x), x.size(), -1)); }
void inverse_inplace(cvec& x) { check(skc_fft(dptr(x), x.size(), 1)); }
void inverse_inplace_unscaled(cvec& x) { check(skc_fft(dptr(x), x.size(), 2)); }
cvec circular_convolve(const cvec& x, const cvec& y) {
    if (x.size() != y.size()) throw std::invalid_argument("circular_convolve: length mismatch");
    cvec fx = x, fy = y;
    forward_inplace(fx);
    forward_inplace(fy);
    for (std::size_t t = 0; t < fx.size(); ++t) fx[t] *= fy[t];
    inverse_inplace(fx);
    return fx;
}
// Every transform the device executed (these calls, contractions, spectra, deflations),
// counted in units of full length-b transforms like the reference's FFTW counter.
std::uint64_t transform_count() { return skc_transform_count(); }
}  // namespace fft

// ---- tensor.hpp ----------------------------------------------------------------------
double DenseTensor3::frobenius_sq() const {
    double s = 0;
    for (double x : entries) s += x * x;
    return s;
}
std::optional<std::array<int, 3>> DenseTensor3::first_asymmetric_triple(double tol) const {
    for (int i = 0; i < n; ++i)
        for (int j = i; j < n; ++j)
            for (int k = j; k < n; ++k) {
                const double ref = at(i, j, k);
                const std::array<std::array<int, 3>, 5> others = {{{i, k, j}, {j, i, k}, {j, k, i}, {k, i, j}, {k, j, i}}};
                for (const auto& p : others)
                    if (std::abs(at(p[0], p[1], p[2]) - ref) > tol) return p;
            }
    return std::nullopt;
}
bool DenseTensor3::is_symmetric(double tol) const { return !first_asymmetric_triple(tol).has_value(); }

void FactoredTensor::add(double a, Eigen::VectorXd u, Eigen::VectorXd v, Eigen::VectorXd w) {
    if (u.size() != n || v.size() != n || w.size() != n)
        throw std::invalid_argument("FactoredTensor: component dimension mismatch");
    components.push_back({a, std::move(u), std::move(v), std::move(w)});
}
void FactoredTensor::add_symmetric(double a, Eigen::VectorXd u) {
    if (u.size() != n) throw std::invalid_argument("FactoredTensor: component dimension mismatch");
    Eigen::VectorXd v = u, w = u;
    components.push_back({a, std::move(u), std::move(v), std::move(w)});
}
CpDecomposition CpDecomposition::symmetric_of(Eigen::VectorXd lambda, Eigen::MatrixXd V) {
    CpDecomposition d;
    d.lambda = std::move(lambda);
    d.A = std::move(V);
    d.B = d.A;
    d.C = d.A;
    return d;
}

// ---- sketch.hpp ----------------------------------------------------------------------
CountSketch sketch_vector(const Eigen::VectorXd& u, const PolyHash& h, const SignGenerator& s) {
    CountSketch cs;
    cs.data.assign(h.buckets(), {0.0, 0.0});
    for (Eigen::Index i = 0; i < u.size(); ++i) cs.data[h.eval(static_cast<std::uint64_t>(i))] += s.value(i) * u[i];
    return cs;
}

// SymTensorSketchSet ------------------------------------------------------------------
SymTensorSketchSet::SymTensorSketchSet(int n, std::uint32_t b, int B, std::uint64_t master_seed) {
    skc_sym_set* h = nullptr;
    check(skc_sym_create(context(), n, b, B, master_seed, &h));
    attach(h);
}
SymTensorSketchSet::~SymTensorSketchSet() = default;
void SymTensorSketchSet::attach(skc_sym_set* h) {
    h_ = std::shared_ptr<skc_sym_set>(h, [](skc_sym_set* p) { skc_sym_destroy(p); });
    std::uint64_t ver = 0;
    check(skc_sym_info(h, &n_, &b_, &B_, &seed_, &ver));
    reps_.clear();
    host_stale_ = true;
    device_stale_ = false;
}
SymTensorSketchSet::SymTensorSketchSet(const SymTensorSketchSet& o) { *this = o; }
SymTensorSketchSet& SymTensorSketchSet::operator=(const SymTensorSketchSet& o) {
    if (this == &o) return *this;
    if (!o.h_) {
        h_.reset();
        n_ = 0;
        B_ = 0;
        return *this;
    }
    o.sync_device();
    std::vector<std::uint64_t> hc(static_cast<std::size_t>(o.B_) * 6), sc(hc.size());
    std::vector<double> data(static_cast<std::size_t>(o.B_) * o.b_ * 2);
    check(skc_sym_coefficients(o.h_.get(), hc.data(), sc.data()));
    check(skc_sym_read_data(o.h_.get(), -1, data.data()));
    skc_sym_set* h = nullptr;
    check(skc_sym_create_from_coefficients(context(), o.n_, o.b_, o.B_, o.seed_, hc.data(), sc.data(), data.data(), &h));
    attach(h);
    version_ = o.version_;
    return *this;
}
void SymTensorSketchSet::pull_host() const {
    if (!h_ || !host_stale_ || device_stale_) return;
    if (reps_.size() != static_cast<std::size_t>(B_)) {
        reps_.assign(static_cast<std::size_t>(B_), Replicate{});
        std::vector<std::uint64_t> hc(static_cast<std::size_t>(B_) * 6), sc(hc.size());
        check(skc_sym_coefficients(h_.get(), hc.data(), sc.data()));
        for (int m = 0; m < B_; ++m) {
            Replicate& r = reps_[m];
            r.h = PolyHash::from_coefficients({hc.begin() + m * 6, hc.begin() + (m + 1) * 6}, b_);
            r.sigma = SignGenerator::from_backing(SignMode::kComplex4,
                                                  PolyHash::from_coefficients({sc.begin() + m * 6, sc.begin() + (m + 1) * 6}, 4));
            r.bucket1.resize(n_);
            r.bucket2.resize(n_);
            r.bucket3.resize(n_);
            r.sexp.resize(n_);
            check(skc_sym_tables(h_.get(), m, r.bucket1.data(), r.bucket2.data(), r.bucket3.data(), r.sexp.data()));
        }
    }
    for (int m = 0; m < B_; ++m) {
        reps_[m].data.resize(b_);
        check(skc_sym_read_data(h_.get(), m, dptr(reps_[m].data)));
    }
    host_stale_ = false;
}
void SymTensorSketchSet::sync_device() const {
    if (!h_ || !device_stale_) return;
    for (int m = 0; m < B_; ++m) {
        if (reps_[m].data.size() != b_) throw std::invalid_argument("mutable_replicate: data length must stay b");
        check(skc_sym_write_data(h_.get(), m, reinterpret_cast<const double*>(reps_[m].data.data())));
    }
    device_stale_ = false;
}
const SymTensorSketchSet::Replicate& SymTensorSketchSet::replicate(int m) const {
    pull_host();
    return reps_.at(static_cast<std::size_t>(m));
}
SymTensorSketchSet::Replicate& SymTensorSketchSet::mutable_replicate(int m) {
    pull_host();
    ++version_;
    device_stale_ = true;
    return reps_.at(static_cast<std::size_t>(m));
}
skc_sym_set* SymTensorSketchSet::device_handle() const {
    sync_device();
    return h_.get();
}
void SymTensorSketchSet::note_device_write(std::uint64_t bumps) {
    version_ += bumps;
    host_stale_ = true;
}
void SymTensorSketchSet::accumulate_dense(const DenseTensor3& T, bool assume_symmetric) {
    if (T.n != n_) throw std::invalid_argument("accumulate_dense: dimension mismatch");
    check(skc_sym_accumulate_dense(device_handle(), T.entries.data(), SKC_F64, SKC_HOST, assume_symmetric ? 1 : 0, 0, n_));
    note_device_write(1);
}
void SymTensorSketchSet::add_scaled_rank1(const Eigen::VectorXd& u, double alpha) {
    if (u.size() != n_) throw std::invalid_argument("add_scaled_rank1: dimension mismatch");
    if (alpha == 0.0) return;
    check(skc_sym_add_scaled_rank1(device_handle(), u.data(), alpha));
    note_device_write(1);
}
double SymTensorSketchSet::recover_entry(int i, int j, int k) const {
    double v = 0;
    check(skc_sym_recover_entry(device_handle(), i, j, k, &v));
    return v;
}
void SymTensorSketchSet::save(const std::string& path) const { check(skc_sym_save(device_handle(), path.c_str())); }
SymTensorSketchSet SymTensorSketchSet::load(const std::string& path) {
    skc_sym_set* h = nullptr;
    check(skc_sym_load(context(), path.c_str(), &h));
    SymTensorSketchSet s;
    s.attach(h);
    return s;
}

// AsymTensorSketchSet -----------------------------------------------------------------
AsymTensorSketchSet::AsymTensorSketchSet(int n, std::uint32_t b, int B, std::uint64_t master_seed) {
    skc_asym_set* h = nullptr;
    check(skc_asym_create(context(), n, b, B, master_seed, &h));
    attach(h);
}
AsymTensorSketchSet::~AsymTensorSketchSet() = default;
void AsymTensorSketchSet::attach(skc_asym_set* h) {
    h_ = std::shared_ptr<skc_asym_set>(h, [](skc_asym_set* p) { skc_asym_destroy(p); });
    std::uint64_t ver = 0;
    check(skc_asym_info(h, &n_, &b_, &B_, &seed_, &ver));
    reps_.clear();
    host_stale_ = true;
    device_stale_ = false;
}
AsymTensorSketchSet::AsymTensorSketchSet(const AsymTensorSketchSet& o) { *this = o; }
AsymTensorSketchSet& AsymTensorSketchSet::operator=(const AsymTensorSketchSet& o) {
    if (this == &o) return *this;
    if (!o.h_) {
        h_.reset();
        n_ = 0;
        B_ = 0;
        return *this;
    }
    o.sync_device();
    std::vector<std::uint64_t> hc(static_cast<std::size_t>(o.B_) * 6), xc(static_cast<std::size_t>(o.B_) * 18);
    std::vector<double> data(static_cast<std::size_t>(o.B_) * o.b_ * 2);
    check(skc_asym_coefficients(o.h_.get(), hc.data(), xc.data()));
    check(skc_asym_read_data(o.h_.get(), -1, data.data()));
    skc_asym_set* h = nullptr;
    check(skc_asym_create_from_coefficients(context(), o.n_, o.b_, o.B_, o.seed_, hc.data(), xc.data(), data.data(), &h));
    attach(h);
    version_ = o.version_;
    return *this;
}
void AsymTensorSketchSet::pull_host() const {
    if (!h_ || !host_stale_ || device_stale_) return;
    if (reps_.size() != static_cast<std::size_t>(B_)) {
        reps_.assign(static_cast<std::size_t>(B_), Replicate{});
        std::vector<std::uint64_t> hc(static_cast<std::size_t>(B_) * 6), xc(static_cast<std::size_t>(B_) * 18);
        check(skc_asym_coefficients(h_.get(), hc.data(), xc.data()));
        std::vector<std::uint32_t> bk(3 * static_cast<std::size_t>(n_));
        std::vector<double> sg(bk.size());
        for (int m = 0; m < B_; ++m) {
            Replicate& r = reps_[m];
            check(skc_asym_tables(h_.get(), m, bk.data(), sg.data()));
            for (int s = 0; s < 3; ++s) {
                const auto h0 = hc.begin() + (m * 3 + s) * 2, x0 = xc.begin() + (m * 3 + s) * 6;
                r.h[s] = PolyHash::from_coefficients({h0, h0 + 2}, b_);
                r.xi[s] = SignGenerator::from_backing(SignMode::kRademacher, PolyHash::from_coefficients({x0, x0 + 6}, 2));
                r.bucket[s].assign(bk.begin() + s * n_, bk.begin() + (s + 1) * n_);
                r.sign[s].assign(sg.begin() + s * n_, sg.begin() + (s + 1) * n_);
            }
        }
    }
    for (int m = 0; m < B_; ++m) {
        reps_[m].data.resize(b_);
        check(skc_asym_read_data(h_.get(), m, dptr(reps_[m].data)));
    }
    host_stale_ = false;
}
void AsymTensorSketchSet::sync_device() const {
    if (!h_ || !device_stale_) return;
    for (int m = 0; m < B_; ++m) {
        if (reps_[m].data.size() != b_) throw std::invalid_argument("mutable_replicate: data length must stay b");
        check(skc_asym_write_data(h_.get(), m, reinterpret_cast<const double*>(reps_[m].data.data())));
    }
    device_stale_ = false;
}
const AsymTensorSketchSet::Replicate& AsymTensorSketchSet::replicate(int m) const {
    pull_host();
    return reps_.at(static_cast<std::size_t>(m));
}
AsymTensorSketchSet::Replicate& AsymTensorSketchSet::mutable_replicate(int m) {
    pull_host();
    ++version_;
    device_stale_ = true;
    return reps_.at(static_cast<std::size_t>(m));
}
skc_asym_set* AsymTensorSketchSet::device_handle() const {
    sync_device();
    return h_.get();
}
void AsymTensorSketchSet::accumulate_dense(const DenseTensor3& T) {
    if (T.n != n_) throw std::invalid_argument("accumulate_dense: dimension mismatch");
    check(skc_asym_accumulate_dense(device_handle(), T.entries.data(), SKC_F64, SKC_HOST, 0, n_));
    ++version_;
    host_stale_ = true;
}
cvec AsymTensorSketchSet::rank1_sketch(int m, const Eigen::VectorXd& u, const Eigen::VectorXd& v,
                                       const Eigen::VectorXd& w) const {
    if (u.size() != n_ || v.size() != n_ || w.size() != n_) throw std::invalid_argument("rank1_sketch: dimension mismatch");
    cvec out(b_);
    check(skc_asym_rank1_sketch(device_handle(), m, u.data(), v.data(), w.data(), dptr(out)));
    return out;
}
void AsymTensorSketchSet::add_rank1(double alpha, const Eigen::VectorXd& u, const Eigen::VectorXd& v,
                                    const Eigen::VectorXd& w) {
    if (u.size() != n_ || v.size() != n_ || w.size() != n_) throw std::invalid_argument("rank1_sketch: dimension mismatch");
    check(skc_asym_add_rank1(device_handle(), alpha, u.data(), v.data(), w.data()));
    ++version_;
    host_stale_ = true;
}
void AsymTensorSketchSet::accumulate_factored(const FactoredTensor& F) {
    if (F.n != n_) throw std::invalid_argument("accumulate_factored: dimension mismatch");
    const std::size_t N = F.components.size(), nn = static_cast<std::size_t>(n_);
    std::vector<double> a(N), U(N * nn), V(N * nn), W(N * nn);
    for (std::size_t c = 0; c < N; ++c) {
        const auto& comp = F.components[c];
        a[c] = comp.weight;
        std::copy(comp.u.data(), comp.u.data() + n_, U.begin() + static_cast<long>(c * nn));
        std::copy(comp.v.data(), comp.v.data() + n_, V.begin() + static_cast<long>(c * nn));
        std::copy(comp.w.data(), comp.w.data() + n_, W.begin() + static_cast<long>(c * nn));
    }
    check(skc_asym_accumulate_factored(device_handle(), static_cast<long long>(N), a.data(), U.data(), V.data(), W.data()));
    ++version_;
    host_stale_ = true;
}
double AsymTensorSketchSet::recover_entry(int i, int j, int k) const {
    double v = 0;
    check(skc_asym_recover_entry(device_handle(), i, j, k, &v));
    return v;
}
void AsymTensorSketchSet::save(const std::string& path) const { check(skc_asym_save(device_handle(), path.c_str())); }
AsymTensorSketchSet AsymTensorSketchSet::load(const std::string& path) {
    skc_asym_set* h = nullptr;
    check(skc_asym_load(context(), path.c_str(), &h));
    AsymTensorSketchSet s;
    s.attach(h);
    return s;
}

// sketch.cpp:412-425: a host helper over a replicate's tables (reference test hook)
SymAuxSketches sym_aux_sketches(const SymTensorSketchSet::Replicate& rep, std::uint32_t b, const Eigen::VectorXd& u) {
    static const std::complex<double> r4[4] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
    SymAuxSketches aux;
    aux.s1.assign(b, {0.0, 0.0});
    aux.s2.assign(b, {0.0, 0.0});
    aux.s3.assign(b, {0.0, 0.0});
    for (Eigen::Index i = 0; i < u.size(); ++i) {
        const double ui = u[i];
        const unsigned e = rep.sexp[static_cast<std::size_t>(i)];
        aux.s1[rep.bucket1[static_cast<std::size_t>(i)]] += r4[e & 3u] * ui;
        aux.s2[rep.bucket2[static_cast<std::size_t>(i)]] += r4[(2u * e) & 3u] * (ui * ui);
        aux.s3[rep.bucket3[static_cast<std::size_t>(i)]] += r4[(3u * e) & 3u] * (ui * ui * ui);
    }
    return aux;
}
cvec sketch_rank1_sym(const SymTensorSketchSet& set, int m, const Eigen::VectorXd& u) {
    if (u.size() != set.n()) throw std::invalid_argument("sketch_rank1_sym: dimension mismatch");
    cvec out(set.b());
    check(skc_sym_rank1_truncated(set.device_handle(), m, u.data(), dptr(out)));
    return out;
}
SketchMode peek_sketch_mode(const std::string& path) {
    int mode = 0;
    check(skc_peek_sketch_mode(path.c_str(), &mode));
    return mode == 1 ? SketchMode::kSym : SketchMode::kAsym;
}

// ---- contraction.hpp -----------------------------------------------------------------
SymContractionWorkspace::SymContractionWorkspace(const SymTensorSketchSet& set) : set_(&set) {}
double SymContractionWorkspace::vvv(const Eigen::VectorXd& u) {
    if (u.size() != set_->n()) throw std::invalid_argument("vvv: dimension mismatch");
    double out = 0;
    check(skc_sym_vvv(set_->device_handle(), u.data(), 1, &out));
    return out;
}
Eigen::VectorXd SymContractionWorkspace::Ivv(const Eigen::VectorXd& u) {
    if (u.size() != set_->n()) throw std::invalid_argument("Ivv: dimension mismatch");
    Eigen::VectorXd out(u.size());
    check(skc_sym_ivv(set_->device_handle(), u.data(), 1, out.data()));
    return out;
}
const cvec& SymContractionWorkspace::cached_transform(int m) {
    spectra_.resize(static_cast<std::size_t>(set_->replicates()));
    cvec& c = spectra_.at(static_cast<std::size_t>(m));
    c.resize(set_->b());
    check(skc_sym_cached_transform(set_->device_handle(), m, dptr(c)));
    return c;
}

AsymContractionWorkspace::AsymContractionWorkspace(const AsymTensorSketchSet& set) : set_(&set) {}
double AsymContractionWorkspace::vvv(const Eigen::VectorXd& u) {
    if (u.size() != set_->n()) throw std::invalid_argument("vvv: dimension mismatch");
    double out = 0;
    check(skc_asym_vvv(set_->device_handle(), u.data(), 1, &out));
    return out;
}
Eigen::VectorXd AsymContractionWorkspace::mode_contraction(int free_mode, const Eigen::VectorXd& x,
                                                           const Eigen::VectorXd& y) {
    if (x.size() != set_->n() || y.size() != set_->n())
        throw std::invalid_argument("mode_contraction: dimension mismatch");
    Eigen::VectorXd out(x.size());
    check(skc_asym_mode_contraction(set_->device_handle(), free_mode, x.data(), y.data(), 1, out.data()));
    return out;
}
Eigen::VectorXd AsymContractionWorkspace::Ivv(const Eigen::VectorXd& u) { return mode_contraction(0, u, u); }
Eigen::VectorXd AsymContractionWorkspace::Ibc(const Eigen::VectorXd& bvec, const Eigen::VectorXd& cvec_) {
    return mode_contraction(0, bvec, cvec_);
}
const cvec& AsymContractionWorkspace::cached_transform(int m) {
    spectra_.resize(static_cast<std::size_t>(set_->replicates()));
    cvec& c = spectra_.at(static_cast<std::size_t>(m));
    c.resize(set_->b());
    check(skc_asym_cached_transform(set_->device_handle(), m, dptr(c)));
    return c;
}

// ---- decompose.hpp -------------------------------------------------------------------
CpDecomposition robust_tpm_fast(SymTensorSketchSet& set, const PowerConfig& cfg) {
    const int n = set.n();
    Eigen::VectorXd lambda(std::max(cfg.k, 0));
    Eigen::MatrixXd V(n, std::max(cfg.k, 0));
    const int st = skc_sym_rtpm(set.device_handle(), cfg.k, cfg.L, cfg.T_iters, cfg.seed, cfg.tol, nullptr,
                                lambda.data(), V.data(), nullptr);
    if (st == SKC_OK) {
        std::uint64_t deflations = 0;
        for (Eigen::Index c = 0; c < lambda.size(); ++c) deflations += lambda[c] != 0.0 ? 1 : 0;
        set.note_device_write(deflations);
    } else if (st == SKC_DEGENERATE) {
        set.note_device_write(0);  // earlier components were already deflated
    }
    check(st);
    return CpDecomposition::symmetric_of(std::move(lambda), std::move(V));
}

CpDecomposition als_fast(const AsymTensorSketchSet& set, const AlsConfig& cfg) {
    const int n = set.n(), k = cfg.k;
    if (k < 1 || cfg.max_iters < 1) throw std::invalid_argument("als: k and max_iters must be positive");
    if (k > n) throw std::invalid_argument("als: target rank exceeds tensor dimension");
    Eigen::VectorXd lambda(k);
    Eigen::MatrixXd A(n, k), B(n, k), C(n, k);  // column-major, as the C-ABI returns them
    int iters = 0;
    check(skc_asym_als(set.device_handle(), k, cfg.max_iters, cfg.tol, cfg.seed, lambda.data(), A.data(), B.data(),
                       C.data(), &iters));
    CpDecomposition d;
    d.lambda = std::move(lambda);
    d.A = std::move(A);
    d.B = std::move(B);
    d.C = std::move(C);
    return d;
}

Eigen::MatrixXd pinv_spectral(const Eigen::MatrixXd& G) {
    // symmetric eigendecomposition by cyclic Jacobi (host), truncation at 1e-10 max|ev|
    const int k = static_cast<int>(G.rows());
    if (G.cols() != k) throw std::invalid_argument("pinv_spectral: matrix must be square");
    std::vector<double> a(G.data(), G.data() + static_cast<std::size_t>(k) * k), v(static_cast<std::size_t>(k) * k, 0.0);
    for (int i = 0; i < k; ++i) v[static_cast<std::size_t>(i) * k + i] = 1.0;
    auto A = [&](int i, int j) -> double& { return a[static_cast<std::size_t>(j) * k + i]; };
    auto Vv = [&](int i, int j) -> double& { return v[static_cast<std::size_t>(j) * k + i]; };
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0, tot = 0.0;
        for (int j = 0; j < k; ++j)
            for (int i = 0; i < k; ++i) {
                tot += A(i, j) * A(i, j);
                if (i != j) off += A(i, j) * A(i, j);
            }
        if (off <= 1e-30 * tot) break;
        for (int p = 0; p < k - 1; ++p)
            for (int q = p + 1; q < k; ++q) {
                const double apq = A(p, q);
                if (apq == 0.0) continue;
                const double th = (A(q, q) - A(p, p)) / (2.0 * apq);
                const double t = (th >= 0 ? 1.0 : -1.0) / (std::abs(th) + std::sqrt(th * th + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int r = 0; r < k; ++r) {
                    const double x = A(r, p), y = A(r, q);
                    A(r, p) = c * x - s * y;
                    A(r, q) = s * x + c * y;
                }
                for (int r = 0; r < k; ++r) {
                    const double x = A(p, r), y = A(q, r);
                    A(p, r) = c * x - s * y;
                    A(q, r) = s * x + c * y;
                }
                for (int r = 0; r < k; ++r) {
                    const double x = Vv(r, p), y = Vv(r, q);
                    Vv(r, p) = c * x - s * y;
                    Vv(r, q) = s * x + c * y;
                }
            }
    }
    double amax = 0.0;
    for (int i = 0; i < k; ++i) amax = std::max(amax, std::abs(A(i, i)));
    const double cutoff = 1e-10 * amax;
    Eigen::MatrixXd P = Eigen::MatrixXd::Zero(k, k);
    for (int q = 0; q < k; ++q) {
        if (!(std::abs(A(q, q)) > cutoff)) continue;
        const double inv = 1.0 / A(q, q);
        for (int j = 0; j < k; ++j)
            for (int i = 0; i < k; ++i) P(i, j) += Vv(i, q) * inv * Vv(j, q);
    }
    return P;
}

// ---- lda.hpp -------------------------------------------------------------------------
long long Corpus::total_tokens() const {
    long long t = 0;
    for (const auto& d : docs) t += d.total;
    return t;
}
namespace {
struct CorpusCsr {
    std::vector<long long> doc_ptr{0};
    std::vector<int> word, count;
    explicit CorpusCsr(const Corpus& c) {
        for (const auto& d : c.docs) {
            word.insert(word.end(), d.word.begin(), d.word.end());
            count.insert(count.end(), d.count.begin(), d.count.end());
            doc_ptr.push_back(static_cast<long long>(word.size()));
        }
    }
    long long D() const { return static_cast<long long>(doc_ptr.size()) - 1; }
};
WhiteningMap whitening_from_rowmajor(int V, int k, const std::vector<double>& W, const std::vector<double>& U,
                                     const std::vector<double>& sv) {
    WhiteningMap wm;
    wm.W.resize(V, k);
    wm.unwhiten.resize(V, k);
    wm.singular_values.resize(k);
    for (int w = 0; w < V; ++w)
        for (int a = 0; a < k; ++a) {
            wm.W(w, a) = W[static_cast<std::size_t>(w) * k + a];
            wm.unwhiten(w, a) = U[static_cast<std::size_t>(w) * k + a];
        }
    for (int a = 0; a < k; ++a) wm.singular_values[a] = sv[a];
    return wm;
}
}  // namespace

Eigen::VectorXd compute_m1(const Corpus& c) {
    CorpusCsr csr(c);
    Eigen::VectorXd m1(c.V);
    check(skc_lda_compute_m1(context(), c.V, csr.D(), csr.doc_ptr.data(), csr.word.data(), csr.count.data(), m1.data()));
    return m1;
}

Eigen::MatrixXd compute_m2(const Corpus& c, double alpha0) {
    CorpusCsr csr(c);
    const int V = c.V;
    Eigen::MatrixXd m2(V, V);
    const int blk = std::min(V, 256);
    std::vector<double> X(static_cast<std::size_t>(V) * blk), Y(X.size());
    for (int c0 = 0; c0 < V; c0 += blk) {
        const int p = std::min(blk, V - c0);
        std::fill(X.begin(), X.end(), 0.0);
        for (int j = 0; j < p; ++j) X[static_cast<std::size_t>(c0 + j) * p + j] = 1.0;
        check(skc_lda_m2_apply(context(), V, csr.D(), csr.doc_ptr.data(), csr.word.data(), csr.count.data(), alpha0, p,
                               X.data(), Y.data()));
        for (int w = 0; w < V; ++w)
            for (int j = 0; j < p; ++j) m2(w, c0 + j) = Y[static_cast<std::size_t>(w) * p + j];
    }
    return m2;
}

WhiteningMap whiten(const Eigen::MatrixXd& m2hat, int k) {
    if (m2hat.rows() != m2hat.cols()) throw std::invalid_argument("whiten: matrix must be square");
    const int V = static_cast<int>(m2hat.rows());
    if (k < 1 || k > V) throw std::invalid_argument("whiten: invalid target rank");
    std::vector<double> M(static_cast<std::size_t>(V) * V);
    for (int i = 0; i < V; ++i)
        for (int j = 0; j < V; ++j) M[static_cast<std::size_t>(i) * V + j] = m2hat(i, j);
    std::vector<double> W(static_cast<std::size_t>(V) * k), U(W.size()), sv(k);
    check(skc_lda_whiten_dense(context(), V, M.data(), k, -1, -1, 0x5EED, W.data(), U.data(), sv.data()));
    return whitening_from_rowmajor(V, k, W, U, sv);
}

WhiteningMap whiten_corpus(const Corpus& c, double alpha0, int k) {
    CorpusCsr csr(c);
    const int V = c.V;
    if (k < 1 || k > V) throw std::invalid_argument("whiten: invalid target rank");
    std::vector<double> W(static_cast<std::size_t>(V) * k), U(W.size()), sv(k);
    check(skc_lda_whiten_corpus(context(), V, csr.D(), csr.doc_ptr.data(), csr.word.data(), csr.count.data(), alpha0, k,
                                -1, -1, 0x5EED, W.data(), U.data(), sv.data()));
    return whitening_from_rowmajor(V, k, W, U, sv);
}

LdaModel recover_params(const CpDecomposition& D, const WhiteningMap& wm, double alpha0) {
    const int k = D.rank();
    if (k < 1) throw std::invalid_argument("recover_params: empty decomposition");
    if (D.A.rows() != wm.W.cols()) throw std::invalid_argument("recover_params: decomposition/whitening rank mismatch");
    const int V = static_cast<int>(wm.W.rows()), r = static_cast<int>(D.A.rows());
    std::vector<double> A(static_cast<std::size_t>(r) * k), U(static_cast<std::size_t>(V) * r), Phi(static_cast<std::size_t>(V) * k);
    for (int i = 0; i < r; ++i)
        for (int j = 0; j < k; ++j) A[static_cast<std::size_t>(i) * k + j] = D.A(i, j);
    for (int w = 0; w < V; ++w)
        for (int j = 0; j < r; ++j) U[static_cast<std::size_t>(w) * r + j] = wm.unwhiten(w, j);
    LdaModel m;
    m.alpha.resize(k);
    check(skc_lda_recover_params(context(), V, k, D.lambda.data(), A.data(), U.data(), alpha0, Phi.data(), m.alpha.data()));
    m.Phi.resize(V, k);
    for (int w = 0; w < V; ++w)
        for (int j = 0; j < k; ++j) m.Phi(w, j) = Phi[static_cast<std::size_t>(w) * k + j];
    return m;
}

Eigen::VectorXd project_to_simplex(const Eigen::VectorXd& y) {
    // one-column recover_params with lambda chosen so mu = y: 0.5 (a0 + 2) lam = 1 at a0 = 0, lam = 1
    const int n = static_cast<int>(y.size());
    double one = 1.0, a = 1.0, alpha = 0.0;
    Eigen::VectorXd out(n);
    check(skc_lda_recover_params(context(), n, 1, &one, &a, y.data(), 0.0, out.data(), &alpha));
    return out;
}

double heldout_likelihood(const LdaModel& m, const Corpus& held, long long* floored_words) {
    CorpusCsr csr(held);
    const int V = m.vocab(), k = m.topics();
    std::vector<double> Phi(static_cast<std::size_t>(V) * k);
    for (int w = 0; w < V; ++w)
        for (int j = 0; j < k; ++j) Phi[static_cast<std::size_t>(w) * k + j] = m.Phi(w, j);
    double ll = 0.0;
    long long fl = 0;
    check(skc_lda_heldout_likelihood(context(), V, k, Phi.data(), held.V, csr.D(), csr.doc_ptr.data(), csr.word.data(),
                                     csr.count.data(), &ll, &fl));
    if (floored_words) *floored_words = fl;
    return ll;
}

StreamStats sketch_whitened_m3(const Corpus& c, const WhiteningMap& wm, double alpha0, SymTensorSketchSet& set) {
    const int k = static_cast<int>(wm.W.cols()), V = c.V;
    if (wm.W.rows() != V) throw std::invalid_argument("sketch_whitened_m3: vocabulary mismatch");
    if (set.n() != k) throw std::invalid_argument("sketch_whitened_m3: set dimension must equal whitening rank");
    std::vector<long long> doc_ptr(1, 0);
    std::vector<int> word, count;
    for (const auto& d : c.docs) {
        word.insert(word.end(), d.word.begin(), d.word.end());
        count.insert(count.end(), d.count.begin(), d.count.end());
        doc_ptr.push_back(static_cast<long long>(word.size()));
    }
    std::vector<double> W(static_cast<std::size_t>(V) * k);  // row-major copy of the column-major map
    for (int w = 0; w < V; ++w)
        for (int a = 0; a < k; ++a) W[static_cast<std::size_t>(w) * k + a] = wm.W(w, a);
    StreamStats stats;
    check(skc_sym_sketch_whitened_m3(set.device_handle(), V, static_cast<long long>(c.docs.size()), doc_ptr.data(),
                                     word.data(), count.data(), W.data(), alpha0, &stats.used, &stats.skipped));
    set.note_device_write(static_cast<std::uint64_t>(set.replicates()));
    return stats;
}

// ---- metrics.hpp (metrics.cpp:8-52) --------------------------------------------------
std::vector<VectorMatch> greedy_match(const Eigen::MatrixXd& recovered, const Eigen::MatrixXd& truth) {
    const int r = static_cast<int>(recovered.cols()), g = static_cast<int>(truth.cols());
    if (g < r) throw std::invalid_argument("greedy_match: fewer truth columns than recovered");
    std::vector<double> cosm(static_cast<std::size_t>(r) * g);
    for (int i = 0; i < r; ++i) {
        const double ni = recovered.col(i).norm();
        for (int j = 0; j < g; ++j) {
            const double nj = truth.col(j).norm();
            cosm[static_cast<std::size_t>(i) * g + j] =
                std::abs(recovered.col(i).dot(truth.col(j))) / std::max(ni * nj, 1e-300);
        }
    }
    std::vector<char> ur(r, 0), ug(g, 0);
    std::vector<VectorMatch> out;
    for (int step = 0; step < r; ++step) {
        double best = -1.0;
        int bi = -1, bj = -1;
        for (int i = 0; i < r; ++i) {
            if (ur[i]) continue;
            for (int j = 0; j < g; ++j) {
                if (ug[j]) continue;
                if (cosm[static_cast<std::size_t>(i) * g + j] > best) {
                    best = cosm[static_cast<std::size_t>(i) * g + j];
                    bi = i;
                    bj = j;
                }
            }
        }
        ur[bi] = 1;
        ug[bj] = 1;
        const double sign = recovered.col(bi).dot(truth.col(bj)) >= 0 ? 1.0 : -1.0;
        double d = 0;
        for (Eigen::Index t = 0; t < truth.rows(); ++t) {
            const double diff = truth(t, bj) - sign * recovered(t, bi);
            d += diff * diff;
        }
        out.push_back({bi, bj, best, d});
    }
    return out;
}
int wrong_vector_count(const std::vector<VectorMatch>& matches, double threshold) {
    int c = 0;
    for (const auto& m : matches) c += m.sq_distance > threshold ? 1 : 0;
    return c;
}

}  // namespace sketchcp
