// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain C++ (+OpenMP) restatement of the reference FFT tensor-sketch hot path
// (arXiv 1506.04448 reference, `sketchcp`, read-only at /root/reference). It is the
// CPU checker for the CUDA product in paper_1506_04448_b200/: only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
// load it. The product path never links or calls it.
//
// Parity status: the reference cannot be compiled here (Eigen3, FFTW3 and doctest
// are absent). This restatement is pinned against every known-answer
// test the reference's own tests hold for the path (tests/test_oracle_pins.py):
// proj/tests/test_hashing.cpp:47-56,65,135-146 and the Monte-Carlo hash tests, the
// FFT tests proj/tests/test_fft.cpp:37-90, and the SPEC.md worked examples. Two
// reference goldens are themselves wrong (test_hashing.cpp:62-66 frozen KAT and
// test_fft.cpp:62-65 b=4 convolution); the oracle follows the reference *code*.
//
// Every function cites the reference file:line it restates. Loop and accumulation
// orders are kept, so the oracle is deterministic at any OpenMP thread count.
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc {

using cd = std::complex<double>;
using cvec = std::vector<cd>;

struct NumericalError : std::runtime_error {  // common.hpp:20-23
    using std::runtime_error::runtime_error;
};
struct DegenerateIterationError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline bool is_power_of_two(std::uint64_t x) { return x != 0 && (x & (x - 1)) == 0; }

// --- rng.hpp:28-46 -----------------------------------------------------------
inline std::uint64_t splitmix64_next(std::uint64_t& state) {
    std::uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

inline std::uint64_t derive_seed(std::uint64_t master, std::uint64_t tag, std::uint64_t i0 = 0,
                                 std::uint64_t i1 = 0) {
    std::uint64_t s = master;
    std::uint64_t out = splitmix64_next(s);
    s ^= tag * 0xD6E8FEB86659FD93ull;
    out ^= splitmix64_next(s);
    s ^= i0 * 0xA5A5A5A5A5A5A5A5ull + 0x0123456789ABCDEFull;
    out ^= splitmix64_next(s);
    s ^= i1 * 0xC2B2AE3D27D4EB4Full + 0x9E3779B97F4A7C15ull;
    out ^= splitmix64_next(s);
    return out;
}

constexpr std::uint64_t kAsymBucketHash = 0x11, kAsymSign = 0x12, kSymBucketHash = 0x21,
                        kSymSign = 0x22, kPowerInit = 0x31, kAlsInit = 0x32;

// --- rng.hpp:51-141 ----------------------------------------------------------
class Rng {
public:
    explicit Rng(std::uint64_t seed) : engine_(seed) {}
    std::uint64_t next_u64() { return engine_(); }
    double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
    double uniform_open() { return (static_cast<double>(engine_() >> 11) + 1.0) * 0x1.0p-53; }
    std::uint64_t uniform_below(std::uint64_t bound) {  // rng.hpp:64-76
        std::uint64_t mask = ~std::uint64_t{0};
        if (bound > 1) {
            unsigned bits = 64 - static_cast<unsigned>(__builtin_clzll(bound - 1));
            mask = (bits >= 64) ? ~std::uint64_t{0} : ((std::uint64_t{1} << bits) - 1);
        } else {
            return 0;
        }
        for (;;) {
            std::uint64_t x = engine_() & mask;
            if (x < bound) return x;
        }
    }
    double gaussian() {  // rng.hpp:79-90
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        double u1 = uniform_open();
        double u2 = uniform();
        double r = std::sqrt(-2.0 * std::log(u1));
        double a = 6.283185307179586476925286766559 * u2;
        spare_ = r * std::sin(a);
        have_spare_ = true;
        return r * std::cos(a);
    }
    // rng.hpp:100-106. Eigen's norm() (vectorised reduction) is replaced by a
    // sequential sum; the order is unpinned by any reference test.
    std::vector<double> unit_sphere(int n) {
        for (;;) {
            std::vector<double> v(n);
            for (int i = 0; i < n; ++i) v[i] = gaussian();
            double s = 0;
            for (double x : v) s += x * x;
            double nrm = std::sqrt(s);
            if (nrm > 1e-12) {
                for (double& x : v) x /= nrm;
                return v;
            }
        }
    }
    double gamma(double shape) {  // rng.hpp:109-123
        if (shape < 1.0) {
            double u = uniform_open();
            return gamma(shape + 1.0) * std::pow(u, 1.0 / shape);
        }
        double d = shape - 1.0 / 3.0;
        double c = 1.0 / std::sqrt(9.0 * d);
        for (;;) {
            double x = gaussian();
            double v = 1.0 + c * x;
            if (v <= 0.0) continue;
            v = v * v * v;
            double u = uniform_open();
            if (std::log(u) < 0.5 * x * x + d - d * v + d * std::log(v)) return d * v;
        }
    }

private:
    std::mt19937_64 engine_;
    double spare_ = 0.0;
    bool have_spare_ = false;
};

// --- hashing.hpp:12-43, hashing.cpp:8-27 --------------------------------------
constexpr std::uint64_t kHashPrime = (std::uint64_t{1} << 31) - 1;

struct PolyHash {
    std::vector<std::uint64_t> coeffs;  // constant term first
    std::uint32_t b = 2;
    static PolyHash from_seed(int independence, std::uint32_t b, std::uint64_t seed) {
        if (independence < 1 || independence > 8)
            throw std::invalid_argument("PolyHash: independence must be in [1, 8]");
        if (b < 2) throw std::invalid_argument("PolyHash: need at least 2 buckets");
        Rng rng(seed);
        PolyHash h;
        h.coeffs.resize(static_cast<std::size_t>(independence));
        for (auto& c : h.coeffs) c = rng.uniform_below(kHashPrime);
        h.b = b;
        return h;
    }
    static PolyHash from_coefficients(std::vector<std::uint64_t> coeffs, std::uint32_t b) {
        if (coeffs.empty()) throw std::invalid_argument("PolyHash: no coefficients");
        if (b < 2) throw std::invalid_argument("PolyHash: need at least 2 buckets");
        for (auto c : coeffs)
            if (c >= kHashPrime) throw std::invalid_argument("PolyHash: coefficient out of range");
        PolyHash h;
        h.coeffs = std::move(coeffs);
        h.b = b;
        return h;
    }
    std::uint32_t eval(std::uint64_t i) const {  // hashing.hpp:29-34
        std::uint64_t acc = 0;
        for (std::size_t d = coeffs.size(); d-- > 0;)
            acc = (acc * (i % kHashPrime) + coeffs[d]) % kHashPrime;
        return static_cast<std::uint32_t>(acc % b);
    }
};

// hashing.hpp:46-50
inline std::uint32_t symmetric_bucket(const PolyHash& h, std::uint64_t i, std::uint64_t j,
                                      std::uint64_t k) {
    std::uint64_t s = std::uint64_t{h.eval(i)} + h.eval(j) + h.eval(k);
    return static_cast<std::uint32_t>(s % h.b);
}

// sketch.cpp:38-45 / contraction.cpp:30-37
inline cd root4(unsigned e) {
    switch (e & 3u) {
        case 0: return {1.0, 0.0};
        case 1: return {0.0, 1.0};
        case 2: return {-1.0, 0.0};
        default: return {0.0, -1.0};
    }
}
// contraction.cpp:40-47
inline double re_rot_conj(unsigned e, cd z) {
    switch (e & 3u) {
        case 0: return z.real();
        case 1: return z.imag();
        case 2: return -z.real();
        default: return -z.imag();
    }
}

// --- fft.hpp:10-26, fft.cpp:40-79 (FFTW semantics, in-tree radix-2) ----------------
// Forward = e^{-2 pi i tk/b} unnormalised; inverse = e^{+...}, scaled 1/b or unscaled.
std::atomic<std::uint64_t> g_transform_count{0};

void check_length(std::size_t b) {
    if (!is_power_of_two(b))
        throw std::invalid_argument("fft: length must be a power of two, got " + std::to_string(b));
}

void fft_core(cvec& x, int sign) {
    const std::size_t n = x.size();
    for (std::size_t i = 1, j = 0; i < n; ++i) {
        std::size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(x[i], x[j]);
    }
    for (std::size_t len = 2; len <= n; len <<= 1) {
        const std::size_t half = len >> 1;
        std::vector<cd> w(half);
        for (std::size_t k = 0; k < half; ++k) {
            // twiddles from long double for ~0.5 ulp accuracy
            long double ang = 2.0L * 3.14159265358979323846264338327950288L * (long double)k / (long double)len;
            w[k] = cd(static_cast<double>(std::cos(ang)), static_cast<double>(sign * std::sin(ang)));
        }
        for (std::size_t s = 0; s < n; s += len)
            for (std::size_t k = 0; k < half; ++k) {
                cd a = x[s + k];
                cd t = x[s + k + half] * w[k];
                x[s + k] = a + t;
                x[s + k + half] = a - t;
            }
    }
}

void forward_inplace(cvec& x) {
    check_length(x.size());
    fft_core(x, -1);
    g_transform_count.fetch_add(1, std::memory_order_relaxed);
}
void inverse_inplace_unscaled(cvec& x) {
    check_length(x.size());
    fft_core(x, +1);
    g_transform_count.fetch_add(1, std::memory_order_relaxed);
}
void inverse_inplace(cvec& x) {
    inverse_inplace_unscaled(x);
    const double s = 1.0 / static_cast<double>(x.size());
    for (auto& v : x) v *= s;
}
cvec circular_convolve(const cvec& x, const cvec& y) {  // fft.cpp:62-71
    if (x.size() != y.size()) throw std::invalid_argument("circular_convolve: length mismatch");
    check_length(x.size());
    cvec fx = x, fy = y;
    forward_inplace(fx);
    forward_inplace(fy);
    for (std::size_t t = 0; t < fx.size(); ++t) fx[t] *= fy[t];
    inverse_inplace(fx);
    return fx;
}

// --- tensor.cpp:16-24 --------------------------------------------------------------
double median_inplace(std::vector<double>& v) {
    if (v.empty()) throw std::invalid_argument("median of empty set");
    std::size_t m = v.size() / 2;
    std::nth_element(v.begin(), v.begin() + m, v.end());
    double hi = v[m];
    if (v.size() % 2 == 1) return hi;
    double lo = *std::max_element(v.begin(), v.begin() + m);
    return 0.5 * (lo + hi);
}

// tensor.cpp:32-43
bool first_asymmetric_triple(const double* T, int n, double tol, int out[3]) {
    auto at = [&](int i, int j, int k) { return T[(static_cast<std::size_t>(i) * n + j) * n + k]; };
    for (int i = 0; i < n; ++i)
        for (int j = i; j < n; ++j)
            for (int k = j; k < n; ++k) {
                double ref = at(i, j, k);
                const std::array<std::array<int, 3>, 5> perms = {
                    {{i, k, j}, {j, i, k}, {j, k, i}, {k, i, j}, {k, j, i}}};
                for (auto& p : perms)
                    if (std::abs(at(p[0], p[1], p[2]) - ref) > tol) {
                        out[0] = p[0];
                        out[1] = p[1];
                        out[2] = p[2];
                        return true;
                    }
            }
    return false;
}

// --- sketch.cpp: symmetric set ------------------------------------------------------
struct SymRep {
    PolyHash h, sigma;  // sigma: complex4 SignGenerator backing (6-wise into 4)
    std::vector<std::uint32_t> bucket1, bucket2, bucket3;
    std::vector<std::uint8_t> sexp;
    cvec data;
};

struct SymSet {
    int n = 0;
    std::uint32_t b = 2;
    int B = 0;
    std::uint64_t seed = 0;
    std::uint64_t version = 0;
    std::vector<SymRep> reps;
};

// sketch.cpp:24-36
void fill_sym_tables(SymRep& rep, int n, std::uint32_t b) {
    rep.bucket1.resize(n);
    rep.bucket2.resize(n);
    rep.bucket3.resize(n);
    rep.sexp.resize(n);
    for (int i = 0; i < n; ++i) {
        std::uint32_t hi = rep.h.eval(i);
        rep.bucket1[i] = hi;
        rep.bucket2[i] = static_cast<std::uint32_t>((2ull * hi) % b);
        rep.bucket3[i] = static_cast<std::uint32_t>((3ull * hi) % b);
        rep.sexp[i] = static_cast<std::uint8_t>(rep.sigma.eval(i));
    }
}

// sketch.cpp:300-313 (SignGenerator ctor hashing.cpp:29-31: 6-wise PolyHash into 4)
SymSet* sym_create(int n, std::uint32_t b, int B, std::uint64_t seed) {
    if (n < 1) throw std::invalid_argument("sketch set: dimension must be positive");
    if (B < 1) throw std::invalid_argument("sketch set: need at least one replicate");
    if (!is_power_of_two(b)) throw std::invalid_argument("sketch set: b must be a power of two");
    auto* s = new SymSet;
    s->n = n;
    s->b = b;
    s->B = B;
    s->seed = seed;
    s->reps.resize(B);
    for (int m = 0; m < B; ++m) {
        auto& rep = s->reps[m];
        rep.h = PolyHash::from_seed(6, b, derive_seed(seed, kSymBucketHash, m));
        rep.sigma = PolyHash::from_seed(6, 4, derive_seed(seed, kSymSign, m));
        fill_sym_tables(rep, n, b);
        rep.data.assign(b, {0.0, 0.0});
    }
    return s;
}

// sketch.cpp:315-345
void sym_accumulate_dense(SymSet& s, const double* T, bool assume_symmetric) {
    const int n = s.n;
    if (!assume_symmetric) {
        int bad[3];
        if (first_asymmetric_triple(T, n, 1e-9, bad))
            throw std::invalid_argument("accumulate_dense: input tensor is not symmetric at (" +
                                        std::to_string(bad[0] + 1) + "," + std::to_string(bad[1] + 1) +
                                        "," + std::to_string(bad[2] + 1) + ")");
    }
    ++s.version;
    const std::uint32_t b = s.b;
#pragma omp parallel for schedule(static)
    for (int m = 0; m < s.B; ++m) {
        auto& rep = s.reps[m];
        for (int i = 0; i < n; ++i) {
            std::uint64_t hi = rep.bucket1[i];
            unsigned ei = rep.sexp[i];
            for (int j = i; j < n; ++j) {
                std::uint64_t hij = hi + rep.bucket1[j];
                unsigned eij = ei + rep.sexp[j];
                const double* row = &T[(static_cast<std::size_t>(i) * n + j) * n];
                for (int k = j; k < n; ++k) {
                    double value = row[k];
                    if (value == 0.0) continue;
                    double mult = (i == j && j == k) ? 1.0 : ((i == j || j == k) ? 3.0 : 6.0);
                    std::uint32_t t = static_cast<std::uint32_t>((hij + rep.bucket1[k]) % b);
                    rep.data[t] += mult * value * root4(eij + rep.sexp[k]);
                }
            }
        }
    }
}

// sketch.cpp:315-345 restricted to rows i in [i0, i1): the same loop order, the partial
// sketch of one i-slice (the multi-GPU shard unit and the bounded CPU-baseline sample).
// T points at row i0 ((i - i0) * n^2 + j * n + k), float64 or float32 (widened exactly,
// as the reference would see the tensor converted to its fp64 DenseTensor3).
template <typename TT>
void sym_accumulate_dense_slice(SymSet& s, const TT* T, int i0, int i1) {
    const int n = s.n;
    ++s.version;
    const std::uint32_t b = s.b;
#pragma omp parallel for schedule(static)
    for (int m = 0; m < s.B; ++m) {
        auto& rep = s.reps[m];
        for (int i = i0; i < i1; ++i) {
            std::uint64_t hi = rep.bucket1[i];
            unsigned ei = rep.sexp[i];
            for (int j = i; j < n; ++j) {
                std::uint64_t hij = hi + rep.bucket1[j];
                unsigned eij = ei + rep.sexp[j];
                const TT* row = &T[(static_cast<std::size_t>(i - i0) * n + j) * n];
                for (int k = j; k < n; ++k) {
                    double value = static_cast<double>(row[k]);
                    if (value == 0.0) continue;
                    double mult = (i == j && j == k) ? 1.0 : ((i == j || j == k) ? 3.0 : 6.0);
                    std::uint32_t t = static_cast<std::uint32_t>((hij + rep.bucket1[k]) % b);
                    rep.data[t] += mult * value * root4(eij + rep.sexp[k]);
                }
            }
        }
    }
}

// BASELINE configs 0-2 planted tensor, restated independently of the product library so
// the CPU arms never load it: lambda ~ U[1,2] and the QR basis from the host Rng streams
// (tags 0x61 / 0x62, modified Gram-Schmidt twice), noise sigma * N(0,1) per sorted triple
// from a counter-based SplitMix64 hash of (a, b, c) and Box-Muller (tag 0x63), mirrored.
// Entries of rows i in [i0, i1) are written to out[(i - i0) * n^2 + j * n + k].
static std::uint64_t gen_mix64(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
void gen_planted_slice(int n, int rank, double sigma, std::uint64_t seed, int i0, int i1, int f32, void* out,
                       double* lambda_out, double* V_out) {
    std::vector<double> lam(rank), V(static_cast<std::size_t>(rank) * n);
    Rng lr(derive_seed(seed, 0x61));
    for (int r = 0; r < rank; ++r) lam[r] = 1.0 + lr.uniform();
    Rng br(derive_seed(seed, 0x62));
    for (int r = 0; r < rank; ++r)
        for (int i = 0; i < n; ++i) V[static_cast<std::size_t>(r) * n + i] = br.gaussian();
    for (int pass = 0; pass < 2; ++pass)
        for (int r = 0; r < rank; ++r) {
            double* v = &V[static_cast<std::size_t>(r) * n];
            for (int q = 0; q < r; ++q) {
                const double* w = &V[static_cast<std::size_t>(q) * n];
                double d = 0;
                for (int i = 0; i < n; ++i) d += v[i] * w[i];
                for (int i = 0; i < n; ++i) v[i] -= d * w[i];
            }
            double ss = 0;
            for (int i = 0; i < n; ++i) ss += v[i] * v[i];
            const double inv = 1.0 / std::sqrt(ss);
            for (int i = 0; i < n; ++i) v[i] *= inv;
        }
    if (lambda_out) std::copy(lam.begin(), lam.end(), lambda_out);
    if (V_out) std::copy(V.begin(), V.end(), V_out);
    const std::uint64_t nseed = derive_seed(seed, 0x63);
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
    for (int i = i0; i < i1; ++i)
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < n; ++k) {
                const int a = std::min(i, std::min(j, k)), c = std::max(i, std::max(j, k)), bb = i + j + k - a - c;
                double s = 0.0;
                for (int r = 0; r < rank; ++r)
                    s += lam[r] * V[static_cast<std::size_t>(r) * n + a] * V[static_cast<std::size_t>(r) * n + bb] *
                         V[static_cast<std::size_t>(r) * n + c];
                if (sigma > 0.0) {
                    const std::uint64_t key = ((static_cast<std::uint64_t>(a) * n + bb) * n + c);
                    const std::uint64_t h1 = gen_mix64(nseed ^ (key * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull));
                    const std::uint64_t h2 = gen_mix64(h1 + 0x9E3779B97F4A7C15ull);
                    const double u1 = (static_cast<double>(h1 >> 11) + 1.0) * 0x1.0p-53;
                    const double u2 = static_cast<double>(h2 >> 11) * 0x1.0p-53;
                    s += sigma * std::sqrt(-2.0 * std::log(u1)) * std::cos(3.141592653589793238462643383279502884 * 2.0 * u2);
                }
                const std::size_t off = (static_cast<std::size_t>(i - i0) * n + j) * n + k;
                if (f32)
                    static_cast<float*>(out)[off] = static_cast<float>(s);
                else
                    static_cast<double*>(out)[off] = s;
            }
}

// sketch.cpp:347-361
void sym_add_scaled_rank1(SymSet& s, const double* u, double alpha) {
    if (alpha == 0.0) return;
    ++s.version;
    const std::uint32_t b = s.b;
#pragma omp parallel for schedule(static)
    for (int m = 0; m < s.B; ++m) {
        auto& rep = s.reps[m];
        cvec su(b, {0.0, 0.0});
        for (int i = 0; i < s.n; ++i) su[rep.bucket1[i]] += root4(rep.sexp[i]) * u[i];
        forward_inplace(su);
        for (auto& z : su) z = z * z * z;
        inverse_inplace(su);
        for (std::uint32_t t = 0; t < b; ++t) rep.data[t] += alpha * su[t];
    }
}

// sketch.cpp:363-377
double sym_recover_entry(const SymSet& s, int i, int j, int k) {
    const int n = s.n;
    if (i < 0 || j < 0 || k < 0 || i >= n || j >= n || k >= n)
        throw std::invalid_argument("recover_entry: index out of range");
    double kappa = (i == j && j == k) ? 1.0 : ((i == j || j == k || i == k) ? 3.0 : 6.0);
    std::vector<double> est(s.B);
    for (int m = 0; m < s.B; ++m) {
        const auto& rep = s.reps[m];
        std::uint32_t t = static_cast<std::uint32_t>(
            (std::uint64_t{rep.bucket1[i]} + rep.bucket1[j] + rep.bucket1[k]) % s.b);
        unsigned e = (4 * 3 - (rep.sexp[i] + rep.sexp[j] + rep.sexp[k])) & 3u;
        est[m] = (root4(e) * rep.data[t]).real() / kappa;
    }
    return median_inplace(est);
}

// sketch.cpp:412-443
void sym_aux_sketches(const SymRep& rep, std::uint32_t b, const double* u, int n, cvec& s1, cvec& s2,
                      cvec& s3) {
    s1.assign(b, {0.0, 0.0});
    s2.assign(b, {0.0, 0.0});
    s3.assign(b, {0.0, 0.0});
    for (int i = 0; i < n; ++i) {
        double ui = u[i];
        s1[rep.bucket1[i]] += root4(rep.sexp[i]) * ui;
        s2[rep.bucket2[i]] += root4(2u * rep.sexp[i]) * (ui * ui);
        s3[rep.bucket3[i]] += root4(3u * rep.sexp[i]) * (ui * ui * ui);
    }
}
cvec sketch_rank1_sym(const SymSet& s, int m, const double* u) {
    const auto& rep = s.reps[m];
    const std::uint32_t b = s.b;
    cvec s1, s2, s3;
    sym_aux_sketches(rep, b, u, s.n, s1, s2, s3);
    cvec f1 = s1;
    forward_inplace(f1);
    cvec f2 = s2;
    forward_inplace(f2);
    cvec acc(b);
    for (std::uint32_t t = 0; t < b; ++t) acc[t] = f1[t] * (f1[t] * f1[t] * (1.0 / 6.0) + f2[t] * 0.5);
    inverse_inplace(acc);
    for (std::uint32_t t = 0; t < b; ++t) acc[t] += (1.0 / 3.0) * s3[t];
    return acc;
}

// --- contraction.cpp:59-181: symmetric workspace ------------------------------------
struct SymWs {
    const SymSet* set;
    std::uint64_t cached_version;
    std::vector<cvec> fourier;
};

// contraction.cpp:62-72
void sym_ensure_fresh(SymWs& ws) {
    if (ws.cached_version == ws.set->version && !ws.fourier.empty()) return;
    const int B = ws.set->B;
    ws.fourier.resize(B);
#pragma omp parallel for schedule(static)
    for (int m = 0; m < B; ++m) {
        ws.fourier[m] = ws.set->reps[m].data;
        forward_inplace(ws.fourier[m]);
    }
    ws.cached_version = ws.set->version;
}

// contraction.cpp:83-126
double sym_vvv(SymWs& ws, const double* u) {
    sym_ensure_fresh(ws);
    const SymSet& s = *ws.set;
    const int n = s.n, B = s.B;
    const std::uint32_t b = s.b;
    std::vector<double> est(B);
#pragma omp parallel for schedule(static) if (!omp_in_parallel())
    for (int m = 0; m < B; ++m) {
        const auto& rep = s.reps[m];
        cvec f1(b, {0.0, 0.0}), f2(b, {0.0, 0.0});
        for (int i = 0; i < n; ++i) {
            double ui = u[i];
            f1[rep.bucket1[i]] += root4(rep.sexp[i]) * ui;
            f2[rep.bucket2[i]] += root4(2u * rep.sexp[i]) * (ui * ui);
        }
        forward_inplace(f1);
        forward_inplace(f2);
        const cd* fT = ws.fourier[m].data();
        double acc1 = 0, acc2 = 0;
        for (std::uint32_t t = 0; t < b; ++t) {
            cd c1 = std::conj(f1[t]);
            cd w1 = fT[t] * c1;
            acc1 += (w1 * c1 * c1).real();
            acc2 += (w1 * std::conj(f2[t])).real();
        }
        double term3 = 0;
        for (int i = 0; i < n; ++i) {
            double u3 = u[i] * u[i] * u[i];
            term3 += u3 * re_rot_conj(3u * rep.sexp[i], rep.data[rep.bucket3[i]]);
        }
        est[m] = (acc1 / 6.0 + acc2 / 2.0) / static_cast<double>(b) + term3 / 3.0;
    }
    return median_inplace(est);
}

// contraction.cpp:128-181
void sym_ivv(SymWs& ws, const double* u, double* result) {
    sym_ensure_fresh(ws);
    const SymSet& s = *ws.set;
    const int n = s.n, B = s.B;
    const std::uint32_t b = s.b;
    std::vector<double> vals(static_cast<std::size_t>(B) * n);
    const double inv_b = 1.0 / static_cast<double>(b);
#pragma omp parallel for schedule(static) if (!omp_in_parallel())
    for (int m = 0; m < B; ++m) {
        const auto& rep = s.reps[m];
        cvec f1(b, {0.0, 0.0}), f2(b, {0.0, 0.0}), z1(b), z2(b);
        for (int i = 0; i < n; ++i) {
            double ui = u[i];
            f1[rep.bucket1[i]] += root4(rep.sexp[i]) * ui;
            f2[rep.bucket2[i]] += root4(2u * rep.sexp[i]) * (ui * ui);
        }
        forward_inplace(f1);
        forward_inplace(f2);
        const cd* fT = ws.fourier[m].data();
        for (std::uint32_t t = 0; t < b; ++t) {
            cd fu = f1[t];
            z1[t] = fT[t] * std::conj(fu * fu + f2[t]);
            z2[t] = fT[t] * std::conj(fu);
        }
        inverse_inplace_unscaled(z1);
        inverse_inplace_unscaled(z2);
        double* out = &vals[static_cast<std::size_t>(m) * n];
        for (int i = 0; i < n; ++i) {
            unsigned e = rep.sexp[i];
            double ui = u[i];
            double v = re_rot_conj(e, z1[rep.bucket1[i]]) * (1.0 / 6.0) * inv_b;
            v += ui * re_rot_conj(2u * e, z2[rep.bucket2[i]]) * (1.0 / 3.0) * inv_b;
            v += ui * ui * re_rot_conj(3u * e, rep.data[rep.bucket3[i]]) * (1.0 / 3.0);
            out[i] = v;
        }
    }
    std::vector<double> tmp(B);
    for (int i = 0; i < n; ++i) {  // contraction.cpp:49-53 strided_median
        for (int m = 0; m < B; ++m) tmp[m] = vals[static_cast<std::size_t>(m) * n + i];
        result[i] = median_inplace(tmp);
    }
}

// --- decompose.cpp:15-40, 83-115: fast RTPM ------------------------------------------
void normalized_or_throw(std::vector<double>& v, double tol) {
    double s = 0;
    for (double x : v) s += x * x;
    double nrm = std::sqrt(s);
    if (!(nrm > tol)) throw DegenerateIterationError("power update produced a vanishing iterate");
    for (double& x : v) x /= nrm;
}

// inits: optional k*L*n initial vectors (component-major, then tau); when null the
// reference's own Rng(derive_seed(seed,0x31,c,tau)).unit_sphere(n) is used.
void robust_tpm_fast(SymSet& s, int k, int L, int T_iters, std::uint64_t seed, double tol,
                     const double* inits, double* lambda, double* V /* n x k col-major */,
                     int* best_taus) {
    const int n = s.n;
    if (k < 1 || L < 1 || T_iters < 1)
        throw std::invalid_argument("power method: k, L and T must be positive");
    if (k > n) throw std::invalid_argument("power method: target rank exceeds tensor dimension");
    SymWs ws{&s, s.version - 1, {}};
    std::vector<double> out(n);
    for (int c = 0; c < k; ++c) {
        std::vector<std::vector<double>> finals(L);
        // restarts are independent (decompose.cpp:93-104): run them on the threads (each
        // contraction then runs serially, same arithmetic); a degenerate iterate throws at
        // the lowest restart index, as the serial loop would
        sym_ensure_fresh(ws);
        std::vector<std::string> err(L);
#pragma omp parallel for schedule(dynamic, 1)
        for (int tau = 0; tau < L; ++tau) {
            std::vector<double> u, out(n);
            if (inits) {
                u.assign(inits + (static_cast<std::size_t>(c) * L + tau) * n,
                         inits + (static_cast<std::size_t>(c) * L + tau + 1) * n);
            } else {
                Rng rng(derive_seed(seed, kPowerInit, c, tau));
                u = rng.unit_sphere(n);
            }
            try {
                for (int t = 0; t < T_iters; ++t) {
                    sym_ivv(ws, u.data(), out.data());
                    u = out;
                    normalized_or_throw(u, tol);
                }
            } catch (const std::exception& e) {
                err[tau] = e.what();
            }
            finals[tau] = u;
        }
        for (int tau = 0; tau < L; ++tau)
            if (!err[tau].empty()) throw DegenerateIterationError(err[tau]);
        double best = -std::numeric_limits<double>::infinity();
        int best_tau = 0;
        std::vector<double> values(L);
#pragma omp parallel for schedule(dynamic, 1)
        for (int tau = 0; tau < L; ++tau) values[tau] = sym_vvv(ws, finals[tau].data());
        for (int tau = 0; tau < L; ++tau) {
            double value = values[tau];
            if (value > best) {
                best = value;
                best_tau = tau;
            }
        }
        lambda[c] = best;
        for (int i = 0; i < n; ++i) V[static_cast<std::size_t>(c) * n + i] = finals[best_tau][i];
        if (best_taus) best_taus[c] = best_tau;
        sym_add_scaled_rank1(s, finals[best_tau].data(), -best);
    }
}

// --- tensor.cpp:67-107 exact contractions; decompose.cpp:22-33,53-81 exact RTPM ---------
double contract_vvv_exact(const double* T, int n, const double* u) {
    double total = 0;
    for (int i = 0; i < n; ++i) {
        const double* ti = T + static_cast<std::size_t>(i) * n * n;
        double acc = 0;
        for (int j = 0; j < n; ++j) {
            const double* tij = ti + static_cast<std::size_t>(j) * n;
            double s = 0;
            for (int k = 0; k < n; ++k) s += tij[k] * u[k];
            acc += u[j] * s;
        }
        total += u[i] * acc;
    }
    return total;
}
void contract_Ivv_exact(const double* T, int n, const double* u, const double* v, double* out) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
        const double* ti = T + static_cast<std::size_t>(i) * n * n;
        double acc = 0;
        for (int j = 0; j < n; ++j) {
            const double* tij = ti + static_cast<std::size_t>(j) * n;
            double s = 0;
            for (int k = 0; k < n; ++k) s += tij[k] * v[k];
            acc += u[j] * s;
        }
        out[i] = acc;
    }
}

// --- sketch.cpp: asymmetric set --------------------------------------------------------
struct AsymRep {
    std::array<PolyHash, 3> h, xi;
    std::array<std::vector<std::uint32_t>, 3> bucket;
    std::array<std::vector<double>, 3> sign;
    cvec data;
};
struct AsymSet {
    int n = 0;
    std::uint32_t b = 2;
    int B = 0;
    std::uint64_t seed = 0;
    std::uint64_t version = 0;
    std::vector<AsymRep> reps;
};

// sketch.cpp:13-22 (xi value: rademacher root, hashing.hpp:73-75)
void fill_asym_tables(AsymRep& rep, int n) {
    for (int s = 0; s < 3; ++s) {
        rep.bucket[s].resize(n);
        rep.sign[s].resize(n);
        for (int i = 0; i < n; ++i) {
            rep.bucket[s][i] = rep.h[s].eval(i);
            rep.sign[s][i] = (rep.xi[s].eval(i) & 1) ? -1.0 : 1.0;
        }
    }
}

// sketch.cpp:155-171
AsymSet* asym_create(int n, std::uint32_t b, int B, std::uint64_t seed) {
    if (n < 1) throw std::invalid_argument("sketch set: dimension must be positive");
    if (B < 1) throw std::invalid_argument("sketch set: need at least one replicate");
    if (!is_power_of_two(b)) throw std::invalid_argument("sketch set: b must be a power of two");
    auto* s = new AsymSet;
    s->n = n;
    s->b = b;
    s->B = B;
    s->seed = seed;
    s->reps.resize(B);
    for (int m = 0; m < B; ++m) {
        auto& rep = s->reps[m];
        for (int sl = 0; sl < 3; ++sl) {
            rep.h[sl] = PolyHash::from_seed(2, b, derive_seed(seed, kAsymBucketHash, m, sl));
            rep.xi[sl] = PolyHash::from_seed(6, 2, derive_seed(seed, kAsymSign, m, sl));
        }
        fill_asym_tables(rep, n);
        rep.data.assign(b, {0.0, 0.0});
    }
    return s;
}

// sketch.cpp:173-193
void asym_accumulate_dense(AsymSet& s, const double* T) {
    ++s.version;
    const int n = s.n;
    const std::uint32_t b = s.b;
#pragma omp parallel for schedule(static)
    for (int m = 0; m < s.B; ++m) {
        auto& rep = s.reps[m];
        for (int i = 0; i < n; ++i) {
            std::uint32_t hi = rep.bucket[0][i];
            double si = rep.sign[0][i];
            for (int j = 0; j < n; ++j) {
                std::uint64_t hij = hi + rep.bucket[1][j];
                double sij = si * rep.sign[1][j];
                const double* row = &T[(static_cast<std::size_t>(i) * n + j) * n];
                for (int k = 0; k < n; ++k) {
                    std::uint32_t t = static_cast<std::uint32_t>((hij + rep.bucket[2][k]) % b);
                    rep.data[t] += sij * rep.sign[2][k] * row[k];
                }
            }
        }
    }
}

// sketch.cpp:195-212
cvec asym_rank1_sketch(const AsymSet& s, int m, const double* u, const double* v, const double* w) {
    const auto& rep = s.reps[m];
    const std::uint32_t b = s.b;
    cvec su(b, {0.0, 0.0}), sv(b, {0.0, 0.0}), sw(b, {0.0, 0.0});
    for (int i = 0; i < s.n; ++i) {
        su[rep.bucket[0][i]] += cd(rep.sign[0][i] * u[i], 0.0);
        sv[rep.bucket[1][i]] += cd(rep.sign[1][i] * v[i], 0.0);
        sw[rep.bucket[2][i]] += cd(rep.sign[2][i] * w[i], 0.0);
    }
    forward_inplace(su);
    forward_inplace(sv);
    forward_inplace(sw);
    for (std::uint32_t t = 0; t < b; ++t) su[t] *= sv[t] * sw[t];
    inverse_inplace(su);
    return su;
}

// sketch.cpp:214-222
void asym_add_rank1(AsymSet& s, double alpha, const double* u, const double* v, const double* w) {
    ++s.version;
#pragma omp parallel for schedule(static)
    for (int m = 0; m < s.B; ++m) {
        cvec r = asym_rank1_sketch(s, m, u, v, w);
        for (std::uint32_t t = 0; t < s.b; ++t) s.reps[m].data[t] += alpha * r[t];
    }
}

// sketch.cpp:224-248 (components as N x n row-major arrays)
void asym_accumulate_factored(AsymSet& s, int N, const double* a, const double* U, const double* Vv,
                              const double* W) {
    ++s.version;
    const int n = s.n;
    const std::uint32_t b = s.b;
#pragma omp parallel for schedule(static)
    for (int m = 0; m < s.B; ++m) {
        auto& rep = s.reps[m];
        cvec su(b), sv(b), sw(b);
        for (int c = 0; c < N; ++c) {
            const double* u = U + static_cast<std::size_t>(c) * n;
            const double* v = Vv + static_cast<std::size_t>(c) * n;
            const double* w = W + static_cast<std::size_t>(c) * n;
            std::fill(su.begin(), su.end(), cd{0.0, 0.0});
            std::fill(sv.begin(), sv.end(), cd{0.0, 0.0});
            std::fill(sw.begin(), sw.end(), cd{0.0, 0.0});
            for (int i = 0; i < n; ++i) {
                su[rep.bucket[0][i]] += cd(rep.sign[0][i] * u[i], 0.0);
                sv[rep.bucket[1][i]] += cd(rep.sign[1][i] * v[i], 0.0);
                sw[rep.bucket[2][i]] += cd(rep.sign[2][i] * w[i], 0.0);
            }
            forward_inplace(su);
            forward_inplace(sv);
            forward_inplace(sw);
            for (std::uint32_t t = 0; t < b; ++t) su[t] *= sv[t] * sw[t];
            inverse_inplace(su);
            for (std::uint32_t t = 0; t < b; ++t) rep.data[t] += a[c] * su[t];
        }
    }
}

// sketch.cpp:250-262
double asym_recover_entry(const AsymSet& s, int i, int j, int k) {
    const int n = s.n;
    if (i < 0 || j < 0 || k < 0 || i >= n || j >= n || k >= n)
        throw std::invalid_argument("recover_entry: index out of range");
    std::vector<double> est(s.B);
    for (int m = 0; m < s.B; ++m) {
        const auto& rep = s.reps[m];
        std::uint32_t t = static_cast<std::uint32_t>(
            (std::uint64_t{rep.bucket[0][i]} + rep.bucket[1][j] + rep.bucket[2][k]) % s.b);
        double sg = rep.sign[0][i] * rep.sign[1][j] * rep.sign[2][k];
        est[m] = sg * rep.data[t].real();
    }
    return median_inplace(est);
}

// --- contraction.cpp:185-304: asymmetric workspace -------------------------------------
struct AsymWs {
    const AsymSet* set;
    std::uint64_t cached_version;
    std::vector<cvec> fourier;
};
void asym_ensure_fresh(AsymWs& ws) {  // contraction.cpp:188-198
    if (ws.cached_version == ws.set->version && !ws.fourier.empty()) return;
    const int B = ws.set->B;
    ws.fourier.resize(B);
#pragma omp parallel for schedule(static)
    for (int m = 0; m < B; ++m) {
        ws.fourier[m] = ws.set->reps[m].data;
        forward_inplace(ws.fourier[m]);
    }
    ws.cached_version = ws.set->version;
}
// contraction.cpp:209-246
double asym_vvv(AsymWs& ws, const double* u) {
    asym_ensure_fresh(ws);
    const AsymSet& s = *ws.set;
    const int n = s.n, B = s.B;
    const std::uint32_t b = s.b;
    std::vector<double> est(B);
#pragma omp parallel for schedule(static)
    for (int m = 0; m < B; ++m) {
        const auto& rep = s.reps[m];
        cvec fx(b, {0.0, 0.0}), fy(b, {0.0, 0.0}), z(b, {0.0, 0.0});
        for (int i = 0; i < n; ++i) {
            fx[rep.bucket[0][i]] += cd(rep.sign[0][i] * u[i], 0.0);
            fy[rep.bucket[1][i]] += cd(rep.sign[1][i] * u[i], 0.0);
            z[rep.bucket[2][i]] += cd(rep.sign[2][i] * u[i], 0.0);
        }
        forward_inplace(fx);
        forward_inplace(fy);
        forward_inplace(z);
        const cd* fT = ws.fourier[m].data();
        double acc = 0;
        for (std::uint32_t t = 0; t < b; ++t) acc += (fT[t] * std::conj(fx[t] * fy[t] * z[t])).real();
        est[m] = acc / static_cast<double>(b);
    }
    return median_inplace(est);
}
// contraction.cpp:248-295
void asym_mode_contraction(AsymWs& ws, int free_mode, const double* x, const double* y, double* result) {
    if (free_mode < 0 || free_mode > 2)
        throw std::invalid_argument("mode_contraction: free_mode must be 0, 1 or 2");
    asym_ensure_fresh(ws);
    const AsymSet& s = *ws.set;
    const int n = s.n, B = s.B;
    const int slot_x = free_mode == 0 ? 1 : 0;
    const int slot_y = free_mode == 2 ? 1 : 2;
    const std::uint32_t b = s.b;
    std::vector<double> vals(static_cast<std::size_t>(B) * n);
    const double inv_b = 1.0 / static_cast<double>(b);
#pragma omp parallel for schedule(static)
    for (int m = 0; m < B; ++m) {
        const auto& rep = s.reps[m];
        cvec fx(b, {0.0, 0.0}), fy(b, {0.0, 0.0}), z(b);
        for (int i = 0; i < n; ++i) {
            fx[rep.bucket[slot_x][i]] += cd(rep.sign[slot_x][i] * x[i], 0.0);
            fy[rep.bucket[slot_y][i]] += cd(rep.sign[slot_y][i] * y[i], 0.0);
        }
        forward_inplace(fx);
        forward_inplace(fy);
        const cd* fT = ws.fourier[m].data();
        for (std::uint32_t t = 0; t < b; ++t) z[t] = fT[t] * std::conj(fx[t] * fy[t]);
        inverse_inplace_unscaled(z);
        double* out = &vals[static_cast<std::size_t>(m) * n];
        for (int i = 0; i < n; ++i)
            out[i] = rep.sign[free_mode][i] * z[rep.bucket[free_mode][i]].real() * inv_b;
    }
    std::vector<double> tmp(B);
    for (int i = 0; i < n; ++i) {
        for (int m = 0; m < B; ++m) tmp[m] = vals[static_cast<std::size_t>(m) * n + i];
        result[i] = median_inplace(tmp);
    }
}

// --- lda.cpp:29-34, 88-100, 145-226: whitened third-moment sketch ----------------------
// Corpus as CSR: doc_ptr[D+1], word[nnz], count[nnz]; W: V x k row-major.
void lda_compute_m1(int V, int D, const long long* doc_ptr, const int* word, const int* count,
                    double* m1) {
    for (int w = 0; w < V; ++w) m1[w] = 0.0;
    long long used = 0;
    for (int d = 0; d < D; ++d) {
        long long total = 0;
        for (long long p = doc_ptr[d]; p < doc_ptr[d + 1]; ++p) total += count[p];
        if (total < 1) continue;
        double scale = 1.0 / static_cast<double>(total);
        for (long long p = doc_ptr[d]; p < doc_ptr[d + 1]; ++p) m1[word[p]] += scale * count[p];
        ++used;
    }
    if (used == 0) throw std::runtime_error("compute_m1: no nonempty documents");
    for (int w = 0; w < V; ++w) m1[w] /= static_cast<double>(used);
}

// --- lda.cpp:102-123: dense M2 = (1/used2) sum_d pair(d)/(m(m-1)) - a0/(a0+1) m1 m1^T --
// pair(a, b) over document positions: c_a c_b, and c_a (c_a - 1) on the diagonal a == b.
void lda_compute_m2(int V, int D, const long long* doc_ptr, const int* word, const int* count, double alpha0,
                    double* m2 /* V x V row-major */) {
    std::vector<double> m1(V);
    lda_compute_m1(V, D, doc_ptr, word, count, m1.data());
    std::fill(m2, m2 + static_cast<std::size_t>(V) * V, 0.0);
    long long used = 0;
    for (int d = 0; d < D; ++d) {
        long long total = 0;
        for (long long q = doc_ptr[d]; q < doc_ptr[d + 1]; ++q) total += count[q];
        if (total < 2) continue;
        ++used;
        const double scale = 1.0 / (static_cast<double>(total) * (total - 1));
        for (long long a = doc_ptr[d]; a < doc_ptr[d + 1]; ++a)
            for (long long b = doc_ptr[d]; b < doc_ptr[d + 1]; ++b) {
                const double pair = (a == b) ? static_cast<double>(count[a]) * (count[a] - 1)
                                             : static_cast<double>(count[a]) * count[b];
                m2[static_cast<std::size_t>(word[a]) * V + word[b]] += scale * pair;
            }
    }
    if (used == 0) throw std::runtime_error("compute_m2: no documents with at least 2 words");
    const double c = alpha0 / (alpha0 + 1.0);
    for (int i = 0; i < V; ++i)
        for (int j = 0; j < V; ++j) {
            double& e = m2[static_cast<std::size_t>(i) * V + j];
            e /= static_cast<double>(used);
            e -= c * m1[i] * m1[j];
        }
}

// Cyclic Jacobi eigensolver for a symmetric matrix: the test oracle standing in for
// Eigen::SelfAdjointEigenSolver (lda.cpp:128). Eigenvalues ascending; column c of the
// row-major evecs is the eigenvector of evals[c] (sign unpinned, as in Eigen).
void sym_eigen_jacobi(int n, const double* A, double* evals, double* evecs) {
    std::vector<long double> a(A, A + static_cast<std::size_t>(n) * n), v(static_cast<std::size_t>(n) * n, 0.0L);
    for (int i = 0; i < n; ++i) v[static_cast<std::size_t>(i) * n + i] = 1.0L;
    auto at = [&](std::vector<long double>& m, int i, int j) -> long double& { return m[static_cast<std::size_t>(i) * n + j]; };
    for (int sweep = 0; sweep < 100; ++sweep) {
        long double off = 0, tot = 0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                tot += at(a, i, j) * at(a, i, j);
                if (i != j) off += at(a, i, j) * at(a, i, j);
            }
        if (off <= 1e-30L * tot) break;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                const long double apq = at(a, p, q);
                if (apq == 0.0L) continue;
                const long double theta = (at(a, q, q) - at(a, p, p)) / (2.0L * apq);
                const long double t = (theta >= 0 ? 1.0L : -1.0L) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0L));
                const long double c = 1.0L / std::sqrt(t * t + 1.0L), s = t * c;
                for (int k = 0; k < n; ++k) {  // A <- A J (columns p, q)
                    const long double akp = at(a, k, p), akq = at(a, k, q);
                    at(a, k, p) = c * akp - s * akq;
                    at(a, k, q) = s * akp + c * akq;
                }
                for (int k = 0; k < n; ++k) {  // A <- J^T A (rows p, q)
                    const long double apk = at(a, p, k), aqk = at(a, q, k);
                    at(a, p, k) = c * apk - s * aqk;
                    at(a, q, k) = s * apk + c * aqk;
                }
                for (int k = 0; k < n; ++k) {
                    const long double vkp = at(v, k, p), vkq = at(v, k, q);
                    at(v, k, p) = c * vkp - s * vkq;
                    at(v, k, q) = s * vkp + c * vkq;
                }
            }
    }
    std::vector<int> ord(n);
    for (int i = 0; i < n; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return at(a, x, x) < at(a, y, y); });
    for (int c = 0; c < n; ++c) {
        evals[c] = static_cast<double>(at(a, ord[c], ord[c]));
        for (int i = 0; i < n; ++i) evecs[static_cast<std::size_t>(i) * n + c] = static_cast<double>(at(v, i, ord[c]));
    }
}

// --- lda.cpp:125-143: whiten(m2hat, k) ---------------------------------------------------
// W[:, c] = u_c / sqrt(ev_c), unwhiten[:, c] = u_c sqrt(ev_c) for the k largest eigenpairs
// (descending); W and unwhiten V x k row-major.
void lda_whiten(int V, const double* m2, int k, double* W, double* unwhiten, double* sv) {
    if (k < 1 || k > V) throw std::invalid_argument("whiten: invalid target rank");
    std::vector<double> ev(V), U(static_cast<std::size_t>(V) * V);
    sym_eigen_jacobi(V, m2, ev.data(), U.data());
    for (int c = 0; c < k; ++c) {
        const double e = ev[V - 1 - c];
        if (!(e > 1e-10))
            throw std::runtime_error("whiten: moment matrix is rank deficient at component " + std::to_string(c + 1) +
                                 " (eigenvalue " + std::to_string(e) + ")");
        sv[c] = e;
        for (int i = 0; i < V; ++i) {
            const double u = U[static_cast<std::size_t>(i) * V + (V - 1 - c)];
            W[static_cast<std::size_t>(i) * k + c] = u / std::sqrt(e);
            unwhiten[static_cast<std::size_t>(i) * k + c] = u * std::sqrt(e);
        }
    }
}

// lda.cpp:250-271 project_to_simplex: sort descending, last prefix index whose value
// exceeds its running threshold, uniform if none.
std::vector<double> project_to_simplex(const double* y, int n) {
    std::vector<double> u(y, y + n);
    std::sort(u.begin(), u.end(), std::greater<double>());
    double css = 0, theta = 0;
    int rho = 0;
    for (int i = 0; i < n; ++i) {
        css += u[i];
        const double t = (css - 1.0) / (i + 1);
        if (u[i] - t > 0) {
            rho = i + 1;
            theta = t;
        }
    }
    std::vector<double> x(n);
    if (rho == 0) {
        std::fill(x.begin(), x.end(), 1.0 / n);
        return x;
    }
    for (int i = 0; i < n; ++i) x[i] = std::max(y[i] - theta, 0.0);
    return x;
}

// lda.cpp:228-248 recover_params: A k x k row-major (column i = component i), unwhiten and
// Phi V x k row-major.
void lda_recover_params(int V, int k, const double* lambda, const double* A, const double* unwhiten, double alpha0,
                        double* Phi, double* alpha) {
    if (k < 1) throw std::invalid_argument("recover_params: empty decomposition");
    std::vector<double> mu(V);
    for (int i = 0; i < k; ++i) {
        const double lam = lambda[i];
        if (lam == 0.0) throw NumericalError("recover_params: zero eigenvalue at component " + std::to_string(i + 1));
        alpha[i] = 4.0 * alpha0 * (alpha0 + 1.0) / ((alpha0 + 2.0) * (alpha0 + 2.0) * lam * lam);
        for (int w = 0; w < V; ++w) {
            double s = 0;
            for (int c = 0; c < k; ++c) s += unwhiten[static_cast<std::size_t>(w) * k + c] * A[static_cast<std::size_t>(c) * k + i];
            mu[w] = 0.5 * (alpha0 + 2.0) * lam * s;
        }
        const std::vector<double> ph = project_to_simplex(mu.data(), V);
        for (int w = 0; w < V; ++w) Phi[static_cast<std::size_t>(w) * k + i] = ph[w];
    }
}

// lda.cpp:273-320 heldout_likelihood (sequential, document order).
double lda_heldout_likelihood(int V, int k, const double* Phi, int Vh, long long D, const long long* doc_ptr,
                              const int* word, const int* count, long long* floored_out) {
    if (Vh > V) throw std::invalid_argument("heldout_likelihood: corpus vocabulary exceeds the model's");
    std::vector<double> gram(static_cast<std::size_t>(k) * k, 0.0);
    for (int a = 0; a < k; ++a)
        for (int b = 0; b < k; ++b) {
            double s = 0;
            for (int w = 0; w < V; ++w) s += Phi[static_cast<std::size_t>(w) * k + a] * Phi[static_cast<std::size_t>(w) * k + b];
            gram[static_cast<std::size_t>(b) * k + a] = s;
        }
    std::vector<double> ev(k), evec(static_cast<std::size_t>(k) * k);
    sym_eigen_jacobi(k, gram.data(), ev.data(), evec.data());
    double lips = -std::numeric_limits<double>::infinity();
    for (double e : ev) lips = std::max(lips, e);
    const double step = lips > 0 ? 1.0 / lips : 1.0;
    long long floored = 0, used = 0;
    double total = 0;
    for (long long d = 0; d < D; ++d) {
        long long tot = 0;
        for (long long q = doc_ptr[d]; q < doc_ptr[d + 1]; ++q) tot += count[q];
        if (tot < 1) continue;
        ++used;
        std::vector<double> pi(k, 1.0 / k);
        if (k == 1) {
            pi.assign(1, 1.0);
        } else {
            std::vector<double> phi_tw(k, 0.0), g(k), nx(k);
            const double inv_m = 1.0 / static_cast<double>(tot);
            for (long long q = doc_ptr[d]; q < doc_ptr[d + 1]; ++q)
                for (int a = 0; a < k; ++a) phi_tw[a] += (inv_m * count[q]) * Phi[static_cast<std::size_t>(word[q]) * k + a];
            for (int it = 0; it < 500; ++it) {
                for (int a = 0; a < k; ++a) {
                    double s = 0;
                    for (int b = 0; b < k; ++b) s += gram[static_cast<std::size_t>(b) * k + a] * pi[b];
                    g[a] = pi[a] - step * (s - phi_tw[a]);
                }
                nx = project_to_simplex(g.data(), k);
                double moved = 0;
                for (int a = 0; a < k; ++a) moved += (nx[a] - pi[a]) * (nx[a] - pi[a]);
                pi.swap(nx);
                if (std::sqrt(moved) <= 1e-8) break;
            }
        }
        double ll = 0;
        for (long long q = doc_ptr[d]; q < doc_ptr[d + 1]; ++q) {
            double p = 0;
            for (int a = 0; a < k; ++a) p += Phi[static_cast<std::size_t>(word[q]) * k + a] * pi[a];
            if (p < 1e-12) {
                p = 1e-12;
                ++floored;
            }
            ll += count[q] * std::log(p);
        }
        total += ll / static_cast<double>(tot);
    }
    if (floored_out) *floored_out = floored;
    if (used == 0) throw NumericalError("heldout_likelihood: empty held-out corpus");
    return total / static_cast<double>(used);
}

void fourier_sketch(const SymRep& rep, std::uint32_t b, const double* v, int k, cvec& out) {
    out.assign(b, {0.0, 0.0});
    for (int i = 0; i < k; ++i) out[rep.bucket1[i]] += root4(rep.sexp[i]) * v[i];
    forward_inplace(out);
}

void lda_sketch_whitened_m3(SymSet& s, int V, int D, const long long* doc_ptr, const int* word,
                            const int* count, const double* W, double alpha0, long long* used_out,
                            long long* skipped_out) {
    const int k = s.n;
    const std::uint32_t b = s.b;
    const int B = s.B;
    long long used = 0, skipped = 0;
    std::vector<double> P, scale1, scale2;
    std::vector<double> coeff1(V, 0.0), sumwn(static_cast<std::size_t>(V) * k, 0.0);
    std::vector<double> p(k);
    for (int d = 0; d < D; ++d) {
        long long total = 0;
        for (long long q = doc_ptr[d]; q < doc_ptr[d + 1]; ++q) total += count[q];
        if (total < 3) {
            ++skipped;
            continue;
        }
        ++used;
        const double m = static_cast<double>(total);
        const double s1 = 1.0 / (m * (m - 1.0) * (m - 2.0));
        const double s2 = alpha0 / ((alpha0 + 2.0) * m * (m - 1.0));
        std::fill(p.begin(), p.end(), 0.0);
        for (long long q = doc_ptr[d]; q < doc_ptr[d + 1]; ++q) {
            const double c = static_cast<double>(count[q]);
            const double* wr = W + static_cast<std::size_t>(word[q]) * k;
            for (int a = 0; a < k; ++a) p[a] += c * wr[a];
        }
        for (long long q = doc_ptr[d]; q < doc_ptr[d + 1]; ++q) {
            int w = word[q];
            double cnt = count[q];
            coeff1[w] += 2.0 * s1 * cnt;
            double* sr = &sumwn[static_cast<std::size_t>(w) * k];
            for (int a = 0; a < k; ++a) sr[a] += s1 * cnt * p[a];
        }
        P.insert(P.end(), p.begin(), p.end());
        scale1.push_back(s1);
        scale2.push_back(s2);
    }
    if (used == 0) throw std::runtime_error("sketch_whitened_m3: no documents with >= 3 words");
    std::vector<double> m1(V), q(k, 0.0);
    lda_compute_m1(V, D, doc_ptr, word, count, m1.data());
    for (int a = 0; a < k; ++a)
        for (int w = 0; w < V; ++w) q[a] += W[static_cast<std::size_t>(w) * k + a] * m1[w];
    const double inv_docs = 1.0 / static_cast<double>(used);
    const double m1_coeff = 2.0 * alpha0 * alpha0 / ((alpha0 + 1.0) * (alpha0 + 2.0));
    ++s.version;
#pragma omp parallel for schedule(static)
    for (int m = 0; m < B; ++m) {
        auto& rep = s.reps[m];
        cvec acc(b, {0.0, 0.0}), cross(b, {0.0, 0.0}), fp, fq, fw, fs;
        for (std::size_t d = 0; d < scale1.size(); ++d) {
            fourier_sketch(rep, b, &P[d * k], k, fp);
            for (std::uint32_t t = 0; t < b; ++t) {
                cd sq = fp[t] * fp[t];
                acc[t] += scale1[d] * (sq * fp[t]);
                cross[t] += scale2[d] * sq;
            }
        }
        fourier_sketch(rep, b, q.data(), k, fq);
        for (std::uint32_t t = 0; t < b; ++t) acc[t] -= 3.0 * cross[t] * fq[t];
        for (int i = 0; i < V; ++i) {
            fourier_sketch(rep, b, W + static_cast<std::size_t>(i) * k, k, fw);
            fourier_sketch(rep, b, &sumwn[static_cast<std::size_t>(i) * k], k, fs);
            for (std::uint32_t t = 0; t < b; ++t) {
                cd w2 = fw[t] * fw[t];
                acc[t] += w2 * (coeff1[i] * fw[t] - 3.0 * fs[t]);
            }
        }
        for (std::uint32_t t = 0; t < b; ++t) acc[t] = acc[t] * inv_docs + m1_coeff * (fq[t] * fq[t] * fq[t]);
        inverse_inplace(acc);
        for (std::uint32_t t = 0; t < b; ++t) rep.data[t] += acc[t];
    }
    if (used_out) *used_out = used;
    if (skipped_out) *skipped_out = skipped;
}

// --- metrics.cpp:8-45 ---------------------------------------------------------------
// recovered: n x r col-major, truth: n x g col-major. out: r rows of (rec, truth, cos, sqdist)
void greedy_match(const double* rec, int r, const double* truth, int g, int n, double* out) {
    if (g < r) throw std::invalid_argument("greedy_match: fewer truth columns than recovered");
    auto col = [n](const double* M, int c) { return M + static_cast<std::size_t>(c) * n; };
    auto dot = [n](const double* a, const double* b) {
        double s = 0;
        for (int i = 0; i < n; ++i) s += a[i] * b[i];
        return s;
    };
    std::vector<double> cosm(static_cast<std::size_t>(r) * g);
    for (int i = 0; i < r; ++i) {
        double ni = std::sqrt(dot(col(rec, i), col(rec, i)));
        for (int j = 0; j < g; ++j) {
            double nj = std::sqrt(dot(col(truth, j), col(truth, j)));
            double denom = std::max(ni * nj, 1e-300);
            cosm[static_cast<std::size_t>(i) * g + j] = std::abs(dot(col(rec, i), col(truth, j))) / denom;
        }
    }
    std::vector<bool> used_r(r, false), used_g(g, false);
    for (int step = 0; step < r; ++step) {
        double best = -1.0;
        int bi = -1, bj = -1;
        for (int i = 0; i < r; ++i) {
            if (used_r[i]) continue;
            for (int j = 0; j < g; ++j) {
                if (used_g[j]) continue;
                double c = cosm[static_cast<std::size_t>(i) * g + j];
                if (c > best) {
                    best = c;
                    bi = i;
                    bj = j;
                }
            }
        }
        used_r[bi] = true;
        used_g[bj] = true;
        double sign = dot(col(rec, bi), col(truth, bj)) >= 0 ? 1.0 : -1.0;
        double d = 0;
        for (int t = 0; t < n; ++t) {
            double diff = col(truth, bj)[t] - sign * col(rec, bi)[t];
            d += diff * diff;
        }
        out[step * 4 + 0] = bi;
        out[step * 4 + 1] = bj;
        out[step * 4 + 2] = best;
        out[step * 4 + 3] = d;
    }
}

thread_local std::string g_err;
thread_local int g_code = 0;

template <typename F>
int guard(F&& f) {
    try {
        f();
        g_code = 0;
        return 0;
    } catch (const DegenerateIterationError& e) {
        g_err = e.what();
        g_code = 3;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        g_code = 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_code = 2;
    }
    return g_code;
}

}  // namespace orc

// =============================== extern "C" API ===============================
// Status codes: 0 ok, 1 invalid_argument, 2 runtime/numerical error, 3 degenerate iteration.
using namespace orc;
extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
int orc_num_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
void orc_set_num_threads(int t) {
#ifdef _OPENMP
    omp_set_num_threads(t);
#else
    (void)t;
#endif
}

std::uint64_t orc_derive_seed(std::uint64_t master, std::uint64_t tag, std::uint64_t i0, std::uint64_t i1) {
    return derive_seed(master, tag, i0, i1);
}
void orc_rng_u64(std::uint64_t seed, int count, std::uint64_t* out) {
    Rng r(seed);
    for (int i = 0; i < count; ++i) out[i] = r.next_u64();
}
void orc_rng_gaussian(std::uint64_t seed, int count, double* out) {
    Rng r(seed);
    for (int i = 0; i < count; ++i) out[i] = r.gaussian();
}
void orc_rng_unit_sphere(std::uint64_t seed, int n, double* out) {
    Rng r(seed);
    auto v = r.unit_sphere(n);
    std::copy(v.begin(), v.end(), out);
}
int orc_polyhash_from_seed(int k, std::uint32_t b, std::uint64_t seed, std::uint64_t* coeffs) {
    return guard([&] {
        auto h = PolyHash::from_seed(k, b, seed);
        std::copy(h.coeffs.begin(), h.coeffs.end(), coeffs);
    });
}
int orc_polyhash_eval(const std::uint64_t* coeffs, int k, std::uint32_t b, const std::uint64_t* idx,
                      int count, std::uint32_t* out) {
    return guard([&] {
        auto h = PolyHash::from_coefficients(std::vector<std::uint64_t>(coeffs, coeffs + k), b);
        for (int i = 0; i < count; ++i) out[i] = h.eval(idx[i]);
    });
}
int orc_symmetric_bucket(const std::uint64_t* coeffs, int k, std::uint32_t b, std::uint64_t i,
                         std::uint64_t j, std::uint64_t kk, std::uint32_t* out) {
    return guard([&] {
        auto h = PolyHash::from_coefficients(std::vector<std::uint64_t>(coeffs, coeffs + k), b);
        *out = symmetric_bucket(h, i, j, kk);
    });
}

// FFT: x is 2b doubles (interleaved re,im), modified in place. dir: -1 forward,
// +1 inverse scaled, +2 inverse unscaled.
int orc_fft(double* x, std::size_t b, int dir) {
    return guard([&] {
        cvec v(b);
        for (std::size_t i = 0; i < b; ++i) v[i] = {x[2 * i], x[2 * i + 1]};
        if (dir == -1)
            forward_inplace(v);
        else if (dir == 1)
            inverse_inplace(v);
        else
            inverse_inplace_unscaled(v);
        for (std::size_t i = 0; i < b; ++i) {
            x[2 * i] = v[i].real();
            x[2 * i + 1] = v[i].imag();
        }
    });
}
int orc_circular_convolve(const double* x, const double* y, std::size_t bx, std::size_t by, double* out) {
    return guard([&] {
        cvec a(bx), c(by);
        for (std::size_t i = 0; i < bx; ++i) a[i] = {x[2 * i], x[2 * i + 1]};
        for (std::size_t i = 0; i < by; ++i) c[i] = {y[2 * i], y[2 * i + 1]};
        cvec z = circular_convolve(a, c);
        for (std::size_t i = 0; i < z.size(); ++i) {
            out[2 * i] = z[i].real();
            out[2 * i + 1] = z[i].imag();
        }
    });
}
std::uint64_t orc_transform_count() { return g_transform_count.load(); }
double orc_median(double* v, int count) {
    std::vector<double> x(v, v + count);
    return median_inplace(x);
}

// ---- symmetric set handle ----
int orc_sym_create(int n, std::uint32_t b, int B, std::uint64_t seed, void** out) {
    return guard([&] { *out = sym_create(n, b, B, seed); });
}
void orc_sym_destroy(void* h) { delete static_cast<SymSet*>(h); }
std::uint64_t orc_sym_version(void* h) { return static_cast<SymSet*>(h)->version; }
int orc_sym_tables(void* h, int m, std::uint32_t* b1, std::uint32_t* b2, std::uint32_t* b3, std::uint8_t* sexp,
                   std::uint64_t* hcoef, std::uint64_t* scoef) {
    return guard([&] {
        auto& s = *static_cast<SymSet*>(h);
        if (m < 0 || m >= s.B) throw std::invalid_argument("replicate index out of range");
        auto& r = s.reps[m];
        std::copy(r.bucket1.begin(), r.bucket1.end(), b1);
        std::copy(r.bucket2.begin(), r.bucket2.end(), b2);
        std::copy(r.bucket3.begin(), r.bucket3.end(), b3);
        std::copy(r.sexp.begin(), r.sexp.end(), sexp);
        std::copy(r.h.coeffs.begin(), r.h.coeffs.end(), hcoef);
        std::copy(r.sigma.coeffs.begin(), r.sigma.coeffs.end(), scoef);
    });
}
int orc_sym_accumulate_dense(void* h, const double* T, int assume_symmetric) {
    return guard([&] { sym_accumulate_dense(*static_cast<SymSet*>(h), T, assume_symmetric != 0); });
}
int orc_sym_accumulate_dense_slice(void* h, const void* T, int f32, int i0, int i1) {
    return guard([&] {
        auto& st = *static_cast<SymSet*>(h);
        if (i0 < 0 || i1 > st.n || i0 > i1) throw std::invalid_argument("accumulate_dense_slice: bad slice");
        if (f32)
            sym_accumulate_dense_slice(st, static_cast<const float*>(T), i0, i1);
        else
            sym_accumulate_dense_slice(st, static_cast<const double*>(T), i0, i1);
    });
}
int orc_gen_planted_slice(int n, int rank, double sigma, std::uint64_t seed, int i0, int i1, int f32, void* out,
                          double* lambda_out, double* V_out) {
    return guard([&] {
        if (n < 1 || rank < 1 || rank > n || i0 < 0 || i1 > n || i0 > i1)
            throw std::invalid_argument("gen_planted_slice: bad arguments");
        gen_planted_slice(n, rank, sigma, seed, i0, i1, f32, out, lambda_out, V_out);
    });
}
int orc_sym_add_scaled_rank1(void* h, const double* u, double alpha) {
    return guard([&] { sym_add_scaled_rank1(*static_cast<SymSet*>(h), u, alpha); });
}
int orc_sym_get_data(void* h, double* out) {  // B x b complex, interleaved
    return guard([&] {
        auto& s = *static_cast<SymSet*>(h);
        for (int m = 0; m < s.B; ++m)
            for (std::uint32_t t = 0; t < s.b; ++t) {
                out[(static_cast<std::size_t>(m) * s.b + t) * 2] = s.reps[m].data[t].real();
                out[(static_cast<std::size_t>(m) * s.b + t) * 2 + 1] = s.reps[m].data[t].imag();
            }
    });
}
int orc_sym_set_data(void* h, const double* in) {  // mutable_replicate: bumps the version
    return guard([&] {
        auto& s = *static_cast<SymSet*>(h);
        for (int m = 0; m < s.B; ++m) {
            ++s.version;
            for (std::uint32_t t = 0; t < s.b; ++t)
                s.reps[m].data[t] = {in[(static_cast<std::size_t>(m) * s.b + t) * 2],
                                     in[(static_cast<std::size_t>(m) * s.b + t) * 2 + 1]};
        }
    });
}
int orc_sym_recover_entry(void* h, int i, int j, int k, double* out) {
    return guard([&] { *out = sym_recover_entry(*static_cast<SymSet*>(h), i, j, k); });
}
int orc_sym_rank1_truncated(void* h, int m, const double* u, double* out) {
    return guard([&] {
        auto& s = *static_cast<SymSet*>(h);
        cvec r = sketch_rank1_sym(s, m, u);
        for (std::uint32_t t = 0; t < s.b; ++t) {
            out[2 * t] = r[t].real();
            out[2 * t + 1] = r[t].imag();
        }
    });
}
int orc_sym_ivv(void* h, const double* u, double* out) {
    return guard([&] {
        auto& s = *static_cast<SymSet*>(h);
        SymWs ws{&s, s.version - 1, {}};
        sym_ivv(ws, u, out);
    });
}
int orc_sym_vvv(void* h, const double* u, double* out) {
    return guard([&] {
        auto& s = *static_cast<SymSet*>(h);
        SymWs ws{&s, s.version - 1, {}};
        *out = sym_vvv(ws, u);
    });
}
// L contractions against one cached spectrum, restarts on the threads (test helpers)
int orc_sym_ivv_batch(void* h, int L, const double* U, double* out) {
    return guard([&] {
        auto& s = *static_cast<SymSet*>(h);
        SymWs ws{&s, s.version - 1, {}};
        sym_ensure_fresh(ws);
#pragma omp parallel for schedule(dynamic, 1)
        for (int l = 0; l < L; ++l) sym_ivv(ws, U + static_cast<std::size_t>(l) * s.n, out + static_cast<std::size_t>(l) * s.n);
    });
}
int orc_sym_vvv_batch(void* h, int L, const double* U, double* out) {
    return guard([&] {
        auto& s = *static_cast<SymSet*>(h);
        SymWs ws{&s, s.version - 1, {}};
        sym_ensure_fresh(ws);
#pragma omp parallel for schedule(dynamic, 1)
        for (int l = 0; l < L; ++l) out[l] = sym_vvv(ws, U + static_cast<std::size_t>(l) * s.n);
    });
}
int orc_sym_cached_transform(void* h, int m, double* out) {
    return guard([&] {
        auto& s = *static_cast<SymSet*>(h);
        cvec f = s.reps[m].data;
        forward_inplace(f);
        for (std::uint32_t t = 0; t < s.b; ++t) {
            out[2 * t] = f[t].real();
            out[2 * t + 1] = f[t].imag();
        }
    });
}
int orc_sym_rtpm(void* h, int k, int L, int T, std::uint64_t seed, double tol, const double* inits,
                 double* lambda, double* V, int* best_taus) {
    return guard([&] { robust_tpm_fast(*static_cast<SymSet*>(h), k, L, T, seed, tol, inits, lambda, V, best_taus); });
}
int orc_lda_recover_params(int V, int k, const double* lambda, const double* A, const double* unwhiten,
                           double alpha0, double* Phi, double* alpha) {
    return guard([&] { lda_recover_params(V, k, lambda, A, unwhiten, alpha0, Phi, alpha); });
}
int orc_lda_heldout_likelihood(int V, int k, const double* Phi, int Vh, long long D, const long long* doc_ptr,
                               const int* word, const int* count, double* ll, long long* floored) {
    return guard([&] { *ll = lda_heldout_likelihood(V, k, Phi, Vh, D, doc_ptr, word, count, floored); });
}
int orc_lda_sketch_whitened_m3(void* h, int V, int D, const long long* doc_ptr, const int* word,
                               const int* count, const double* W, double alpha0, long long* used,
                               long long* skipped) {
    return guard([&] {
        lda_sketch_whitened_m3(*static_cast<SymSet*>(h), V, D, doc_ptr, word, count, W, alpha0, used, skipped);
    });
}

// ---- asymmetric set handle ----
int orc_asym_create(int n, std::uint32_t b, int B, std::uint64_t seed, void** out) {
    return guard([&] { *out = asym_create(n, b, B, seed); });
}
void orc_asym_destroy(void* h) { delete static_cast<AsymSet*>(h); }
int orc_asym_tables(void* h, int m, std::uint32_t* bucket /*3n*/, double* sign /*3n*/, std::uint64_t* hcoef /*3x2*/,
                    std::uint64_t* xcoef /*3x6*/) {
    return guard([&] {
        auto& s = *static_cast<AsymSet*>(h);
        if (m < 0 || m >= s.B) throw std::invalid_argument("replicate index out of range");
        auto& r = s.reps[m];
        for (int sl = 0; sl < 3; ++sl) {
            std::copy(r.bucket[sl].begin(), r.bucket[sl].end(), bucket + static_cast<std::size_t>(sl) * s.n);
            std::copy(r.sign[sl].begin(), r.sign[sl].end(), sign + static_cast<std::size_t>(sl) * s.n);
            std::copy(r.h[sl].coeffs.begin(), r.h[sl].coeffs.end(), hcoef + sl * 2);
            std::copy(r.xi[sl].coeffs.begin(), r.xi[sl].coeffs.end(), xcoef + sl * 6);
        }
    });
}
int orc_asym_accumulate_dense(void* h, const double* T) {
    return guard([&] { asym_accumulate_dense(*static_cast<AsymSet*>(h), T); });
}
int orc_asym_add_rank1(void* h, double alpha, const double* u, const double* v, const double* w) {
    return guard([&] { asym_add_rank1(*static_cast<AsymSet*>(h), alpha, u, v, w); });
}
int orc_asym_accumulate_factored(void* h, int N, const double* a, const double* U, const double* V,
                                 const double* W) {
    return guard([&] { asym_accumulate_factored(*static_cast<AsymSet*>(h), N, a, U, V, W); });
}
int orc_asym_rank1_sketch(void* h, int m, const double* u, const double* v, const double* w, double* out) {
    return guard([&] {
        auto& s = *static_cast<AsymSet*>(h);
        cvec r = asym_rank1_sketch(s, m, u, v, w);
        for (std::uint32_t t = 0; t < s.b; ++t) {
            out[2 * t] = r[t].real();
            out[2 * t + 1] = r[t].imag();
        }
    });
}
int orc_asym_get_data(void* h, double* out) {
    return guard([&] {
        auto& s = *static_cast<AsymSet*>(h);
        for (int m = 0; m < s.B; ++m)
            for (std::uint32_t t = 0; t < s.b; ++t) {
                out[(static_cast<std::size_t>(m) * s.b + t) * 2] = s.reps[m].data[t].real();
                out[(static_cast<std::size_t>(m) * s.b + t) * 2 + 1] = s.reps[m].data[t].imag();
            }
    });
}
int orc_asym_recover_entry(void* h, int i, int j, int k, double* out) {
    return guard([&] { *out = asym_recover_entry(*static_cast<AsymSet*>(h), i, j, k); });
}
int orc_asym_vvv(void* h, const double* u, double* out) {
    return guard([&] {
        auto& s = *static_cast<AsymSet*>(h);
        AsymWs ws{&s, s.version - 1, {}};
        *out = asym_vvv(ws, u);
    });
}
int orc_asym_mode_contraction(void* h, int free_mode, const double* x, const double* y, double* out) {
    return guard([&] {
        auto& s = *static_cast<AsymSet*>(h);
        AsymWs ws{&s, s.version - 1, {}};
        asym_mode_contraction(ws, free_mode, x, y, out);
    });
}

// decompose.cpp:44-51 + 117-205: pinv_spectral and als_fast restated (test oracle).
int orc_pinv_spectral(int k, const double* G, double* P) {
    return guard([&] {
        std::vector<double> ev(k), U(static_cast<std::size_t>(k) * k);
        sym_eigen_jacobi(k, G, ev.data(), U.data());
        double amax = 0.0;
        for (double e : ev) amax = std::max(amax, std::fabs(e));
        const double cutoff = 1e-10 * amax;
        for (int i = 0; i < k; ++i)
            for (int j = 0; j < k; ++j) {
                double s = 0.0;
                for (int q = 0; q < k; ++q)
                    if (std::fabs(ev[q]) > cutoff)
                        s += U[static_cast<std::size_t>(i) * k + q] * (1.0 / ev[q]) * U[static_cast<std::size_t>(j) * k + q];
                P[static_cast<std::size_t>(i) * k + j] = s;
            }
    });
}
int orc_asym_als(void* h, int k, int max_iters, double tol, std::uint64_t seed, double* lambda_out, double* A_out,
                 double* B_out, double* C_out, int* iters_out) {
    return guard([&] {
        auto& s = *static_cast<AsymSet*>(h);
        const int n = s.n;
        if (k < 1 || max_iters < 1) throw std::invalid_argument("als: k and max_iters must be positive");
        if (k > n) throw std::invalid_argument("als: target rank exceeds tensor dimension");
        // factors column-major n x k
        std::vector<double> F[3];
        for (auto& f : F) f.assign(static_cast<std::size_t>(n) * k, 0.0);
        for (int r = 0; r < k; ++r) {
            Rng rng(derive_seed(seed, kAlsInit, r));
            for (int f = 0; f < 3; ++f) {
                auto v = rng.unit_sphere(n);
                std::copy(v.begin(), v.end(), F[f].begin() + static_cast<std::size_t>(r) * n);
            }
        }
        AsymWs ws{&s, s.version - 1, {}};
        std::vector<double> lambda(k, 1.0), lambda_prev(k, 1.0), M(static_cast<std::size_t>(n) * k), P(static_cast<std::size_t>(k) * k);
        int it = 0;
        for (; it < max_iters;) {
            for (int mode = 0; mode < 3; ++mode) {
                const int f1 = mode == 0 ? 1 : 0, f2 = mode == 2 ? 1 : 2;
                for (int r = 0; r < k; ++r)
                    asym_mode_contraction(ws, mode, F[f1].data() + static_cast<std::size_t>(r) * n,
                                          F[f2].data() + static_cast<std::size_t>(r) * n, M.data() + static_cast<std::size_t>(r) * n);
                std::vector<double> G(static_cast<std::size_t>(k) * k);
                for (int a = 0; a < k; ++a)
                    for (int b = 0; b < k; ++b) {
                        double g1 = 0.0, g2 = 0.0;
                        for (int i = 0; i < n; ++i) {
                            g1 += F[f1][static_cast<std::size_t>(a) * n + i] * F[f1][static_cast<std::size_t>(b) * n + i];
                            g2 += F[f2][static_cast<std::size_t>(a) * n + i] * F[f2][static_cast<std::size_t>(b) * n + i];
                        }
                        G[static_cast<std::size_t>(a) * k + b] = g1 * g2;
                    }
                if (orc_pinv_spectral(k, G.data(), P.data()) != 0) throw std::runtime_error(g_err);
                std::vector<double> prev = F[mode];
                for (int r = 0; r < k; ++r) {
                    double nrm2 = 0.0;
                    for (int i = 0; i < n; ++i) {
                        double v = 0.0;
                        for (int q = 0; q < k; ++q) v += M[static_cast<std::size_t>(q) * n + i] * P[static_cast<std::size_t>(q) * k + r];
                        F[mode][static_cast<std::size_t>(r) * n + i] = v;
                        nrm2 += v * v;
                    }
                    const double nrm = std::sqrt(nrm2);
                    lambda[r] = nrm;
                    for (int i = 0; i < n; ++i) {
                        double& x = F[mode][static_cast<std::size_t>(r) * n + i];
                        x = nrm > 0 ? x / nrm : prev[static_cast<std::size_t>(r) * n + i];
                    }
                }
            }
            ++it;
            double dn = 0.0, pn = 0.0;
            for (int r = 0; r < k; ++r) {
                dn += (lambda[r] - lambda_prev[r]) * (lambda[r] - lambda_prev[r]);
                pn += lambda_prev[r] * lambda_prev[r];
            }
            if (std::sqrt(dn) / std::max(std::sqrt(pn), 1e-300) < tol) break;
            lambda_prev = lambda;
        }
        std::copy(lambda.begin(), lambda.end(), lambda_out);
        std::copy(F[0].begin(), F[0].end(), A_out);
        std::copy(F[1].begin(), F[1].end(), B_out);
        std::copy(F[2].begin(), F[2].end(), C_out);
        if (iters_out) *iters_out = it;
    });
}

// ---- exact contractions (accuracy oracle) and metrics ----
double orc_contract_vvv_exact(const double* T, int n, const double* u) { return contract_vvv_exact(T, n, u); }
void orc_contract_Ivv_exact(const double* T, int n, const double* u, const double* v, double* out) {
    contract_Ivv_exact(T, n, u, v, out);
}
int orc_first_asymmetric_triple(const double* T, int n, double tol, int* out) {
    return first_asymmetric_triple(T, n, tol, out) ? 1 : 0;
}
int orc_greedy_match(const double* rec, int r, const double* truth, int g, int n, double* out) {
    return guard([&] { greedy_match(rec, r, truth, g, n, out); });
}

int orc_lda_compute_m1(int V, int D, const long long* doc_ptr, const int* word, const int* count, double* m1) {
    return guard([&] { lda_compute_m1(V, D, doc_ptr, word, count, m1); });
}
int orc_lda_compute_m2(int V, int D, const long long* doc_ptr, const int* word, const int* count, double alpha0,
                       double* m2) {
    return guard([&] { lda_compute_m2(V, D, doc_ptr, word, count, alpha0, m2); });
}
int orc_sym_eigen(int n, const double* A, double* evals, double* evecs) {
    return guard([&] { sym_eigen_jacobi(n, A, evals, evecs); });
}
int orc_lda_whiten(int V, const double* m2, int k, double* W, double* unwhiten, double* sv) {
    return guard([&] { lda_whiten(V, m2, k, W, unwhiten, sv); });
}

}  // extern "C"
