// C entry points over the reference's own classes (proj/include/sketchcp, compiled
// verbatim from /root/reference/proj/src into oracle/_ref by oracle/Makefile's `ref`
// target). Test infrastructure: tests/test_ref_pins.py runs the same inputs through this
// library and through the oracle restatement (oracle/sketchcp_oracle.cpp) to pin the
// oracle to the reference itself. Never linked into the product.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "sketchcp/contraction.hpp"
#include "sketchcp/decompose.hpp"
#include "sketchcp/fft.hpp"
#include "sketchcp/hashing.hpp"
#include "sketchcp/rng.hpp"
#include "sketchcp/sketch.hpp"
#include "sketchcp/tensor.hpp"

using namespace sketchcp;

namespace {
thread_local std::string g_err;
template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
Eigen::VectorXd vec(const double* u, int n) {
    Eigen::VectorXd v(n);
    for (int i = 0; i < n; ++i) v[i] = u[i];
    return v;
}
DenseTensor3 dense(const double* T, int n) {
    DenseTensor3 D(n);
    std::memcpy(D.entries.data(), T, sizeof(double) * static_cast<std::size_t>(n) * n * n);
    return D;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint64_t ref_derive_seed(std::uint64_t master, std::uint64_t tag, std::uint64_t i0, std::uint64_t i1) {
    return derive_seed(master, tag, i0, i1);
}
int ref_unit_sphere(std::uint64_t seed, int n, double* out) {
    return guard([&] {
        Rng r(seed);
        Eigen::VectorXd v = r.unit_sphere(n);
        for (int i = 0; i < n; ++i) out[i] = v[i];
    });
}
int ref_fft(double* x, std::size_t b, int dir) {
    return guard([&] {
        cvec v(b);
        for (std::size_t t = 0; t < b; ++t) v[t] = {x[2 * t], x[2 * t + 1]};
        if (dir < 0) fft::forward_inplace(v);
        else fft::inverse_inplace(v);
        for (std::size_t t = 0; t < b; ++t) {
            x[2 * t] = v[t].real();
            x[2 * t + 1] = v[t].imag();
        }
    });
}

// ---- SymTensorSketchSet / SymContractionWorkspace / robust_tpm_fast ----
int ref_sym_create(int n, std::uint32_t b, int B, std::uint64_t seed, void** out) {
    return guard([&] { *out = new SymTensorSketchSet(n, b, B, seed); });
}
void ref_sym_destroy(void* h) { delete static_cast<SymTensorSketchSet*>(h); }
int ref_sym_tables(void* h, int m, std::uint32_t* b1, std::uint32_t* b2, std::uint32_t* b3, std::uint8_t* sexp) {
    return guard([&] {
        const auto& r = static_cast<SymTensorSketchSet*>(h)->replicate(m);
        std::copy(r.bucket1.begin(), r.bucket1.end(), b1);
        std::copy(r.bucket2.begin(), r.bucket2.end(), b2);
        std::copy(r.bucket3.begin(), r.bucket3.end(), b3);
        std::copy(r.sexp.begin(), r.sexp.end(), sexp);
    });
}
int ref_sym_accumulate_dense(void* h, const double* T, int assume_symmetric) {
    return guard([&] {
        auto& s = *static_cast<SymTensorSketchSet*>(h);
        s.accumulate_dense(dense(T, s.n()), assume_symmetric != 0);
    });
}
int ref_sym_add_scaled_rank1(void* h, const double* u, double alpha) {
    return guard([&] {
        auto& s = *static_cast<SymTensorSketchSet*>(h);
        s.add_scaled_rank1(vec(u, s.n()), alpha);
    });
}
int ref_sym_get_data(void* h, double* out) {
    return guard([&] {
        const auto& s = *static_cast<SymTensorSketchSet*>(h);
        for (int m = 0; m < s.replicates(); ++m)
            for (std::uint32_t t = 0; t < s.b(); ++t) {
                out[(static_cast<std::size_t>(m) * s.b() + t) * 2] = s.replicate(m).data[t].real();
                out[(static_cast<std::size_t>(m) * s.b() + t) * 2 + 1] = s.replicate(m).data[t].imag();
            }
    });
}
int ref_sym_set_data(void* h, const double* in) {
    return guard([&] {
        auto& s = *static_cast<SymTensorSketchSet*>(h);
        for (int m = 0; m < s.replicates(); ++m) {
            auto& d = s.mutable_replicate(m).data;
            for (std::uint32_t t = 0; t < s.b(); ++t)
                d[t] = {in[(static_cast<std::size_t>(m) * s.b() + t) * 2],
                        in[(static_cast<std::size_t>(m) * s.b() + t) * 2 + 1]};
        }
    });
}
int ref_sym_recover_entry(void* h, int i, int j, int k, double* out) {
    return guard([&] { *out = static_cast<SymTensorSketchSet*>(h)->recover_entry(i, j, k); });
}
int ref_sym_ivv(void* h, const double* u, double* out) {
    return guard([&] {
        auto& s = *static_cast<SymTensorSketchSet*>(h);
        SymContractionWorkspace ws(s);
        Eigen::VectorXd r = ws.Ivv(vec(u, s.n()));
        for (int i = 0; i < s.n(); ++i) out[i] = r[i];
    });
}
int ref_sym_vvv(void* h, const double* u, double* out) {
    return guard([&] {
        auto& s = *static_cast<SymTensorSketchSet*>(h);
        SymContractionWorkspace ws(s);
        *out = ws.vvv(vec(u, s.n()));
    });
}
int ref_sym_rtpm(void* h, int k, int L, int T_iters, std::uint64_t seed, double tol, double* lambda, double* V) {
    return guard([&] {
        auto& s = *static_cast<SymTensorSketchSet*>(h);
        PowerConfig cfg;
        cfg.k = k;
        cfg.L = L;
        cfg.T_iters = T_iters;
        cfg.b = s.b();
        cfg.B = s.replicates();
        cfg.seed = seed;
        cfg.tol = tol;
        CpDecomposition d = robust_tpm_fast(s, cfg);
        for (int c = 0; c < k; ++c) {
            lambda[c] = d.lambda[c];
            for (int i = 0; i < s.n(); ++i) V[static_cast<std::size_t>(c) * s.n() + i] = d.A(i, c);
        }
    });
}

// ---- AsymTensorSketchSet / AsymContractionWorkspace ----
int ref_asym_create(int n, std::uint32_t b, int B, std::uint64_t seed, void** out) {
    return guard([&] { *out = new AsymTensorSketchSet(n, b, B, seed); });
}
void ref_asym_destroy(void* h) { delete static_cast<AsymTensorSketchSet*>(h); }
int ref_asym_accumulate_dense(void* h, const double* T) {
    return guard([&] {
        auto& s = *static_cast<AsymTensorSketchSet*>(h);
        s.accumulate_dense(dense(T, s.n()));
    });
}
int ref_asym_get_data(void* h, double* out) {
    return guard([&] {
        const auto& s = *static_cast<AsymTensorSketchSet*>(h);
        for (int m = 0; m < s.replicates(); ++m)
            for (std::uint32_t t = 0; t < s.b(); ++t) {
                out[(static_cast<std::size_t>(m) * s.b() + t) * 2] = s.replicate(m).data[t].real();
                out[(static_cast<std::size_t>(m) * s.b() + t) * 2 + 1] = s.replicate(m).data[t].imag();
            }
    });
}
int ref_asym_vvv(void* h, const double* u, double* out) {
    return guard([&] {
        auto& s = *static_cast<AsymTensorSketchSet*>(h);
        AsymContractionWorkspace ws(s);
        *out = ws.vvv(vec(u, s.n()));
    });
}
int ref_asym_mode_contraction(void* h, int free_mode, const double* x, const double* y, double* out) {
    return guard([&] {
        auto& s = *static_cast<AsymTensorSketchSet*>(h);
        AsymContractionWorkspace ws(s);
        Eigen::VectorXd r = ws.mode_contraction(free_mode, vec(x, s.n()), vec(y, s.n()));
        for (int i = 0; i < s.n(); ++i) out[i] = r[i];
    });
}

}  // extern "C"
