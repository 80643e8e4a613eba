// CPU emulation of the CTA-local FFT passes in skc_fft.cuh: each pass is run for
// every work item in turn (items of one pass touch disjoint elements), and the
// result is checked against a direct O(N^2) DFT. Exit code 0 = pass.
#include <complex>
#include <cstdio>
#include <random>
#include <vector>
#include "../../paper_1506_04448_b200/csrc/skc_fft.cuh"
using namespace skc;
int main() {
    int fails = 0;
    std::mt19937_64 rng(5);
    std::normal_distribution<double> nd;
    for (int logb : {1, 2, 3, 4, 5, 7, 8, 11, 12, 13}) {
        const int b = 1 << logb;
        std::vector<double2> tw(b);
        for (int k = 0; k < b; ++k) {
            long double a = 2.0L * 3.14159265358979323846264338327950288L * k / b;
            tw[k] = mk((double)cosl(a), (double)sinl(a));
        }
        for (int logN : {logb, logb > 3 ? logb - 2 : logb}) {
            const int N = 1 << logN;
            const int S = b / N;
            std::vector<std::complex<double>> x(b);
            for (auto& z : x) z = {nd(rng), nd(rng)};
            // reference full DFT
            std::vector<std::complex<double>> F(b);
            for (int f = 0; f < b; ++f) {
                std::complex<long double> s = 0;
                for (int t = 0; t < b; ++t) {
                    long double a = -2.0L * 3.14159265358979323846264338327950288L * ((long long)f * t % b) / b;
                    s += std::complex<long double>(x[t].real(), x[t].imag()) * std::complex<long double>(cosl(a), sinl(a));
                }
                F[f] = {(double)s.real(), (double)s.imag()};
            }
            PassPlan pl = make_plan(N);
            // local table w_N^k as used by the templated device drivers (index with logN)
            std::vector<double2> twl(N);
            for (int k = 0; k < N; ++k) twl[k] = tw[static_cast<size_t>(k) * S];
            const bool use_local = (logN % 2) == 1 || N == b;  // exercise both indexings
            double maxerr = 0, maxinv = 0;
            std::vector<std::complex<double>> back(b, 0.0);
            for (int r = 0; r < S; ++r) {
                std::vector<double2> sm(padded_len(N), mk(0, 0));
                for (int t = 0; t < b; ++t) {
                    double2 w = conj(tw[((long long)r * t) % b]);
                    double2 v = cmul(mk(x[t].real(), x[t].imag()), w);
                    int tp = t % N;
                    sm[pad16(tp)] = cadd(sm[pad16(tp)], v);
                }
                for (int p = 0; p < pl.npass; ++p) {
                    int items = N >> pl.logr[p];
                    for (int w = 0; w < items; ++w)
                        dif_pass_dispatch(pl.logr[p], sm.data(), w, pl.h[p], use_local ? twl.data() : tw.data(),
                                          use_local ? logN : logb);
                }
                for (int j = 0; j < N; ++j) {
                    int f = r + S * (int)bitrev(j, logN);
                    double2 got = sm[pad16(j)];
                    maxerr = std::max(maxerr, std::abs(std::complex<double>(got.x, got.y) - F[f]) / std::sqrt((double)b));
                }
                for (int p = pl.npass - 1; p >= 0; --p) {
                    int items = N >> pl.logr[p];
                    for (int w = 0; w < items; ++w)
                        dit_pass_dispatch(pl.logr[p], sm.data(), w, pl.h[p], use_local ? twl.data() : tw.data(),
                                          use_local ? logN : logb);
                }
                for (int t = 0; t < b; ++t) {
                    double2 v = cmul(sm[pad16(t % N)], tw[((long long)r * t) % b]);
                    back[t] += std::complex<double>(v.x, v.y);
                }
            }
            for (int t = 0; t < b; ++t) maxinv = std::max(maxinv, std::abs(back[t] / (double)b - x[t]));
            bool ok = maxerr < 1e-13 && maxinv < 1e-13;
            if (!ok) ++fails;
            if (plan_npass(logN) != pl.npass) { ++fails; std::printf("constexpr plan mismatch\n"); }
            for (int p = 0; p < pl.npass; ++p)
                if (plan_logr(logN, p) != pl.logr[p] || plan_h(logN, p) != pl.h[p]) { ++fails; std::printf("plan mismatch\n"); }
            std::printf("b=%6d N=%6d S=%3d passes=%d fwd_err=%.2e inv_err=%.2e %s\n", b, N, S, pl.npass, maxerr, maxinv, ok ? "ok" : "FAIL");
        }
    }
    return fails ? 1 : 0;
}
