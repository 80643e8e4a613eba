// FFTW3 stand-in (see fftw3.h): iterative radix-2 DIT over a long-double twiddle table.
// Test infrastructure for oracle/_ref only.
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstdlib>
#include <vector>

struct fftw_plan_s {
    int n, sign;
    std::vector<std::complex<double>> tw;  // e^{sign 2 pi i k / n}, k < n/2
    std::vector<int> rev;
};

fftw_complex* fftw_alloc_complex(unsigned long n) {
    return static_cast<fftw_complex*>(std::aligned_alloc(64, ((n * sizeof(fftw_complex)) + 63) / 64 * 64));
}
void fftw_free(void* p) { std::free(p); }

fftw_plan fftw_plan_dft_1d(int n, fftw_complex*, fftw_complex*, int sign, unsigned) {
    auto* p = new fftw_plan_s;
    p->n = n;
    p->sign = sign;
    const long double two_pi = 6.283185307179586476925286766559005768L;
    p->tw.resize(static_cast<std::size_t>(n / 2 > 0 ? n / 2 : 1));
    for (int k = 0; k < n / 2; ++k) {
        const long double a = two_pi * static_cast<long double>(k) / static_cast<long double>(n);
        p->tw[k] = {static_cast<double>(cosl(a)), static_cast<double>(sign * sinl(a))};
    }
    int lg = 0;
    while ((1 << lg) < n) ++lg;
    p->rev.resize(n);
    for (int i = 0; i < n; ++i) {
        int r = 0;
        for (int b = 0; b < lg; ++b)
            if (i & (1 << b)) r |= 1 << (lg - 1 - b);
        p->rev[i] = r;
    }
    return p;
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    const int n = p->n;
    auto* x = reinterpret_cast<std::complex<double>*>(out);
    auto* xi = reinterpret_cast<std::complex<double>*>(in);
    if (x != xi)
        for (int i = 0; i < n; ++i) x[i] = xi[i];
    for (int i = 0; i < n; ++i)
        if (i < p->rev[i]) std::swap(x[i], x[p->rev[i]]);
    for (int len = 2; len <= n; len <<= 1) {
        const int half = len / 2, step = n / len;
        for (int s = 0; s < n; s += len)
            for (int k = 0; k < half; ++k) {
                const std::complex<double> w = p->tw[static_cast<std::size_t>(k) * step];
                const std::complex<double> a = x[s + k], b = x[s + k + half] * w;
                x[s + k] = a + b;
                x[s + k + half] = a - b;
            }
    }
}

void fftw_destroy_plan(fftw_plan p) { delete p; }
