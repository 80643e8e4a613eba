// Host dense linear algebra shared by whitening, recovery and ALS: symmetric
// eigensolvers, simplex projection and the spectral pseudoinverse.
#include "skc_abi_impl.hpp"

namespace skcabi {

// Householder tridiagonalisation + implicit shifted QL (O(p^3); the textbook method),
// symmetric row-major input; vecs[i*n + c] = component i of the eigenvector of vals[c]
// (ascending). Returns false if an eigenvalue fails to converge.
bool sym_eigen_ql_rowmajor(int n, std::vector<double> a, std::vector<double>& vals, std::vector<double>& vecs) {
    auto A = [&](int i, int j) -> double& { return a[(size_t)i * n + j]; };
    std::vector<double> d(n), e(n);
    for (int i = n - 1; i > 0; --i) {
        const int l = i - 1;
        double h = 0.0, scale = 0.0;
        if (l > 0) {
            for (int k = 0; k <= l; ++k) scale += std::fabs(A(i, k));
            if (scale == 0.0) {
                e[i] = A(i, l);
            } else {
                for (int k = 0; k <= l; ++k) {
                    A(i, k) /= scale;
                    h += A(i, k) * A(i, k);
                }
                double f = A(i, l);
                double g = (f >= 0.0) ? -std::sqrt(h) : std::sqrt(h);
                e[i] = scale * g;
                h -= f * g;
                A(i, l) = f - g;
                f = 0.0;
                for (int j = 0; j <= l; ++j) {
                    A(j, i) = A(i, j) / h;
                    g = 0.0;
                    for (int k = 0; k <= j; ++k) g += A(j, k) * A(i, k);
                    for (int k = j + 1; k <= l; ++k) g += A(k, j) * A(i, k);
                    e[j] = g / h;
                    f += e[j] * A(i, j);
                }
                const double hh = f / (h + h);
                for (int j = 0; j <= l; ++j) {
                    f = A(i, j);
                    e[j] = g = e[j] - hh * f;
                    for (int k = 0; k <= j; ++k) A(j, k) -= (f * e[k] + g * A(i, k));
                }
            }
        } else {
            e[i] = A(i, l);
        }
        d[i] = h;
    }
    d[0] = 0.0;
    e[0] = 0.0;
    for (int i = 0; i < n; ++i) {
        const int l = i - 1;
        if (d[i] != 0.0) {
            for (int j = 0; j <= l; ++j) {
                double g = 0.0;
                for (int k = 0; k <= l; ++k) g += A(i, k) * A(k, j);
                for (int k = 0; k <= l; ++k) A(k, j) -= g * A(k, i);
            }
        }
        d[i] = A(i, i);
        A(i, i) = 1.0;
        for (int j = 0; j <= l; ++j) A(j, i) = A(i, j) = 0.0;
    }
    // implicit QL on (d, e) accumulating into A (columns = eigenvectors)
    for (int i = 1; i < n; ++i) e[i - 1] = e[i];
    e[n - 1] = 0.0;
    for (int l = 0; l < n; ++l) {
        int iter = 0, m;
        do {
            for (m = l; m < n - 1; ++m) {
                const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
                if (std::fabs(e[m]) <= 1e-16 * dd) break;
            }
            if (m != l) {
                if (iter++ == 100) return false;
                double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
                double r = std::hypot(g, 1.0);
                g = d[m] - d[l] + e[l] / (g + (g >= 0.0 ? std::fabs(r) : -std::fabs(r)));
                double s = 1.0, c = 1.0, p = 0.0;
                int i;
                for (i = m - 1; i >= l; --i) {
                    double f = s * e[i];
                    const double b = c * e[i];
                    e[i + 1] = (r = std::hypot(f, g));
                    if (r == 0.0) {
                        d[i + 1] -= p;
                        e[m] = 0.0;
                        break;
                    }
                    s = f / r;
                    c = g / r;
                    g = d[i + 1] - p;
                    r = (d[i] - g) * s + 2.0 * c * b;
                    d[i + 1] = g + (p = s * r);
                    g = c * r - b;
                    for (int k = 0; k < n; ++k) {
                        f = A(k, i + 1);
                        A(k, i + 1) = s * A(k, i) + c * f;
                        A(k, i) = c * A(k, i) - s * f;
                    }
                }
                if (r == 0.0 && i >= l) continue;
                d[l] -= p;
                e[l] = g;
                e[m] = 0.0;
            }
        } while (m != l);
    }
    std::vector<int> ord(n);
    for (int i = 0; i < n; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return d[x] < d[y]; });
    vals.resize(n);
    vecs.assign((size_t)n * n, 0.0);
    for (int c = 0; c < n; ++c) {
        vals[c] = d[ord[c]];
        for (int i = 0; i < n; ++i) vecs[(size_t)i * n + c] = A(i, ord[c]);
    }
    return true;
}

// Symmetric eigensolver used by the host-side small problems (col-major output like
// jacobi_eigen): tridiagonal QL, with the Jacobi sweep as fallback.
void jacobi_eigen(int p, std::vector<double> a, std::vector<double>& vals, std::vector<double>& vecs);
void sym_eigen_host(int p, const std::vector<double>& a, std::vector<double>& vals, std::vector<double>& vecs) {
    std::vector<double> rm;
    if (sym_eigen_ql_rowmajor(p, a, vals, rm)) {  // symmetric: row-major == col-major input
        vecs.assign(static_cast<size_t>(p) * p, 0.0);
        for (int c = 0; c < p; ++c)
            for (int i = 0; i < p; ++i) vecs[static_cast<size_t>(c) * p + i] = rm[static_cast<size_t>(i) * p + c];
        return;
    }
    jacobi_eigen(p, a, vals, vecs);
}

// Cyclic Jacobi for a small symmetric matrix (col-major p x p): ascending eigenvalues,
// column c of vecs the eigenvector of vals[c].
void jacobi_eigen(int p, std::vector<double> a, std::vector<double>& vals, std::vector<double>& vecs) {
    vecs.assign(static_cast<size_t>(p) * p, 0.0);
    for (int i = 0; i < p; ++i) vecs[static_cast<size_t>(i) * p + i] = 1.0;
    auto A = [&](int i, int j) -> double& { return a[static_cast<size_t>(j) * p + i]; };
    auto Vv = [&](int i, int j) -> double& { return vecs[static_cast<size_t>(j) * p + i]; };
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0, tot = 0.0;
        for (int j = 0; j < p; ++j)
            for (int i = 0; i < p; ++i) {
                tot += A(i, j) * A(i, j);
                if (i != j) off += A(i, j) * A(i, j);
            }
        if (off <= 1e-30 * tot) break;
        for (int P = 0; P < p - 1; ++P)
            for (int Q = P + 1; Q < p; ++Q) {
                const double apq = A(P, Q);
                if (apq == 0.0) continue;
                const double theta = (A(Q, Q) - A(P, P)) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double cs = 1.0 / std::sqrt(t * t + 1.0), sn = t * cs;
                for (int k = 0; k < p; ++k) {
                    const double akp = A(k, P), akq = A(k, Q);
                    A(k, P) = cs * akp - sn * akq;
                    A(k, Q) = sn * akp + cs * akq;
                }
                for (int k = 0; k < p; ++k) {
                    const double apk = A(P, k), aqk = A(Q, k);
                    A(P, k) = cs * apk - sn * aqk;
                    A(Q, k) = sn * apk + cs * aqk;
                }
                for (int k = 0; k < p; ++k) {
                    const double vkp = Vv(k, P), vkq = Vv(k, Q);
                    Vv(k, P) = cs * vkp - sn * vkq;
                    Vv(k, Q) = sn * vkp + cs * vkq;
                }
            }
    }
    std::vector<int> ord(p);
    for (int i = 0; i < p; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return A(x, x) < A(y, y); });
    std::vector<double> sorted(static_cast<size_t>(p) * p);
    vals.resize(p);
    for (int c = 0; c < p; ++c) {
        vals[c] = A(ord[c], ord[c]);
        for (int i = 0; i < p; ++i) sorted[static_cast<size_t>(c) * p + i] = Vv(i, ord[c]);
    }
    vecs.swap(sorted);
}

// lda.cpp:250-271: Euclidean projection onto the probability simplex (sort-based)
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
    if (rho == 0) {  // all mass collapsed: uniform (lda.cpp:262-265)
        std::fill(x.begin(), x.end(), 1.0 / n);
        return x;
    }
    for (int i = 0; i < n; ++i) x[i] = std::max(y[i] - theta, 0.0);
    return x;
}

// decompose.cpp:44-51 pinv_spectral: symmetric pseudoinverse with spectral truncation at
// 1e-10 of the largest |eigenvalue|. G is symmetric PSD here (Hadamard product of Grams):
// when its Cholesky pivots show it is well conditioned the pseudoinverse is the inverse,
// computed by Cholesky; otherwise the eigen-decomposition route (Jacobi) truncates.
std::vector<double> pinv_spectral_host(int k, const std::vector<double>& G /* col-major */) {
    std::vector<double> L(static_cast<size_t>(k) * k, 0.0);
    bool ok = true;
    double gmax = 0.0;
    for (int i = 0; i < k; ++i) gmax = std::max(gmax, std::fabs(G[static_cast<size_t>(i) * k + i]));
    for (int j = 0; j < k && ok; ++j) {
        double s = G[static_cast<size_t>(j) * k + j];
        for (int q = 0; q < j; ++q) s -= L[static_cast<size_t>(q) * k + j] * L[static_cast<size_t>(q) * k + j];
        if (!(s > 1e-8 * gmax)) {  // margin above the 1e-10 spectral cutoff
            ok = false;
            break;
        }
        L[static_cast<size_t>(j) * k + j] = std::sqrt(s);
        for (int i = j + 1; i < k; ++i) {
            double t = G[static_cast<size_t>(j) * k + i];
            for (int q = 0; q < j; ++q) t -= L[static_cast<size_t>(q) * k + i] * L[static_cast<size_t>(q) * k + j];
            L[static_cast<size_t>(j) * k + i] = t / L[static_cast<size_t>(j) * k + j];
        }
    }
    std::vector<double> P(static_cast<size_t>(k) * k, 0.0);
    if (ok) {
        // columns of G^{-1}: solve L L^T x = e_c
        std::vector<double> y(k);
        for (int c = 0; c < k; ++c) {
            for (int i = 0; i < k; ++i) {
                double s = (i == c) ? 1.0 : 0.0;
                for (int q = 0; q < i; ++q) s -= L[static_cast<size_t>(q) * k + i] * y[q];
                y[i] = s / L[static_cast<size_t>(i) * k + i];
            }
            for (int i = k - 1; i >= 0; --i) {
                double s = y[i];
                for (int q = i + 1; q < k; ++q) s -= L[static_cast<size_t>(i) * k + q] * P[static_cast<size_t>(c) * k + q];
                P[static_cast<size_t>(c) * k + i] = s / L[static_cast<size_t>(i) * k + i];
            }
        }
        return P;
    }
    std::vector<double> ev, U;
    sym_eigen_host(k, G, ev, U);
    double amax = 0.0;
    for (double e : ev) amax = std::max(amax, std::fabs(e));
    const double cutoff = 1e-10 * amax;
    for (int q = 0; q < k; ++q) {
        const double e = ev[q];
        if (!(std::fabs(e) > cutoff)) continue;
        const double inv = 1.0 / e;
        for (int j = 0; j < k; ++j)
            for (int i = 0; i < k; ++i)
                P[static_cast<size_t>(j) * k + i] += U[static_cast<size_t>(q) * k + i] * inv * U[static_cast<size_t>(q) * k + j];
    }
    return P;
}

}  // namespace skcabi
