// Asymmetric sketch sets (sketch.hpp SketchSet), their mode contractions and the fast
// sketched ALS (decompose.cpp:117-205) over the C-ABI.
#include "skc_abi_impl.hpp"

namespace skcabi {

void init_asym_device(skc_asym_set* s, const double* data_host) {
    skc_context* ctx = s->ctx;
    ctx->use();
    const cudaStream_t st = ctx->stream;
    const size_t B3n = static_cast<size_t>(s->B) * 3 * s->n;
    s->d_hcoef.upload(s->hcoef.data(), s->hcoef.size(), st);
    s->d_xcoef.upload(s->xcoef.data(), s->xcoef.size(), st);
    s->bucket.alloc(B3n);
    s->packed.alloc(B3n);
    s->sign.alloc(B3n);
    s->perm.alloc(B3n);
    launch_asym_tables(st, s->d_hcoef.p, s->d_xcoef.p, s->n, s->b, s->B, s->bucket.p, s->sign.p, s->packed.p);
    ctx->check_launch();
    s->N = local_length(s->b);
    s->logN = ilog2(static_cast<unsigned>(s->N));
    s->S = static_cast<int>(s->b / static_cast<std::uint32_t>(s->N));
    s->logb = ilog2(s->b);
    launch_sort_perm(st, s->bucket.p, s->B * 3, s->n, static_cast<std::uint32_t>(s->N - 1), s->perm.p);
    s->plan.alloc(B3n);
    launch_make_plan(st, s->perm.p, s->bucket.p, nullptr, 0, s->packed.p, s->B * 3, s->n, s->plan.p);
    ctx->check_launch();
    const size_t Bb = static_cast<size_t>(s->B) * s->b;
    s->data.alloc(Bb);
    s->spec.alloc(Bb);
    if (data_host)
        CK(cudaMemcpyAsync(s->data.p, data_host, Bb * sizeof(double2), cudaMemcpyHostToDevice, st));
    else
        CK(cudaMemsetAsync(s->data.p, 0, Bb * sizeof(double2), st));
    ctx->tw(s->b);
    ctx->sync();
}

}  // namespace skcabi

extern "C" {

// ---- asymmetric set ----
int skc_asym_create(skc_context* ctx, int n, uint32_t b, int B, uint64_t master_seed, skc_asym_set** out) {
    return guard([&] {
        check_vec(ctx, "context");
        validate_set_args(n, b, B);
        auto s = std::make_unique<skc_asym_set>();
        s->ctx = ctx;
        s->n = n;
        s->b = b;
        s->B = B;
        s->seed = master_seed;
        s->hcoef.resize(static_cast<size_t>(B) * 3 * 2);
        s->xcoef.resize(static_cast<size_t>(B) * 3 * 6);
        for (int m = 0; m < B; ++m)  // sketch.cpp:161-167
            for (int sl = 0; sl < 3; ++sl) {
                poly_coefficients(2, derive_seed(master_seed, seed_tag::kAsymBucketHash, m, sl),
                                  &s->hcoef[(m * 3 + sl) * 2]);
                poly_coefficients(6, derive_seed(master_seed, seed_tag::kAsymSign, m, sl), &s->xcoef[(m * 3 + sl) * 6]);
            }
        init_asym_device(s.get(), nullptr);
        *out = s.release();
    });
}
int skc_asym_create_from_coefficients(skc_context* ctx, int n, uint32_t b, int B, uint64_t master_seed,
                                      const uint64_t* hcoef, const uint64_t* xcoef, const double* data_host,
                                      skc_asym_set** out) {
    return guard([&] {
        check_vec(ctx, "context");
        validate_set_args(n, b, B);
        check_vec(hcoef, "hcoef");
        check_vec(xcoef, "xcoef");
        for (int x = 0; x < B * 6; ++x) require(hcoef[x] < kHashPrime, "PolyHash: coefficient out of range");
        for (int x = 0; x < B * 18; ++x) require(xcoef[x] < kHashPrime, "PolyHash: coefficient out of range");
        auto s = std::make_unique<skc_asym_set>();
        s->ctx = ctx;
        s->n = n;
        s->b = b;
        s->B = B;
        s->seed = master_seed;
        s->hcoef.assign(hcoef, hcoef + static_cast<size_t>(B) * 6);
        s->xcoef.assign(xcoef, xcoef + static_cast<size_t>(B) * 18);
        init_asym_device(s.get(), data_host);
        *out = s.release();
    });
}
int skc_asym_destroy(skc_asym_set* s) {
    return guard([&] {
        if (!s) return;
        s->ctx->use();
        s->ctx->sync();
        delete s;
    });
}
int skc_asym_info(const skc_asym_set* s, int* n, uint32_t* b, int* B, uint64_t* seed, uint64_t* version) {
    return guard([&] {
        check_vec(s, "set");
        if (n) *n = s->n;
        if (b) *b = s->b;
        if (B) *B = s->B;
        if (seed) *seed = s->seed;
        if (version) *version = s->version;
    });
}
int skc_asym_tables(const skc_asym_set* s, int m, uint32_t* bucket, double* sign) {
    return guard([&] {
        check_vec(s, "set");
        require(m >= 0 && m < s->B, "replicate index out of range");
        s->ctx->use();
        const size_t off = static_cast<size_t>(m) * 3 * s->n, cnt = static_cast<size_t>(3) * s->n;
        if (bucket) CK(cudaMemcpyAsync(bucket, s->bucket.p + off, cnt * 4, cudaMemcpyDeviceToHost, s->ctx->stream));
        if (sign) CK(cudaMemcpyAsync(sign, s->sign.p + off, cnt * 8, cudaMemcpyDeviceToHost, s->ctx->stream));
        s->ctx->sync();
    });
}
int skc_asym_coefficients(const skc_asym_set* s, uint64_t* hcoef, uint64_t* xcoef) {
    return guard([&] {
        check_vec(s, "set");
        if (hcoef) std::copy(s->hcoef.begin(), s->hcoef.end(), hcoef);
        if (xcoef) std::copy(s->xcoef.begin(), s->xcoef.end(), xcoef);
    });
}
int skc_asym_accumulate_dense(skc_asym_set* s, const void* T, int dtype, int location, int i0, int i1) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(T, "accumulate_dense: tensor");
        require(dtype == SKC_F64 || dtype == SKC_F32, "accumulate_dense: dtype must be SKC_F64 or SKC_F32");
        require(location == SKC_HOST || location == SKC_DEVICE, "accumulate_dense: bad location");
        require(0 <= i0 && i0 <= i1 && i1 <= s->n, "accumulate_dense: slice out of range");
        require(s->n <= 65535, "accumulate_dense: n above 65535 is not supported");
        skc_context* ctx = s->ctx;
        ctx->use();
        bool zc = false;
        const void* Td = stage_tensor(ctx, T, s->n, dtype, location, false, i0, i1, false, nullptr, &zc);
        s->version++;  // sketch.cpp:175
        run_dense_build(ctx, Td, s->n, dtype, false, i0, i1, s->B, s->b, s->packed.p, s->data.p, zc);
        ctx->sync();
    });
}

static void asym_factored_device(skc_asym_set* s, const double* ad, const double* Ud, const double* Vd,
                                 const double* Wd, long long Ncomp, double alpha, int m_only, double2* dst,
                                 bool overwrite) {
    skc_context* ctx = s->ctx;
    const int Bm = m_only >= 0 ? 1 : s->B;
    const int per_rep = Bm * s->S;
    int chunks = static_cast<int>(std::max<long long>(1, std::min<long long>(Ncomp, (4ll * ctx->sms + per_rep - 1) / per_rep)));
    ctx->freq_acc.alloc(static_cast<size_t>(chunks) * per_rep * s->N * 2);
    ctx->tmp.alloc(static_cast<size_t>(s->B) * s->b);
    AsymView v = s->view();
    launch_asym_factored_accumulate(ctx->stream, v, ad, Ud, Vd, Wd, Ncomp, chunks, m_only, ctx->freq_acc.p);
    ctx->check_launch();
    // reduce into tmp slot of replicate (m_only or all)
    double2* tmp = ctx->tmp.p;
    launch_freq_reduce_inverse(ctx->stream, ctx->freq_acc.p, chunks, Bm, s->S, s->N, s->logN, s->b, s->logb, v.twl,
                               tmp);
    ctx->check_launch();
    // combine: for m_only the tmp holds one replicate at index 0
    launch_combine_residues(ctx->stream, tmp, Bm, s->S, s->N, s->b, v.tw, alpha, -1, overwrite,
                            dst + (m_only >= 0 ? static_cast<size_t>(m_only) * s->b * 0 : 0));
    ctx->check_launch();
}

int skc_asym_add_rank1(skc_asym_set* s, double alpha, const double* u, const double* v, const double* w) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(u, "add_rank1: u");
        check_vec(v, "add_rank1: v");
        check_vec(w, "add_rank1: w");
        skc_context* ctx = s->ctx;
        ctx->use();
        s->version++;  // sketch.cpp:216
        const int n = s->n;
        std::vector<double> h(3 * static_cast<size_t>(n));
        std::copy(u, u + n, h.begin());
        std::copy(v, v + n, h.begin() + n);
        std::copy(w, w + n, h.begin() + 2 * n);
        ctx->X.upload(h.data(), h.size(), ctx->stream);
        asym_factored_device(s, nullptr, ctx->X.p, ctx->X.p + n, ctx->X.p + 2 * n, 1, alpha, -1, s->data.p, false);
        ctx->sync();
    });
}
int skc_asym_accumulate_factored(skc_asym_set* s, long long N, const double* a, const double* U, const double* V,
                                 const double* W) {
    return guard([&] {
        check_vec(s, "set");
        require(N >= 0, "accumulate_factored: negative component count");
        skc_context* ctx = s->ctx;
        ctx->use();
        s->version++;  // sketch.cpp:226
        if (N == 0) return;
        check_vec(a, "accumulate_factored: a");
        check_vec(U, "accumulate_factored: U");
        check_vec(V, "accumulate_factored: V");
        check_vec(W, "accumulate_factored: W");
        const size_t Nn = static_cast<size_t>(N) * s->n;
        std::vector<double> h(3 * Nn + static_cast<size_t>(N));
        std::copy(U, U + Nn, h.begin());
        std::copy(V, V + Nn, h.begin() + Nn);
        std::copy(W, W + Nn, h.begin() + 2 * Nn);
        std::copy(a, a + N, h.begin() + 3 * Nn);
        ctx->X.upload(h.data(), h.size(), ctx->stream);
        asym_factored_device(s, ctx->X.p + 3 * Nn, ctx->X.p, ctx->X.p + Nn, ctx->X.p + 2 * Nn, N, 1.0, -1, s->data.p,
                             false);
        ctx->sync();
    });
}
int skc_asym_rank1_sketch(skc_asym_set* s, int m, const double* u, const double* v, const double* w,
                          double* out_host) {
    return guard([&] {
        check_vec(s, "set");
        require(m >= 0 && m < s->B, "replicate index out of range");
        check_vec(u, "rank1_sketch: u");
        check_vec(v, "rank1_sketch: v");
        check_vec(w, "rank1_sketch: w");
        skc_context* ctx = s->ctx;
        ctx->use();
        const int n = s->n;
        std::vector<double> h(3 * static_cast<size_t>(n));
        std::copy(u, u + n, h.begin());
        std::copy(v, v + n, h.begin() + n);
        std::copy(w, w + n, h.begin() + 2 * n);
        ctx->X.upload(h.data(), h.size(), ctx->stream);
        DevBuf<double2> out;
        out.alloc(s->b);
        asym_factored_device(s, nullptr, ctx->X.p, ctx->X.p + n, ctx->X.p + 2 * n, 1, 1.0, m, out.p, true);
        CK(cudaMemcpyAsync(out_host, out.p, s->b * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
    });
}
int skc_asym_read_data(const skc_asym_set* s, int m, double* out_host) {
    return guard([&] {
        check_vec(s, "set");
        require(m < s->B, "replicate index out of range");
        s->ctx->use();
        const size_t off = m < 0 ? 0 : static_cast<size_t>(m) * s->b;
        const size_t cnt = m < 0 ? static_cast<size_t>(s->B) * s->b : s->b;
        CK(cudaMemcpyAsync(out_host, s->data.p + off, cnt * sizeof(double2), cudaMemcpyDeviceToHost, s->ctx->stream));
        s->ctx->sync();
    });
}
int skc_asym_write_data(skc_asym_set* s, int m, const double* in_host) {
    return guard([&] {
        check_vec(s, "set");
        require(m < s->B, "replicate index out of range");
        s->ctx->use();
        const size_t off = m < 0 ? 0 : static_cast<size_t>(m) * s->b;
        const size_t cnt = m < 0 ? static_cast<size_t>(s->B) * s->b : s->b;
        CK(cudaMemcpyAsync(s->data.p + off, in_host, cnt * sizeof(double2), cudaMemcpyHostToDevice, s->ctx->stream));
        s->version++;
        s->ctx->sync();
    });
}
int skc_asym_data_device(skc_asym_set* s, void** dev_ptr, size_t* bytes) {
    return guard([&] {
        check_vec(s, "set");
        *dev_ptr = s->data.p;
        *bytes = static_cast<size_t>(s->B) * s->b * sizeof(double2);
    });
}
int skc_asym_bump_version(skc_asym_set* s) {
    return guard([&] {
        check_vec(s, "set");
        s->version++;
    });
}
int skc_asym_recover_entry(const skc_asym_set* s, int i, int j, int k, double* out) {
    return guard([&] {  // sketch.cpp:250-262
        check_vec(s, "set");
        const int n = s->n;
        if (i < 0 || j < 0 || k < 0 || i >= n || j >= n || k >= n)
            fail(kInvalidArgument, "recover_entry: index out of range");
        s->ctx->use();
        std::vector<double> est(s->B);
        for (int m = 0; m < s->B; ++m) {
            const int idx[3] = {i, j, k};
            std::uint32_t bk[3];
            double sg[3];
            for (int q = 0; q < 3; ++q) {
                const size_t off = (static_cast<size_t>(m) * 3 + q) * n + idx[q];
                CK(cudaMemcpy(&bk[q], s->bucket.p + off, 4, cudaMemcpyDeviceToHost));
                CK(cudaMemcpy(&sg[q], s->sign.p + off, 8, cudaMemcpyDeviceToHost));
            }
            const std::uint32_t t = static_cast<std::uint32_t>((std::uint64_t{bk[0]} + bk[1] + bk[2]) % s->b);
            double2 z;
            CK(cudaMemcpy(&z, s->data.p + static_cast<size_t>(m) * s->b + t, sizeof(double2), cudaMemcpyDeviceToHost));
            est[m] = sg[0] * sg[1] * sg[2] * z.x;
        }
        std::size_t mid = est.size() / 2;
        std::nth_element(est.begin(), est.begin() + mid, est.end());
        double hi = est[mid];
        if (est.size() % 2 == 1) {
            *out = hi;
        } else {
            double lo = *std::max_element(est.begin(), est.begin() + mid);
            *out = 0.5 * (lo + hi);
        }
    });
}
int skc_asym_mode_contraction(skc_asym_set* s, int free_mode, const double* X_host, const double* Y_host, int L,
                              double* out_host) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(X_host, "mode_contraction: x");
        check_vec(Y_host, "mode_contraction: y");
        if (free_mode < 0 || free_mode > 2)
            fail(kInvalidArgument, "mode_contraction: free_mode must be 0, 1 or 2");  // contraction.cpp:253-254
        require(L >= 1, "mode_contraction: need at least one vector pair");
        require(s->B <= 128, "median over more than 128 replicates is not supported");
        skc_context* ctx = s->ctx;
        ctx->use();
        const size_t Ln = static_cast<size_t>(L) * s->n;
        std::vector<double> h(2 * Ln);
        std::copy(X_host, X_host + Ln, h.begin());
        std::copy(Y_host, Y_host + Ln, h.begin() + Ln);
        ctx->U.upload(h.data(), h.size(), ctx->stream);
        s->ensure_fresh();
        ctx->part.alloc(static_cast<size_t>(L) * s->B * s->S * s->n);
        launch_asym_mode(ctx->stream, s->view(), free_mode, ctx->U.p, ctx->U.p + Ln, L, ctx->part.p);
        ctx->check_launch();
        ctx->values.alloc(Ln);
        launch_median_rows(ctx->stream, ctx->part.p, L, s->B, s->S, s->n, ctx->values.p, nullptr, 0.0, nullptr);
        ctx->check_launch();
        CK(cudaMemcpyAsync(out_host, ctx->values.p, Ln * 8, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
    });
}
int skc_asym_vvv(skc_asym_set* s, const double* U_host, int L, double* out_host) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(U_host, "vvv: u");
        require(L >= 1, "vvv: need at least one vector");
        require(s->B <= 128, "median over more than 128 replicates is not supported");
        skc_context* ctx = s->ctx;
        ctx->use();
        ctx->U.upload(U_host, static_cast<size_t>(L) * s->n, ctx->stream);
        s->ensure_fresh();
        ctx->part.alloc(static_cast<size_t>(L) * s->B * s->S);
        launch_asym_vvv(ctx->stream, s->view(), ctx->U.p, L, ctx->part.p);
        ctx->check_launch();
        ctx->values.alloc(static_cast<size_t>(L));
        launch_asym_vvv_finish(ctx->stream, ctx->part.p, L, s->B, s->S, s->b, ctx->values.p);
        ctx->check_launch();
        CK(cudaMemcpyAsync(out_host, ctx->values.p, static_cast<size_t>(L) * 8, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
    });
}
int skc_asym_cached_transform(skc_asym_set* s, int m, double* out_host) {
    return guard([&] {
        check_vec(s, "set");
        require(m >= 0 && m < s->B, "replicate index out of range");
        s->ctx->use();
        s->ensure_fresh();
        spectrum_to_host(s->ctx, s->spec.p, m, s->b, s->N, s->logN, s->S, out_host);
    });
}

// als_fast(set, cfg) (decompose.cpp:117-205): CP-ALS where each factor column update is a
// batched sketched mode contraction (contraction.cpp:248-295) of the other two factors'
// columns. Factors stay on the device (column-major n x k); the k x k Grams are DGEMMs,
// the spectral pseudoinverse is host math. A, B, C out: n x k column-major.
int skc_asym_als(skc_asym_set* s, int k, int max_iters, double tol, uint64_t seed, double* lambda_out, double* A_out,
                 double* B_out, double* C_out, int* iters_out) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(lambda_out, "als: lambda");
        check_vec(A_out, "als: A");
        check_vec(B_out, "als: B");
        check_vec(C_out, "als: C");
        if (k < 1 || max_iters < 1) fail(kInvalidArgument, "als: k and max_iters must be positive");  // decompose.cpp:125-126
        if (k > s->n) fail(kInvalidArgument, "als: target rank exceeds tensor dimension");         // decompose.cpp:127
        require(s->B <= 128, "median over more than 128 replicates is not supported");
        skc_context* ctx = s->ctx;
        ctx->use();
        const int n = s->n;
        const size_t nk = static_cast<size_t>(n) * k;
        // als_init (decompose.cpp:124-138): one Rng per component r, A/B/C columns in turn
        std::vector<double> h(3 * nk);
        for (int r = 0; r < k; ++r) {
            Rng rng(derive_seed(seed, seed_tag::kAlsInit, static_cast<std::uint64_t>(r)));
            for (int f = 0; f < 3; ++f) rng.unit_sphere(n, h.data() + f * nk + static_cast<size_t>(r) * n);
        }
        DevBuf<double> F, M, prev, G1, G2, P, lam;
        F.upload(h.data(), h.size(), ctx->stream);
        M.alloc(nk);
        prev.alloc(nk);
        G1.alloc(static_cast<size_t>(k) * k);
        G2.alloc(static_cast<size_t>(k) * k);
        P.alloc(static_cast<size_t>(k) * k);
        lam.alloc(static_cast<size_t>(k));
        double* fac[3] = {F.p, F.p + nk, F.p + 2 * nk};
        s->ensure_fresh();
        ctx->part.alloc(static_cast<size_t>(k) * s->B * s->S * n);
        std::vector<double> g1(static_cast<size_t>(k) * k), g2(g1.size()), G(g1.size());
        std::vector<double> lambda(k, 1.0), lambda_prev(k, 1.0);  // s.lambda = Ones (decompose.cpp:129)
        int it = 0;
        for (; it < max_iters;) {
            for (int mode = 0; mode < 3; ++mode) {
                const int f1 = mode == 0 ? 1 : 0, f2 = mode == 2 ? 1 : 2;
                // M[:, r] = T(free mode, F1[:, r], F2[:, r]) for all r at once
                launch_asym_mode(ctx->stream, s->view(), mode, fac[f1], fac[f2], k, ctx->part.p);
                launch_median_rows(ctx->stream, ctx->part.p, k, s->B, s->S, n, M.p, nullptr, 0.0, nullptr);
                ctx->check_launch();
                // G = (F1' F1) .* (F2' F2)
                dgemm_cm(ctx, true, false, k, k, n, fac[f1], n, fac[f1], n, G1.p, k);
                dgemm_cm(ctx, true, false, k, k, n, fac[f2], n, fac[f2], n, G2.p, k);
                CK(cudaMemcpyAsync(g1.data(), G1.p, g1.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
                CK(cudaMemcpyAsync(g2.data(), G2.p, g2.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
                ctx->sync();
                for (size_t q = 0; q < G.size(); ++q) G[q] = g1[q] * g2[q];
                const std::vector<double> Pinv = pinv_spectral_host(k, G);
                CK(cudaMemcpyAsync(P.p, Pinv.data(), Pinv.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
                // target = M * pinv(G); normalize_columns(target, prev, lambda)
                CK(cudaMemcpyAsync(prev.p, fac[mode], nk * 8, cudaMemcpyDeviceToDevice, ctx->stream));
                dgemm_cm(ctx, false, false, n, k, k, M.p, n, P.p, k, fac[mode], n);
                launch_normalize_columns(ctx->stream, n, k, fac[mode], prev.p, lam.p);
                ctx->check_launch();
            }
            CK(cudaMemcpyAsync(lambda.data(), lam.p, static_cast<size_t>(k) * 8, cudaMemcpyDeviceToHost, ctx->stream));
            ctx->sync();
            ++it;
            double dn = 0.0, pn = 0.0;
            for (int r = 0; r < k; ++r) {
                dn += (lambda[r] - lambda_prev[r]) * (lambda[r] - lambda_prev[r]);
                pn += lambda_prev[r] * lambda_prev[r];
            }
            if (std::sqrt(dn) / std::max(std::sqrt(pn), 1e-300) < tol) break;  // decompose.cpp:184-186
            lambda_prev = lambda;
        }
        std::copy(lambda.begin(), lambda.end(), lambda_out);
        CK(cudaMemcpyAsync(A_out, fac[0], nk * 8, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(B_out, fac[1], nk * 8, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(C_out, fac[2], nk * 8, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
        if (iters_out) *iters_out = it;
    });
}

}  // extern "C"
