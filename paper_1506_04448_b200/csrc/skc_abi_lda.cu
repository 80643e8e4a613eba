// Spectral LDA (lda.hpp/lda.cpp) over the C-ABI: corpus upload and transpose, M1 / implicit
// M2, randomized whitening, sketch_whitened_m3, recovery, held-out likelihood and the
// device-resident corpus handle. Kernels in skc_lda.cu and skc_whiten.cu.
#include "skc_abi_impl.hpp"

namespace skcabi {

void upload_corpus(skc_context* ctx, int V, long long D, const long long* doc_ptr, const int* word, const int* count,
                   CorpusDev& c, const std::string& who, bool check_counts) {
    require(V >= 1 && D >= 0, who + ": invalid corpus dimensions");
    check_vec(doc_ptr, (who + ": doc_ptr").c_str());
    const long long nnz = doc_ptr[D];
    require(doc_ptr[0] == 0 && nnz >= 0, who + ": doc_ptr must start at 0");
    if (nnz > 0) {
        check_vec(word, (who + ": word").c_str());
        check_vec(count, (who + ": count").c_str());
    }
    for (long long d = 0; d < D; ++d)  // O(D) host check keeps device reads in bounds
        if (doc_ptr[d + 1] < doc_ptr[d]) fail(kInvalidArgument, who + ": doc_ptr must be non-decreasing");
    // device-side validation, totals, stable word-major transpose, used-document list
    // and word-pass chunks (corpus_gpu_build, skc_whiten.cu)
    constexpr long long kWordChunk = 64;
    const cudaStream_t st = ctx->stream;
    const size_t nz = static_cast<size_t>(std::max<long long>(nnz, 1));
    const size_t Dz = static_cast<size_t>(std::max<long long>(D, 1));
    c.V = V;
    c.D = D;
    c.nnz = nnz;
    c.doc_ptr.upload(doc_ptr, static_cast<size_t>(D) + 1, st);
    const int zero = 0;
    c.word.upload(nnz > 0 ? word : &zero, nz, st);
    c.count.upload(nnz > 0 ? count : &zero, nz, st);
    c.cptr.alloc(static_cast<size_t>(V) + 1);
    c.cdoc.alloc(nz);
    c.ccount.alloc(nz);
    c.total.alloc(Dz);
    c.used_docs.alloc(Dz);
    c.word_chunk.alloc(static_cast<size_t>(V) + 1);
    const size_t max_chunks = static_cast<size_t>(nnz / kWordChunk + V + 1);
    c.chunk_lo.alloc(max_chunks);
    c.chunk_hi.alloc(max_chunks);
    DevBuf<unsigned long long> stats;
    stats.alloc(8);
    DevBuf<unsigned char> temp;
    const size_t tb = corpus_gpu_temp_bytes(V, D, nnz);
    temp.alloc(tb);
    corpus_gpu_build(st, V, D, nnz, c.doc_ptr.p, c.word.p, c.count.p, check_counts, c.total.p, c.cptr.p, c.cdoc.p,
                     c.ccount.p, c.used_docs.p, stats.p, kWordChunk, c.word_chunk.p, c.chunk_lo.p, c.chunk_hi.p,
                     temp.p, tb);
    ctx->check_launch();
    unsigned long long hs[8];
    CK(cudaMemcpyAsync(hs, stats.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    long long nchunks = 0;
    CK(cudaMemcpyAsync(&nchunks, c.word_chunk.p + V, sizeof(long long), cudaMemcpyDeviceToHost, st));
    ctx->sync();
    if (hs[0]) fail(kInvalidArgument, who + ": doc_ptr must be non-decreasing");
    if (hs[1]) fail(kInvalidArgument, who + ": word id out of range");
    if (hs[2]) fail(kInvalidArgument, who + ": negative count");
    c.used1 = static_cast<long long>(hs[3]);
    c.used2 = static_cast<long long>(hs[4]);
    c.used3 = static_cast<long long>(hs[5]);
    c.nchunks = nchunks;
    c.total.alloc(static_cast<size_t>(std::max<long long>(D, 1)));
    c.s2.alloc(static_cast<size_t>(std::max<long long>(D, 1)));
    c.invm.alloc(static_cast<size_t>(std::max<long long>(D, 1)));
    c.diag.alloc(static_cast<size_t>(V));
    c.m1p.alloc(static_cast<size_t>(V));
    launch_corpus_prep(st, V, D, c.doc_ptr.p, c.count.p, c.cptr.p, c.cdoc.p, c.ccount.p, c.total.p, c.s2.p, c.invm.p,
                       c.diag.p, c.m1p.p);
    ctx->check_launch();
}

// reference error order: compute_m2 calls compute_m1 first (lda.cpp:89-99, 103, 120)
void check_corpus_m1(const CorpusDev& c) {
    if (c.D == 0) fail(kNumericalError, "compute_m1: empty corpus");
    if (c.used1 == 0) fail(kNumericalError, "compute_m1: no nonempty documents");
}
void check_corpus_m2(const CorpusDev& c) {
    check_corpus_m1(c);
    if (c.used2 == 0) fail(kNumericalError, "compute_m2: no documents with at least 2 words");
}

struct M2Work {
    DevBuf<double> Z, part, mx;
};
void m2_apply(skc_context* ctx, const CorpusDev& c, double alpha0, int p, const double* Xd, double* Yd, M2Work& w) {
    w.Z.alloc(static_cast<size_t>(std::max<long long>(c.D, 1)) * p);
    w.part.alloc(static_cast<size_t>(std::max<long long>(std::max<long long>(c.nchunks, (c.V + 511) / 512), 1)) * p);
    w.mx.alloc(static_cast<size_t>(p));
    launch_m2_apply(ctx->stream, c.V, c.D, p, c.doc_ptr.p, c.word.p, c.count.p, c.cdoc.p, c.ccount.p, c.nchunks,
                    c.chunk_lo.p, c.chunk_hi.p, c.word_chunk.p, c.s2.p, c.diag.p, c.m1p.p,
                    1.0 / static_cast<double>(c.used1), 1.0 / static_cast<double>(c.used2), alpha0 / (alpha0 + 1.0),
                    Xd, w.Z.p, w.part.p, w.mx.p, Yd);
    ctx->check_launch();
}

// Q (V x p row-major = p x V col-major) = orthonormal basis of range(Y): CholeskyQR2 with
// DGEMM Gram products; modified Gram-Schmidt on the host (with random completion) when
// the Gram matrix is not numerically positive definite (rank-deficient block).
struct OrthWork {
    DevBuf<double> G, Rinv, tmp;
};
void orthonormalize(skc_context* ctx, int V, int p, const double* Yd, double* Qd, OrthWork& w, Rng& rng) {
    w.G.alloc(static_cast<size_t>(p) * p);
    w.Rinv.alloc(static_cast<size_t>(p) * p);
    w.tmp.alloc(static_cast<size_t>(V) * p);
    std::vector<double> G(static_cast<size_t>(p) * p), Ri(static_cast<size_t>(p) * p);
    const double* src = Yd;
    for (int pass = 0; pass < 2; ++pass) {
        dgemm_cm(ctx, false, true, p, p, V, src, p, src, p, w.G.p, p);
        CK(cudaMemcpyAsync(G.data(), w.G.p, G.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
        // Cholesky G = R^T R (R upper, col-major)
        bool ok = true;
        double gmax = 0.0;
        for (int i = 0; i < p; ++i) gmax = std::max(gmax, G[static_cast<size_t>(i) * p + i]);
        std::vector<double> R(static_cast<size_t>(p) * p, 0.0);
        for (int j = 0; j < p && ok; ++j) {
            for (int i = 0; i <= j; ++i) {
                double s = G[static_cast<size_t>(j) * p + i];
                for (int k = 0; k < i; ++k) s -= R[static_cast<size_t>(i) * p + k] * R[static_cast<size_t>(j) * p + k];
                if (i == j) {
                    if (!(s > 1e-12 * gmax)) {
                        ok = false;
                        break;
                    }
                    R[static_cast<size_t>(j) * p + j] = std::sqrt(s);
                } else {
                    R[static_cast<size_t>(j) * p + i] = s / R[static_cast<size_t>(i) * p + i];
                }
            }
        }
        if (!ok) {
            // host modified Gram-Schmidt (twice) with random completion of null directions
            std::vector<double> Y(static_cast<size_t>(V) * p);
            CK(cudaMemcpyAsync(Y.data(), src, Y.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
            ctx->sync();
            auto col = [&](int c, int r) -> double& { return Y[static_cast<size_t>(r) * p + c]; };
            double ymax = 0.0;
            for (double x : Y) ymax = std::max(ymax, std::fabs(x));
            for (int c = 0; c < p; ++c) {
                for (int attempt = 0; attempt < 8; ++attempt) {
                    for (int rep = 0; rep < 2; ++rep)
                        for (int c2 = 0; c2 < c; ++c2) {
                            double d = 0.0;
                            for (int r = 0; r < V; ++r) d += col(c2, r) * col(c, r);
                            for (int r = 0; r < V; ++r) col(c, r) -= d * col(c2, r);
                        }
                    double nr = 0.0;
                    for (int r = 0; r < V; ++r) nr += col(c, r) * col(c, r);
                    nr = std::sqrt(nr);
                    if (nr > 1e-10 * std::max(ymax, 1e-300) && nr > 0.0) {
                        for (int r = 0; r < V; ++r) col(c, r) /= nr;
                        break;
                    }
                    for (int r = 0; r < V; ++r) col(c, r) = rng.gaussian();
                    ymax = 1.0;
                }
            }
            CK(cudaMemcpyAsync(Qd, Y.data(), Y.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
            ctx->sync();
            return;
        }
        // Rinv (upper) by back substitution, col-major
        std::fill(Ri.begin(), Ri.end(), 0.0);
        for (int j = 0; j < p; ++j) {
            Ri[static_cast<size_t>(j) * p + j] = 1.0 / R[static_cast<size_t>(j) * p + j];
            for (int i = j - 1; i >= 0; --i) {
                double s = 0.0;
                for (int k = i + 1; k <= j; ++k) s += R[static_cast<size_t>(k) * p + i] * Ri[static_cast<size_t>(j) * p + k];
                Ri[static_cast<size_t>(j) * p + i] = -s / R[static_cast<size_t>(i) * p + i];
            }
        }
        CK(cudaMemcpyAsync(w.Rinv.p, Ri.data(), Ri.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        // Q^T = Rinv^T Y^T  (col-major: (p x V) = (p x p)^T (p x V))
        double* dst = (pass == 0) ? w.tmp.p : Qd;
        dgemm_cm(ctx, true, false, p, V, p, w.Rinv.p, p, src, p, dst, p);
        src = dst;
    }
}

// whiten (lda.cpp:125-143) for an operator apply(X, Y): Y = M2 X on V x p device blocks.
template <typename Apply>
void whiten_randomized(skc_context* ctx, int V, int k, int oversample, int iters, std::uint64_t seed, Apply apply,
                       double* W_out, double* U_out, double* sv_out) {
    require(k >= 1 && k <= V, "whiten: invalid target rank");
    if (oversample < 0) oversample = std::max(16, k / 4);
    if (iters < 0) iters = 12;
    const int p = std::min(V, (k + oversample + 31) / 32 * 32);
    auto tick = [](const char*) {};  // (phase marks of the whitening pipeline)
    Rng rng(derive_seed(seed, seed_tag::kWhitenProbe));  // host stream: MGS completion only
    DevBuf<double> Q, Y;
    Q.alloc(static_cast<size_t>(V) * p);
    Y.alloc(static_cast<size_t>(V) * p);
    // Gaussian start block on the device (counter-based, deterministic)
    launch_gaussian_fill(ctx->stream, derive_seed(seed, seed_tag::kWhitenProbe), static_cast<long long>(V) * p, Y.p);
    tick("omega");
    OrthWork ow;
    orthonormalize(ctx, V, p, Y.p, Q.p, ow, rng);
    tick("orth0");
    for (int it = 0; it < iters; ++it) {
        apply(Q.p, Y.p, p);
        tick("apply");
        orthonormalize(ctx, V, p, Y.p, Q.p, ow, rng);
        tick("orth");
    }
    apply(Q.p, Y.p, p);
    // Rayleigh-Ritz: H = Q^T M2 Q (p x p)
    DevBuf<double> Hd;
    Hd.alloc(static_cast<size_t>(p) * p);
    dgemm_cm(ctx, false, true, p, p, V, Q.p, p, Y.p, p, Hd.p, p);
    std::vector<double> H(static_cast<size_t>(p) * p);
    CK(cudaMemcpyAsync(H.data(), Hd.p, H.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    for (int i = 0; i < p; ++i)
        for (int j = i + 1; j < p; ++j) {
            const double s = 0.5 * (H[static_cast<size_t>(j) * p + i] + H[static_cast<size_t>(i) * p + j]);
            H[static_cast<size_t>(j) * p + i] = H[static_cast<size_t>(i) * p + j] = s;
        }
    tick("rayleigh");
    std::vector<double> ev, U;
    sym_eigen_host(p, H, ev, U);
    tick("eigen");
    std::vector<double> Uk(static_cast<size_t>(p) * k), fw(k), fu(k);
    for (int c = 0; c < k; ++c) {
        const double e = ev[p - 1 - c];
        if (!(e > 1e-10))  // lda.cpp:133-136
            fail(kNumericalError, "whiten: moment matrix is rank deficient at component " + std::to_string(c + 1) +
                                      " (eigenvalue " + std::to_string(e) + ")");
        sv_out[c] = e;
        fw[c] = 1.0 / std::sqrt(e);
        fu[c] = std::sqrt(e);
        std::copy(U.begin() + static_cast<size_t>(p - 1 - c) * p, U.begin() + static_cast<size_t>(p - c) * p,
                  Uk.begin() + static_cast<size_t>(c) * p);
    }
    DevBuf<double> Ukd, Vk, fwd, fud, out;
    Ukd.upload(Uk.data(), Uk.size(), ctx->stream);
    Vk.alloc(static_cast<size_t>(V) * k);
    // Vk (V x k row-major = k x V col-major) = Uk^T (k x p) Q^T (p x V)
    dgemm_cm(ctx, true, false, k, V, p, Ukd.p, p, Q.p, p, Vk.p, k);
    fwd.upload(fw.data(), fw.size(), ctx->stream);
    fud.upload(fu.data(), fu.size(), ctx->stream);
    out.alloc(static_cast<size_t>(V) * k);
    launch_scale_cols(ctx->stream, V, k, Vk.p, fwd.p, out.p);
    CK(cudaMemcpyAsync(W_out, out.p, static_cast<size_t>(V) * k * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    launch_scale_cols(ctx->stream, V, k, Vk.p, fud.p, out.p);
    CK(cudaMemcpyAsync(U_out, out.p, static_cast<size_t>(V) * k * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
}

// sketch_whitened_m3 (lda.cpp:145-226) on an uploaded corpus.
// Shard mode (global_m1 != null): the document sums run over this corpus only, while the
// normalisation 1/D_used (global_used) and q = W^T m1 (global_m1, V, already averaged)
// are the whole corpus'; add_q_cubed selects the one shard that adds c_m1 F(q)^3. The
// sketch is linear in the per-document terms, so summing the shards' data reproduces the
// full sketch_whitened_m3.
void sketch_whitened_m3_dev(skc_sym_set* s, CorpusDev& c, const double* W, double alpha0, long long* used_out,
                            long long* skipped_out, long long global_used, const double* global_m1,
                            bool add_q_cubed) {
    check_vec(W, "sketch_whitened_m3: W");
    const int k = s->n;  // lda.cpp:149-151: set dimension must equal the whitening rank
    require(k <= 2048, "sketch_whitened_m3: whitening rank above 2048 is not supported on the device path");
    const bool shard = global_m1 != nullptr;
    const long long used = c.used3, skipped = c.D - c.used3, used1 = c.used1;
    const long long norm_used = shard ? global_used : used;
    if (norm_used <= 0) fail(kNumericalError, "sketch_whitened_m3: no documents with >= 3 words");  // lda.cpp:186
    const int V = c.V;
    const long long D = c.D;
    skc_context* ctx = s->ctx;
    ctx->use();
    const cudaStream_t st = ctx->stream;
    DevBuf<long long> d_total;
    DevBuf<double> d_W, d_P, d_s1, d_s2, d_coeff1, d_sumwn, d_m1, d_q, d_acc, d_cross, d_vpart;
    d_W.upload(W, static_cast<size_t>(V) * k, st);
    d_vpart.alloc(static_cast<size_t>(std::max<long long>(c.nchunks, 1)) * (k + 2));
    d_P.alloc(static_cast<size_t>(std::max<long long>(D, 1)) * k);
    d_s1.alloc(static_cast<size_t>(std::max<long long>(D, 1)));
    d_s2.alloc(static_cast<size_t>(std::max<long long>(D, 1)));
    d_total.alloc(static_cast<size_t>(std::max<long long>(D, 1)));
    d_coeff1.alloc(static_cast<size_t>(V));
    d_sumwn.alloc(static_cast<size_t>(V) * k);
    d_m1.alloc(static_cast<size_t>(V));
    d_q.alloc(static_cast<size_t>(k));
    {
        SKC_PROF(ctx, "lda_docs");
        launch_lda_docs(st, k, D, c.doc_ptr.p, c.word.p, c.count.p, d_W.p, alpha0, d_P.p, d_s1.p, d_s2.p, d_total.p);
    }
    {
        SKC_PROF(ctx, "lda_vocab");
        launch_lda_vocab_chunked(st, k, V, c.nchunks, c.chunk_lo.p, c.chunk_hi.p, c.word_chunk.p, c.cdoc.p, c.ccount.p,
                                 d_P.p, d_s1.p, d_total.p, d_vpart.p, d_coeff1.p, d_sumwn.p, d_m1.p);
    }
    if (shard) {
        d_m1.upload(global_m1, static_cast<size_t>(V), st);
        launch_lda_q(st, k, V, d_W.p, d_m1.p, 1.0, d_q.p);
    } else {
        launch_lda_q(st, k, V, d_W.p, d_m1.p, 1.0 / static_cast<double>(used1), d_q.p);
    }
    ctx->check_launch();
    const int per_rep = s->B * s->S;
    // ~4 waves of 2 resident CTAs per SM for each of the two item kinds
    const int chunks_d = wave_chunks(ctx->sms, per_rep, used);
    const int chunks_v = std::max(1, static_cast<int>(std::min<long long>(V, (8ll * ctx->sms) / per_rep)));
    d_acc.alloc(static_cast<size_t>(chunks_d + chunks_v) * per_rep * s->N * 2);
    d_cross.alloc(static_cast<size_t>(chunks_d) * per_rep * s->N * 2);
    SymView v = s->view();
    {
        SKC_PROF(ctx, "lda_accumulate");
        launch_lda_accumulate(st, v, used, c.used_docs.p, d_P.p, d_s1.p, d_s2.p, V, d_W.p, d_coeff1.p, d_sumwn.p,
                              chunks_d, chunks_v, d_acc.p, d_cross.p);
    }
    ctx->check_launch();
    ctx->tmp.alloc(static_cast<size_t>(s->B) * s->b);
    const double inv_docs = 1.0 / static_cast<double>(norm_used);
    const double m1_coeff =
        add_q_cubed ? 2.0 * alpha0 * alpha0 / ((alpha0 + 1.0) * (alpha0 + 2.0)) : 0.0;  // lda.cpp:191
    launch_lda_finish(st, v, d_acc.p, d_cross.p, chunks_d + chunks_v, chunks_d, d_q.p, inv_docs, m1_coeff, ctx->tmp.p);
    ctx->check_launch();
    launch_combine_residues(st, ctx->tmp.p, s->B, s->S, s->N, s->b, v.tw, 1.0, -1, false, s->data.p);
    ctx->check_launch();
    s->version += static_cast<std::uint64_t>(s->B);  // mutable_replicate(m) per replicate (lda.cpp:197)
    ctx->sync();
    if (used_out) *used_out = used;
    if (skipped_out) *skipped_out = skipped;
}


}  // namespace skcabi

// opaque handle of include/sketchcp_b200.h
struct skc_lda_corpus {
    skc_context* ctx = nullptr;
    CorpusDev dev;
};

extern "C" {

int skc_sym_sketch_whitened_m3(skc_sym_set* s, int V, long long D, const long long* doc_ptr, const int* word,
                               const int* count, const double* W, double alpha0, long long* used_out,
                               long long* skipped_out) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(W, "sketch_whitened_m3: W");
        s->ctx->use();
        CorpusDev c;
        upload_corpus(s->ctx, V, D, doc_ptr, word, count, c, "sketch_whitened_m3", false);
        sketch_whitened_m3_dev(s, c, W, alpha0, used_out, skipped_out);
    });
}

// ---- LDA moments and whitening (lda.cpp:88-143) ----------------------------------------
int skc_lda_compute_m1(skc_context* ctx, int V, long long D, const long long* doc_ptr, const int* word,
                       const int* count, double* m1_out) {
    return guard([&] {
        check_vec(ctx, "context");
        check_vec(m1_out, "compute_m1: out");
        ctx->use();
        CorpusDev c;
        upload_corpus(ctx, V, D, doc_ptr, word, count, c);
        check_corpus_m1(c);
        CK(cudaMemcpyAsync(m1_out, c.m1p.p, static_cast<size_t>(V) * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
        ctx->sync();
        for (int w = 0; w < V; ++w) m1_out[w] /= static_cast<double>(c.used1);  // lda.cpp:99
    });
}

int skc_lda_m2_apply(skc_context* ctx, int V, long long D, const long long* doc_ptr, const int* word,
                     const int* count, double alpha0, int p, const double* X, double* Y) {
    return guard([&] {
        check_vec(ctx, "context");
        check_vec(X, "m2_apply: X");
        check_vec(Y, "m2_apply: Y");
        require(p >= 1, "m2_apply: p must be positive");
        ctx->use();
        CorpusDev c;
        upload_corpus(ctx, V, D, doc_ptr, word, count, c);
        check_corpus_m2(c);
        DevBuf<double> Xd, Yd;
        Xd.upload(X, static_cast<size_t>(V) * p, ctx->stream);
        Yd.alloc(static_cast<size_t>(V) * p);
        M2Work w;
        m2_apply(ctx, c, alpha0, p, Xd.p, Yd.p, w);
        CK(cudaMemcpyAsync(Y, Yd.p, static_cast<size_t>(V) * p * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
    });
}

int skc_lda_whiten_corpus(skc_context* ctx, int V, long long D, const long long* doc_ptr, const int* word,
                          const int* count, double alpha0, int k, int oversample, int iters, uint64_t seed,
                          double* W, double* unwhiten, double* singular_values) {
    return guard([&] {
        check_vec(ctx, "context");
        check_vec(W, "whiten: W");
        check_vec(unwhiten, "whiten: unwhiten");
        check_vec(singular_values, "whiten: singular_values");
        ctx->use();
        CorpusDev c;
        upload_corpus(ctx, V, D, doc_ptr, word, count, c);
        check_corpus_m2(c);
        require(k >= 1 && k <= V, "whiten: invalid target rank");
        M2Work w;
        SKC_PROF(ctx, "lda_whiten");
        whiten_randomized(
            ctx, V, k, oversample, iters, seed,
            [&](const double* Xd, double* Yd, int p) { m2_apply(ctx, c, alpha0, p, Xd, Yd, w); }, W, unwhiten,
            singular_values);
    });
}

int skc_lda_whiten_dense(skc_context* ctx, int V, const double* m2, int k, int oversample, int iters, uint64_t seed,
                         double* W, double* unwhiten, double* singular_values) {
    return guard([&] {
        check_vec(ctx, "context");
        check_vec(m2, "whiten: m2hat");
        check_vec(W, "whiten: W");
        check_vec(unwhiten, "whiten: unwhiten");
        check_vec(singular_values, "whiten: singular_values");
        require(V >= 1, "whiten: matrix must be square");
        require(k >= 1 && k <= V, "whiten: invalid target rank");
        ctx->use();
        // SelfAdjointEigenSolver reads the lower triangle: symmetrise from it
        std::vector<double> M(static_cast<size_t>(V) * V);
        for (int i = 0; i < V; ++i)
            for (int j = 0; j <= i; ++j)
                M[static_cast<size_t>(i) * V + j] = M[static_cast<size_t>(j) * V + i] = m2[static_cast<size_t>(i) * V + j];
        DevBuf<double> Md;
        Md.upload(M.data(), M.size(), ctx->stream);
        whiten_randomized(
            ctx, V, k, oversample, iters, seed,
            [&](const double* Xd, double* Yd, int p) {
                // Y^T (p x V) = X^T (p x V) M2 (V x V)
                dgemm_cm(ctx, false, false, p, V, V, Xd, p, Md.p, V, Yd, p);
            },
            W, unwhiten, singular_values);
    });
}

// lda.cpp:228-248: topics and prior from the whitened CP decomposition (host math, O(V k)).
int skc_lda_recover_params(skc_context* ctx, int V, int k, const double* lambda, const double* A,
                           const double* unwhiten, double alpha0, double* Phi, double* alpha) {
    return guard([&] {
        check_vec(ctx, "context");
        require(k >= 1, "recover_params: empty decomposition");
        check_vec(lambda, "recover_params: lambda");
        check_vec(A, "recover_params: A");
        check_vec(unwhiten, "recover_params: unwhiten");
        check_vec(Phi, "recover_params: Phi");
        check_vec(alpha, "recover_params: alpha");
        require(V >= 1, "recover_params: decomposition/whitening rank mismatch");
        for (int i = 0; i < k; ++i) {  // lda.cpp:236-241
            const double lam = lambda[i];
            if (lam == 0.0) fail(kNumericalError, "recover_params: zero eigenvalue at component " + std::to_string(i + 1));
            alpha[i] = 4.0 * alpha0 * (alpha0 + 1.0) / ((alpha0 + 2.0) * (alpha0 + 2.0) * lam * lam);
        }
        ctx->use();
        DevBuf<double> dl, dA, dU, mu, dP;
        dl.upload(lambda, static_cast<size_t>(k), ctx->stream);
        dA.upload(A, static_cast<size_t>(k) * k, ctx->stream);
        dU.upload(unwhiten, static_cast<size_t>(V) * k, ctx->stream);
        mu.alloc(static_cast<size_t>(V) * k);
        dP.alloc(static_cast<size_t>(V) * k);
        launch_lda_recover_params(ctx->stream, V, k, dl.p, dA.p, dU.p, alpha0, mu.p, dP.p);
        ctx->check_launch();
        CK(cudaMemcpyAsync(Phi, dP.p, sizeof(double) * V * k, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
    });
}

// lda.cpp:273-320: mean per-document held-out log-likelihood; the mixtures by projected
// gradient on the device (one warp per document, skc_lda_post.cu); the step from the
// largest eigenvalue of the k x k Gram (host Jacobi); the sum in document order.
int skc_lda_heldout_likelihood(skc_context* ctx, int V, int k, const double* Phi, int Vh, long long D,
                               const long long* doc_ptr, const int* word, const int* count, double* ll_out,
                               long long* floored_out) {
    return guard([&] {
        check_vec(ctx, "context");
        check_vec(Phi, "heldout_likelihood: Phi");
        check_vec(doc_ptr, "heldout_likelihood: doc_ptr");
        check_vec(ll_out, "heldout_likelihood: out");
        require(Vh <= V, "heldout_likelihood: corpus vocabulary exceeds the model's");
        require(k >= 1 && k <= 128, "heldout_likelihood: the device path supports k <= 128");
        require(D >= 0 && doc_ptr[0] == 0, "heldout_likelihood: doc_ptr must start at 0");
        const long long nnz = doc_ptr[D];
        for (long long q = 0; q < nnz; ++q)
            require(word[q] >= 0 && word[q] < Vh, "heldout_likelihood: word index out of range");
        ctx->use();
        DevBuf<double> dP, G, per;
        DevBuf<long long> dptr, fl;
        DevBuf<int> dw, dc;
        dP.upload(Phi, static_cast<size_t>(V) * k, ctx->stream);
        G.alloc(static_cast<size_t>(k) * k);
        launch_phi_gram(ctx->stream, V, k, dP.p, G.p);
        std::vector<double> gram(static_cast<size_t>(k) * k);
        CK(cudaMemcpyAsync(gram.data(), G.p, sizeof(double) * k * k, cudaMemcpyDeviceToHost, ctx->stream));
        dptr.upload(doc_ptr, static_cast<size_t>(D) + 1, ctx->stream);
        dw.upload(word, static_cast<size_t>(std::max<long long>(nnz, 1)), ctx->stream);
        dc.upload(count, static_cast<size_t>(std::max<long long>(nnz, 1)), ctx->stream);
        per.alloc(static_cast<size_t>(std::max<long long>(D, 1)));
        fl.alloc(static_cast<size_t>(std::max<long long>(D, 1)));
        ctx->sync();
        std::vector<double> ev, U;
        sym_eigen_host(k, gram, ev, U);
        const double lips = ev.empty() ? 0.0 : ev.back();
        const double step = lips > 0 ? 1.0 / lips : 1.0;
        if (D > 0) {
            launch_lda_heldout(ctx->stream, k, D, dptr.p, dw.p, dc.p, dP.p, G.p, step, per.p, fl.p);
            ctx->check_launch();
        }
        std::vector<double> hp(static_cast<size_t>(std::max<long long>(D, 1)));
        std::vector<long long> hf(static_cast<size_t>(std::max<long long>(D, 1)));
        if (D > 0) {
            CK(cudaMemcpyAsync(hp.data(), per.p, sizeof(double) * D, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaMemcpyAsync(hf.data(), fl.p, sizeof(long long) * D, cudaMemcpyDeviceToHost, ctx->stream));
        }
        ctx->sync();
        double total = 0.0;
        long long nused = 0, floored = 0;
        for (long long d = 0; d < D; ++d)
            if (!std::isnan(hp[d])) {
                total += hp[d];
                ++nused;
                floored += hf[d];
            }
        if (floored_out) *floored_out = floored;
        if (nused == 0) fail(kNumericalError, "heldout_likelihood: empty held-out corpus");
        *ll_out = total / static_cast<double>(nused);
    });
}

// ---- device-resident corpus handle (upload + transpose once, reuse across calls) ------
int skc_lda_corpus_create(skc_context* ctx, int V, long long D, const long long* doc_ptr, const int* word,
                          const int* count, skc_lda_corpus** out) {
    return guard([&] {
        check_vec(ctx, "context");
        check_vec(out, "lda_corpus_create: out");
        ctx->use();
        auto c = std::make_unique<skc_lda_corpus>();
        c->ctx = ctx;
        upload_corpus(ctx, V, D, doc_ptr, word, count, c->dev, "lda", true);
        ctx->sync();
        *out = c.release();
    });
}
int skc_lda_corpus_destroy(skc_lda_corpus* c) {
    return guard([&] {
        if (!c) return;
        c->ctx->use();
        delete c;
    });
}
int skc_lda_corpus_info(const skc_lda_corpus* c, int* V, long long* D, long long* nnz, long long* used3) {
    return guard([&] {
        check_vec(c, "corpus");
        if (V) *V = c->dev.V;
        if (D) *D = c->dev.D;
        if (nnz) *nnz = c->dev.nnz;
        if (used3) *used3 = c->dev.used3;
    });
}
int skc_lda_whiten_corpus_handle(skc_lda_corpus* c, double alpha0, int k, int oversample, int iters, uint64_t seed,
                                 double* W, double* unwhiten, double* singular_values) {
    return guard([&] {
        check_vec(c, "corpus");
        check_vec(W, "whiten: W");
        check_vec(unwhiten, "whiten: unwhiten");
        check_vec(singular_values, "whiten: singular_values");
        skc_context* ctx = c->ctx;
        ctx->use();
        check_corpus_m2(c->dev);
        require(k >= 1 && k <= c->dev.V, "whiten: invalid target rank");
        M2Work w;
        SKC_PROF(ctx, "lda_whiten");
        whiten_randomized(
            ctx, c->dev.V, k, oversample, iters, seed,
            [&](const double* Xd, double* Yd, int p) { m2_apply(ctx, c->dev, alpha0, p, Xd, Yd, w); }, W, unwhiten,
            singular_values);
    });
}
int skc_sym_sketch_whitened_m3_corpus(skc_sym_set* s, skc_lda_corpus* c, const double* W, double alpha0,
                                      long long* used_out, long long* skipped_out) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(c, "corpus");
        require(s->ctx == c->ctx, "sketch_whitened_m3: set and corpus belong to different contexts");
        sketch_whitened_m3_dev(s, c->dev, W, alpha0, used_out, skipped_out);
    });
}

// Document-shard form of sketch_whitened_m3 for multi-GPU runs (distributed.py).
int skc_sym_sketch_whitened_m3_shard(skc_sym_set* s, int V, long long D, const long long* doc_ptr, const int* word,
                                     const int* count, const double* W, double alpha0, long long global_used,
                                     const double* global_m1, int add_q_cubed, long long* used_out,
                                     long long* skipped_out) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(W, "sketch_whitened_m3: W");
        check_vec(global_m1, "sketch_whitened_m3: global m1");
        require(global_used >= 1, "sketch_whitened_m3: no documents with >= 3 words");
        s->ctx->use();
        CorpusDev c;
        upload_corpus(s->ctx, V, D, doc_ptr, word, count, c, "sketch_whitened_m3", false);
        sketch_whitened_m3_dev(s, c, W, alpha0, used_out, skipped_out, global_used, global_m1, add_q_cubed != 0);
    });
}

}  // extern "C"
