// Symmetric sketch sets (sketch.hpp SymmetricSketchSet), sketched contractions
// (contraction.hpp) and the RTPM driver (decompose.hpp) over the C-ABI.
#include "skc_abi_impl.hpp"

namespace skcabi {

// Upload coefficients, derive tables on the device, sort scatter permutations.
void init_sym_device(skc_sym_set* s, const double* data_host) {
    skc_context* ctx = s->ctx;
    ctx->use();
    const cudaStream_t st = ctx->stream;
    const size_t Bn = static_cast<size_t>(s->B) * s->n;
    s->d_hcoef.upload(s->hcoef.data(), s->hcoef.size(), st);
    s->d_scoef.upload(s->scoef.data(), s->scoef.size(), st);
    s->bucket1.alloc(Bn);
    s->bucket2.alloc(Bn);
    s->bucket3.alloc(Bn);
    s->packed.alloc(Bn);
    s->sexp.alloc(Bn);
    s->perm1.alloc(Bn);
    s->perm2.alloc(Bn);
    launch_sym_tables(st, s->d_hcoef.p, s->d_scoef.p, s->n, s->b, s->B, s->bucket1.p, s->bucket2.p, s->bucket3.p,
                      s->sexp.p, s->packed.p);
    ctx->check_launch();
    s->N = local_length(s->b);
    s->logN = ilog2(static_cast<unsigned>(s->N));
    s->S = static_cast<int>(s->b / static_cast<std::uint32_t>(s->N));
    s->logb = ilog2(s->b);
    launch_sort_perm(st, s->bucket1.p, s->B, s->n, static_cast<std::uint32_t>(s->N - 1), s->perm1.p);
    launch_sort_perm(st, s->bucket2.p, s->B, s->n, static_cast<std::uint32_t>(s->N - 1), s->perm2.p);
    s->plan1.alloc(Bn);
    s->plan2.alloc(Bn);
    launch_make_plan(st, s->perm1.p, s->bucket1.p, s->sexp.p, 1, nullptr, s->B, s->n, s->plan1.p);
    launch_make_plan(st, s->perm2.p, s->bucket2.p, s->sexp.p, 2, nullptr, s->B, s->n, s->plan2.p);
    ctx->check_launch();
    {
        // residue twiddles for the contraction scatter/gather (coalesced instead of
        // dependent random reads of the b-entry table); skipped above 256 MB
        const size_t cnt = static_cast<size_t>(s->B) * s->S * s->n;
        if (4 * cnt * sizeof(double2) <= (size_t(256) << 20)) {
            s->stw1.alloc(cnt);
            s->stw2.alloc(cnt);
            s->gtw1.alloc(cnt);
            s->gtw2.alloc(cnt);
            ctx->tw(s->b);
            SymView v = s->view();
            v.data = nullptr;
            v.spec = nullptr;
            launch_sym_twiddle_tables(st, v, s->stw1.p, s->stw2.p, s->gtw1.p, s->gtw2.p);
            ctx->check_launch();
        }
    }
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

// Symmetry check of the reference (tensor.cpp:32-43) — first failing (i,j,k,perm) in
// the reference's loop order, found on the device.
__global__ void k_first_asym(const void* T, int dtype, int n, double tol, unsigned long long* best) {
    long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= (long long)n * n * n) return;
    int i = static_cast<int>(idx / ((long long)n * n)), j = static_cast<int>((idx / n) % n), k = static_cast<int>(idx % n);
    if (!(i <= j && j <= k)) return;
    auto at = [&](int a, int b2, int c) -> double {
        size_t off = (static_cast<size_t>(a) * n + b2) * n + c;
        return dtype == 0 ? static_cast<const double*>(T)[off] : static_cast<double>(static_cast<const float*>(T)[off]);
    };
    const double ref = at(i, j, k);
    const int perms[5][3] = {{i, k, j}, {j, i, k}, {j, k, i}, {k, i, j}, {k, j, i}};
    for (int p = 0; p < 5; ++p)
        if (fabs(at(perms[p][0], perms[p][1], perms[p][2]) - ref) > tol) {
            // loop order: (i, j, k) lexicographic among sorted triples, then perm
            unsigned long long key = (static_cast<unsigned long long>(idx) << 3) | static_cast<unsigned long long>(p);
            atomicMin(best, key);
            return;
        }
}

}  // namespace skcabi

extern "C" {

// ---- symmetric set ----
int skc_sym_create(skc_context* ctx, int n, uint32_t b, int B, uint64_t master_seed, skc_sym_set** out) {
    return guard([&] {
        check_vec(ctx, "context");
        validate_set_args(n, b, B);
        auto s = std::make_unique<skc_sym_set>();
        s->ctx = ctx;
        s->n = n;
        s->b = b;
        s->B = B;
        s->seed = master_seed;
        s->hcoef.resize(static_cast<size_t>(B) * 6);
        s->scoef.resize(static_cast<size_t>(B) * 6);
        for (int m = 0; m < B; ++m) {  // sketch.cpp:307-309
            poly_coefficients(6, derive_seed(master_seed, seed_tag::kSymBucketHash, m), &s->hcoef[m * 6]);
            poly_coefficients(6, derive_seed(master_seed, seed_tag::kSymSign, m), &s->scoef[m * 6]);
        }
        init_sym_device(s.get(), nullptr);
        *out = s.release();
    });
}
int skc_sym_create_from_coefficients(skc_context* ctx, int n, uint32_t b, int B, uint64_t master_seed,
                                     const uint64_t* hcoef, const uint64_t* scoef, const double* data_host,
                                     skc_sym_set** out) {
    return guard([&] {
        check_vec(ctx, "context");
        validate_set_args(n, b, B);
        check_vec(hcoef, "hcoef");
        check_vec(scoef, "scoef");
        for (int x = 0; x < B * 6; ++x)
            require(hcoef[x] < kHashPrime && scoef[x] < kHashPrime, "PolyHash: coefficient out of range");
        auto s = std::make_unique<skc_sym_set>();
        s->ctx = ctx;
        s->n = n;
        s->b = b;
        s->B = B;
        s->seed = master_seed;
        s->hcoef.assign(hcoef, hcoef + static_cast<size_t>(B) * 6);
        s->scoef.assign(scoef, scoef + static_cast<size_t>(B) * 6);
        init_sym_device(s.get(), data_host);
        *out = s.release();
    });
}
int skc_sym_destroy(skc_sym_set* s) {
    return guard([&] {
        if (!s) return;
        s->ctx->use();
        s->ctx->sync();
        delete s;
    });
}
int skc_sym_info(const skc_sym_set* s, int* n, uint32_t* b, int* B, uint64_t* seed, uint64_t* version) {
    return guard([&] {
        check_vec(s, "set");
        if (n) *n = s->n;
        if (b) *b = s->b;
        if (B) *B = s->B;
        if (seed) *seed = s->seed;
        if (version) *version = s->version;
    });
}
int skc_sym_tables(const skc_sym_set* s, int m, uint32_t* bucket1, uint32_t* bucket2, uint32_t* bucket3,
                   uint8_t* sexp) {
    return guard([&] {
        check_vec(s, "set");
        require(m >= 0 && m < s->B, "replicate index out of range");
        s->ctx->use();
        const size_t off = static_cast<size_t>(m) * s->n, bytes = static_cast<size_t>(s->n) * 4;
        cudaStream_t st = s->ctx->stream;
        if (bucket1) CK(cudaMemcpyAsync(bucket1, s->bucket1.p + off, bytes, cudaMemcpyDeviceToHost, st));
        if (bucket2) CK(cudaMemcpyAsync(bucket2, s->bucket2.p + off, bytes, cudaMemcpyDeviceToHost, st));
        if (bucket3) CK(cudaMemcpyAsync(bucket3, s->bucket3.p + off, bytes, cudaMemcpyDeviceToHost, st));
        if (sexp) CK(cudaMemcpyAsync(sexp, s->sexp.p + off, s->n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}
int skc_sym_coefficients(const skc_sym_set* s, uint64_t* hcoef, uint64_t* scoef) {
    return guard([&] {
        check_vec(s, "set");
        if (hcoef) std::copy(s->hcoef.begin(), s->hcoef.end(), hcoef);
        if (scoef) std::copy(s->scoef.begin(), s->scoef.end(), scoef);
    });
}

}  // extern "C"
namespace skcabi {
// first_asymmetric_triple (tensor.cpp:32-45) over a device-visible n^3 tensor; throws
// the reference's invalid_argument message at the first failure.
void check_symmetric(skc_context* ctx, const void* Td, int dtype, int n) {
    ctx->asym_key.alloc(1);
    unsigned long long init = ~0ull;
    CK(cudaMemcpyAsync(ctx->asym_key.p, &init, 8, cudaMemcpyHostToDevice, ctx->stream));
    long long tot = static_cast<long long>(n) * n * n;
    k_first_asym<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, ctx->stream>>>(Td, dtype, n, 1e-9, ctx->asym_key.p);
    count_launch();
    ctx->check_launch();
    unsigned long long key = 0;
    CK(cudaMemcpyAsync(&key, ctx->asym_key.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    if (key != ~0ull) {
        const long long idx = static_cast<long long>(key >> 3);
        const int p = static_cast<int>(key & 7);
        const int i = static_cast<int>(idx / ((long long)n * n)), j = static_cast<int>((idx / n) % n),
                  k = static_cast<int>(idx % n);
        const int perms[5][3] = {{i, k, j}, {j, i, k}, {j, k, i}, {k, i, j}, {k, j, i}};
        fail(kInvalidArgument, "accumulate_dense: input tensor is not symmetric at (" + std::to_string(perms[p][0] + 1) +
                                   "," + std::to_string(perms[p][1] + 1) + "," + std::to_string(perms[p][2] + 1) + ")");
    }
}
}  // namespace skcabi
extern "C" {

int skc_sym_accumulate_dense(skc_sym_set* s, const void* T, int dtype, int location, int assume_symmetric, int i0,
                             int i1) {
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
        const void* Td = stage_tensor(ctx, T, s->n, dtype, location, true, i0, i1, !assume_symmetric, nullptr, &zc);
        if (!assume_symmetric) check_symmetric(ctx, Td, dtype, s->n);
        s->version++;  // sketch.cpp:324
        {
            SKC_PROF(ctx, "build_total");
            run_dense_build(ctx, Td, s->n, dtype, true, i0, i1, s->B, s->b, s->packed.p, s->data.p, zc);
        }
        ctx->sync();
    });
}

}  // extern "C"
namespace skcabi {
// Frequency-domain rank-1 / moment accumulation shared by add_scaled_rank1,
// accumulate_moment and RTPM deflation. X: device N x n.
// Frequency-domain accumulation of sum_s w_s F(CS(x_s))^3 over Nsamp samples, reduced over
// chunks and inverted per residue into ctx->tmp (B x b, linear in the samples).
void sym_moment_partial(skc_sym_set* s, const double* Xd, const double* wd, long long Nsamp) {
    skc_context* ctx = s->ctx;
    const int per_rep = s->B * s->S;
    const int chunks = wave_chunks(ctx->sms, per_rep, Nsamp);
    ctx->freq_acc.alloc(static_cast<size_t>(chunks) * per_rep * s->N * 2);
    ctx->tmp.alloc(static_cast<size_t>(s->B) * s->b);
    SymView v = s->view();
    {
        SKC_PROF(ctx, "moment");
        launch_sym_moment_accumulate(ctx->stream, v, Xd, wd, 1.0, Nsamp, chunks, ctx->freq_acc.p);
    }
    ctx->check_launch();
    {
        SKC_PROF(ctx, "freq_inverse");
        launch_freq_reduce_inverse(ctx->stream, ctx->freq_acc.p, chunks, s->B, s->S, s->N, s->logN, s->b, s->logb,
                                   v.twl, ctx->tmp.p);
    }
    ctx->check_launch();
}
// data += alpha x (residue combination of ctx->tmp)
void sym_moment_combine(skc_sym_set* s, double alpha) {
    skc_context* ctx = s->ctx;
    SymView v = s->view();
    {
        SKC_PROF(ctx, "combine");
        launch_combine_residues(ctx->stream, ctx->tmp.p, s->B, s->S, s->N, s->b, v.tw, alpha, -1, false, s->data.p);
    }
    ctx->check_launch();
}
static void sym_moment_device(skc_sym_set* s, const double* Xd, const double* wd, double alpha, long long Nsamp) {
    sym_moment_partial(s, Xd, wd, Nsamp);
    sym_moment_combine(s, alpha);
}
}  // namespace skcabi
extern "C" {

int skc_sym_add_scaled_rank1(skc_sym_set* s, const double* u_host, double alpha) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(u_host, "add_scaled_rank1: u");
        if (alpha == 0.0) return;  // sketch.cpp:349
        skc_context* ctx = s->ctx;
        ctx->use();
        s->version++;
        ctx->X.upload(u_host, s->n, ctx->stream);
        sym_moment_device(s, ctx->X.p, nullptr, alpha, 1);
        ctx->sync();
    });
}

int skc_sym_accumulate_moment(skc_sym_set* s, const double* X, const double* w, long long N, int location) {
    return guard([&] {
        check_vec(s, "set");
        require(N >= 0, "accumulate_moment: negative sample count");
        if (N == 0) return;
        check_vec(X, "accumulate_moment: X");
        skc_context* ctx = s->ctx;
        ctx->use();
        const double* Xd = X;
        const double* wd = w;
        if (location == SKC_HOST) {
            ctx->X.upload(X, static_cast<size_t>(N) * s->n, ctx->stream);
            Xd = ctx->X.p;
            if (w) {
                ctx->values.upload(w, static_cast<size_t>(N), ctx->stream);
                wd = ctx->values.p;
            }
        }
        s->version++;
        sym_moment_device(s, Xd, wd, 1.0, N);
        ctx->sync();
    });
}

int skc_sym_aux_sketches(const skc_sym_set* s, int m, const double* u_host, double* s1, double* s2, double* s3) {
    return guard([&] {  // sketch.cpp:412-425
        check_vec(s, "set");
        check_vec(u_host, "sym_aux_sketches: u");
        require(m >= 0 && m < s->B, "replicate index out of range");
        skc_context* ctx = s->ctx;
        ctx->use();
        ctx->X.upload(u_host, s->n, ctx->stream);
        ctx->tmp.alloc(3 * static_cast<size_t>(s->b));
        launch_sym_aux(ctx->stream, s->view(), m, ctx->X.p, ctx->tmp.p);
        ctx->check_launch();
        const size_t bytes = s->b * sizeof(double2);
        if (s1) CK(cudaMemcpyAsync(s1, ctx->tmp.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        if (s2) CK(cudaMemcpyAsync(s2, ctx->tmp.p + s->b, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        if (s3) CK(cudaMemcpyAsync(s3, ctx->tmp.p + 2 * static_cast<size_t>(s->b), bytes, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
    });
}

int skc_sym_rank1_truncated(const skc_sym_set* s, int m, const double* u_host, double* out_host) {
    return guard([&] {  // sketch.cpp:427-443
        check_vec(s, "set");
        check_vec(u_host, "sketch_rank1_sym: u");
        check_vec(out_host, "sketch_rank1_sym: out");
        require(m >= 0 && m < s->B, "replicate index out of range");
        skc_context* ctx = s->ctx;
        ctx->use();
        const cudaStream_t st = ctx->stream;
        const SymView v = s->view();
        ctx->X.upload(u_host, s->n, st);
        DevBuf<double2> aux, spec2, acc, tmp, out;
        aux.alloc(3 * static_cast<size_t>(s->b));
        spec2.alloc(2 * static_cast<size_t>(s->b));
        acc.alloc(s->b);
        tmp.alloc(s->b);
        out.alloc(s->b);
        launch_sym_aux(st, v, m, ctx->X.p, aux.p);
        // forward transforms of s1 and s2 (two "replicates" in local residue layout)
        launch_spectrum(st, aux.p, s->b, s->logb, 2, s->N, s->logN, s->S, v.tw, v.twl, spec2.p);
        launch_rank1_trunc_product(st, spec2.p, static_cast<long long>(s->b), acc.p);
        launch_freq_reduce_inverse(st, reinterpret_cast<const double*>(acc.p), 1, 1, s->S, s->N, s->logN, s->b,
                                   s->logb, v.twl, tmp.p);
        launch_combine_residues(st, tmp.p, 1, s->S, s->N, s->b, v.tw, 1.0, -1, true, out.p);
        launch_add_third(st, aux.p + 2 * static_cast<size_t>(s->b), s->b, out.p);
        ctx->check_launch();
        CK(cudaMemcpyAsync(out_host, out.p, s->b * sizeof(double2), cudaMemcpyDeviceToHost, st));
        ctx->sync();
    });
}

int skc_sym_read_data(const skc_sym_set* s, int m, double* out_host) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(out_host, "read_data: out");
        require(m < s->B, "replicate index out of range");
        s->ctx->use();
        const size_t off = m < 0 ? 0 : static_cast<size_t>(m) * s->b;
        const size_t cnt = m < 0 ? static_cast<size_t>(s->B) * s->b : s->b;
        CK(cudaMemcpyAsync(out_host, s->data.p + off, cnt * sizeof(double2), cudaMemcpyDeviceToHost, s->ctx->stream));
        s->ctx->sync();
    });
}
int skc_sym_write_data(skc_sym_set* s, int m, const double* in_host) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(in_host, "write_data: in");
        require(m < s->B, "replicate index out of range");
        s->ctx->use();
        const size_t off = m < 0 ? 0 : static_cast<size_t>(m) * s->b;
        const size_t cnt = m < 0 ? static_cast<size_t>(s->B) * s->b : s->b;
        CK(cudaMemcpyAsync(s->data.p + off, in_host, cnt * sizeof(double2), cudaMemcpyHostToDevice, s->ctx->stream));
        s->version++;
        s->ctx->sync();
    });
}
int skc_sym_data_device(skc_sym_set* s, void** dev_ptr, size_t* bytes) {
    return guard([&] {
        check_vec(s, "set");
        *dev_ptr = s->data.p;
        *bytes = static_cast<size_t>(s->B) * s->b * sizeof(double2);
    });
}
int skc_sym_bump_version(skc_sym_set* s) {
    return guard([&] {
        check_vec(s, "set");
        s->version++;
    });
}
int skc_sym_recover_entry(const skc_sym_set* s, int i, int j, int k, double* out) {
    // sketch.cpp:363-377 — O(B) gather of host-visible data; computed from the
    // device tables and data copied back per replicate.
    return guard([&] {
        check_vec(s, "set");
        const int n = s->n;
        if (i < 0 || j < 0 || k < 0 || i >= n || j >= n || k >= n)
            fail(kInvalidArgument, "recover_entry: index out of range");
        s->ctx->use();
        const double kappa = (i == j && j == k) ? 1.0 : ((i == j || j == k || i == k) ? 3.0 : 6.0);
        std::vector<double> est(s->B);
        std::vector<std::uint32_t> b1(3);
        std::vector<std::uint8_t> se(3);
        for (int m = 0; m < s->B; ++m) {
            const int idx[3] = {i, j, k};
            for (int q = 0; q < 3; ++q) {
                CK(cudaMemcpy(&b1[q], s->bucket1.p + static_cast<size_t>(m) * n + idx[q], 4, cudaMemcpyDeviceToHost));
                CK(cudaMemcpy(&se[q], s->sexp.p + static_cast<size_t>(m) * n + idx[q], 1, cudaMemcpyDeviceToHost));
            }
            const std::uint32_t t =
                static_cast<std::uint32_t>((std::uint64_t{b1[0]} + b1[1] + b1[2]) % s->b);
            double2 z;
            CK(cudaMemcpy(&z, s->data.p + static_cast<size_t>(m) * s->b + t, sizeof(double2), cudaMemcpyDeviceToHost));
            const unsigned e = (4 * 3 - (se[0] + se[1] + se[2])) & 3u;
            // (root4(e) * z).real()
            double re;
            switch (e) {
                case 0: re = z.x; break;
                case 1: re = -z.y; break;
                case 2: re = -z.x; break;
                default: re = z.y; break;
            }
            est[m] = re / kappa;
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

// ---- symmetric contractions ----
static void sym_contract_batch(skc_sym_set* s, const double* Ud, int L, int mode) {
    skc_context* ctx = s->ctx;
    s->ensure_fresh();
    const size_t per = (mode == 0) ? static_cast<size_t>(s->n) : 3;
    ctx->part.alloc(static_cast<size_t>(L) * s->B * s->S * per);
    SKC_PROF(ctx, "sym_contract");
    launch_sym_contract(ctx->stream, s->view(), Ud, L, mode, ctx->part.p);
    ctx->check_launch();
}

int skc_sym_ivv(skc_sym_set* s, const double* U_host, int L, double* out_host) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(U_host, "Ivv: U");
        check_vec(out_host, "Ivv: out");
        require(L >= 1, "Ivv: need at least one vector");
        require(s->B <= 128, "median over more than 128 replicates is not supported");
        skc_context* ctx = s->ctx;
        ctx->use();
        ctx->U.upload(U_host, static_cast<size_t>(L) * s->n, ctx->stream);
        sym_contract_batch(s, ctx->U.p, L, 0);
        ctx->values.alloc(static_cast<size_t>(L) * s->n);
        {
            SKC_PROF(ctx, "median");
            launch_median_rows(ctx->stream, ctx->part.p, L, s->B, s->S, s->n, ctx->values.p, nullptr, 0.0, nullptr);
        }
        ctx->check_launch();
        CK(cudaMemcpyAsync(out_host, ctx->values.p, static_cast<size_t>(L) * s->n * 8, cudaMemcpyDeviceToHost,
                           ctx->stream));
        ctx->sync();
    });
}
int skc_sym_vvv(skc_sym_set* s, const double* U_host, int L, double* out_host) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(U_host, "vvv: U");
        check_vec(out_host, "vvv: out");
        require(L >= 1, "vvv: need at least one vector");
        require(s->B <= 128, "median over more than 128 replicates is not supported");
        skc_context* ctx = s->ctx;
        ctx->use();
        ctx->U.upload(U_host, static_cast<size_t>(L) * s->n, ctx->stream);
        sym_contract_batch(s, ctx->U.p, L, 1);
        ctx->values.alloc(static_cast<size_t>(L));
        {
            SKC_PROF(ctx, "vvv_finish");
            launch_sym_vvv_finish(ctx->stream, ctx->part.p, L, s->B, s->S, s->b, ctx->values.p);
        }
        ctx->check_launch();
        CK(cudaMemcpyAsync(out_host, ctx->values.p, static_cast<size_t>(L) * 8, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
    });
}

int skc_sym_cached_transform(skc_sym_set* s, int m, double* out_host) {
    return guard([&] {
        check_vec(s, "set");
        require(m >= 0 && m < s->B, "replicate index out of range");
        s->ctx->use();
        s->ensure_fresh();
        spectrum_to_host(s->ctx, s->spec.p, m, s->b, s->N, s->logN, s->S, out_host);
    });
}

}  // extern "C"
namespace skcabi {
// ---- RTPM ----
// Runs T power steps on L restarts resident at ctx->U (device) and the median vvv of
// the finals into ctx->values. Degenerate flags accumulate in ctx->flags.
static void rtpm_restarts_launches(skc_sym_set* s, int L, int T_iters, double tol) {
    skc_context* ctx = s->ctx;
    CK(cudaMemsetAsync(ctx->flags.p, 0, sizeof(int) * L, ctx->stream));
    const SymView v = s->view();
    for (int t = 0; t < T_iters; ++t) {
        {
            SKC_PROF(ctx, "sym_contract");
            launch_sym_contract(ctx->stream, v, ctx->U.p, L, 0, ctx->part.p);
        }
        SKC_PROF(ctx, "median");
        launch_median_rows(ctx->stream, ctx->part.p, L, s->B, s->S, s->n, nullptr, ctx->U.p, tol, ctx->flags.p,
                           ctx->values.p);
    }
    launch_sym_contract(ctx->stream, v, ctx->U.p, L, 1, ctx->part.p);
    launch_sym_vvv_finish(ctx->stream, ctx->part.p, L, s->B, s->S, s->b, ctx->values.p);
}
void rtpm_restarts_device(skc_sym_set* s, int L, int T_iters, double tol) {
    skc_context* ctx = s->ctx;
    s->ensure_fresh();
    ctx->flags.alloc(static_cast<size_t>(L));
    ctx->part.alloc(static_cast<size_t>(L) * s->B * s->S * std::max(s->n, 3));
    ctx->values.alloc(static_cast<size_t>(L) * s->n);
    if (ctx->prof_on) {  // per-kernel event scopes: launch directly
        rtpm_restarts_launches(s, L, T_iters, tol);
        ctx->check_launch();
        return;
    }
    // The T power steps and the selection values are one CUDA graph, captured once per
    // (set, L, T, tol, buffers) and replayed per component: 2T + 3 launches per replay.
    std::uint64_t tolbits;
    std::memcpy(&tolbits, &tol, sizeof(tolbits));
    const std::vector<std::uint64_t> key = {static_cast<std::uint64_t>(L),
                                            static_cast<std::uint64_t>(T_iters), tolbits,
                                            reinterpret_cast<std::uint64_t>(ctx->U.p),
                                            reinterpret_cast<std::uint64_t>(ctx->part.p),
                                            reinterpret_cast<std::uint64_t>(ctx->values.p),
                                            reinterpret_cast<std::uint64_t>(ctx->flags.p),
                                            reinterpret_cast<std::uint64_t>(s->spec.p),
                                            reinterpret_cast<std::uint64_t>(s->data.p)};
    auto it = s->rtpm_graphs.find(key);
    if (it == s->rtpm_graphs.end()) {
        // attributes and lazily built tables are set up by one direct run
        rtpm_restarts_launches(s, L, T_iters, tol);
        ctx->check_launch();
        const std::uint64_t l0 = launch_count(), f0 = transform_units();
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        rtpm_restarts_launches(s, L, T_iters, tol);
        CK(cudaStreamEndCapture(ctx->stream, &g));
        skc_sym_set::RtpmGraph rg;
        CK(cudaGraphInstantiate(&rg.exec, g, 0));
        cudaGraphDestroy(g);
        rg.launches = launch_count() - l0;
        rg.transforms = transform_units() - f0;
        if (s->rtpm_graphs.size() > 16) {  // bounded cache
            for (auto& e : s->rtpm_graphs) cudaGraphExecDestroy(e.second.exec);
            s->rtpm_graphs.clear();
        }
        s->rtpm_graphs[key] = rg;
        return;  // the direct run above computed this call's results
    }
    CK(cudaGraphLaunch(it->second.exec, ctx->stream));
    count_replay(it->second.launches, it->second.transforms);
}
void check_degenerate(skc_context* ctx, int L) {
    std::vector<int> f(L);
    CK(cudaMemcpyAsync(f.data(), ctx->flags.p, sizeof(int) * L, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    for (int x : f)
        if (x) fail(kDegenerate, "power update produced a vanishing iterate");  // decompose.cpp:37-38
}
}  // namespace skcabi
extern "C" {

int skc_sym_rtpm(skc_sym_set* s, int k, int L, int T_iters, uint64_t seed, double tol, const double* inits,
                 double* lambda, double* V, int* best_tau) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(lambda, "rtpm: lambda");
        check_vec(V, "rtpm: V");
        // decompose.cpp:15-20
        if (k < 1 || L < 1 || T_iters < 1) fail(kInvalidArgument, "power method: k, L and T must be positive");
        if (k > s->n) fail(kInvalidArgument, "power method: target rank exceeds tensor dimension");
        require(s->B <= 128, "median over more than 128 replicates is not supported");
        skc_context* ctx = s->ctx;
        ctx->use();
        const int n = s->n;
        const size_t Ln = static_cast<size_t>(L) * n;
        // inits Rng(derive_seed(seed, 0x31, c, tau)).unit_sphere(n) (decompose.cpp:96-97) in
        // pinned double buffers: component c+1's are drawn on the host (restarts in
        // parallel, each stream independent) while the device runs component c
        double* pin[2] = {nullptr, nullptr};
        if (!inits) {
            pin[0] = ctx->pinned_doubles(2 * Ln);
            pin[1] = pin[0] + Ln;
        }
        auto draw = [&](int c, double* dst) {
#pragma omp parallel for schedule(static)
            for (int t = 0; t < L; ++t) {
                Rng rng(derive_seed(seed, seed_tag::kPowerInit, static_cast<std::uint64_t>(c), static_cast<std::uint64_t>(t)));
                rng.unit_sphere(n, dst + static_cast<size_t>(t) * n);
            }
        };
        if (!inits) draw(0, pin[0]);
        ctx->ints.alloc(16);
        ctx->dbl.alloc(4);
        ctx->X.alloc(static_cast<size_t>(n));
        for (int c = 0; c < k; ++c) {
            const double* U0 = inits ? inits + static_cast<size_t>(c) * Ln : pin[c & 1];
            ctx->U.upload(U0, Ln, ctx->stream);
            rtpm_restarts_device(s, L, T_iters, tol);
            launch_argmax_first(ctx->stream, ctx->values.p, L, ctx->ints.p + 2, ctx->dbl.p);
            ctx->check_launch();
            if (!inits && c + 1 < k) draw(c + 1, pin[(c + 1) & 1]);  // overlaps the device work
            int bt = 0;
            double lam = 0.0;
            CK(cudaMemcpyAsync(&bt, ctx->ints.p + 2, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaMemcpyAsync(&lam, ctx->dbl.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
            check_degenerate(ctx, L);  // synchronises
            lambda[c] = lam;
            if (best_tau) best_tau[c] = bt;
            CK(cudaMemcpyAsync(V + static_cast<size_t>(c) * n, ctx->U.p + static_cast<size_t>(bt) * n, n * 8,
                               cudaMemcpyDeviceToHost, ctx->stream));
            // deflation: add_scaled_rank1(v, -lambda) (decompose.cpp:112)
            if (lam != 0.0) {
                CK(cudaMemcpyAsync(ctx->X.p, ctx->U.p + static_cast<size_t>(bt) * n, n * 8, cudaMemcpyDeviceToDevice,
                                   ctx->stream));
                s->version++;
                sym_moment_device(s, ctx->X.p, nullptr, -lam, 1);
            }
            ctx->sync();
        }
    });
}

int skc_sym_rtpm_restarts(skc_sym_set* s, const double* U0_host, int L, int T_iters, double tol, double* finals_out,
                          double* values_out) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(U0_host, "rtpm_restarts: U0");
        require(L >= 1 && T_iters >= 1, "power method: k, L and T must be positive");
        require(s->B <= 128, "median over more than 128 replicates is not supported");
        skc_context* ctx = s->ctx;
        ctx->use();
        ctx->U.upload(U0_host, static_cast<size_t>(L) * s->n, ctx->stream);
        rtpm_restarts_device(s, L, T_iters, tol);
        if (finals_out)
            CK(cudaMemcpyAsync(finals_out, ctx->U.p, static_cast<size_t>(L) * s->n * 8, cudaMemcpyDeviceToHost,
                               ctx->stream));
        if (values_out)
            CK(cudaMemcpyAsync(values_out, ctx->values.p, static_cast<size_t>(L) * 8, cudaMemcpyDeviceToHost,
                               ctx->stream));
        check_degenerate(ctx, L);
    });
}

}  // extern "C"
