// C-ABI implementation (include/sketchcp_b200.h), core unit: context, profiling, seeds and
// hashing, standalone transforms, the sketch file container and the planted-tensor
// generators. Host C++ orchestration of the sm_100a kernels; validation, error messages
// and exception taxonomy follow the reference (proj/include/sketchcp/*.hpp).
#include "skc_abi_impl.hpp"

namespace skcabi {

// natural-order spectrum of replicate m from the residue/bit-reversed layout
void spectrum_to_host(skc_context* ctx, const double2* spec, int m, std::uint32_t b, int N, int logN, int S,
                             double* out) {
    std::vector<double2> loc(b);
    CK(cudaMemcpyAsync(loc.data(), spec + static_cast<size_t>(m) * b, b * sizeof(double2), cudaMemcpyDeviceToHost,
                       ctx->stream));
    ctx->sync();
    for (int r = 0; r < S; ++r)
        for (int j = 0; j < N; ++j) {
            const std::uint32_t f = static_cast<std::uint32_t>(r) + static_cast<std::uint32_t>(S) * bitrev(j, logN);
            out[2 * f] = loc[static_cast<size_t>(r) * N + j].x;
            out[2 * f + 1] = loc[static_cast<size_t>(r) * N + j].y;
        }
}

}  // namespace skcabi

extern "C" {

const char* skc_last_error(void) { return g_last_error.c_str(); }
int skc_version(void) { return 1; }
uint64_t skc_kernel_launch_count(void) { return launch_count(); }
uint64_t skc_transform_count(void) { return transform_units(); }

int skc_device_count(int* out) {
    return guard([&] {
        int c = 0;
        cudaError_t e = cudaGetDeviceCount(&c);
        if (e != cudaSuccess) c = 0;
        *out = c;
    });
}

int skc_context_create(int device, skc_context** out) {
    return guard([&] {
        check_vec(out, "skc_context_create");
        int count = 0;
        cudaError_t e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess || count == 0)
            fail(kCudaError, "no CUDA device available (this library has no CPU fallback)");
        require(device >= 0 && device < count, "skc_context_create: device index out of range");
        CK(cudaSetDevice(device));
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10)
            fail(kCudaError, std::string("device ") + prop.name + " is not sm_100-class; this library targets sm_100a");
        auto ctx = std::make_unique<skc_context>();
        ctx->device = device;
        ctx->sms = prop.multiProcessorCount;
        ctx->smem_optin = static_cast<int>(prop.sharedMemPerBlockOptin);
        CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        *out = ctx.release();
    });
}
int skc_context_destroy(skc_context* ctx) {
    return guard([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        if (ctx->stream2) cudaStreamSynchronize(ctx->stream2);
        if (ctx->comm) ncclCommDestroy(ctx->comm);
        if (ctx->host_ints) cudaFreeHost(ctx->host_ints);
        if (ctx->host_dbl) cudaFreeHost(ctx->host_dbl);
        for (auto& r : ctx->prof) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
        if (ctx->ev_order) cudaEventDestroy(ctx->ev_order);
        cudaStream_t st = ctx->stream, st2 = ctx->stream2;
        cudaEvent_t ev[5];
        for (int c = 0; c < 5; ++c) ev[c] = ctx->ev_q[c];
        delete ctx;
        cudaStreamDestroy(st);
        if (st2) cudaStreamDestroy(st2);
        for (int c = 0; c < 5; ++c)
            if (ev[c]) cudaEventDestroy(ev[c]);
    });
}
int skc_context_synchronize(skc_context* ctx) {
    return guard([&] {
        check_vec(ctx, "context");
        ctx->use();
        ctx->sync();
    });
}
int skc_profile_enable(skc_context* ctx, int on) {
    return guard([&] {
        check_vec(ctx, "context");
        ctx->use();
        ctx->prof_on = on != 0;
        // pre-create events so timed loops under profiling pay no event creation
        while (ctx->prof_on && ctx->ev_pool.size() < 512) {
            cudaEvent_t e = nullptr;
            CK(cudaEventCreate(&e));
            ctx->ev_pool.push_back(e);
        }
    });
}
int skc_profile_reset(skc_context* ctx) {
    return guard([&] {
        check_vec(ctx, "context");
        ctx->use();
        ctx->sync();
        for (auto& r : ctx->prof) {  // back to the pool
            ctx->ev_pool.push_back(r.a);
            ctx->ev_pool.push_back(r.b);
        }
        ctx->prof.clear();
    });
}
int skc_profile_get(skc_context* ctx, const char* kernel, double* total_ms, uint64_t* launches) {
    return guard([&] {
        check_vec(ctx, "context");
        check_vec(kernel, "kernel name");
        ctx->use();
        ctx->sync();
        double tot = 0.0;
        std::uint64_t cnt = 0;
        for (auto& r : ctx->prof)
            if (r.name == kernel) {
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, r.a, r.b));
                tot += ms;
                ++cnt;
            }
        if (total_ms) *total_ms = tot;
        if (launches) *launches = cnt;
    });
}
int skc_context_stream(skc_context* ctx, void** stream_out) {
    return guard([&] {
        check_vec(ctx, "context");
        *stream_out = reinterpret_cast<void*>(ctx->stream);
    });
}

int skc_context_wait_stream(skc_context* ctx, void* producer) {
    return guard([&] {
        check_vec(ctx, "context");
        ctx->use();
        if (!ctx->ev_order) CK(cudaEventCreateWithFlags(&ctx->ev_order, cudaEventDisableTiming));
        CK(cudaEventRecord(ctx->ev_order, static_cast<cudaStream_t>(producer)));
        CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_order, 0));
    });
}

int skc_context_build_retries(skc_context* ctx, long long* out) {
    return guard([&] {
        check_vec(ctx, "context");
        check_vec(out, "out");
        *out = ctx->build_two_limb_retries;
    });
}
int skc_context_build_banded(skc_context* ctx, long long* out) {
    return guard([&] {
        check_vec(ctx, "context");
        check_vec(out, "out");
        *out = ctx->build_banded;
    });
}

uint64_t skc_derive_seed(uint64_t master, uint64_t tag, uint64_t i0, uint64_t i1) {
    return derive_seed(master, tag, i0, i1);
}
int skc_unit_sphere(uint64_t seed, int n, double* out) {
    return guard([&] {
        require(n >= 1, "unit_sphere: n must be positive");
        Rng(seed).unit_sphere(n, out);
    });
}
int skc_power_inits(uint64_t seed, int n, int c0, int k, int tau0, int L, double* out) {
    return guard([&] {
        require(n >= 1 && k >= 0 && L >= 0, "power_inits: invalid sizes");
        for (int c = 0; c < k; ++c)
            for (int t = 0; t < L; ++t) {
                Rng rng(derive_seed(seed, seed_tag::kPowerInit, static_cast<std::uint64_t>(c0 + c),
                                    static_cast<std::uint64_t>(tau0 + t)));
                rng.unit_sphere(n, out + (static_cast<size_t>(c) * L + t) * n);
            }
    });
}
int skc_poly_coefficients(int independence, uint64_t seed, uint64_t* out) {
    return guard([&] {
        require(independence >= 1 && independence <= 8, "PolyHash: independence must be in [1, 8]");
        poly_coefficients(independence, seed, out);
    });
}
uint32_t skc_poly_eval(const uint64_t* coeffs, int k, uint32_t b, uint64_t i) { return poly_eval(coeffs, k, b, i); }

// ---- standalone transforms: fft::* (fft.hpp:15-26) on the device -------------------------
static skc_context* process_context() {
    static std::mutex mu;
    static skc_context* ctx = nullptr;
    std::lock_guard<std::mutex> lk(mu);
    if (!ctx) {
        skc_context* c = nullptr;
        const int st = skc_context_create(0, &c);
        if (st != kOk) fail(st, g_last_error);
        ctx = c;
    }
    return ctx;
}

// dir: -1 forward (unnormalised, e^{-2 pi i}), +1 inverse scaled by 1/b, +2 inverse unscaled.
static void device_fft(skc_context* ctx, double* x, std::size_t b, int dir) {
    if (!is_pow2(b))  // fft.cpp:40-44
        fail(kInvalidArgument, "fft: length must be a power of two, got " + std::to_string(b));
    require(b <= (1u << 28), "fft: length above 2^28 is not supported");
    require(dir == -1 || dir == 1 || dir == 2, "fft: direction must be -1, +1 or +2");
    ctx->use();
    const cudaStream_t st = ctx->stream;
    const std::uint32_t bb = static_cast<std::uint32_t>(b);
    if (bb == 1) return;  // length-1 transform is the identity
    const int N = local_length(bb), logN = ilog2(static_cast<unsigned>(N)), S = static_cast<int>(bb / N);
    const int logb = ilog2(bb);
    DevBuf<double2> in, out;
    in.alloc(b);
    out.alloc(b);
    if (dir == -1) {
        in.upload(reinterpret_cast<const double2*>(x), b, st);
        launch_spectrum(st, in.p, bb, logb, 1, N, logN, S, ctx->tw(bb), ctx->twl(N), out.p);
        ctx->check_launch();
        spectrum_to_host(ctx, out.p, 0, bb, N, logN, S, x);
    } else {
        std::vector<double2> lay(b);
        for (int r = 0; r < S; ++r)
            for (int j = 0; j < N; ++j) {
                const std::size_t f = static_cast<std::size_t>(r) + static_cast<std::size_t>(S) * bitrev(j, logN);
                lay[static_cast<std::size_t>(r) * N + j] = double2{x[2 * f], x[2 * f + 1]};
            }
        in.upload(lay.data(), b, st);
        launch_freq_reduce_inverse(st, reinterpret_cast<const double*>(in.p), 1, 1, S, N, logN, bb, logb, ctx->twl(N),
                                   out.p);
        launch_combine_residues(st, out.p, 1, S, N, bb, ctx->tw(bb), 1.0, -1, true, in.p, dir == 1);
        ctx->check_launch();
        CK(cudaMemcpyAsync(x, in.p, b * sizeof(double2), cudaMemcpyDeviceToHost, st));
        ctx->sync();
    }
}

int skc_fft(double* x_host, size_t b, int dir) {
    return guard([&] {
        check_vec(x_host, "fft: x");
        device_fft(process_context(), x_host, b, dir);
    });
}

// ---- sketch file container (sketch.cpp:47-141, 264-296, 379-410, 445-449) -----------------
// little-endian: magic "SKCPSKT\0", u64 version 1, mode (0 asym, 1 sym), n, b, B, seed; then
// per replicate the hash coefficient lists (count + values) and the complex data.
namespace {
const char kMagic[8] = {'S', 'K', 'C', 'P', 'S', 'K', 'T', '\0'};
void put_u64(std::ostream& os, std::uint64_t v) {
    unsigned char buf[8];
    for (int i = 0; i < 8; ++i) buf[i] = static_cast<unsigned char>(v >> (8 * i));
    os.write(reinterpret_cast<const char*>(buf), 8);
}
std::uint64_t get_u64(std::istream& is) {
    unsigned char buf[8];
    is.read(reinterpret_cast<char*>(buf), 8);
    if (!is) fail(kFormatError, "sketch file: truncated");
    std::uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<std::uint64_t>(buf[i]) << (8 * i);
    return v;
}
void put_coeffs(std::ostream& os, const std::uint64_t* c, int k) {
    put_u64(os, static_cast<std::uint64_t>(k));
    for (int d = 0; d < k; ++d) put_u64(os, c[d]);
}
void get_coeffs(std::istream& is, int expect, std::uint64_t* out) {
    const std::uint64_t cnt = get_u64(is);
    if (cnt == 0 || cnt > 16) fail(kFormatError, "sketch file: bad hash coefficient count");
    if (cnt != static_cast<std::uint64_t>(expect))
        fail(kFormatError, "sketch file: unexpected hash independence for this sketch kind");
    for (std::uint64_t d = 0; d < cnt; ++d) {
        out[d] = get_u64(is);
        if (out[d] >= kHashPrime) fail(kInvalidArgument, "PolyHash: coefficient out of range");
    }
}
void put_data(std::ostream& os, const std::vector<double>& d) {
    for (double x : d) {
        std::uint64_t bits;
        std::memcpy(&bits, &x, 8);
        put_u64(os, bits);
    }
}
void get_data(std::istream& is, std::vector<double>& d) {
    for (double& x : d) {
        const std::uint64_t bits = get_u64(is);
        std::memcpy(&x, &bits, 8);
    }
}
struct FileHeader {
    std::uint64_t mode, n, b, B, seed;
};
FileHeader read_header(std::istream& is) {
    char magic[8];
    is.read(magic, 8);
    if (!is || std::memcmp(magic, kMagic, 8) != 0) fail(kFormatError, "sketch file: bad magic");
    if (get_u64(is) != 1) fail(kFormatError, "sketch file: unsupported version");
    FileHeader h;
    h.mode = get_u64(is);
    if (h.mode > 1) fail(kFormatError, "sketch file: unknown mode");
    h.n = get_u64(is);
    h.b = get_u64(is);
    h.B = get_u64(is);
    h.seed = get_u64(is);
    if (h.n == 0 || h.B == 0 || !is_pow2(h.b)) fail(kFormatError, "sketch file: invalid header");
    return h;
}
void write_header(std::ostream& os, std::uint64_t mode, std::uint64_t n, std::uint64_t b, std::uint64_t B,
                  std::uint64_t seed) {
    os.write(kMagic, 8);
    put_u64(os, 1);
    put_u64(os, mode);
    put_u64(os, n);
    put_u64(os, b);
    put_u64(os, B);
    put_u64(os, seed);
}
}  // namespace

int skc_peek_sketch_mode(const char* path, int* mode) {
    return guard([&] {
        check_vec(path, "path");
        std::ifstream is(path, std::ios::binary);
        if (!is) fail(kFormatError, std::string("cannot open sketch file: ") + path);
        *mode = static_cast<int>(read_header(is).mode);
    });
}

int skc_sym_save(const skc_sym_set* s, const char* path) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(path, "path");
        std::vector<double> data(static_cast<size_t>(s->B) * s->b * 2);
        s->ctx->use();
        CK(cudaMemcpyAsync(data.data(), s->data.p, data.size() * 8, cudaMemcpyDeviceToHost, s->ctx->stream));
        s->ctx->sync();
        std::ofstream os(path, std::ios::binary);
        if (!os) fail(kFormatError, std::string("cannot write sketch file: ") + path);
        write_header(os, 1, s->n, s->b, s->B, s->seed);
        std::vector<double> rep(2 * static_cast<size_t>(s->b));
        for (int m = 0; m < s->B; ++m) {
            put_coeffs(os, &s->hcoef[m * 6], 6);
            put_coeffs(os, &s->scoef[m * 6], 6);
            std::copy(data.begin() + static_cast<long>(m) * 2 * s->b, data.begin() + static_cast<long>(m + 1) * 2 * s->b,
                      rep.begin());
            put_data(os, rep);
        }
        if (!os) fail(kFormatError, std::string("write failure on sketch file: ") + path);
    });
}

int skc_sym_load(skc_context* ctx, const char* path, skc_sym_set** out) {
    return guard([&] {
        check_vec(ctx, "context");
        check_vec(path, "path");
        std::ifstream is(path, std::ios::binary);
        if (!is) fail(kFormatError, std::string("cannot open sketch file: ") + path);
        const FileHeader h = read_header(is);
        if (h.mode != 1) fail(kFormatError, std::string(path) + ": not a symmetric sketch file");
        require(h.n <= 0x7fffffffull && h.B <= 0x7fffffffull && h.b <= (1ull << 28), "sketch file: dimensions too large");
        const int n = static_cast<int>(h.n), B = static_cast<int>(h.B);
        const std::uint32_t b = static_cast<std::uint32_t>(h.b);
        std::vector<std::uint64_t> hc(static_cast<size_t>(B) * 6), sc(static_cast<size_t>(B) * 6);
        std::vector<double> data(static_cast<size_t>(B) * b * 2), rep(2 * static_cast<size_t>(b));
        for (int m = 0; m < B; ++m) {
            get_coeffs(is, 6, &hc[m * 6]);
            get_coeffs(is, 6, &sc[m * 6]);
            get_data(is, rep);
            std::copy(rep.begin(), rep.end(), data.begin() + static_cast<long>(m) * 2 * b);
        }
        const int st = skc_sym_create_from_coefficients(ctx, n, b, B, h.seed, hc.data(), sc.data(), data.data(), out);
        if (st != kOk) fail(st, g_last_error);
    });
}

int skc_asym_save(const skc_asym_set* s, const char* path) {
    return guard([&] {
        check_vec(s, "set");
        check_vec(path, "path");
        std::vector<double> data(static_cast<size_t>(s->B) * s->b * 2);
        s->ctx->use();
        CK(cudaMemcpyAsync(data.data(), s->data.p, data.size() * 8, cudaMemcpyDeviceToHost, s->ctx->stream));
        s->ctx->sync();
        std::ofstream os(path, std::ios::binary);
        if (!os) fail(kFormatError, std::string("cannot write sketch file: ") + path);
        write_header(os, 0, s->n, s->b, s->B, s->seed);
        std::vector<double> rep(2 * static_cast<size_t>(s->b));
        for (int m = 0; m < s->B; ++m) {
            for (int sl = 0; sl < 3; ++sl) put_coeffs(os, &s->hcoef[(m * 3 + sl) * 2], 2);
            for (int sl = 0; sl < 3; ++sl) put_coeffs(os, &s->xcoef[(m * 3 + sl) * 6], 6);
            std::copy(data.begin() + static_cast<long>(m) * 2 * s->b, data.begin() + static_cast<long>(m + 1) * 2 * s->b,
                      rep.begin());
            put_data(os, rep);
        }
        if (!os) fail(kFormatError, std::string("write failure on sketch file: ") + path);
    });
}

int skc_asym_load(skc_context* ctx, const char* path, skc_asym_set** out) {
    return guard([&] {
        check_vec(ctx, "context");
        check_vec(path, "path");
        std::ifstream is(path, std::ios::binary);
        if (!is) fail(kFormatError, std::string("cannot open sketch file: ") + path);
        const FileHeader h = read_header(is);
        if (h.mode != 0) fail(kFormatError, std::string(path) + ": not an asymmetric sketch file");
        require(h.n <= 0x7fffffffull && h.B <= 0x7fffffffull && h.b <= (1ull << 28), "sketch file: dimensions too large");
        const int n = static_cast<int>(h.n), B = static_cast<int>(h.B);
        const std::uint32_t b = static_cast<std::uint32_t>(h.b);
        std::vector<std::uint64_t> hc(static_cast<size_t>(B) * 6), xc(static_cast<size_t>(B) * 18);
        std::vector<double> data(static_cast<size_t>(B) * b * 2), rep(2 * static_cast<size_t>(b));
        for (int m = 0; m < B; ++m) {
            for (int sl = 0; sl < 3; ++sl) get_coeffs(is, 2, &hc[(m * 3 + sl) * 2]);
            for (int sl = 0; sl < 3; ++sl) get_coeffs(is, 6, &xc[(m * 3 + sl) * 6]);
            get_data(is, rep);
            std::copy(rep.begin(), rep.end(), data.begin() + static_cast<long>(m) * 2 * b);
        }
        const int st = skc_asym_create_from_coefficients(ctx, n, b, B, h.seed, hc.data(), xc.data(), data.data(), out);
        if (st != kOk) fail(st, g_last_error);
    });
}

// ---- generators ----
static void planted_factors(int n, int rank, std::uint64_t seed, double* lambda, double* V) {
    Rng lr(derive_seed(seed, seed_tag::kGenLambda));
    for (int r = 0; r < rank; ++r) lambda[r] = 1.0 + lr.uniform();  // U[1,2]
    Rng br(derive_seed(seed, seed_tag::kGenBasis));
    for (int r = 0; r < rank; ++r)
        for (int i = 0; i < n; ++i) V[static_cast<size_t>(r) * n + i] = br.gaussian();
    // modified Gram-Schmidt, two passes (orthonormal columns = Q of a QR)
    for (int pass = 0; pass < 2; ++pass)
        for (int r = 0; r < rank; ++r) {
            double* v = V + static_cast<size_t>(r) * n;
            for (int q = 0; q < r; ++q) {
                const double* w = V + static_cast<size_t>(q) * n;
                double d = 0;
                for (int i = 0; i < n; ++i) d += v[i] * w[i];
                for (int i = 0; i < n; ++i) v[i] -= d * w[i];
            }
            double s = 0;
            for (int i = 0; i < n; ++i) s += v[i] * v[i];
            const double inv = 1.0 / std::sqrt(s);
            for (int i = 0; i < n; ++i) v[i] *= inv;
        }
}

int skc_gen_planted_tensor(int n, int rank, double sigma, uint64_t seed, int dtype, void* T_out, double* lambda_out,
                           double* V_out) {
    return guard([&] {
        require(n >= 1 && rank >= 1 && rank <= n, "gen_planted_tensor: need 1 <= rank <= n");
        require(dtype == SKC_F64 || dtype == SKC_F32, "gen_planted_tensor: bad dtype");
        check_vec(T_out, "gen_planted_tensor: T");
        std::vector<double> lam(rank), V(static_cast<size_t>(rank) * n);
        planted_factors(n, rank, seed, lam.data(), V.data());
        if (lambda_out) std::copy(lam.begin(), lam.end(), lambda_out);
        if (V_out) std::copy(V.begin(), V.end(), V_out);
        // noise for the sorted triples in loop order, mirrored (tensor.cpp:228-244 convention)
        Rng nr(derive_seed(seed, seed_tag::kGenNoise));
        auto put = [&](size_t off, double x) {
            if (dtype == SKC_F64)
                static_cast<double*>(T_out)[off] = x;
            else
                static_cast<float*>(T_out)[off] = static_cast<float>(x);
        };
        for (int i = 0; i < n; ++i)
            for (int j = i; j < n; ++j)
                for (int k = j; k < n; ++k) {
                    double s = 0;
                    for (int r = 0; r < rank; ++r)
                        s += lam[r] * V[static_cast<size_t>(r) * n + i] * V[static_cast<size_t>(r) * n + j] *
                             V[static_cast<size_t>(r) * n + k];
                    if (sigma > 0) s += sigma * nr.gaussian();
                    const int p[6][3] = {{i, j, k}, {i, k, j}, {j, i, k}, {j, k, i}, {k, i, j}, {k, j, i}};
                    for (auto& q : p) put((static_cast<size_t>(q[0]) * n + q[1]) * n + q[2], s);
                }
    });
}

int skc_gen_planted_tensor_device(skc_context* ctx, int n, int rank, double sigma, uint64_t seed, int dtype,
                                  void* dev_out, double* lambda_out, double* V_out) {
    return guard([&] {
        check_vec(ctx, "context");
        require(n >= 1 && rank >= 1 && rank <= n, "gen_planted_tensor: need 1 <= rank <= n");
        require(dtype == SKC_F64 || dtype == SKC_F32, "gen_planted_tensor: bad dtype");
        ctx->use();
        std::vector<double> lam(rank), V(static_cast<size_t>(rank) * n);
        planted_factors(n, rank, seed, lam.data(), V.data());
        if (lambda_out) std::copy(lam.begin(), lam.end(), lambda_out);
        if (V_out) std::copy(V.begin(), V.end(), V_out);
        DevBuf<double> dl, dv;
        dl.upload(lam.data(), lam.size(), ctx->stream);
        dv.upload(V.data(), V.size(), ctx->stream);
        launch_gen_planted(ctx->stream, n, rank, dl.p, dv.p, sigma, derive_seed(seed, seed_tag::kGenNoise), dtype,
                           dev_out);
        ctx->check_launch();
        ctx->sync();
    });
}

}  // extern "C"
