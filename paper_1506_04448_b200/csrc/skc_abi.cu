// C-ABI implementation (include/sketchcp_b200.h): host C++ orchestration of the
// sm_100a kernels in skc_kernels.cu. Mirrors the reference classes in
// proj/include/sketchcp/{sketch,contraction,decompose}.hpp: validation, error
// messages and exception taxonomy follow the reference; compute runs only on the GPU.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <fstream>
#include <tuple>
#include <vector>

#include "../../include/sketchcp_b200.h"
#include "skc_fft.cuh"
#include "skc_host.hpp"
#include "skc_internal.hpp"

using namespace skc;

namespace {

thread_local std::string g_last_error;

#define CK(call)                                                                                     \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess) {                                                                     \
            int code_ = (e_ == cudaErrorMemoryAllocation) ? kOutOfMemory : kCudaError;               \
            fail(code_, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call);        \
        }                                                                                            \
    } while (0)

template <typename F>
int guard(F&& f) {
    try {
        f();
        return kOk;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return kOutOfMemory;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return kNumericalError;
    }
}

// RAII device buffer.
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t count = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        count = 0;
    }
    void alloc(size_t c) {
        if (c <= count && p) return;
        release();
        if (c == 0) c = 1;
        CK(cudaMalloc(&p, c * sizeof(T)));
        count = c;
    }
    void upload(const T* h, size_t c, cudaStream_t st) {
        alloc(c);
        CK(cudaMemcpyAsync(p, h, c * sizeof(T), cudaMemcpyHostToDevice, st));
    }
};

// integer knob from the environment, clamped to [lo, hi] (A/B experiment hooks)
int env_int(const char* name, int dflt, int lo, int hi) {
    const char* e = std::getenv(name);
    if (!e) return dflt;
    return std::min(hi, std::max(lo, std::atoi(e)));
}

int local_length(std::uint32_t b) {
    static int pref = [] {
        const char* e = std::getenv("SKC_LOCAL_N");
        int v = e ? std::atoi(e) : 2048;
        if (v < 2 || !is_pow2(static_cast<std::uint64_t>(v)) || v > 4096) v = 2048;
        return v;
    }();
    return static_cast<int>(std::min<std::uint32_t>(b, static_cast<std::uint32_t>(pref)));
}

std::vector<double> host_twiddles(std::uint32_t b) {
    std::vector<double> tw(2 * static_cast<size_t>(b));
    const long double two_pi = 6.283185307179586476925286766559005768L;
    for (std::uint32_t k = 0; k < b; ++k) {
        long double a = two_pi * static_cast<long double>(k) / static_cast<long double>(b);
        tw[2 * k] = static_cast<double>(cosl(a));
        tw[2 * k + 1] = static_cast<double>(sinl(a));
    }
    return tw;
}

}  // namespace

// ============================ context ============================================
struct skc_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t stream2 = nullptr;  // pipelined zero-copy builds: main pass of chunk c
    cudaEvent_t ev_q[5] = {};        // chunk c quantized / all chunks done
    cublasHandle_t cublas = nullptr;  // LDA whitening block products (lazy)
    int sms = 148;
    int smem_optin = 227 * 1024;
    std::map<std::uint32_t, std::unique_ptr<DevBuf<double2>>> twiddles;
    // dense-build row tables keyed by (n, i0, i1, sym)
    struct RowTab {
        DevBuf<std::uint32_t> rows;
        DevBuf<long long> offs;  // packed-stream offset of each row (= cum[row])
        std::vector<long long> cum;  // cumulative entries per row (host)
        int nrows = 0;

    };
    std::map<std::tuple<int, int, int, bool>, std::unique_ptr<RowTab>> rowtabs;
    // scratch
    DevBuf<unsigned char> tensor_stage;
    DevBuf<long long> qbuf;
    DevBuf<short> rowF;
    DevBuf<double> prepass;
    DevBuf<int> ints;  // [0] scale exp, [1] nonfinite, [2] best tau, [3..] misc
    DevBuf<double> dbl;  // [0] best value
    DevBuf<int> build_ints;                // per-type row counters of the dense build
    DevBuf<unsigned long long> build_acc;  // exact fixed-point slot accumulators
    DevBuf<double> U, part, values, freq_acc, X;
    DevBuf<double2> tmp;
    DevBuf<int> flags;
    DevBuf<unsigned long long> asym_key;

    // per-kernel event profiling (skc_profile_*)
    struct ProfRec {
        std::string name;
        cudaEvent_t a, b;
    };
    bool prof_on = false;
    std::vector<ProfRec> prof;

    void use() const { CK(cudaSetDevice(device)); }
    // w_N^k tables for the CTA-local transforms (contiguous; the full-b table would be
    // read at stride S)
    const double2* twl(int N) { return tw(static_cast<std::uint32_t>(N)); }
    const double2* tw(std::uint32_t b) {
        auto it = twiddles.find(b);
        if (it != twiddles.end()) return it->second->p;
        auto buf = std::make_unique<DevBuf<double2>>();
        std::vector<double> h = host_twiddles(b);
        buf->upload(reinterpret_cast<const double2*>(h.data()), b, stream);
        CK(cudaStreamSynchronize(stream));
        const double2* p = buf->p;
        twiddles[b] = std::move(buf);
        return p;
    }
    RowTab& rowtab(int n, int i0, int i1, bool sym) {
        auto key = std::make_tuple(n, i0, i1, sym);
        auto it = rowtabs.find(key);
        if (it != rowtabs.end()) return *it->second;
        auto rt = std::make_unique<RowTab>();
        std::vector<std::uint32_t> rows;
        rt->cum.push_back(0);
        for (int i = i0; i < i1; ++i)
            for (int j = sym ? i : 0; j < n; ++j) {
                rows.push_back((static_cast<std::uint32_t>(i) << 16) | static_cast<std::uint32_t>(j));
                rt->cum.push_back(rt->cum.back() + (sym ? (n - j) : n));
            }
        rt->nrows = static_cast<int>(rows.size());
        rt->rows.upload(rows.data(), rows.size(), stream);
        rt->offs.upload(rt->cum.data(), rows.size(), stream);
        CK(cudaStreamSynchronize(stream));
        RowTab& ref = *rt;
        rowtabs[key] = std::move(rt);
        return ref;
    }
    void sync() { CK(cudaStreamSynchronize(stream)); }
    void check_launch() { CK(cudaGetLastError()); }
};

// Records a CUDA event pair around the launches in its scope when profiling is on.
struct ProfScope {
    skc_context* c;
    const char* name;
    cudaEvent_t a = nullptr;
    ProfScope(skc_context* ctx, const char* nm) : c(ctx), name(nm) {
        if (!c->prof_on) return;
        CK(cudaEventCreate(&a));
        CK(cudaEventRecord(a, c->stream));
    }
    ~ProfScope() {
        if (!c->prof_on || !a) return;
        cudaEvent_t b = nullptr;
        if (cudaEventCreate(&b) != cudaSuccess) return;
        cudaEventRecord(b, c->stream);
        c->prof.push_back({name, a, b});
    }
};
#define SKC_CAT2(a, b) a##b
#define SKC_CAT(a, b) SKC_CAT2(a, b)
#define SKC_PROF(ctx, nm) ProfScope SKC_CAT(prof_scope_, __LINE__)(ctx, nm)

// ============================ sets ===============================================
struct skc_sym_set {
    skc_context* ctx = nullptr;
    int n = 0;
    std::uint32_t b = 2;
    int logb = 1;
    int B = 0;
    std::uint64_t seed = 0;
    std::uint64_t version = 0;
    std::vector<std::uint64_t> hcoef, scoef;  // B x 6 each
    DevBuf<std::uint64_t> d_hcoef, d_scoef;
    DevBuf<std::uint32_t> bucket1, bucket2, bucket3, packed, perm1, perm2;
    DevBuf<uint2> plan1, plan2;
    DevBuf<double2> stw1, stw2, gtw1, gtw2;  // residue twiddle tables (may stay empty)
    DevBuf<std::uint8_t> sexp;
    DevBuf<double2> data, spec;
    int N = 2, logN = 1, S = 1;
    std::uint64_t spec_version = ~0ull;
    bool spec_valid = false;

    SymView view() const {
        SymView v;
        v.n = n;
        v.b = b;
        v.logb = logb;
        v.B = B;
        v.bucket1 = bucket1.p;
        v.bucket2 = bucket2.p;
        v.bucket3 = bucket3.p;
        v.sexp = sexp.p;
        v.packed = packed.p;
        v.tw = ctx->tw(b);
        v.twl = ctx->twl(N);
        v.N = N;
        v.logN = logN;
        v.S = S;
        v.plan1 = plan1.p;
        v.plan2 = plan2.p;
        v.data = data.p;
        v.spec = spec.p;
        v.stw1 = stw1.p;
        v.stw2 = stw2.p;
        v.gtw1 = gtw1.p;
        v.gtw2 = gtw2.p;
        return v;
    }
    // contraction.cpp:62-72: refresh cached spectra when the version moved.
    void ensure_fresh() {
        if (spec_valid && spec_version == version) return;
        SKC_PROF(ctx, "spectrum");
        launch_spectrum(ctx->stream, data.p, b, logb, B, N, logN, S, ctx->tw(b), ctx->twl(N), spec.p);
        ctx->check_launch();
        spec_version = version;
        spec_valid = true;
    }
};

struct skc_asym_set {
    skc_context* ctx = nullptr;
    int n = 0;
    std::uint32_t b = 2;
    int logb = 1;
    int B = 0;
    std::uint64_t seed = 0;
    std::uint64_t version = 0;
    std::vector<std::uint64_t> hcoef, xcoef;  // B x 3 x 2, B x 3 x 6
    DevBuf<std::uint64_t> d_hcoef, d_xcoef;
    DevBuf<std::uint32_t> bucket, packed, perm;
    DevBuf<uint2> plan;
    DevBuf<double> sign;
    DevBuf<double2> data, spec;
    int N = 2, logN = 1, S = 1;
    std::uint64_t spec_version = ~0ull;
    bool spec_valid = false;

    AsymView view() const {
        AsymView v;
        v.n = n;
        v.b = b;
        v.logb = logb;
        v.B = B;
        v.bucket = bucket.p;
        v.sign = sign.p;
        v.packed = packed.p;
        v.tw = ctx->tw(b);
        v.twl = ctx->twl(N);
        v.N = N;
        v.logN = logN;
        v.S = S;
        v.plan = plan.p;
        v.data = data.p;
        v.spec = spec.p;
        return v;
    }
    void ensure_fresh() {
        if (spec_valid && spec_version == version) return;
        SKC_PROF(ctx, "spectrum");
        launch_spectrum(ctx->stream, data.p, b, logb, B, N, logN, S, ctx->tw(b), ctx->twl(N), spec.p);
        ctx->check_launch();
        spec_version = version;
        spec_valid = true;
    }
};

namespace {

void validate_set_args(int n, std::uint32_t b, int B) {
    // sketch.cpp:157-159 / 302-304
    require(n >= 1, "sketch set: dimension must be positive");
    require(B >= 1, "sketch set: need at least one replicate");
    require(is_pow2(b), "sketch set: b must be a power of two");
    require(b >= 2, "PolyHash: need at least 2 buckets");
    require(b <= (1u << 28), "sketch set: b above 2^28 is not supported by the packed bucket tables");
}

void check_vec(const void* p, const char* what) { require(p != nullptr, std::string(what) + ": null pointer"); }

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

// ---- dense build orchestration ------------------------------------------------------
// Device-visible view of the input tensor. Device pointers are used as is. Pinned
// (page-locked, UVA-mapped) host memory is read in place by the quantize pass, so only
// the bytes the build reads cross the bus. Pageable host memory is staged, copying only
// the row blocks the build reads (sym: T[i][i:n][:], asym: T[i0:i1]) unless the full
// tensor is needed by the symmetry check.
const void* stage_tensor(skc_context* ctx, const void* T, int n, int dtype, int location, bool sym, int i0, int i1,
                         bool need_full, size_t* h2d_bytes, bool* zero_copy = nullptr) {
    if (h2d_bytes) *h2d_bytes = 0;
    if (zero_copy) *zero_copy = false;
    if (location == SKC_DEVICE) return T;
    const size_t es = dtype == SKC_F64 ? 8 : 4;
    const size_t n2 = static_cast<size_t>(n) * n;
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, T) == cudaSuccess && attr.type == cudaMemoryTypeHost &&
        attr.devicePointer != nullptr) {
        if (zero_copy) *zero_copy = true;
        return attr.devicePointer;
    }
    cudaGetLastError();  // clear a failed attribute query on pageable memory
    ctx->tensor_stage.alloc(n2 * n * es);
    unsigned char* dst = ctx->tensor_stage.p;
    const unsigned char* src = static_cast<const unsigned char*>(T);
    size_t moved = 0;
    if (need_full) {
        CK(cudaMemcpyAsync(dst, src, n2 * n * es, cudaMemcpyHostToDevice, ctx->stream));
        moved = n2 * n * es;
    } else if (sym) {
        for (int i = i0; i < i1; ++i) {
            const size_t off = (static_cast<size_t>(i) * n + i) * n * es, len = static_cast<size_t>(n - i) * n * es;
            CK(cudaMemcpyAsync(dst + off, src + off, len, cudaMemcpyHostToDevice, ctx->stream));
            moved += len;
        }
    } else {
        const size_t off = static_cast<size_t>(i0) * n2 * es, len = static_cast<size_t>(i1 - i0) * n2 * es;
        CK(cudaMemcpyAsync(dst + off, src + off, len, cudaMemcpyHostToDevice, ctx->stream));
        moved = len;
    }
    if (h2d_bytes) *h2d_bytes = moved;
    return dst;
}

void run_dense_build(skc_context* ctx, const void* Tdev, int n, int dtype, bool sym, int i0, int i1, int B,
                     std::uint32_t b, const std::uint32_t* packed, double2* data, bool zero_copy) {
    if (i0 >= i1) return;
    skc_context::RowTab& rt = ctx->rowtab(n, i0, i1, sym);
    if (rt.nrows == 0) return;
    const long long total_slots = static_cast<long long>(B) * (sym ? 2ll * b : static_cast<long long>(b));
    // slots per CTA limited by shared memory (limbs + per-replicate hash tables)
    int G = 1;
    for (;; ++G) {
        long long spc = ((total_slots + G - 1) / G + 31) / 32 * 32;
        const long long spr0 = sym ? 2ll * b : static_cast<long long>(b);
        int Rg = 1;
        for (int g = 0; g < G; ++g) {
            const long long lo = g * spc, hi = std::min(lo + spc, total_slots);
            if (hi > lo) Rg = std::max(Rg, static_cast<int>((hi - 1) / spr0 - lo / spr0 + 1));
        }
        if (Rg <= 16 && build_smem_bytes(spc, Rg, n) <= static_cast<size_t>(ctx->smem_optin - 1024)) break;
        if (G > 4096) fail(kInvalidArgument, "accumulate_dense: sketch set too large for the dense build");
    }
    long long spc = (total_slots + G - 1) / G;
    spc = (spc + 31) / 32 * 32;
    if (const char* e = std::getenv("SKC_BUILD_SPC")) {  // experiment hook: forced window size
        const long long f = std::atoll(e) / 32 * 32;
        if (f >= 32 && f <= spc * 4 && build_smem_bytes(f, 16, n) <= static_cast<size_t>(ctx->smem_optin - 1024)) {
            spc = f;
            G = static_cast<int>((total_slots + spc - 1) / spc);
        }
    }
    const long long spr = sym ? 2ll * b : static_cast<long long>(b);
    int R = 1;
    std::vector<int> Rg(G, 1);
    for (int g = 0; g < G; ++g) {
        const long long lo = g * spc, hi = std::min(lo + spc, total_slots);
        if (hi > lo) Rg[g] = static_cast<int>((hi - 1) / spr - lo / spr + 1);
        R = std::max(R, Rg[g]);
    }
    require(R <= 16, "accumulate_dense: slot range spans too many replicates");
    const long long tot = rt.cum.back();
    const int P = std::max(1, ctx->sms);  // one persistent CTA per SM, rows handed out dynamically
    ctx->build_ints.alloc(static_cast<size_t>(G));
    ctx->build_acc.alloc(static_cast<size_t>(total_slots));
    ctx->qbuf.alloc(static_cast<size_t>(std::max<long long>(1, tot)));
    ctx->rowF.alloc(static_cast<size_t>(rt.nrows));
    ctx->prepass.alloc(kPrepassBlocks);
    ctx->ints.alloc(16);

    BuildPlan p;
    p.n = n;
    p.sym = sym;
    p.dtype = dtype;
    p.rowtab = rt.rows.p;
    p.nrows = rt.nrows;
    p.P = P;
    p.G = G;
    p.next_row = ctx->build_ints.p;
    p.acc = ctx->build_acc.p;
    static const bool row_variant = [] {
        const char* e = std::getenv("SKC_BUILD_KERNEL");
        return e && std::string(e) == "rows";
    }();
    // flat kernel's doubled SYM tables need bucket sums below bit 30: b <= 2^27 (larger
    // sets take the row-walk kernel, which uses the plain packed form)
    p.flat = !row_variant && (!sym || b <= (1u << 27));
    static const bool trace_on = std::getenv("SKC_BUILD_TRACE") != nullptr;
    DevBuf<unsigned long long> trace;
    p.trace = nullptr;
    if (trace_on) {
        trace.alloc(3 * static_cast<size_t>(P));
        p.trace = trace.p;
    }
    p.total_slots = total_slots;
    p.slots_per_cta = static_cast<int>(spc);
    p.R = R;
    p.bmask = b - 1;
    p.B = B;
    p.packed = packed;
    p.rowoff = rt.offs.p;
    p.qbuf = ctx->qbuf.p;
    p.rowF = ctx->rowF.p;
    p.prepass_partials = ctx->prepass.p;
    p.scale_exp = ctx->ints.p;
    p.nonfinite = ctx->ints.p + 1;
    p.data_as_double = reinterpret_cast<double*>(data);
    // Zero-copy host input: the quantize pass is bus-bound, so the rows are cut into K
    // chunks and chunk c+1 is read over PCIe (a few SMs, wide blocks) while the main pass
    // of chunk c runs on the other SMs (second stream). Each chunk keeps its own exponent
    // and exact accumulator; the finalize sums the K chunk sketches in order.
    static const bool pipe_on = [] {
        const char* e = std::getenv("SKC_BUILD_PIPELINE");  // "0": A/B switch for the chunked path
        return !(e && std::string(e) == "0");
    }();
    const int K = (pipe_on && zero_copy && rt.nrows >= 4096 &&
                   sizeof(double) * 32 * (size_t)n <= (size_t)ctx->smem_optin - 1024)
                      ? env_int("SKC_BUILD_K", 4, 2, 4)
                      : 1;
    if (K > 1) {
        const int qsms = env_int("SKC_BUILD_QSMS", 16, 1, 64);  // SMs given to the bus-bound quantize pass
        p.P = std::max(1, ctx->sms - qsms);
        p.prepass_threads = 1024;
        p.prepass_blocks = qsms;
        p.prepass_warps = 32;
        ctx->build_acc.alloc(static_cast<size_t>(K) * total_slots);
        ctx->build_ints.alloc(static_cast<size_t>(K) * G);
        ctx->ints.alloc(16);
        ctx->prepass.alloc(static_cast<size_t>(K) * qsms);
        if (!ctx->stream2) CK(cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking));
        if (!ctx->ev_q[0])
            for (int c = 0; c < 5; ++c) CK(cudaEventCreateWithFlags(&ctx->ev_q[c], cudaEventDisableTiming));
        // decreasing chunk sizes: chunk c's main pass (~0.4x the bus time of its rows) hides
        // under chunk c+1's bus reads, and the exposed tail (last main pass) stays short
        static const double kFrac4[5] = {0.0, 0.42, 0.72, 0.90, 1.0};
        std::vector<int> rb(K + 1, 0);
        for (int c = 1; c < K; ++c) {
            const long long target = (K == 4) ? static_cast<long long>(static_cast<double>(tot) * kFrac4[c]) : tot * c / K;
            rb[c] = static_cast<int>(std::lower_bound(rt.cum.begin(), rt.cum.end(), target) - rt.cum.begin());
            rb[c] = std::min(std::max(rb[c], rb[c - 1]), rt.nrows);
        }
        rb[K] = rt.nrows;
        CK(cudaMemsetAsync(p.nonfinite, 0, sizeof(int), ctx->stream));
        {
            SKC_PROF(ctx, "build_pipelined");
            static const bool ptrace = std::getenv("SKC_PIPE_TRACE") != nullptr;
            cudaEvent_t te[4][5];
            if (ptrace)
                for (auto& row : te)
                    for (auto& e : row) CK(cudaEventCreate(&e));
            if (ptrace) CK(cudaEventRecord(te[0][0], ctx->stream));
            for (int c = 0; c < K; ++c) {
                BuildPlan pc = p;
                pc.rowtab = rt.rows.p + rb[c];
                pc.rowoff = rt.offs.p + rb[c];
                pc.rowF = ctx->rowF.p + rb[c];
                pc.nrows = rb[c + 1] - rb[c];
                pc.prepass_partials = ctx->prepass.p + static_cast<size_t>(c) * qsms;
                pc.scale_exp = ctx->ints.p + 4 + c;
                pc.reset_nonfinite = false;
                pc.acc = ctx->build_acc.p + static_cast<size_t>(c) * total_slots;
                pc.next_row = ctx->build_ints.p + static_cast<size_t>(c) * G;
                if (ptrace) CK(cudaEventRecord(te[0][c + 1 < 5 ? c + 1 : 4], ctx->stream));
                if (pc.nrows > 0) launch_build_prepass(ctx->stream, Tdev, pc);
                if (ptrace) CK(cudaEventRecord(te[1][c], ctx->stream));
                CK(cudaEventRecord(ctx->ev_q[c], ctx->stream));
                CK(cudaStreamWaitEvent(ctx->stream2, ctx->ev_q[c], 0));
                if (pc.nrows > 0) {
                    if (ptrace) CK(cudaEventRecord(te[2][c], ctx->stream2));
                    launch_build_main(ctx->stream2, Tdev, pc);
                    if (ptrace) CK(cudaEventRecord(te[3][c], ctx->stream2));
                } else {
                    CK(cudaMemsetAsync(pc.acc, 0, sizeof(unsigned long long) * (size_t)total_slots, ctx->stream2));
                }
            }
            CK(cudaEventRecord(ctx->ev_q[K], ctx->stream2));
            CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_q[K], 0));
            BuildPlan pf = p;
            pf.acc = ctx->build_acc.p;
            launch_build_finalize_multi(ctx->stream, pf, K, ctx->ints.p + 4);
            if (ptrace) {
                ctx->sync();
                for (int c = 0; c < K && c < 4; ++c) {
                    float q0, q1, m0, m1;
                    cudaEventElapsedTime(&q0, te[0][0], te[0][c + 1 < 5 ? c + 1 : 4]);
                    cudaEventElapsedTime(&q1, te[0][0], te[1][c]);
                    cudaEventElapsedTime(&m0, te[0][0], te[2][c]);
                    cudaEventElapsedTime(&m1, te[0][0], te[3][c]);
                    std::fprintf(stderr, "chunk %d quantize %.3f-%.3f ms main %.3f-%.3f ms\n", c, q0, q1, m0, m1);
                }
                for (auto& row : te)
                    for (auto& e : row) cudaEventDestroy(e);
            }
        }
        ctx->check_launch();
    } else {
        {
            SKC_PROF(ctx, "build_prepass");
            launch_build_prepass(ctx->stream, Tdev, p);
        }
        ctx->check_launch();
        {
            SKC_PROF(ctx, "build_main");
            launch_build_main(ctx->stream, Tdev, p);
        }
        ctx->check_launch();
        {
            SKC_PROF(ctx, "build_finalize");
            launch_build_finalize(ctx->stream, p);  // device-side no-op when nonfinite
        }
        ctx->check_launch();
    }
    int nonfinite = 0;
    CK(cudaMemcpyAsync(&nonfinite, p.nonfinite, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    // Fixed-point accumulation cannot carry NaN/Inf the way the reference's
    // floating-point sum would; reject instead of producing a wrong sketch.
    if (nonfinite) fail(kInvalidArgument, "accumulate_dense: tensor has a non-finite entry");
    if (trace_on) {
        std::vector<unsigned long long> t(3 * static_cast<size_t>(P));
        CK(cudaMemcpy(t.data(), trace.p, t.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        unsigned long long t0 = ~0ull;
        for (int x = 0; x < P; ++x) t0 = std::min(t0, t[3 * x]);
        std::fprintf(stderr, "build trace: G=%d spc=%lld P=%d\n", G, spc, P);
        for (int x = 0; x < P; ++x)
            std::fprintf(stderr, "cta %3d start %7.1f us dur %7.1f us switches %llu\n", x, (t[3 * x] - t0) * 1e-3,
                         (t[3 * x + 1] - t[3 * x]) * 1e-3, t[3 * x + 2]);
    }
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


// ---- LDA moments and whitening (lda.cpp:88-143; kernels in skc_whiten.cu) ---------------
#define CB(call)                                                                                      \
    do {                                                                                              \
        cublasStatus_t st_ = (call);                                                                  \
        if (st_ != CUBLAS_STATUS_SUCCESS)                                                             \
            fail(kCudaError, std::string("cuBLAS error ") + std::to_string(static_cast<int>(st_)) + " at " #call); \
    } while (0)

cublasHandle_t cublas_of(skc_context* ctx) {
    if (!ctx->cublas) CB(cublasCreate(&ctx->cublas));
    CB(cublasSetStream(ctx->cublas, ctx->stream));
    return ctx->cublas;
}

// Corpus on the device: CSR (document-major) and its word-major transpose, per-document
// weights and per-word diagonal / M1 sums.
struct CorpusDev {
    int V = 0;
    long long D = 0, nnz = 0, used1 = 0, used2 = 0, used3 = 0;
    DevBuf<long long> used_docs;  // documents with >= 3 tokens (sketch_whitened_m3, lda.cpp:164-168)
    DevBuf<long long> doc_ptr, cptr, cdoc, total;
    DevBuf<int> word, count, ccount;
    DevBuf<double> s2, invm, diag, m1p;
    // word-pass chunks (load balance over Zipf-heavy words): [chunk_lo, chunk_hi) CSC
    // ranges, word w owns chunks [word_chunk[w], word_chunk[w+1])
    long long nchunks = 0;
    DevBuf<long long> chunk_lo, chunk_hi, word_chunk;
};

void upload_corpus(skc_context* ctx, int V, long long D, const long long* doc_ptr, const int* word, const int* count,
                   CorpusDev& c, const std::string& who = "lda", bool check_counts = true) {
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

// Q (V x p row-major = p x V col-major) = orthonormal basis of range(Y): CholeskyQR2 with
// DGEMM Gram products; modified Gram-Schmidt on the host (with random completion) when
// the Gram matrix is not numerically positive definite (rank-deficient block).
struct OrthWork {
    DevBuf<double> G, Rinv, tmp;
};
void orthonormalize(skc_context* ctx, int V, int p, const double* Yd, double* Qd, OrthWork& w, Rng& rng) {
    cublasHandle_t h = cublas_of(ctx);
    const double one = 1.0, zero = 0.0;
    w.G.alloc(static_cast<size_t>(p) * p);
    w.Rinv.alloc(static_cast<size_t>(p) * p);
    w.tmp.alloc(static_cast<size_t>(V) * p);
    std::vector<double> G(static_cast<size_t>(p) * p), Ri(static_cast<size_t>(p) * p);
    const double* src = Yd;
    for (int pass = 0; pass < 2; ++pass) {
        CB(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, p, p, V, &one, src, p, src, p, &zero, w.G.p, p));
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
        CB(cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, p, V, p, &one, w.Rinv.p, p, src, p, &zero, dst, p));
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
    static const bool trace = std::getenv("SKC_WHITEN_TRACE") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto tick = [&](const char* what) {
        if (!trace) return;
        ctx->sync();
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "whiten %-12s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
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
    cublasHandle_t h = cublas_of(ctx);
    const double one = 1.0, zero = 0.0;
    DevBuf<double> Hd;
    Hd.alloc(static_cast<size_t>(p) * p);
    CB(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, p, p, V, &one, Q.p, p, Y.p, p, &zero, Hd.p, p));
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
    CB(cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, k, V, p, &one, Ukd.p, p, Q.p, p, &zero, Vk.p, k));
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

// sketch_whitened_m3 (lda.cpp:145-226) on an uploaded corpus.
// Shard mode (global_m1 != null): the document sums run over this corpus only, while the
// normalisation 1/D_used (global_used) and q = W^T m1 (global_m1, V, already averaged)
// are the whole corpus'; add_q_cubed selects the one shard that adds c_m1 F(q)^3. The
// sketch is linear in the per-document terms, so summing the shards' data reproduces the
// full sketch_whitened_m3.
void sketch_whitened_m3_dev(skc_sym_set* s, CorpusDev& c, const double* W, double alpha0, long long* used_out,
                            long long* skipped_out, long long global_used = -1, const double* global_m1 = nullptr,
                            bool add_q_cubed = true) {
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
    const int chunks_d = std::max(1, static_cast<int>(std::min<long long>(std::max<long long>(used, 1), (8ll * ctx->sms) / per_rep)));
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

}  // namespace

// ============================ C-ABI ==============================================
struct skc_lda_corpus {
    skc_context* ctx = nullptr;
    CorpusDev dev;
};

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
        if (ctx->cublas) cublasDestroy(ctx->cublas);
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
        ctx->prof_on = on != 0;
    });
}
int skc_profile_reset(skc_context* ctx) {
    return guard([&] {
        check_vec(ctx, "context");
        ctx->use();
        ctx->sync();
        for (auto& r : ctx->prof) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
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
        if (!assume_symmetric) {
            ctx->asym_key.alloc(1);
            unsigned long long init = ~0ull;
            CK(cudaMemcpyAsync(ctx->asym_key.p, &init, 8, cudaMemcpyHostToDevice, ctx->stream));
            long long tot = static_cast<long long>(s->n) * s->n * s->n;
            k_first_asym<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, ctx->stream>>>(Td, dtype, s->n, 1e-9,
                                                                                           ctx->asym_key.p);
            count_launch();
            ctx->check_launch();
            unsigned long long key = 0;
            CK(cudaMemcpyAsync(&key, ctx->asym_key.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
            ctx->sync();
            if (key != ~0ull) {
                const long long idx = static_cast<long long>(key >> 3);
                const int p = static_cast<int>(key & 7);
                const int n = s->n;
                const int i = static_cast<int>(idx / ((long long)n * n)), j = static_cast<int>((idx / n) % n),
                          k = static_cast<int>(idx % n);
                const int perms[5][3] = {{i, k, j}, {j, i, k}, {j, k, i}, {k, i, j}, {k, j, i}};
                fail(kInvalidArgument, "accumulate_dense: input tensor is not symmetric at (" +
                                           std::to_string(perms[p][0] + 1) + "," + std::to_string(perms[p][1] + 1) +
                                           "," + std::to_string(perms[p][2] + 1) + ")");
            }
        }
        s->version++;  // sketch.cpp:324
        run_dense_build(ctx, Td, s->n, dtype, true, i0, i1, s->B, s->b, s->packed.p, s->data.p, zc);
        ctx->sync();
    });
}

// Frequency-domain rank-1 / moment accumulation shared by add_scaled_rank1,
// accumulate_moment and RTPM deflation. X: device N x n.
static void sym_moment_device(skc_sym_set* s, const double* Xd, const double* wd, double alpha, long long Nsamp) {
    skc_context* ctx = s->ctx;
    const int per_rep = s->B * s->S;
    // ~4 waves of 2 resident CTAs per SM; one sample per chunk at most
    int chunks = static_cast<int>(std::max<long long>(1, std::min<long long>(Nsamp, (8ll * ctx->sms) / per_rep)));
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
    {
        SKC_PROF(ctx, "combine");
        launch_combine_residues(ctx->stream, ctx->tmp.p, s->B, s->S, s->N, s->b, v.tw, alpha, -1, false, s->data.p);
    }
    ctx->check_launch();
}

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
        launch_median_rows(ctx->stream, ctx->part.p, L, s->B, s->S, s->n, ctx->values.p, nullptr, 0.0, nullptr);
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
        launch_sym_vvv_finish(ctx->stream, ctx->part.p, L, s->B, s->S, s->b, ctx->values.p);
        ctx->check_launch();
        CK(cudaMemcpyAsync(out_host, ctx->values.p, static_cast<size_t>(L) * 8, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
    });
}

// natural-order spectrum of replicate m from the residue/bit-reversed layout
static void spectrum_to_host(skc_context* ctx, const double2* spec, int m, std::uint32_t b, int N, int logN, int S,
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

int skc_sym_cached_transform(skc_sym_set* s, int m, double* out_host) {
    return guard([&] {
        check_vec(s, "set");
        require(m >= 0 && m < s->B, "replicate index out of range");
        s->ctx->use();
        s->ensure_fresh();
        spectrum_to_host(s->ctx, s->spec.p, m, s->b, s->N, s->logN, s->S, out_host);
    });
}

// ---- RTPM ----
// Runs T power steps on L restarts resident at ctx->U (device) and the median vvv of
// the finals into ctx->values. Degenerate flags accumulate in ctx->flags.
static void rtpm_restarts_device(skc_sym_set* s, int L, int T_iters, double tol) {
    skc_context* ctx = s->ctx;
    s->ensure_fresh();
    ctx->flags.alloc(static_cast<size_t>(L));
    CK(cudaMemsetAsync(ctx->flags.p, 0, sizeof(int) * L, ctx->stream));
    ctx->part.alloc(static_cast<size_t>(L) * s->B * s->S * std::max(s->n, 3));
    const SymView v = s->view();
    for (int t = 0; t < T_iters; ++t) {
        {
            SKC_PROF(ctx, "sym_contract");
            launch_sym_contract(ctx->stream, v, ctx->U.p, L, 0, ctx->part.p);
        }
        SKC_PROF(ctx, "median");
        ctx->values.alloc(static_cast<size_t>(L) * s->n);
        launch_median_rows(ctx->stream, ctx->part.p, L, s->B, s->S, s->n, nullptr, ctx->U.p, tol, ctx->flags.p,
                           ctx->values.p);
    }
    ctx->check_launch();
    launch_sym_contract(ctx->stream, v, ctx->U.p, L, 1, ctx->part.p);
    ctx->values.alloc(static_cast<size_t>(L));
    launch_sym_vvv_finish(ctx->stream, ctx->part.p, L, s->B, s->S, s->b, ctx->values.p);
    ctx->check_launch();
}

static void check_degenerate(skc_context* ctx, int L) {
    std::vector<int> f(L);
    CK(cudaMemcpyAsync(f.data(), ctx->flags.p, sizeof(int) * L, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    for (int x : f)
        if (x) fail(kDegenerate, "power update produced a vanishing iterate");  // decompose.cpp:37-38
}

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
        std::vector<double> gen;
        if (!inits) {
            gen.resize(static_cast<size_t>(L) * n);
        }
        ctx->ints.alloc(16);
        ctx->dbl.alloc(4);
        ctx->X.alloc(static_cast<size_t>(n));
        for (int c = 0; c < k; ++c) {
            const double* U0;
            if (inits) {
                U0 = inits + static_cast<size_t>(c) * L * n;
            } else {
                for (int t = 0; t < L; ++t) {
                    Rng rng(derive_seed(seed, seed_tag::kPowerInit, static_cast<std::uint64_t>(c),
                                        static_cast<std::uint64_t>(t)));
                    rng.unit_sphere(n, gen.data() + static_cast<size_t>(t) * n);
                }
                U0 = gen.data();
            }
            ctx->U.upload(U0, static_cast<size_t>(L) * n, ctx->stream);
            rtpm_restarts_device(s, L, T_iters, tol);
            launch_argmax_first(ctx->stream, ctx->values.p, L, ctx->ints.p + 2, ctx->dbl.p);
            ctx->check_launch();
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
        cublasHandle_t h = cublas_of(ctx);
        const double one = 1.0, zero = 0.0;
        whiten_randomized(
            ctx, V, k, oversample, iters, seed,
            [&](const double* Xd, double* Yd, int p) {
                // Y^T (p x V) = X^T (p x V) M2 (V x V)
                CB(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, p, V, V, &one, Xd, p, Md.p, V, &zero, Yd, p));
            },
            W, unwhiten, singular_values);
    });
}


// lda.cpp:228-248: topics and prior from the whitened CP decomposition (host math, O(V k)).
int skc_lda_recover_params(int V, int k, const double* lambda, const double* A, const double* unwhiten, double alpha0,
                           double* Phi, double* alpha) {
    return guard([&] {
        require(k >= 1, "recover_params: empty decomposition");
        check_vec(lambda, "recover_params: lambda");
        check_vec(A, "recover_params: A");
        check_vec(unwhiten, "recover_params: unwhiten");
        check_vec(Phi, "recover_params: Phi");
        check_vec(alpha, "recover_params: alpha");
        require(V >= 1, "recover_params: decomposition/whitening rank mismatch");
        std::vector<double> mu(V);
        for (int i = 0; i < k; ++i) {
            const double lam = lambda[i];
            if (lam == 0.0) fail(kNumericalError, "recover_params: zero eigenvalue at component " + std::to_string(i + 1));
            alpha[i] = 4.0 * alpha0 * (alpha0 + 1.0) / ((alpha0 + 2.0) * (alpha0 + 2.0) * lam * lam);
            for (int w = 0; w < V; ++w) {  // mu = 0.5 (a0 + 2) lam * unwhiten A[:, i]
                double s = 0.0;
                for (int c = 0; c < k; ++c) s += unwhiten[static_cast<size_t>(w) * k + c] * A[static_cast<size_t>(c) * k + i];
                mu[w] = 0.5 * (alpha0 + 2.0) * lam * s;
            }
            const std::vector<double> ph = project_to_simplex(mu.data(), V);
            for (int w = 0; w < V; ++w) Phi[static_cast<size_t>(w) * k + i] = ph[w];
        }
    });
}

// lda.cpp:273-320: mean per-document held-out log-likelihood, mixtures by simplex-
// projected gradient (500 steps, stop at |step| <= 1e-8). Documents in parallel
// (each is independent; the final sum runs in document order).
int skc_lda_heldout_likelihood(int V, int k, const double* Phi, int Vh, long long D, const long long* doc_ptr,
                               const int* word, const int* count, double* ll_out, long long* floored_out) {
    return guard([&] {
        check_vec(Phi, "heldout_likelihood: Phi");
        check_vec(doc_ptr, "heldout_likelihood: doc_ptr");
        check_vec(ll_out, "heldout_likelihood: out");
        require(Vh <= V, "heldout_likelihood: corpus vocabulary exceeds the model's");
        std::vector<double> gram(static_cast<size_t>(k) * k, 0.0);
        for (int a = 0; a < k; ++a)
            for (int b = 0; b < k; ++b) {
                double s = 0.0;
                for (int w = 0; w < V; ++w) s += Phi[static_cast<size_t>(w) * k + a] * Phi[static_cast<size_t>(w) * k + b];
                gram[static_cast<size_t>(b) * k + a] = s;
            }
        std::vector<double> ev, U;
        sym_eigen_host(k, gram, ev, U);
        const double lips = ev.empty() ? 0.0 : ev.back();
        const double step = lips > 0 ? 1.0 / lips : 1.0;
        std::vector<double> per(static_cast<size_t>(std::max<long long>(D, 1)), 0.0);
        std::vector<long long> fl(static_cast<size_t>(std::max<long long>(D, 1)), 0);
        std::vector<char> used(static_cast<size_t>(std::max<long long>(D, 1)), 0);
#pragma omp parallel for schedule(dynamic, 16)
        for (long long d = 0; d < D; ++d) {
            long long tot = 0;
            for (long long q = doc_ptr[d]; q < doc_ptr[d + 1]; ++q) tot += count[q];
            if (tot < 1) continue;
            used[d] = 1;
            std::vector<double> pi(k, 1.0 / k);
            if (k > 1) {
                std::vector<double> phi_tw(k, 0.0), grad(k), next(k);
                const double inv_m = 1.0 / static_cast<double>(tot);
                for (long long q = doc_ptr[d]; q < doc_ptr[d + 1]; ++q)
                    for (int a = 0; a < k; ++a)
                        phi_tw[a] += (inv_m * count[q]) * Phi[static_cast<size_t>(word[q]) * k + a];
                for (int it = 0; it < 500; ++it) {
                    for (int a = 0; a < k; ++a) {
                        double s = 0.0;
                        for (int b = 0; b < k; ++b) s += gram[static_cast<size_t>(b) * k + a] * pi[b];
                        grad[a] = pi[a] - step * (s - phi_tw[a]);
                    }
                    next = project_to_simplex(grad.data(), k);
                    double moved = 0.0;
                    for (int a = 0; a < k; ++a) moved += (next[a] - pi[a]) * (next[a] - pi[a]);
                    pi.swap(next);
                    if (std::sqrt(moved) <= 1e-8) break;
                }
            } else {
                pi.assign(1, 1.0);
            }
            double ll = 0.0;
            for (long long q = doc_ptr[d]; q < doc_ptr[d + 1]; ++q) {
                double pw = 0.0;
                for (int a = 0; a < k; ++a) pw += Phi[static_cast<size_t>(word[q]) * k + a] * pi[a];
                if (pw < 1e-12) {
                    pw = 1e-12;
                    ++fl[d];
                }
                ll += count[q] * std::log(pw);
            }
            per[d] = ll / static_cast<double>(tot);
        }
        double total = 0.0;
        long long nused = 0, floored = 0;
        for (long long d = 0; d < D; ++d)
            if (used[d]) {
                total += per[d];
                ++nused;
                floored += fl[d];
            }
        if (floored_out) *floored_out = floored;
        if (nused == 0) fail(kNumericalError, "heldout_likelihood: empty held-out corpus");
        *ll_out = total / static_cast<double>(nused);
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
        cublasHandle_t hb = cublas_of(ctx);
        const double one = 1.0, zero = 0.0;
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
                CB(cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, k, k, n, &one, fac[f1], n, fac[f1], n, &zero, G1.p, k));
                CB(cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, k, k, n, &one, fac[f2], n, fac[f2], n, &zero, G2.p, k));
                CK(cudaMemcpyAsync(g1.data(), G1.p, g1.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
                CK(cudaMemcpyAsync(g2.data(), G2.p, g2.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
                ctx->sync();
                for (size_t q = 0; q < G.size(); ++q) G[q] = g1[q] * g2[q];
                const std::vector<double> Pinv = pinv_spectral_host(k, G);
                CK(cudaMemcpyAsync(P.p, Pinv.data(), Pinv.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
                // target = M * pinv(G); normalize_columns(target, prev, lambda)
                CK(cudaMemcpyAsync(prev.p, fac[mode], nk * 8, cudaMemcpyDeviceToDevice, ctx->stream));
                CB(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, n, k, k, &one, M.p, n, P.p, k, &zero, fac[mode], n));
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
