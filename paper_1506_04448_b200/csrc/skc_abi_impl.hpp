// Shared internals of the C-ABI translation units (skc_abi*.cu): error plumbing,
// device buffers, the context and the sketch-set objects behind the opaque handles of
// include/sketchcp_b200.h. Not a public header.
#pragma once
#include <nccl.h>
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

namespace skcabi {

inline thread_local std::string g_last_error;

#define CK(call)                                                                                     \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess) {                                                                     \
            int code_ = (e_ == cudaErrorMemoryAllocation) ? kOutOfMemory : kCudaError;               \
            fail(code_, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call);        \
        }                                                                                            \
    } while (0)

template <typename F>
inline int guard(F&& f) {
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

// Local transform length: CTA-local FFTs of N = min(b, 2048) points, S = b / N residues
// (2048 measured fastest for the config-1 contraction against 1024 and 4096).
inline int local_length(std::uint32_t b) { return static_cast<int>(std::min<std::uint32_t>(b, 2048u)); }

inline std::vector<double> host_twiddles(std::uint32_t b) {
    std::vector<double> tw(2 * static_cast<size_t>(b));
    const long double two_pi = 6.283185307179586476925286766559005768L;
    for (std::uint32_t k = 0; k < b; ++k) {
        long double a = two_pi * static_cast<long double>(k) / static_cast<long double>(b);
        tw[2 * k] = static_cast<double>(cosl(a));
        tw[2 * k + 1] = static_cast<double>(sinl(a));
    }
    return tw;
}

}  // namespace skcabi
using namespace skcabi;

// ============================ context ============================================
struct skc_context {
    int device = 0;
    // NCCL communicator over the replicas of a set on several GPUs (skc_group_create or
    // skc_context_comm_init); nranks 1 without one
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1;
    DevBuf<double> gathered;  // all-gathered pre-pass partials / restart values
    cudaStream_t stream = nullptr;
    cudaStream_t stream2 = nullptr;  // pipelined zero-copy builds: main pass of chunk c
    cudaEvent_t ev_q[5] = {};        // chunk c quantized / all chunks done
    cudaEvent_t ev_order = nullptr;  // skc_context_wait_stream
    DevBuf<double> gemm_ws;  // split-K partials of the block products (dgemm_cm)
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
    int* host_ints = nullptr;  // pinned host scratch for small synchronous readbacks (DMA, no staging)
    double* host_dbl = nullptr;  // pinned host scratch for RTPM inits (grown on demand)
    size_t host_dbl_n = 0;
    double* pinned_doubles(size_t count) {
        if (count > host_dbl_n) {
            if (host_dbl) cudaFreeHost(host_dbl);
            host_dbl = nullptr;
            host_dbl_n = 0;
            CK(cudaMallocHost(reinterpret_cast<void**>(&host_dbl), count * sizeof(double)));
            host_dbl_n = count;
        }
        return host_dbl;
    }
    int* pinned_ints() {
        if (!host_ints) CK(cudaMallocHost(reinterpret_cast<void**>(&host_ints), 16 * sizeof(int)));
        return host_ints;
    }
    DevBuf<double> dbl;  // [0] best value
    DevBuf<int> build_ints;                // per-type row counters of the dense build
    DevBuf<unsigned long long> build_acc;  // exact fixed-point slot accumulators
    bool build_scratch_clean = false;      // build_acc / build_ints are all zero (finalize re-zeroes them)
    bool build_ovf_clean = false;          // ints[3] (one-limb overflow flag) is zero
    long long build_two_limb_retries = 0;  // one-limb builds redone with two limbs (overflow)
    long long build_banded = 0;            // builds redone in magnitude bands (high dynamic range)
    const void* build_acc_clean_p = nullptr;  // the buffers (pointer, size) that were cleared
    const void* build_ints_clean_p = nullptr;
    size_t build_acc_clean_n = 0, build_ints_clean_n = 0;
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
    std::vector<cudaEvent_t> ev_pool;  // recycled profiling events (creation costs host time in timed loops)
    cudaEvent_t pooled_event() {
        if (!ev_pool.empty()) {
            cudaEvent_t e = ev_pool.back();
            ev_pool.pop_back();
            return e;
        }
        cudaEvent_t e = nullptr;
        CK(cudaEventCreate(&e));
        return e;
    }

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
        a = c->pooled_event();
        CK(cudaEventRecord(a, c->stream));
    }
    ~ProfScope() {
        if (!c->prof_on || !a) return;
        cudaEvent_t b = nullptr;
        if (!c->ev_pool.empty()) {
            b = c->ev_pool.back();
            c->ev_pool.pop_back();
        } else if (cudaEventCreate(&b) != cudaSuccess) {
            return;
        }
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
    // CUDA graphs of the RTPM power-step loop on this set, keyed by what the captured
    // launches bake in besides the set's own buffers (shape, tolerance, context scratch)
    struct RtpmGraph {
        cudaGraphExec_t exec = nullptr;
        std::uint64_t launches = 0, transforms = 0;
    };
    std::map<std::vector<std::uint64_t>, RtpmGraph> rtpm_graphs;
    skc_sym_set() = default;
    skc_sym_set(const skc_sym_set&) = delete;
    skc_sym_set& operator=(const skc_sym_set&) = delete;
    ~skc_sym_set() {
        for (auto& g : rtpm_graphs)
            if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
    }
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

namespace skcabi {

inline void validate_set_args(int n, std::uint32_t b, int B) {
    // sketch.cpp:157-159 / 302-304
    require(n >= 1, "sketch set: dimension must be positive");
    require(B >= 1, "sketch set: need at least one replicate");
    require(is_pow2(b), "sketch set: b must be a power of two");
    require(b >= 2, "PolyHash: need at least 2 buckets");
    require(b <= (1u << 28), "sketch set: b above 2^28 is not supported by the packed bucket tables");
}

inline void check_vec(const void* p, const char* what) { require(p != nullptr, std::string(what) + ": null pointer"); }

// ---- LDA moments and whitening (lda.cpp:88-143; kernels in skc_whiten.cu) ---------------
// Column-major DGEMM in cuBLAS's argument convention (alpha 1, beta 0), on the repo's own
// kernel (skc_gemm.cu): C (m x n, ldc) = op(A) op(B), op(A) m x k, op(B) k x n.
inline void dgemm_cm(skc_context* ctx, bool ta, bool tb, int m, int n, int k, const double* A, int lda,
                     const double* B, int ldb, double* C, int ldc) {
    const int z = k > 0 ? dgemm_slices(m, n, k, ctx->sms) : 1;
    if (z > 1) ctx->gemm_ws.alloc(static_cast<size_t>(z) * m * n);
    launch_dgemm(ctx->stream, ctx->sms, m, n, k, A, ta ? lda : 1, ta ? 1 : lda, B, tb ? ldb : 1, tb ? 1 : ldb, C, 1, ldc,
                 ctx->gemm_ws.p);
    ctx->check_launch();
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

// Sample/document chunks of the frequency-domain accumulation kernels (2 resident
// 256-thread CTAs per SM, per_rep = B*S CTAs per chunk): at least ~4 waves, rounded up
// to a chunk count whose grid fills its last wave to >= 99% (config 3: 14 chunks = 3.78
// waves -> 22 = 5.95 waves; a 10-full-wave grid measured 6% faster than 14 chunks).
// At most `cap` chunks (one sample or document per chunk).
inline int wave_chunks(int sms, int per_rep, long long cap) {
    const long long resident = 2ll * sms;
    const long long c0 = std::max<long long>(1, (8ll * sms) / per_rep);
    const long long w0 = (c0 * per_rep + resident - 1) / resident;
    long long chunks = c0;
    for (long long w = w0; w <= 4 * w0; ++w) {
        const long long c = (w * resident) / per_rep;
        if (c >= c0 && static_cast<double>(c * per_rep) >= 0.99 * static_cast<double>(w * resident)) {
            chunks = c;
            break;
        }
    }
    return static_cast<int>(std::max<long long>(1, std::min<long long>(std::max<long long>(cap, 1), chunks)));
}

// ---- cross-unit helpers ----------------------------------------------------------------
// skc_abi_build.cu
const void* stage_tensor(skc_context* ctx, const void* T, int n, int dtype, int location, bool sym, int i0, int i1,
                         bool need_full, size_t* h2d_bytes, bool* zero_copy = nullptr);
void run_dense_build(skc_context* ctx, const void* Tdev, int n, int dtype, bool sym, int i0, int i1, int B,
                     std::uint32_t b, const std::uint32_t* packed, double2* data, bool zero_copy, bool two_limb = false);
void ensure_build_scratch_clean(skc_context* ctx);
void run_dense_build_banded(skc_context* ctx, const void* Tdev, int n, int dtype, bool sym, int i0, int i1, int B,
                            std::uint32_t b, const std::uint32_t* packed, double2* data, bool zero_copy);
skc_context::RowTab& prepare_dense_build(skc_context* ctx, int n, int dtype, bool sym, int i0, int i1, int B,
                                         std::uint32_t b, const std::uint32_t* packed, double2* data, bool zero_copy,
                                         bool two_limb, BuildPlan& p);
// skc_abi_sym.cu
void check_symmetric(skc_context* ctx, const void* Td, int dtype, int n);
void sym_moment_partial(skc_sym_set* s, const double* Xd, const double* wd, long long Nsamp);
void sym_moment_combine(skc_sym_set* s, double alpha);
void rtpm_restarts_device(skc_sym_set* s, int L, int T_iters, double tol);
void check_degenerate(skc_context* ctx, int L);
// skc_abi_lda.cu
void upload_corpus(skc_context* ctx, int V, long long D, const long long* doc_ptr, const int* word, const int* count,
                   CorpusDev& c, const std::string& who = "lda", bool check_counts = true);
void sketch_whitened_m3_dev(skc_sym_set* s, CorpusDev& c, const double* W, double alpha0, long long* used_out,
                            long long* skipped_out, long long global_used = -1, const double* global_m1 = nullptr,
                            bool add_q_cubed = true);
// skc_abi.cu
void spectrum_to_host(skc_context* ctx, const double2* spec, int m, std::uint32_t b, int N, int logN, int S,
                      double* out);
// skc_abi_linalg.cu
bool sym_eigen_ql_rowmajor(int n, std::vector<double> a, std::vector<double>& vals, std::vector<double>& vecs);
void sym_eigen_host(int p, const std::vector<double>& a, std::vector<double>& vals, std::vector<double>& vecs);
void jacobi_eigen(int p, std::vector<double> a, std::vector<double>& vals, std::vector<double>& vecs);
std::vector<double> project_to_simplex(const double* y, int n);
std::vector<double> pinv_spectral_host(int k, const std::vector<double>& G);

}  // namespace skcabi
