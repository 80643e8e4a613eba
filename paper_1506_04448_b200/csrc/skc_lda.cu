// LDA whitened third-moment sketch on sm_100a — sketch_whitened_m3
// (proj/src/lda.cpp:145-226, with compute_m1 lda.cpp:88-100).
//
//   doc pass      p_d = W^T n_d (k-vector), s1_d = 1/(m(m-1)(m-2)), s2_d = a0/((a0+2) m(m-1))
//                 for documents with m >= 3 (lda.cpp:163-185)      -> k_lda_docs (warp/doc)
//   vocab sums    coeff1_w = sum_d 2 s1_d c_dw, sumwn_w = sum_d s1_d c_dw p_d, in ascending d
//                 through the word-major transpose (deterministic)  -> k_lda_vocab (warp/word)
//   m1, q         m1 = mean_d n_d/m_d (m_d >= 1), q = W^T m1        -> k_lda_m1, k_lda_q
//   spectra       acc = sum_d s1 F(p)^3 + sum_w F(w)^2 (coeff1 F(w) - 3 F(sumwn_w)),
//                 cross = sum_d s2 F(p)^2                          -> k_lda_accumulate
//                 acc = (acc - 3 cross F(q)) / D + c_m1 F(q)^3; data += IFFT(acc) -> k_lda_finish
// All transforms use the residue-split local FFT of skc_fft.cuh.
#include <cuda_runtime.h>

#include "skc_fft.cuh"
#include "skc_host.hpp"
#include "skc_internal.hpp"

namespace skc {

namespace {
inline unsigned cdiv_l(long long a, long long b) { return static_cast<unsigned>((a + b - 1) / b); }
constexpr int kThreads = 256;

__device__ __forceinline__ void zero_sm(double2* sm, int count) {
    for (int x = threadIdx.x; x < count; x += blockDim.x) sm[x] = mk(0.0, 0.0);
}

// Deterministic scatter of a dense k-vector through the set's bucket1 plan: every
// contribution is computed independently (all loads in flight), then each run head sums
// its run in plan order. Two vectors (A: valA, B: valB) may be scattered at once.
// scratch: up to 2k double2 + 2k keys.
template <typename ValA, typename ValB>
__device__ __forceinline__ void scatter_dense2(double2* yA, ValA valA, double2* yB, ValB valB, const uint2* __restrict__ plan,
                                               int n, int N, int r, std::uint32_t bmask, const double2* __restrict__ tw,
                                               double2* scr, std::uint32_t* keys, const double2* __restrict__ stw) {
    const std::uint32_t nmask = static_cast<std::uint32_t>(N - 1);
    const int tot = yB ? 2 * n : n;
    for (int x = threadIdx.x; x < tot; x += blockDim.x) {
        const bool b = x >= n;
        const int q = b ? x - n : x;
        const uint2 e = plan[q];
        const double val = b ? valB(e.x) : valA(e.x);
        // plan-order residue twiddle of this (m, r) when the set has the table (coalesced)
        const double2 w = stw ? stw[q] : conj(tw[(static_cast<std::uint32_t>(r) * (e.y & 0x0FFFFFFFu)) & bmask]);
        scr[x] = cmul(root4_times(e.y >> 28, val), w);
        keys[x] = e.y & nmask;
    }
    __syncthreads();
    for (int x = threadIdx.x; x < tot; x += blockDim.x) {
        const int lo = (x >= n) ? n : 0;
        const std::uint32_t key = keys[x];
        if (x > lo && keys[x - 1] == key) continue;
        double2 acc = scr[x];
        for (int x2 = x + 1; x2 < lo + n && keys[x2] == key; ++x2) acc = cadd(acc, scr[x2]);
        ((x >= n) ? yB : yA)[pad16(static_cast<int>(key))] = acc;
    }
}
template <typename ValFn>
__device__ __forceinline__ void scatter_dense(double2* y, const uint2* __restrict__ plan, int n, int N, int r,
                                              std::uint32_t bmask, const double2* __restrict__ tw, ValFn val,
                                              double2* scr, std::uint32_t* keys, const double2* __restrict__ stw) {
    scatter_dense2(y, val, static_cast<double2*>(nullptr), val, plan, n, N, r, bmask, tw, scr, keys, stw);
}
}  // namespace

// ---- document pass: one warp per document ------------------------------------------
__global__ void k_lda_docs(int k, long long D, const long long* __restrict__ doc_ptr, const int* __restrict__ word,
                           const int* __restrict__ count, const double* __restrict__ W, double alpha0,
                           double* __restrict__ P, double* __restrict__ s1, double* __restrict__ s2,
                           long long* __restrict__ total_out) {
    const long long d = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (d >= D) return;
    const long long b0 = doc_ptr[d], b1 = doc_ptr[d + 1];
    long long tot = 0;
    for (long long q = b0 + lane; q < b1; q += 32) tot += count[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0) total_out[d] = tot;
    const double m = static_cast<double>(tot);
    const bool used = tot >= 3;
    if (lane == 0) {
        s1[d] = used ? 1.0 / (m * (m - 1.0) * (m - 2.0)) : 0.0;
        s2[d] = used ? alpha0 / ((alpha0 + 2.0) * m * (m - 1.0)) : 0.0;
    }
    // p = sum_q c_q W[word_q]  (lda.cpp:172-174, words in document order)
    for (int a = lane; a < k; a += 32) {
        double acc = 0.0;
        if (used)
            for (long long q = b0; q < b1; ++q) acc += static_cast<double>(count[q]) * W[(size_t)word[q] * k + a];
        P[(size_t)d * k + a] = acc;
    }
}

// ---- vocabulary accumulators through the word-major transpose ------------------------
// cptr[V+1], cdoc[nnz] (ascending d per word), ccount[nnz]
__global__ void k_lda_vocab(int k, int V, const long long* __restrict__ cptr, const long long* __restrict__ cdoc,
                            const int* __restrict__ ccount, const double* __restrict__ P, const double* __restrict__ s1,
                            const long long* __restrict__ total, double* __restrict__ coeff1,
                            double* __restrict__ sumwn, double* __restrict__ m1_partial) {
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= V) return;
    const long long b0 = cptr[w], b1 = cptr[w + 1];
    for (int a = lane; a < k; a += 32) {
        double acc = 0.0;
        for (long long q = b0; q < b1; ++q) {
            const long long d = cdoc[q];
            const double c = s1[d] * static_cast<double>(ccount[q]);
            if (c != 0.0) acc += c * P[(size_t)d * k + a];
        }
        sumwn[(size_t)w * k + a] = acc;
    }
    if (lane == 0) {
        double c1 = 0.0, m1 = 0.0;
        for (long long q = b0; q < b1; ++q) {
            const long long d = cdoc[q];
            c1 += 2.0 * s1[d] * static_cast<double>(ccount[q]);                                       // lda.cpp:178
            if (total[d] >= 1) m1 += (1.0 / static_cast<double>(total[d])) * static_cast<double>(ccount[q]);  // lda.cpp:94-95
        }
        coeff1[w] = c1;
        m1_partial[w] = m1;
    }
}

// Chunked vocabulary pass (load balance over Zipf-heavy words): a warp per <= 64-entry
// chunk of a word's CSC range writes partial (sumwn[0..k), coeff1, m1); a warp per word
// adds its chunks in order. Same sums as k_lda_vocab in a fixed chunked order.
__global__ void k_lda_vocab_chunks(int k, long long nchunks, const long long* __restrict__ chunk_lo,
                                   const long long* __restrict__ chunk_hi, const long long* __restrict__ cdoc,
                                   const int* __restrict__ ccount, const double* __restrict__ P,
                                   const double* __restrict__ s1, const long long* __restrict__ total,
                                   double* __restrict__ part) {
    const long long ck = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (ck >= nchunks) return;
    const long long q0 = chunk_lo[ck], q1 = chunk_hi[ck];
    double* o = part + (size_t)ck * (k + 2);
    for (int a = lane; a < k; a += 32) {
        double acc = 0.0;
        for (long long q = q0; q < q1; ++q) {
            const long long d = cdoc[q];
            const double c = s1[d] * static_cast<double>(ccount[q]);
            if (c != 0.0) acc += c * P[(size_t)d * k + a];
        }
        o[a] = acc;
    }
    if (lane == 0) {
        double c1 = 0.0, m1 = 0.0;
        for (long long q = q0; q < q1; ++q) {
            const long long d = cdoc[q];
            c1 += 2.0 * s1[d] * static_cast<double>(ccount[q]);                                       // lda.cpp:178
            if (total[d] >= 1) m1 += (1.0 / static_cast<double>(total[d])) * static_cast<double>(ccount[q]);  // lda.cpp:94-95
        }
        o[k] = c1;
        o[k + 1] = m1;
    }
}
__global__ void k_lda_vocab_finish(int k, int V, const long long* __restrict__ word_chunk,
                                   const double* __restrict__ part, double* __restrict__ coeff1,
                                   double* __restrict__ sumwn, double* __restrict__ m1_partial) {
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= V) return;
    const long long c0 = word_chunk[w], c1e = word_chunk[w + 1];
    for (int a = lane; a < k + 2; a += 32) {
        double acc = 0.0;
        for (long long ck = c0; ck < c1e; ++ck) acc += part[(size_t)ck * (k + 2) + a];
        if (a < k)
            sumwn[(size_t)w * k + a] = acc;
        else if (a == k)
            coeff1[w] = acc;
        else
            m1_partial[w] = acc;
    }
}
void launch_lda_vocab_chunked(cudaStream_t st, int k, int V, long long nchunks, const long long* chunk_lo,
                              const long long* chunk_hi, const long long* word_chunk, const long long* cdoc,
                              const int* ccount, const double* P, const double* s1, const long long* total,
                              double* part, double* coeff1, double* sumwn, double* m1_partial) {
    if (nchunks > 0)
        k_lda_vocab_chunks<<<cdiv_l(nchunks * 32, kThreads), kThreads, 0, st>>>(k, nchunks, chunk_lo, chunk_hi, cdoc,
                                                                              ccount, P, s1, total, part);
    k_lda_vocab_finish<<<cdiv_l((long long)V * 32, kThreads), kThreads, 0, st>>>(k, V, word_chunk, part, coeff1,
                                                                                 sumwn, m1_partial);
    count_launch();
    count_launch();
}

// q[a] = sum_w W[w][a] * m1[w] / used1 (lda.cpp:188-189); one block per a, fixed order.
__global__ void k_lda_q(int k, int V, const double* __restrict__ W, const double* __restrict__ m1_partial,
                        double inv_used1, double* __restrict__ q) {
    __shared__ double red[kThreads / 32];
    const int a = blockIdx.x;
    double acc = 0.0;
    for (int w = threadIdx.x; w < V; w += blockDim.x) acc += W[(size_t)w * k + a] * (m1_partial[w] * inv_used1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < kThreads / 32; ++i) s += red[i];
        q[a] = s;
    }
}

// ---- frequency-domain accumulation: CTA per (chunk, m, r) -----------------------------
// Two kernels, two resident CTAs per SM each:
//   documents (used ones only, via the host-built index list): ACC += s1 F(p)^3,
//                                                               CR  += s2 F(p)^2
//   vocabulary words: ACC += F(w)^2 (coeff1 F(w) - 3 F(sumwn))
// The item-invariant scatter metadata of (m, r) (weight, local key, index) is built once
// per CTA; item rows are double-buffered into shared memory with cp.async; the local
// arrays are re-zeroed by the accumulate pass, so each item costs one barrier before and
// one after its transform.
struct ScatterMeta {
    double2* wv;
    std::uint32_t* keys;
    std::uint32_t* idx;
};
__device__ __forceinline__ void build_meta(const ScatterMeta& mt, const uint2* __restrict__ plan,
                                           const double2* __restrict__ stw, const double2* __restrict__ tw, int n, int N,
                                           int r, std::uint32_t bmask) {
    const std::uint32_t nmask = static_cast<std::uint32_t>(N - 1);
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        const uint2 e = plan[q];
        const double2 w = stw ? stw[q] : conj(tw[(static_cast<std::uint32_t>(r) * (e.y & 0x0FFFFFFFu)) & bmask]);
        mt.wv[q] = cmul(root4_times(e.y >> 28, 1.0), w);
        mt.keys[q] = e.y & nmask;
        mt.idx[q] = e.x;
    }
}
// run heads sum wv[q] val[idx[q]] in plan order (deterministic) into y (all-zero before)
__device__ __forceinline__ void scatter_meta(double2* y, const ScatterMeta& mt, const double* val, int n) {
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        const std::uint32_t key = mt.keys[q];
        if (q > 0 && mt.keys[q - 1] == key) continue;
        double2 a = mk(0.0, 0.0);
        for (int q2 = q; q2 < n && mt.keys[q2] == key; ++q2) {
            const double x = val[mt.idx[q2]];
            const double2 w = mt.wv[q2];
            a = cadd(a, mk(w.x * x, w.y * x));
        }
        y[pad16(static_cast<int>(key))] = a;
    }
}
__device__ __forceinline__ void async_row(double* dst, const double* src, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const std::uint32_t da = static_cast<std::uint32_t>(__cvta_generic_to_shared(dst + i));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(da), "l"(src + i) : "memory");
    }
}

template <int LOGN>
__global__ void __launch_bounds__(kThreads, 2)
    k_lda_acc_docs(SymView v, long long Du, const long long* __restrict__ used_docs, const double* __restrict__ P,
                   const double* __restrict__ s1, const double* __restrict__ s2, int chunks, double* __restrict__ acc_out,
                   double* __restrict__ cross_out) {
    extern __shared__ double2 sm[];
    constexpr int N = 1 << LOGN;
    constexpr int stride = N + (N >> 4) + 1;
    const int S = v.S, n = v.n, B = v.B;
    const int r = blockIdx.x % S;
    const int m = (blockIdx.x / S) % B;
    const int ch = blockIdx.x / (S * B);
    double2* A = sm;
    double2* ACC = sm + stride;
    double2* CR = ACC + stride;  // ACC and CR padded like A (the fused last DIF pass writes 16 consecutive positions per thread)
    ScatterMeta mt{CR + stride, nullptr, nullptr};
    mt.keys = reinterpret_cast<std::uint32_t*>(mt.wv + n);
    mt.idx = mt.keys + n;
    double* rows = reinterpret_cast<double*>(mt.idx + n);  // 2 x n (2n u32: 8-byte aligned)
    const long long per = (Du + chunks - 1) / chunks;
    const long long i0 = (long long)ch * per, i1 = min(Du, i0 + per);
    zero_sm(A, stride);
    zero_sm(ACC, 2 * stride);
    build_meta(mt, v.plan1 + (size_t)m * n, v.stw1 ? v.stw1 + ((size_t)m * S + r) * n : nullptr, v.tw, n, N, r,
               v.b - 1);
    if (i0 < i1) async_row(rows, P + (size_t)used_docs[i0] * n, n);
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (long long it = i0; it < i1; ++it) {
        if (it + 1 < i1) async_row(rows + (size_t)((it + 1 - i0) & 1) * n, P + (size_t)used_docs[it + 1] * n, n);
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        const long long d = used_docs[it];
        scatter_meta(A, mt, rows + (size_t)((it - i0) & 1) * n, n);
        __syncthreads();
        const double a1 = s1[d], a2 = s2[d];
        // the last DIF pass feeds the accumulators directly (no extra pass over A)
        dif_local_epilogue<LOGN, 4>(A, v.twl, [&](int j, double2 f) {
            A[pad16(j)] = mk(0.0, 0.0);
            const double2 sq = cmul(f, f);
            ACC[pad16(j)] = cadd(ACC[pad16(j)], cscale(cmul(sq, f), a1));  // lda.cpp:205
            CR[pad16(j)] = cadd(CR[pad16(j)], cscale(sq, a2));              // lda.cpp:206
        });
    }
    __syncthreads();
    double2* ao = reinterpret_cast<double2*>(acc_out) + (((size_t)ch * B + m) * S + r) * N;
    double2* co = reinterpret_cast<double2*>(cross_out) + (((size_t)ch * B + m) * S + r) * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
        ao[j] = ACC[pad16(j)];
        co[j] = CR[pad16(j)];
    }
}

// Paired-document form of k_lda_acc_docs for local length 2048 (config 4: b = 2^14). Two
// documents go through a 16 x 16 x 8 pass plan together (2 x 128 radix-16 items for the 256
// threads; one document left half of them idle), the closing radix-8 pass gives a thread the
// same 8 consecutive outputs of both, so ACC lives in 8 complex registers; CR stays in shared
// memory (padded like A), and the array ACC used to take holds the second document. Items
// are taken in the bank-conflict-free order of k_sym_moment_pair (skc_kernels.cu).
template <int LOGN>
__global__ void __launch_bounds__((1 << LOGN) / 8, 2)
    k_lda_acc_docs_pair(SymView v, long long Du, const long long* __restrict__ used_docs, const double* __restrict__ P,
                        const double* __restrict__ s1, const double* __restrict__ s2, int chunks,
                        double* __restrict__ acc_out, double* __restrict__ cross_out) {
    extern __shared__ double2 sm[];
    constexpr int N = 1 << LOGN, NT = N / 8;
    constexpr int stride = N + (N >> 4) + 1;
    static_assert(LOGN >= 8 && (LOGN - 3) % 4 == 0, "16 x ... x 16 x 8 pass plan");
    const int S = v.S, n = v.n, B = v.B;
    const int r = blockIdx.x % S;
    const int m = (blockIdx.x / S) % B;
    const int ch = blockIdx.x / (S * B);
    double2* A0 = sm;
    double2* A1 = sm + stride;
    double2* CR = A1 + stride;
    ScatterMeta mt{CR + stride, nullptr, nullptr};
    mt.keys = reinterpret_cast<std::uint32_t*>(mt.wv + n);
    mt.idx = mt.keys + n;
    double* rows = reinterpret_cast<double*>(mt.idx + n);  // the pair's rows (2n u32 before: 8-byte aligned)
    const long long per = (Du + chunks - 1) / chunks;
    const long long i0 = (long long)ch * per, i1 = min(Du, i0 + per);
    zero_sm(A0, 3 * stride);
    build_meta(mt, v.plan1 + (size_t)m * n, v.stw1 ? v.stw1 + ((size_t)m * S + r) * n : nullptr, v.tw, n, N, r,
               v.b - 1);
    auto fetch = [&](long long it) {
        if (it < i1) async_row(rows, P + (size_t)used_docs[it] * n, n);
        if (it + 1 < i1) async_row(rows + n, P + (size_t)used_docs[it + 1] * n, n);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double2 accr[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) accr[q] = mk(0.0, 0.0);
    const int wi = static_cast<int>((threadIdx.x & ~15u) | ((threadIdx.x & 7u) << 1) | ((threadIdx.x >> 3) & 1u));
    fetch(i0);
    for (long long it = i0; it < i1; it += 2) {
        const int cnt = static_cast<int>(min(2ll, i1 - it));
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        for (int q = threadIdx.x; q < n; q += NT) {  // run heads, both documents (plan order)
            const std::uint32_t key = mt.keys[q];
            if (q > 0 && mt.keys[q - 1] == key) continue;
            double2 a0 = mk(0.0, 0.0), a1 = mk(0.0, 0.0);
            for (int q2 = q; q2 < n && mt.keys[q2] == key; ++q2) {
                const int i = static_cast<int>(mt.idx[q2]);
                const double2 wq = mt.wv[q2];
                const double x0 = rows[i], x1 = cnt > 1 ? rows[n + i] : 0.0;
                a0 = cadd(a0, mk(wq.x * x0, wq.y * x0));
                a1 = cadd(a1, mk(wq.x * x1, wq.y * x1));
            }
            A0[pad16(static_cast<int>(key))] = a0;
            if (cnt > 1) A1[pad16(static_cast<int>(key))] = a1;
        }
        __syncthreads();
        fetch(it + 2);  // the rows are consumed: the next pair lands during the passes
        constexpr int NP16 = (LOGN - 3) / 4;
#pragma unroll
        for (int pz = 0; pz < NP16; ++pz) {
            const int h = (N >> 1) >> (4 * pz);
            for (int w = threadIdx.x; w < cnt * (N / 16); w += NT) {
                const int a = w / (N / 16);
                dif_pass_item<4>(a ? A1 : A0, w - a * (N / 16), h, v.twl, LOGN);
            }
            __syncthreads();
        }
#pragma unroll 1
        for (int c = 0; c < cnt; ++c) {
            double2* A = c ? A1 : A0;
            const long long d = used_docs[it + c];
            const double a1 = s1[d], a2 = s2[d];
            double2 z[8];
            int base, g;
            dif_item_core<3, true>(A, wi, 4, v.twl, LOGN, z, base, g);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int pj = pad16(base + q * g);
                A[pj] = mk(0.0, 0.0);
                const double2 sq = cmul(z[q], z[q]);
                accr[q] = cadd(accr[q], cscale(cmul(sq, z[q]), a1));  // lda.cpp:205
                CR[pj] = cadd(CR[pj], cscale(sq, a2));               // lda.cpp:206
            }
        }
        // (the next scatter is behind the barrier at the top of the loop)
    }
    __syncthreads();
    double2* ao = reinterpret_cast<double2*>(acc_out) + (((size_t)ch * B + m) * S + r) * N;
    double2* co = reinterpret_cast<double2*>(cross_out) + (((size_t)ch * B + m) * S + r) * N;
#pragma unroll
    for (int q = 0; q < 8; ++q) ao[8 * wi + q] = accr[q];
    for (int j = threadIdx.x; j < N; j += NT) co[j] = CR[pad16(j)];
}

template <int LOGN>
__global__ void __launch_bounds__(kThreads, 2)
    k_lda_acc_vocab(SymView v, int V, const double* __restrict__ W, const double* __restrict__ coeff1,
                    const double* __restrict__ sumwn, int chunks, double* __restrict__ acc_out) {
    extern __shared__ double2 sm[];
    constexpr int N = 1 << LOGN;
    constexpr int stride = N + (N >> 4) + 1;
    const int S = v.S, n = v.n, B = v.B;
    const int r = blockIdx.x % S;
    const int m = (blockIdx.x / S) % B;
    const int ch = blockIdx.x / (S * B);
    double2* A = sm;
    double2* Bw = sm + stride;
    double2* ACC = sm + 2 * stride;
    ScatterMeta mt{ACC + N, nullptr, nullptr};
    mt.keys = reinterpret_cast<std::uint32_t*>(mt.wv + n);
    mt.idx = mt.keys + n;
    double* rows = reinterpret_cast<double*>(mt.idx + n);  // 2 x (W row, sumwn row)
    const long long per = ((long long)V + chunks - 1) / chunks;
    const long long i0 = (long long)ch * per, i1 = min((long long)V, i0 + per);
    zero_sm(A, 2 * stride);
    zero_sm(ACC, N);
    build_meta(mt, v.plan1 + (size_t)m * n, v.stw1 ? v.stw1 + ((size_t)m * S + r) * n : nullptr, v.tw, n, N, r,
               v.b - 1);
    auto fetch = [&](long long w, int buf) {
        async_row(rows + (size_t)buf * 2 * n, W + (size_t)w * n, n);
        async_row(rows + (size_t)buf * 2 * n + n, sumwn + (size_t)w * n, n);
    };
    if (i0 < i1) fetch(i0, 0);
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (long long w = i0; w < i1; ++w) {
        if (w + 1 < i1) fetch(w + 1, static_cast<int>((w + 1 - i0) & 1));
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        const double* row = rows + (size_t)((w - i0) & 1) * 2 * n;
        scatter_meta(A, mt, row, n);
        scatter_meta(Bw, mt, row + n, n);
        __syncthreads();
        dif_local<LOGN>(sm, 2, v.twl);
        const double c1 = coeff1[w];
        for (int j = threadIdx.x; j < N; j += blockDim.x) {
            const double2 fw = A[pad16(j)], fs = Bw[pad16(j)];
            A[pad16(j)] = mk(0.0, 0.0);
            Bw[pad16(j)] = mk(0.0, 0.0);
            const double2 w2 = cmul(fw, fw);
            ACC[j] = cadd(ACC[j], cmul(w2, csub(cscale(fw, c1), cscale(fs, 3.0))));  // lda.cpp:216-217
        }
    }
    __syncthreads();
    double2* ao = reinterpret_cast<double2*>(acc_out) + (((size_t)ch * B + m) * S + r) * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) ao[j] = ACC[j];
}

// Vocabulary pass at local length 2048 on the 16 x 16 x 8 plan: a word's two arrays (F(w),
// F(sumwn)) already fill the radix-16 passes (2 x 128 items); the closing radix-8 pass hands
// a thread the same 8 outputs of both, so the product (lda.cpp:216-217) is formed and
// accumulated in registers: no pointwise pass over the arrays and no shared-memory ACC.
template <int LOGN>
__global__ void __launch_bounds__((1 << LOGN) / 8, 2)
    k_lda_acc_vocab_reg(SymView v, int V, const double* __restrict__ W, const double* __restrict__ coeff1,
                        const double* __restrict__ sumwn, int chunks, double* __restrict__ acc_out) {
    extern __shared__ double2 sm[];
    constexpr int N = 1 << LOGN, NT = N / 8;
    constexpr int stride = N + (N >> 4) + 1;
    static_assert(LOGN >= 8 && (LOGN - 3) % 4 == 0, "16 x ... x 16 x 8 pass plan");
    const int S = v.S, n = v.n, B = v.B;
    const int r = blockIdx.x % S;
    const int m = (blockIdx.x / S) % B;
    const int ch = blockIdx.x / (S * B);
    double2* A = sm;
    double2* Bw = sm + stride;
    ScatterMeta mt{Bw + stride, nullptr, nullptr};
    mt.keys = reinterpret_cast<std::uint32_t*>(mt.wv + n);
    mt.idx = mt.keys + n;
    double* rows = reinterpret_cast<double*>(mt.idx + n);  // 2 x (W row, sumwn row)
    const long long per = ((long long)V + chunks - 1) / chunks;
    const long long i0 = (long long)ch * per, i1 = min((long long)V, i0 + per);
    zero_sm(A, 2 * stride);
    build_meta(mt, v.plan1 + (size_t)m * n, v.stw1 ? v.stw1 + ((size_t)m * S + r) * n : nullptr, v.tw, n, N, r,
               v.b - 1);
    auto fetch = [&](long long w, int buf) {
        async_row(rows + (size_t)buf * 2 * n, W + (size_t)w * n, n);
        async_row(rows + (size_t)buf * 2 * n + n, sumwn + (size_t)w * n, n);
    };
    double2 accr[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) accr[q] = mk(0.0, 0.0);
    const int wi = static_cast<int>((threadIdx.x & ~15u) | ((threadIdx.x & 7u) << 1) | ((threadIdx.x >> 3) & 1u));
    if (i0 < i1) fetch(i0, 0);
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (long long w = i0; w < i1; ++w) {
        if (w + 1 < i1) fetch(w + 1, static_cast<int>((w + 1 - i0) & 1));
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        const double* row = rows + (size_t)((w - i0) & 1) * 2 * n;
        scatter_meta(A, mt, row, n);
        scatter_meta(Bw, mt, row + n, n);
        __syncthreads();
        constexpr int NP16 = (LOGN - 3) / 4;
#pragma unroll
        for (int pz = 0; pz < NP16; ++pz) {
            const int h = (N >> 1) >> (4 * pz);
            for (int it = threadIdx.x; it < 2 * (N / 16); it += NT) {
                const int a = it / (N / 16);
                dif_pass_item<4>(a ? Bw : A, it - a * (N / 16), h, v.twl, LOGN);
            }
            __syncthreads();
        }
        const double c1 = coeff1[w];
        double2 zw[8], zs[8];
        int base, g;
        dif_item_core<3, true>(A, wi, 4, v.twl, LOGN, zw, base, g);
        dif_item_core<3, true>(Bw, wi, 4, v.twl, LOGN, zs, base, g);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int pj = pad16(base + q * g);
            A[pj] = mk(0.0, 0.0);
            Bw[pj] = mk(0.0, 0.0);
            const double2 w2 = cmul(zw[q], zw[q]);
            accr[q] = cadd(accr[q], cmul(w2, csub(cscale(zw[q], c1), cscale(zs[q], 3.0))));  // lda.cpp:216-217
        }
        // (the next scatter is behind the barrier at the top of the loop)
    }
    double2* ao = reinterpret_cast<double2*>(acc_out) + (((size_t)ch * B + m) * S + r) * N;
#pragma unroll
    for (int q = 0; q < 8; ++q) ao[8 * wi + q] = accr[q];
}

// acc = (sum acc - 3 sum cross F(q)) / D + c_m1 F(q)^3 (lda.cpp:211, 220-221), inverse DIT.
template <int LOGN>
__global__ void __launch_bounds__(kThreads, 1)
    k_lda_finish(SymView v, const double* __restrict__ acc_in, const double* __restrict__ cross_in, int chunks_acc,
                 int chunks_cross, const double* __restrict__ q, double inv_docs, double m1_coeff,
                 double2* __restrict__ tmp) {
    extern __shared__ double2 sm[];
    constexpr int N = 1 << LOGN;
    const int S = v.S, n = v.n, B = v.B;
    const int r = blockIdx.x % S, m = blockIdx.x / S;
    double2* scr = sm + (N + (N >> 4) + 1);
    std::uint32_t* keys = reinterpret_cast<std::uint32_t*>(scr + 2 * n);
    zero_sm(sm, N + (N >> 4) + 1);
    __syncthreads();
    scatter_dense(sm, v.plan1 + (size_t)m * n, n, N, r, v.b - 1, v.tw, [&](std::uint32_t i) { return q[i]; }, scr, keys,
                  v.stw1 ? v.stw1 + ((size_t)m * S + r) * n : nullptr);
    __syncthreads();
    dif_local<LOGN>(sm, 1, v.twl);
    const double2* ai = reinterpret_cast<const double2*>(acc_in);
    const double2* ci = reinterpret_cast<const double2*>(cross_in);
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
        double2 a = mk(0.0, 0.0), c = mk(0.0, 0.0);
        for (int h = 0; h < chunks_acc; ++h) a = cadd(a, ai[(((size_t)h * B + m) * S + r) * N + j]);
        for (int h = 0; h < chunks_cross; ++h) c = cadd(c, ci[(((size_t)h * B + m) * S + r) * N + j]);
        const double2 fq = sm[pad16(j)];
        a = csub(a, cscale(cmul(c, fq), 3.0));
        sm[pad16(j)] = cadd(cscale(a, inv_docs), cscale(cmul(cmul(fq, fq), fq), m1_coeff));
    }
    __syncthreads();
    dit_local<LOGN>(sm, 1, v.twl);
    double2* o = tmp + ((size_t)m * S + r) * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) o[j] = sm[pad16(j)];
}

void launch_lda_docs(cudaStream_t st, int k, long long D, const long long* doc_ptr, const int* word, const int* count,
                     const double* W, double alpha0, double* P, double* s1, double* s2, long long* total) {
    k_lda_docs<<<cdiv_l(D * 32, kThreads), kThreads, 0, st>>>(k, D, doc_ptr, word, count, W, alpha0, P, s1, s2, total);
    count_launch();
}
void launch_lda_vocab(cudaStream_t st, int k, int V, const long long* cptr, const long long* cdoc, const int* ccount,
                      const double* P, const double* s1, const long long* total, double* coeff1, double* sumwn,
                      double* m1_partial) {
    k_lda_vocab<<<cdiv_l((long long)V * 32, kThreads), kThreads, 0, st>>>(k, V, cptr, cdoc, ccount, P, s1, total,
                                                                        coeff1, sumwn, m1_partial);
    count_launch();
}
void launch_lda_q(cudaStream_t st, int k, int V, const double* W, const double* m1_partial, double inv_used1,
                  double* q) {
    k_lda_q<<<k, kThreads, 0, st>>>(k, V, W, m1_partial, inv_used1, q);
    count_launch();
}

#define SKC_LOGN_SWITCH_L(logN, X) \
    switch (logN) {                \
        case 1: X(1); break;       \
        case 2: X(2); break;       \
        case 3: X(3); break;       \
        case 4: X(4); break;       \
        case 5: X(5); break;       \
        case 6: X(6); break;       \
        case 7: X(7); break;       \
        case 8: X(8); break;       \
        case 9: X(9); break;       \
        case 10: X(10); break;     \
        case 11: X(11); break;     \
        case 12: X(12); break;     \
        default: break;            \
    }

#ifdef SKC_LDA_NOPAIR  // experiment builds: the one-document kernel at every length
constexpr bool kPairDocs = false;
#else
constexpr bool kPairDocs = true;
#endif
// acc: (chunks_d + chunks_v) partial spectra (documents first), cross: chunks_d.
void launch_lda_accumulate(cudaStream_t st, const SymView& v, long long Du, const long long* used_docs, const double* P,
                           const double* s1, const double* s2, int V, const double* W, const double* coeff1,
                           const double* sumwn, int chunks_d, int chunks_v, double* acc, double* cross) {
    const size_t meta = (sizeof(double2) + 2 * sizeof(std::uint32_t)) * (size_t)v.n;
    const size_t smem_d = sizeof(double2) * (3 * padded_len(v.N)) + meta + 2 * sizeof(double) * (size_t)v.n;
    const size_t smem_v = sizeof(double2) * (2 * padded_len(v.N) + v.N) + meta + 4 * sizeof(double) * (size_t)v.n;
    const unsigned grid_d = (unsigned)((long long)chunks_d * v.B * v.S);
    const unsigned grid_v = (unsigned)((long long)chunks_v * v.B * v.S);
    double* acc_v = acc + (size_t)chunks_d * v.B * v.S * v.N * 2;
    if (Du <= 0) {  // a document shard with no used documents contributes nothing
        cudaMemsetAsync(acc, 0, sizeof(double) * (size_t)chunks_d * v.B * v.S * v.N * 2, st);
        cudaMemsetAsync(cross, 0, sizeof(double) * (size_t)chunks_d * v.B * v.S * v.N * 2, st);
    }
#define L_(LG)                                                                                                      \
    {                                                                                                               \
        cudaFuncSetAttribute(k_lda_acc_docs<LG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_d);         \
        cudaFuncSetAttribute(k_lda_acc_vocab<LG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_v);        \
        if (Du > 0 && (LG != 11 || !kPairDocs)) k_lda_acc_docs<LG><<<grid_d, kThreads, smem_d, st>>>(v, Du, used_docs, P, s1, s2, chunks_d, acc, cross); \
        if (V > 0 && (LG != 11 || !kPairDocs)) k_lda_acc_vocab<LG><<<grid_v, kThreads, smem_v, st>>>(v, V, W, coeff1, sumwn, chunks_v, acc_v); \
    }
    if (Du > 0 && v.logN == 11 && kPairDocs) {  // local length 2048: paired documents, ACC in registers (launched first)
        cudaFuncSetAttribute(k_lda_acc_docs_pair<11>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_d);
        k_lda_acc_docs_pair<11><<<grid_d, 256, smem_d, st>>>(v, Du, used_docs, P, s1, s2, chunks_d, acc, cross);
    }
    if (V > 0 && v.logN == 11 && kPairDocs) {  // local length 2048: product accumulated in registers
        cudaFuncSetAttribute(k_lda_acc_vocab_reg<11>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_v);
        k_lda_acc_vocab_reg<11><<<grid_v, 256, smem_v, st>>>(v, V, W, coeff1, sumwn, chunks_v, acc_v);
    }
    SKC_LOGN_SWITCH_L(v.logN, L_)
#undef L_
    count_launch();
    count_launch();
    count_transforms((std::uint64_t)(Du + 2ll * V) * v.B * v.S, v.S);
}
void launch_lda_finish(cudaStream_t st, const SymView& v, const double* acc, const double* cross, int chunks_acc,
                       int chunks_cross, const double* q, double inv_docs, double m1_coeff, double2* tmp) {
    const size_t smem = sizeof(double2) * padded_len(v.N) + (sizeof(double2) + 4) * 2 * (size_t)v.n;
#define L_(LG)                                                                                               \
    {                                                                                                        \
        cudaFuncSetAttribute(k_lda_finish<LG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);      \
        k_lda_finish<LG><<<v.B * v.S, kThreads, smem, st>>>(v, acc, cross, chunks_acc, chunks_cross, q, inv_docs,   \
                                                            m1_coeff, tmp);                                          \
    }
    SKC_LOGN_SWITCH_L(v.logN, L_)
#undef L_
    count_launch();
    count_transforms((std::uint64_t)v.B * v.S * 2, v.S);
}

}  // namespace skc
