// K6: LDA moments and whitening on sm_100a (lda.cpp:88-143).
//
// The reference forms M2 densely (V x V, 20 GB at V = 5e4) and calls a full
// SelfAdjointEigenSolver. Here M2 is never formed. It is applied to a V x p block as
//
//   M2 X = (1/used2) [ C^T (S2 (C X)) - diag(sum_d s2_d n_d) X ] - a0/(a0+1) m1 (m1^T X),
//
// where C is the D x V count matrix, S2 = diag(1/(m_d (m_d - 1))) over documents with
// m_d >= 2, and m1 = (1/used1) sum_{m_d >= 1} n_d / m_d. This equals the reference's
// position-pair sum, pair(a, a) = c_a (c_a - 1), exactly, duplicates included. Top-k
// eigenpairs come from randomized subspace iteration with Rayleigh-Ritz (host code in
// skc_abi_lda.cu; the block products use the FP64 kernel of skc_gemm.cu).
//
//   k_corpus_docs   per document: m_d, s2_d, 1/m_d                       (thread/doc)
//   k_m2_word_prep  per word: diag_w = sum s2_d c_dw, m1_w (CSC, fixed order)  (thread/word)
//   k_m2_docs       Z[d, :] = s2_d sum_q c_q X[w_q, :]                     (warp/doc)
//   k_colsum        mx = m1^T X                                           (block/32 cols)
//   k_m2_word_chunks / k_m2_word_finish
//                   Y[w, :] = (sum_{d in w} c Z[d, :] - diag_w X[w, :]) / used2 - a m1_w mx
//                   (warp per <= 64-entry chunk of a word's CSC range, then warp per word)
// Every sum runs in a fixed order, so the operator is deterministic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cub/cub.cuh>

#include "skc_host.hpp"
#include "skc_internal.hpp"

namespace skc {

namespace {
inline unsigned cdiv_w(long long a, long long b) { return static_cast<unsigned>((a + b - 1) / b); }
}  // namespace

__global__ void k_corpus_docs(long long D, const long long* __restrict__ doc_ptr, const int* __restrict__ count,
                              long long* __restrict__ total, double* __restrict__ s2, double* __restrict__ invm) {
    const long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (d >= D) return;
    long long t = 0;
    for (long long q = doc_ptr[d]; q < doc_ptr[d + 1]; ++q) t += count[q];
    total[d] = t;
    const double m = static_cast<double>(t);
    s2[d] = t >= 2 ? 1.0 / (m * (m - 1.0)) : 0.0;  // lda.cpp:111
    invm[d] = t >= 1 ? 1.0 / m : 0.0;              // lda.cpp:94
}

__global__ void k_m2_word_prep(int V, const long long* __restrict__ cptr, const long long* __restrict__ cdoc,
                               const int* __restrict__ ccount, const double* __restrict__ s2,
                               const double* __restrict__ invm, double* __restrict__ diag, double* __restrict__ m1p) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= V) return;
    double dg = 0.0, m = 0.0;
    for (long long q = cptr[w]; q < cptr[w + 1]; ++q) {
        const long long d = cdoc[q];
        const double c = static_cast<double>(ccount[q]);
        dg += s2[d] * c;
        m += invm[d] * c;
    }
    diag[w] = dg;
    m1p[w] = m;
}

__global__ void k_m2_docs(long long D, int p, const long long* __restrict__ doc_ptr, const int* __restrict__ word,
                          const int* __restrict__ count, const double* __restrict__ s2, const double* __restrict__ X,
                          double* __restrict__ Z) {
    const long long d = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (d >= D) return;
    const double sd = s2[d];
    const long long q0 = doc_ptr[d], q1 = doc_ptr[d + 1];
    for (int c0 = 0; c0 < p; c0 += 128) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        if (sd != 0.0) {
            for (long long q = q0; q < q1; ++q) {
                const double cnt = static_cast<double>(count[q]);
                const double* xr = X + (size_t)word[q] * p;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int c = c0 + lane + 32 * u;
                    if (c < p) acc[u] += cnt * xr[c];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = c0 + lane + 32 * u;
            if (c < p) Z[(size_t)d * p + c] = sd * acc[u];
        }
    }
}

// mx[c] = sum_w m1_w X[w, c] with m1_w = m1p_w / used1, in two deterministic stages:
// block (rb, cg) sums rows [rb*RB, (rb+1)*RB) of column group cg (8 warps striding the
// rows, warp partials combined in order) into part[rb][c]; then k_colsum_final adds the
// row-block partials in order.
constexpr int kColsumRows = 512;
__global__ void k_colsum(int V, int p, const double* __restrict__ m1p, double inv_used1, const double* __restrict__ X,
                         double* __restrict__ part) {
    __shared__ double sp[8][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = blockIdx.y * 32 + lane;
    const int r0 = blockIdx.x * kColsumRows, r1 = min(V, r0 + kColsumRows);
    double acc = 0.0;
    if (c < p)
        for (int w = r0 + warp; w < r1; w += 8) acc += (m1p[w] * inv_used1) * X[(size_t)w * p + c];
    sp[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && c < p) {
        double s = 0.0;
        for (int i = 0; i < 8; ++i) s += sp[i][lane];
        part[(size_t)blockIdx.x * p + c] = s;
    }
}
__global__ void k_colsum_final(int nb, int p, const double* __restrict__ part, double* __restrict__ mx) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= p) return;
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[(size_t)b * p + c];
    mx[c] = s;
}

// Word pass split for load balance: a word's CSC range is cut into chunks of at most
// kWordChunk entries (frequent words are Zipf-heavy); a warp per chunk writes its partial
// sum, and a warp per word adds its chunks in order and applies the diagonal and rank-1
// terms. Deterministic for any chunking of the same corpus.
__global__ void k_m2_word_chunks(long long nchunks, int p, const long long* __restrict__ chunk_lo,
                                 const long long* __restrict__ chunk_hi, const long long* __restrict__ cdoc,
                                 const int* __restrict__ ccount, const double* __restrict__ Z,
                                 double* __restrict__ part) {
    const long long ck = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (ck >= nchunks) return;
    const long long q0 = chunk_lo[ck], q1 = chunk_hi[ck];
    for (int c0 = 0; c0 < p; c0 += 128) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (long long q = q0; q < q1; ++q) {
            const double cnt = static_cast<double>(ccount[q]);
            const double* zr = Z + (size_t)cdoc[q] * p;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c = c0 + lane + 32 * u;
                if (c < p) acc[u] += cnt * zr[c];
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = c0 + lane + 32 * u;
            if (c < p) part[(size_t)ck * p + c] = acc[u];
        }
    }
}
__global__ void k_m2_word_finish(int V, int p, const long long* __restrict__ word_chunk, const double* __restrict__ part,
                                 const double* __restrict__ diag, const double* __restrict__ m1p, double inv_used1,
                                 double inv_used2, double a, const double* __restrict__ mx, const double* __restrict__ X,
                                 double* __restrict__ Y) {
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= V) return;
    const double dg = diag[w];
    const double m1w = m1p[w] * inv_used1;
    for (int c = lane; c < p; c += 32) {
        double acc = 0.0;
        for (long long ck = word_chunk[w]; ck < word_chunk[w + 1]; ++ck) acc += part[(size_t)ck * p + c];
        const size_t idx = (size_t)w * p + c;
        Y[idx] = (acc - dg * X[idx]) * inv_used2 - a * m1w * mx[c];
    }
}

// W[w, c] = Vk[w, c] * f[c] (row-major V x k): scaling of the Ritz vectors
__global__ void k_scale_cols(long long rows, int k, const double* __restrict__ in, const double* __restrict__ f,
                             double* __restrict__ out) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= rows * k) return;
    out[i] = in[i] * f[i % k];
}

// ALS normalize_columns (decompose.cpp:145-155) on a column-major n x k factor: lambda[r]
// = ||col r|| (fixed-order block reduction); col /= norm, or the previous column when the
// norm is zero.
__global__ void k_normalize_columns(int n, double* __restrict__ F, const double* __restrict__ prev,
                                    double* __restrict__ lambda) {
    __shared__ double red[8];
    const int r = blockIdx.x;
    double* col = F + (size_t)r * n;
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += 256) acc += col[i] * col[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    __shared__ double nrm_s;
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < 8; ++i) s += red[i];
        nrm_s = sqrt(s);
        lambda[r] = nrm_s;
    }
    __syncthreads();
    const double nrm = nrm_s;
    for (int i = threadIdx.x; i < n; i += 256) col[i] = nrm > 0 ? col[i] / nrm : prev[(size_t)r * n + i];
}
// Counter-based Gaussian block: element t from two splitmix64 draws keyed by (seed, t)
// and the Box-Muller cosine branch (deterministic; only the start of the subspace
// iteration, so device libm rounding is immaterial).
__device__ __forceinline__ unsigned long long smix(unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__global__ void k_gaussian_fill(unsigned long long seed, long long count, double* __restrict__ out) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= count) return;
    const unsigned long long a = smix(seed ^ smix(2ull * (unsigned long long)t));
    const unsigned long long b = smix(seed ^ smix(2ull * (unsigned long long)t + 1ull));
    const double u1 = (static_cast<double>(a >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
    const double u2 = static_cast<double>(b >> 11) * 0x1.0p-53;          // [0, 1)
    out[t] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}
void launch_gaussian_fill(cudaStream_t st, unsigned long long seed, long long count, double* out) {
    k_gaussian_fill<<<cdiv_w(count, 256), 256, 0, st>>>(seed, count, out);
    count_launch();
}

void launch_normalize_columns(cudaStream_t st, int n, int k, double* F, const double* prev, double* lambda) {
    k_normalize_columns<<<k, 256, 0, st>>>(n, F, prev, lambda);
    count_launch();
}

void launch_corpus_prep(cudaStream_t st, int V, long long D, const long long* doc_ptr, const int* count,
                        const long long* cptr, const long long* cdoc, const int* ccount, long long* total, double* s2,
                        double* invm, double* diag, double* m1p) {
    if (D > 0) k_corpus_docs<<<cdiv_w(D, 256), 256, 0, st>>>(D, doc_ptr, count, total, s2, invm);
    k_m2_word_prep<<<cdiv_w(V, 256), 256, 0, st>>>(V, cptr, cdoc, ccount, s2, invm, diag, m1p);
    count_launch();
    count_launch();
}

void launch_m2_apply(cudaStream_t st, int V, long long D, int p, const long long* doc_ptr, const int* word,
                     const int* count, const long long* cdoc, const int* ccount, long long nchunks,
                     const long long* chunk_lo, const long long* chunk_hi, const long long* word_chunk,
                     const double* s2, const double* diag, const double* m1p, double inv_used1, double inv_used2,
                     double a, const double* X, double* Z, double* part, double* mx, double* Y) {
    if (D > 0) k_m2_docs<<<cdiv_w(D * 32, 256), 256, 0, st>>>(D, p, doc_ptr, word, count, s2, X, Z);
    {
        const int nb = static_cast<int>(cdiv_w(V, kColsumRows));
        // (part is free here: the chunk pass below overwrites it after mx is final)
        k_colsum<<<dim3(nb, cdiv_w(p, 32)), 256, 0, st>>>(V, p, m1p, inv_used1, X, part);
        k_colsum_final<<<cdiv_w(p, 128), 128, 0, st>>>(nb, p, part, mx);
        count_launch();
    }
    if (nchunks > 0)
        k_m2_word_chunks<<<cdiv_w(nchunks * 32, 256), 256, 0, st>>>(nchunks, p, chunk_lo, chunk_hi, cdoc, ccount, Z,
                                                                    part);
    k_m2_word_finish<<<cdiv_w((long long)V * 32, 256), 256, 0, st>>>(V, p, word_chunk, part, diag, m1p, inv_used1,
                                                                     inv_used2, a, mx, X, Y);
    count_launch();
    count_launch();
    count_launch();
    count_launch();
}

void launch_scale_cols(cudaStream_t st, long long rows, int k, const double* in, const double* f, double* out) {
    k_scale_cols<<<cdiv_w(rows * k, 256), 256, 0, st>>>(rows, k, in, f, out);
    count_launch();
}

}  // namespace skc

// ---- device corpus preparation (replaces the host transpose for large corpora) -------
// Validation, per-document totals and the word histogram in one document pass; a stable
// radix sort of (word, entry index) pairs gives the word-major transpose with documents
// ascending inside each word (the order of the host counting sort), so every per-word sum
// downstream runs in the same order as before. cub is used for the scan / sort / select
// primitives of this setup step only.

namespace skc {
namespace {
__global__ void k_corpus_docs_scan(long long D, int V, const long long* __restrict__ doc_ptr, const int* __restrict__ word,
                                   const int* __restrict__ count, int check_counts, long long* __restrict__ total,
                                   unsigned int* __restrict__ doc_of, unsigned long long* __restrict__ hist,
                                   unsigned long long* __restrict__ stats, unsigned char* __restrict__ used3_flag) {
    const long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (d >= D) return;
    const long long q0 = doc_ptr[d], q1 = doc_ptr[d + 1];
    if (q1 < q0) {
        atomicAdd(&stats[0], 1ull);
        total[d] = 0;
        used3_flag[d] = 0;
        return;
    }
    long long t = 0;
    bool bw = false, bc = false;
    for (long long q = q0; q < q1; ++q) {
        const int w = word[q];
        doc_of[q] = static_cast<unsigned int>(d);
        if (w < 0 || w >= V) {
            bw = true;
            continue;
        }
        if (check_counts && count[q] < 0) bc = true;
        t += count[q];
        atomicAdd(&hist[w], 1ull);
    }
    if (bw) atomicAdd(&stats[1], 1ull);
    if (bc) atomicAdd(&stats[2], 1ull);
    total[d] = t;
    if (t >= 1) atomicAdd(&stats[3], 1ull);
    if (t >= 2) atomicAdd(&stats[4], 1ull);
    used3_flag[d] = t >= 3;
}
__global__ void k_iota_u32(long long n, unsigned int* __restrict__ out) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) out[i] = static_cast<unsigned int>(i);
}
__global__ void k_corpus_gather(long long nnz, const unsigned int* __restrict__ order,
                                const unsigned int* __restrict__ doc_of, const int* __restrict__ count,
                                long long* __restrict__ cdoc, int* __restrict__ ccount) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= nnz) return;
    const unsigned int q = order[i];
    cdoc[i] = doc_of[q];
    ccount[i] = count[q];
}
__global__ void k_word_nchunks(int V, const long long* __restrict__ cptr, long long chunk, long long* __restrict__ nch) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= V) return;
    nch[w] = (cptr[w + 1] - cptr[w] + chunk - 1) / chunk;
}
__global__ void k_word_chunks(int V, const long long* __restrict__ cptr, const long long* __restrict__ wc, long long chunk,
                              long long* __restrict__ lo, long long* __restrict__ hi) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= V) return;
    long long k = wc[w];
    for (long long q = cptr[w]; q < cptr[w + 1]; q += chunk, ++k) {
        lo[k] = q;
        hi[k] = min(q + chunk, cptr[w + 1]);
    }
}
template <typename T>
__global__ void k_cast_to_ll(long long n, const T* __restrict__ in, long long* __restrict__ out) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) out[i] = static_cast<long long>(in[i]);
}
}  // namespace

// temp layout: [doc_of u32 nnz][order_in u32 nnz][keys_out u32 nnz][order_out u32 nnz]
//              [hist u64 V+1][nch ll V+1][flags u8 D][cub temp]
size_t corpus_gpu_temp_bytes(int V, long long D, long long nnz) {
    size_t sort_b = 0, scan_b = 0, sel_b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_b, (const unsigned int*)nullptr, (unsigned int*)nullptr,
                                    (const unsigned int*)nullptr, (unsigned int*)nullptr, static_cast<int>(std::max<long long>(nnz, 1)));
    cub::DeviceScan::ExclusiveSum(nullptr, scan_b, (const long long*)nullptr, (long long*)nullptr, V + 1);
    cub::DeviceSelect::Flagged(nullptr, sel_b, cub::CountingInputIterator<long long>(0), (const unsigned char*)nullptr,
                               (long long*)nullptr, (long long*)nullptr, static_cast<int>(std::max<long long>(D, 1)));
    const size_t nz = static_cast<size_t>(std::max<long long>(nnz, 1));
    // + 256-byte alignment slack for each of the 8 carved regions
    return 16 * nz + 2 * 8 * (static_cast<size_t>(V) + 1) + static_cast<size_t>(std::max<long long>(D, 1)) +
           std::max(sort_b, std::max(scan_b, sel_b)) + 8 * 256;
}

void corpus_gpu_build(cudaStream_t st, int V, long long D, long long nnz, const long long* doc_ptr, const int* word,
                      const int* count, bool check_counts, long long* total, long long* cptr, long long* cdoc,
                      int* ccount, long long* used_docs, unsigned long long* stats, long long chunk,
                      long long* word_chunk, long long* chunk_lo, long long* chunk_hi, void* temp, size_t temp_bytes) {
    const size_t nz = static_cast<size_t>(std::max<long long>(nnz, 1));
    unsigned char* t = static_cast<unsigned char*>(temp);
    auto carve = [&](size_t bytes) {
        unsigned char* p = t;
        t += (bytes + 255) / 256 * 256;
        return p;
    };
    unsigned int* doc_of = reinterpret_cast<unsigned int*>(carve(4 * nz));
    unsigned int* order_in = reinterpret_cast<unsigned int*>(carve(4 * nz));
    unsigned int* keys_out = reinterpret_cast<unsigned int*>(carve(4 * nz));
    unsigned int* order_out = reinterpret_cast<unsigned int*>(carve(4 * nz));
    unsigned long long* hist = reinterpret_cast<unsigned long long*>(carve(8 * (static_cast<size_t>(V) + 1)));
    long long* nch = reinterpret_cast<long long*>(carve(8 * (static_cast<size_t>(V) + 1)));
    unsigned char* flags = carve(static_cast<size_t>(std::max<long long>(D, 1)));
    void* cub_tmp = t;
    size_t cub_b = temp_bytes - static_cast<size_t>(t - static_cast<unsigned char*>(temp));
    cudaMemsetAsync(hist, 0, 8 * (static_cast<size_t>(V) + 1), st);
    cudaMemsetAsync(stats, 0, 8 * 8, st);
    if (D > 0)
        k_corpus_docs_scan<<<cdiv_w(D, 256), 256, 0, st>>>(D, V, doc_ptr, word, count, check_counts ? 1 : 0, total,
                                                            doc_of, hist, stats, flags);
    // cptr = exclusive scan of the histogram (V + 1 entries, last = nnz of valid words)
    k_cast_to_ll<unsigned long long><<<cdiv_w(V + 1, 256), 256, 0, st>>>(V + 1, hist, nch);
    cub::DeviceScan::ExclusiveSum(cub_tmp, cub_b, nch, cptr, V + 1, st);
    if (nnz > 0) {
        // stable sort of entry indices by word: documents stay ascending within each word
        k_iota_u32<<<cdiv_w(nnz, 256), 256, 0, st>>>(nnz, order_in);
        int bits = 1;
        while ((1ll << bits) < V) ++bits;
        cub::DeviceRadixSort::SortPairs(cub_tmp, cub_b, reinterpret_cast<const unsigned int*>(word), keys_out, order_in,
                                        order_out, static_cast<int>(nnz), 0, bits, st);
        k_corpus_gather<<<cdiv_w(nnz, 256), 256, 0, st>>>(nnz, order_out, doc_of, count, cdoc, ccount);
    }
    // used-document list (>= 3 tokens), ascending
    if (D > 0)
        cub::DeviceSelect::Flagged(cub_tmp, cub_b, cub::CountingInputIterator<long long>(0), flags, used_docs,
                                   reinterpret_cast<long long*>(&stats[5]), static_cast<int>(D), st);
    // word-pass chunk lists
    k_word_nchunks<<<cdiv_w(V, 256), 256, 0, st>>>(V, cptr, chunk, nch);
    cub::DeviceScan::ExclusiveSum(cub_tmp, cub_b, nch, word_chunk, V + 1, st);
    k_word_chunks<<<cdiv_w(V, 256), 256, 0, st>>>(V, cptr, word_chunk, chunk, chunk_lo, chunk_hi);
    for (int i = 0; i < 8; ++i) count_launch();
}

}  // namespace skc
