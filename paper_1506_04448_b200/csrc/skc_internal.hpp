// Internal interface between the C-ABI orchestration (skc_abi*.cu) and the
// kernels (skc_kernels.cu). Device pointers only; every launch goes on `st`.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "skc_fft.cuh"

namespace skc {

// Per-set device view used by the sketch kernels.
struct SymView {
    int n;
    std::uint32_t b;
    int logb;
    int B;
    const std::uint32_t* bucket1;  // B x n
    const std::uint32_t* bucket2;
    const std::uint32_t* bucket3;
    const std::uint8_t* sexp;
    const std::uint32_t* packed;  // h | e << 30
    const double2* tw;            // w_b^k, k in [0, b)
    const double2* twl;           // w_N^k, k in [0, N) (local transforms)
    // residue split
    int N, logN, S;
    const uint2* plan1;  // B x n: (i, h_i | e_i << 28) sorted by (h_i mod N, i)
    const uint2* plan2;  // B x n: (i, 2h_i mod b | 2e_i << 28) sorted by (2h_i mod N, i)
    const double2* data;         // B x b time domain
    const double2* spec;         // B x S x N local bit-reversed spectra
    // residue twiddles per (m, r): scatter (plan order) conj(w_b^{r t}), gather (index
    // order) w_b^{r t}; B x S x n each, or null (then taken from tw on the fly)
    const double2* stw1;
    const double2* stw2;
    const double2* gtw1;
    const double2* gtw2;
    int lpb = 4;  // restarts per CTA of the contraction kernels (set per launch)
};

struct AsymView {
    int n;
    std::uint32_t b;
    int logb;
    int B;
    const std::uint32_t* bucket;  // B x 3 x n
    const double* sign;           // B x 3 x n (+-1)
    const std::uint32_t* packed;  // B x 3 x n: h | neg << 31
    const double2* tw;
    const double2* twl;
    int N, logN, S;
    const uint2* plan;  // B x 3 x n: (i, h_s(i) | neg << 31) sorted by (h_s(i) mod N, i)
    const double2* data;
    const double2* spec;
};

std::uint64_t launch_count();
void count_launch();
void count_replay(std::uint64_t launches, std::uint64_t transforms);
std::uint64_t launch_count();
std::uint64_t transform_units();
std::uint64_t transform_units();          // local FFTs executed, in units of length-N transforms
void count_transforms(std::uint64_t local_ffts, int S);  // accumulate S-split counts

// tables
void launch_sym_tables(cudaStream_t st, const std::uint64_t* hcoef, const std::uint64_t* scoef, int n,
                       std::uint32_t b, int B, std::uint32_t* b1, std::uint32_t* b2, std::uint32_t* b3,
                       std::uint8_t* sexp, std::uint32_t* packed);
void launch_asym_tables(cudaStream_t st, const std::uint64_t* hcoef, const std::uint64_t* xcoef, int n,
                        std::uint32_t b, int B, std::uint32_t* bucket, double* sign, std::uint32_t* packed);
// keys: nrep x n table; perm[rep][rank] = i sorted by (keys & mask, i)
void launch_sort_perm(cudaStream_t st, const std::uint32_t* keys, int nrep, int n, std::uint32_t mask,
                      std::uint32_t* perm);
// plan[q] = (i, bucket_i | ((sexp_i * sexp_mult) & 3) << 28 | sign bit of packed_i) for i = perm[q]
void launch_make_plan(cudaStream_t st, const std::uint32_t* perm, const std::uint32_t* bucket, const std::uint8_t* sexp,
                      int sexp_mult, const std::uint32_t* packed, int nrep, int n, uint2* plan);

// dense build (skc_build.cu)
struct BuildPlan {
    int n;
    bool sym;
    int dtype;  // 0 f64, 1 f32
    const std::uint32_t* rowtab;  // packed (i << 16 | j) rows of the stream
    int nrows;
    // work split: G contiguous slot ranges ("types"), P persistent CTAs with dynamic
    // row hand-out per type (next_row counters) and migration between types
    int P, G;
    int* next_row;               // 2G ints: G row counters, then G per-window CTA counts
    int lock_rows = 0x3fffffff;  // class-list windows stay within this many rows of each other
    int cls_bits = -1;           // >= 0: class-list kernel, windows = (replicate, [parity,] bucket mod 2^cls_bits)
    bool one_limb = false;       // class-list kernel: one biased 32-bit limb per slot (fp32 input)
    int* ovf = nullptr;          // one-limb overflow flag (= nonfinite + 2)
    int xsrc_mode = 0;           // 0: pre-pass writes the fixed-point stream (contiguous-window kernels);
                                 // 1: class-list kernel reads the device-resident T (pre-pass: sums only);
                                 // 2: pre-pass writes a packed raw copy of the rows (bus-read T)
    unsigned long long* acc;     // total_slots exact fixed-point accumulators
    long long total_slots;   // B x 2b (sym) or B x b (asym)
    int slots_per_cta;
    int R;                   // max replicates a slot range overlaps
    std::uint32_t bmask;
    int B;
    const std::uint32_t* packed;  // sym: B x n (h | e << 30); asym: B x 3 x n (h | neg << 31)
    const long long* rowoff;      // packed-stream offset of each row
    long long* qbuf;              // packed fixed-point stream (quantize pass)
    short* rowF;                  // per-row exponent of qbuf
    double* prepass_partials;     // nseg segments of [prepass_blocks L1 sums, prepass_blocks maxima]
    int nseg = 1;                 // > 1: all-gathered partials of nseg ranks (multi-GPU build)
    int prepass_blocks = 1024, prepass_threads = 256, prepass_warps = 8;
    bool reset_nonfinite = true;
    bool pdl = false;  // main and finalize launched programmatically dependent (single-stream build)
    int* scale_exp;               // device int
    int* nonfinite;               // device int
    double* data_as_double;       // B x b x 2
    long long total_entries = 0;  // entries of the whole build (all ranks' slices)
    double rho_max = 0.0;         // resolution bound of the build (0: by limbs; +inf: band passes)
    double band_lo = 0.0, band_hi = INFINITY;  // magnitude band of kappa|T| (HDR band passes)
};
// Exponent histogram of kappa|T| over a build's rows (HDR builds): hist[e + kExpBias] counts
// the entries with 2^e <= kappa|T| < 2^(e+1), zeros not counted.
constexpr int kExpBias = 1100, kExpBins = 2200;
void launch_build_exp_hist(cudaStream_t st, const void* T, const BuildPlan& p, unsigned long long* hist);
constexpr int kPrepassBlocks = 1024;
size_t build_smem_bytes(long long slots_per_cta, int R, int n);
size_t cls_smem_bytes(std::uint32_t b, int tbits, int n, bool sym, bool one_limb);
void launch_build_prepass(cudaStream_t st, const void* T, const BuildPlan& p);
void launch_build_main(cudaStream_t st, const void* T, const BuildPlan& p);
void launch_build_finalize(cudaStream_t st, const BuildPlan& p);
void launch_build_finalize_multi(cudaStream_t st, const BuildPlan& p, int K, const int* scale_exps, int* counters,
                                 int ncounters);

// LDA moments / whitening (skc_whiten.cu)
void launch_corpus_prep(cudaStream_t st, int V, long long D, const long long* doc_ptr, const int* count,
                        const long long* cptr, const long long* cdoc, const int* ccount, long long* total, double* s2,
                        double* invm, double* diag, double* m1p);
void launch_m2_apply(cudaStream_t st, int V, long long D, int p, const long long* doc_ptr, const int* word,
                     const int* count, const long long* cdoc, const int* ccount, long long nchunks,
                     const long long* chunk_lo, const long long* chunk_hi, const long long* word_chunk,
                     const double* s2, const double* diag, const double* m1p, double inv_used1, double inv_used2,
                     double a, const double* X, double* Z, double* part, double* mx, double* Y);
// FP64 C = op(A) op(B) with element strides (skc_gemm.cu); split-K partials in ws
// (dgemm_slices(M, N, K, sms) x M x N doubles when more than one slice)
int dgemm_slices(int M, int N, int K, int sms);
void launch_dgemm(cudaStream_t st, int sms, int M, int N, int K, const double* A, long long ai, long long ak,
                  const double* B, long long bk, long long bj, double* C, long long ci, long long cj, double* ws);
void launch_scale_cols(cudaStream_t st, long long rows, int k, const double* in, const double* f, double* out);
void launch_normalize_columns(cudaStream_t st, int n, int k, double* F, const double* prev, double* lambda);
void launch_gaussian_fill(cudaStream_t st, unsigned long long seed, long long count, double* out);
// device corpus preparation (skc_whiten.cu): stats[0..5] = bad doc_ptr, bad word, negative
// count, docs >= 1 token, docs >= 2 tokens, docs >= 3 tokens
size_t corpus_gpu_temp_bytes(int V, long long D, long long nnz);
void corpus_gpu_build(cudaStream_t st, int V, long long D, long long nnz, const long long* doc_ptr, const int* word,
                      const int* count, bool check_counts, long long* total, long long* cptr, long long* cdoc,
                      int* ccount, long long* used_docs, unsigned long long* stats, long long chunk,
                      long long* word_chunk, long long* chunk_lo, long long* chunk_hi, void* temp, size_t temp_bytes);

// residue twiddle tables of a symmetric set (SymView::stw*/gtw*)
void launch_sym_twiddle_tables(cudaStream_t st, const SymView& v, double2* stw1, double2* stw2, double2* gtw1,
                               double2* gtw2);

// spectra: spec[m][r][j] = local DIF of residue r of data[m]
void launch_spectrum(cudaStream_t st, const double2* data, std::uint32_t b, int logb, int B, int N, int logN,
                     int S, const double2* tw, const double2* twl, double2* spec);

// symmetric contractions. mode 0: Ivv partials (L x B x S x n); mode 1: vvv
// partials (L x B x S x 3: acc1, acc2, term3).
void launch_sym_contract(cudaStream_t st, const SymView& v, const double* U, int L, int mode, double* out);
// medians: part L x B x S x n -> out L x n (and optional normalisation into Unext)
void launch_median_rows(cudaStream_t st, const double* part, int L, int B, int S, int n, double* out,
                        double* Unext, double tol, int* flags, double* scratch = nullptr);
void launch_sym_vvv_finish(cudaStream_t st, const double* part, int L, int B, int S, std::uint32_t b,
                           double* values);
void launch_asym_vvv_finish(cudaStream_t st, const double* part, int L, int B, int S, std::uint32_t b,
                            double* values);
void launch_argmax_first(cudaStream_t st, const double* values, int L, int* best, double* best_value);

// deflation / rank-1 / factored / moment accumulation (frequency domain)
// acc[chunk][m][r][N] partial spectra; then reduce+DIT -> tmp[m][r][N]; combine -> data.
// acc[chunk][m][r][j] = sum over samples s in chunk of wscale * w[s] * F_r(CS_m(x_s))[j]^3
// (w may be null: weight 1). chunks * B * S CTAs.
void launch_sym_moment_accumulate(cudaStream_t st, const SymView& v, const double* X, const double* w,
                                  double wscale, long long Nsamp, int chunks, double* acc);
void launch_freq_reduce_inverse(cudaStream_t st, const double* acc, int chunks, int B, int S, int N, int logN,
                                std::uint32_t b, int logb, const double2* twl, double2* tmp);
void launch_combine_residues(cudaStream_t st, const double2* tmp, int B, int S, int N, std::uint32_t b,
                             const double2* tw, double alpha, int m_only, bool overwrite, double2* dst,
                             bool scaled = true);
void launch_asym_factored_accumulate(cudaStream_t st, const AsymView& v, const double* a, const double* U,
                                     const double* V, const double* W, long long Ncomp, int chunks, int m_only,
                                     double* acc);

// asymmetric contractions
void launch_asym_mode(cudaStream_t st, const AsymView& v, int free_mode, const double* X, const double* Y, int L,
                      double* part);
void launch_asym_vvv(cudaStream_t st, const AsymView& v, const double* U, int L, double* part);

// sym_aux_sketches / sketch_rank1_sym (sketch.cpp:412-443)
void launch_sym_aux(cudaStream_t st, const SymView& v, int m, const double* u, double2* out /* 3 x b */);
void launch_rank1_trunc_product(cudaStream_t st, const double2* spec2, long long len, double2* acc);
void launch_add_third(cudaStream_t st, const double2* s3, std::uint32_t b, double2* out);

// LDA recover_params / heldout_likelihood (skc_lda_post.cu)
void launch_lda_recover_params(cudaStream_t st, int V, int k, const double* lambda, const double* A,
                               const double* unwhiten, double alpha0, double* mu, double* Phi);
void launch_phi_gram(cudaStream_t st, int V, int k, const double* Phi, double* G);
bool launch_lda_heldout(cudaStream_t st, int k, long long D, const long long* doc_ptr, const int* word, const int* count,
                        const double* Phi, const double* G, double step, double* per, long long* floored);
// LDA whitened third moment (skc_lda.cu)
void launch_lda_docs(cudaStream_t st, int k, long long D, const long long* doc_ptr, const int* word, const int* count,
                     const double* W, double alpha0, double* P, double* s1, double* s2, long long* total);
void launch_lda_vocab_chunked(cudaStream_t st, int k, int V, long long nchunks, const long long* chunk_lo,
                              const long long* chunk_hi, const long long* word_chunk, const long long* cdoc,
                              const int* ccount, const double* P, const double* s1, const long long* total,
                              double* part, double* coeff1, double* sumwn, double* m1_partial);
void launch_lda_vocab(cudaStream_t st, int k, int V, const long long* cptr, const long long* cdoc, const int* ccount,
                      const double* P, const double* s1, const long long* total, double* coeff1, double* sumwn,
                      double* m1_partial);
void launch_lda_q(cudaStream_t st, int k, int V, const double* W, const double* m1_partial, double inv_used1,
                  double* q);
void launch_lda_accumulate(cudaStream_t st, const SymView& v, long long Du, const long long* used_docs, const double* P,
                           const double* s1, const double* s2, int V, const double* W, const double* coeff1,
                           const double* sumwn, int chunks_d, int chunks_v, double* acc, double* cross);
void launch_lda_finish(cudaStream_t st, const SymView& v, const double* acc, const double* cross, int chunks_acc,
                       int chunks_cross, const double* q, double inv_docs, double m1_coeff, double2* tmp);

// generators
void launch_gen_planted(cudaStream_t st, int n, int rank, const double* lambda, const double* V, double sigma,
                        std::uint64_t seed, int dtype, void* out);

}  // namespace skc
