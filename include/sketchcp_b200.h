/*
 * sketchcp_b200.h — C-ABI of the B200-native FFT tensor-sketch hot path.
 *
 * This is the drop-in boundary for the reference C++ library `sketchcp`
 * (arXiv 1506.04448 reference, proj/include/sketchcp/). The reference has no
 * FFI layer; its path is reached through C++ classes. Each entry point below
 * names the reference member it replaces (file:line under proj/). The reference's
 * C++ classes (SymTensorSketchSet, SymContractionWorkspace, robust_tpm_fast, ...)
 * are re-implemented as thin host wrappers over these functions (see
 * INTEGRATION.md for the C++ and ctypes bindings).
 *
 * Conventions
 *  - Plain pointers and sizes only. Complex arrays are interleaved (re, im) fp64,
 *    i.e. std::complex<double> layout. Dense tensors are row-major (i,j,k) at
 *    (i*n + j)*n + k, like DenseTensor3 (tensor.hpp:15-28).
 *  - Every function returns a status code (SKC_OK = 0). On failure the message is
 *    available from skc_last_error() (thread-local). Status codes map onto the
 *    reference exception taxonomy (common.hpp:15-27):
 *      SKC_INVALID_ARGUMENT  -> std::invalid_argument
 *      SKC_NUMERICAL_ERROR   -> sketchcp::NumericalError
 *      SKC_DEGENERATE        -> sketchcp::DegenerateIterationError
 *      SKC_FORMAT_ERROR      -> sketchcp::FormatError
 *  - All calls are synchronous at the boundary unless the name ends in _async.
 *  - `host` arguments are host pointers; `dev` arguments are device pointers on
 *    the context's device. A `location` argument selects between the two
 *    (SKC_HOST / SKC_DEVICE).
 *  - There is no CPU fallback: on a machine without a usable sm_100 device every
 *    compute entry point fails with SKC_CUDA_ERROR.
 */
#ifndef SKETCHCP_B200_H
#define SKETCHCP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SKC_OK = 0,
    SKC_INVALID_ARGUMENT = 1,
    SKC_NUMERICAL_ERROR = 2,
    SKC_DEGENERATE = 3,
    SKC_FORMAT_ERROR = 4,
    SKC_CUDA_ERROR = 5,
    SKC_OUT_OF_MEMORY = 6
};
enum { SKC_HOST = 0, SKC_DEVICE = 1 };
enum { SKC_F64 = 0, SKC_F32 = 1 };

typedef struct skc_context skc_context;
typedef struct skc_sym_set skc_sym_set;
typedef struct skc_asym_set skc_asym_set;

/* ---- errors / library ---------------------------------------------------- */
const char* skc_last_error(void);
int skc_version(void);
/* Number of CUDA kernels this library has launched so far (process-wide). */
uint64_t skc_kernel_launch_count(void);
/* Number of local FFTs executed on the device so far; the analogue of
 * fft::transform_count() (fft.hpp:25) counted in units of full length-b
 * transforms. */
uint64_t skc_transform_count(void);

/* ---- context: one per device; owns a stream and scratch -------------------- */
int skc_context_create(int device, skc_context** out);
int skc_context_destroy(skc_context* ctx);
int skc_context_synchronize(skc_context* ctx);
/* The stream all work of this context is enqueued on (cudaStream_t). */
int skc_context_stream(skc_context* ctx, void** stream_out);
/* Orders all later work of this context after everything already enqueued on
 * `producer` (a cudaStream_t; NULL = the legacy default stream): an event is
 * recorded on `producer` and the context stream waits on it, with no host sync.
 * Ordering contract for device pointers: every entry point that takes a device
 * pointer reads it on the context stream, so a caller whose input is produced
 * on another stream (e.g. a framework's current stream) calls this first.
 * Results are complete when the entry point returns (synchronous API) unless the
 * entry point says otherwise. */
int skc_context_wait_stream(skc_context* ctx, void* producer);
/* Dense builds of fp32 tensors run with one 32-bit limb per sketch slot; a build whose
 * limb could overflow (a partial sum reached 2^30, i.e. ~2^8 same-signed full-scale adds
 * to one slot in one pass) or whose entries need a finer scale is discarded and repeated
 * exactly with two limbs. Number of such repeats so far. */
int skc_context_build_retries(skc_context* ctx, long long* out);
/* Dense builds redone in magnitude bands: tensors whose entries span more magnitudes than
 * one exact fixed-point scale resolves to ~2^-34 of each bucket (high dynamic range). */
int skc_context_build_banded(skc_context* ctx, long long* out);
int skc_device_count(int* out);
/* Per-kernel device timing with CUDA events on the context stream (off by
 * default). skc_profile_get sums the recorded durations of one kernel family
 * ("build_prepass", "build_main", "build_finalize", "spectrum", "sym_contract",
 * "median", "moment", "freq_inverse", "combine", "asym_mode", "asym_vvv",
 * "asym_factored") since the last reset. */
int skc_profile_enable(skc_context* ctx, int on);
int skc_profile_reset(skc_context* ctx);
int skc_profile_get(skc_context* ctx, const char* kernel, double* total_ms, uint64_t* launches);

/* ---- host-side helpers (no device needed) --------------------------------- */
/* derive_seed (rng.hpp:35-46) */
uint64_t skc_derive_seed(uint64_t master, uint64_t tag, uint64_t i0, uint64_t i1);
/* Rng(seed).unit_sphere(n) (rng.hpp:100-106) */
int skc_unit_sphere(uint64_t seed, int n, double* out);
/* RTPM initial vectors: out[(c*L + tau)*n + i] = Rng(derive_seed(seed,0x31,c,tau)).unit_sphere(n)
 * for c in [c0, c0+k), tau in [tau0, tau0+L)  (decompose.cpp:99-100) */
int skc_power_inits(uint64_t seed, int n, int c0, int k, int tau0, int L, double* out);
/* PolyHash::from_seed coefficients (hashing.cpp:8-16) and eval (hashing.hpp:29-34) */
int skc_poly_coefficients(int independence, uint64_t seed, uint64_t* out);
uint32_t skc_poly_eval(const uint64_t* coeffs, int k, uint32_t b, uint64_t i);

/* ---- symmetric sketch set: SymTensorSketchSet (sketch.hpp:87-136) --------- */
/* SymTensorSketchSet(n, b, B, master_seed) (sketch.cpp:300-313). Hash
 * coefficients are drawn on the host (bit-exact mt19937_64 stream); the bucket /
 * sign tables are derived on the device from them. */
int skc_sym_create(skc_context* ctx, int n, uint32_t b, int B, uint64_t master_seed, skc_sym_set** out);
/* Construction from stored coefficients (SymTensorSketchSet::load, sketch.cpp:391-410):
 * hcoef B*6 (bucket hash), scoef B*6 (complex4 sign hash), data B*b complex or NULL. */
int skc_sym_create_from_coefficients(skc_context* ctx, int n, uint32_t b, int B, uint64_t master_seed,
                                     const uint64_t* hcoef, const uint64_t* scoef, const double* data_host,
                                     skc_sym_set** out);
int skc_sym_destroy(skc_sym_set* s);
/* n(), b(), replicates(), master_seed(), version() (sketch.hpp:100-104) */
int skc_sym_info(const skc_sym_set* s, int* n, uint32_t* b, int* B, uint64_t* master_seed, uint64_t* version);
/* Device-derived tables of replicate m, copied to the host (Replicate fields,
 * sketch.hpp:89-95): bucket1=h, bucket2=2h mod b, bucket3=3h mod b, sexp. */
int skc_sym_tables(const skc_sym_set* s, int m, uint32_t* bucket1, uint32_t* bucket2, uint32_t* bucket3,
                   uint8_t* sexp);
int skc_sym_coefficients(const skc_sym_set* s, uint64_t* hcoef, uint64_t* scoef);
/* accumulate_dense(T, assume_symmetric) (sketch.cpp:315-345) restricted to the
 * i-slice [i0, i1) of the sorted-triple loop (i0=0, i1=n for the whole tensor;
 * slices let ranks shard the build). T is the full n^3 tensor (row-major), fp64
 * or fp32 (dtype), on the host or the device. Without assume_symmetric the
 * symmetry check of the reference (tolerance 1e-9, tensor.cpp:32-43) runs first. */
int skc_sym_accumulate_dense(skc_sym_set* s, const void* T, int dtype, int location, int assume_symmetric,
                             int i0, int i1);
/* add_scaled_rank1(u, alpha) (sketch.cpp:347-361); u host n-vector. */
int skc_sym_add_scaled_rank1(skc_sym_set* s, const double* u_host, double alpha);
/* Frequency-domain accumulation of a factored symmetric moment:
 *   data += sum_i w_i * (full symmetric sketch of x_i^(x)3)
 * X: N x n row-major samples (fp64) on host or device, w: N weights (same location).
 * Mathematically N calls of add_scaled_rank1(x_i, w_i) with one inverse transform
 * per replicate at the end, the pattern of lda.cpp:195-223. */
int skc_sym_accumulate_moment(skc_sym_set* s, const double* X, const double* w, long long N, int location);
/* sketch_whitened_m3(corpus, W, alpha0, set) (lda.cpp:145-226). Corpus in CSR form
 * (doc_ptr[D+1] with doc_ptr[0] = 0, word[nnz], count[nnz]) and the whitening map W
 * (V x k row-major, k == set n), all host arrays. used/skipped receive StreamStats
 * (lda.hpp:57-60). Documents shorter than 3 tokens are skipped (lda.cpp:164-167). */
int skc_sym_sketch_whitened_m3(skc_sym_set* s, int V, long long D, const long long* doc_ptr, const int* word,
                               const int* count, const double* W, double alpha0, long long* used,
                               long long* skipped);
/* als_fast(set, AlsConfig{k, max_iters, tol, seed}) (decompose.cpp:117-205): CP-ALS with
 * batched sketched mode contractions. lambda[k]; A, B, C n x k column-major; iters_out
 * (may be null) receives the number of sweeps run. */
int skc_asym_als(skc_asym_set* s, int k, int max_iters, double tol, uint64_t seed, double* lambda, double* A,
                 double* B, double* C, int* iters_out);

/* ---- LDA moments and whitening (lda.cpp:88-143) -------------------------------------
 * Corpus arguments as for skc_sym_sketch_whitened_m3 (host CSR). Matrices are row-major.
 * compute_m1 (lda.cpp:88-100): m1[V] = mean over documents with >= 1 token of n_d / m_d. */
int skc_lda_compute_m1(skc_context* ctx, int V, long long D, const long long* doc_ptr, const int* word,
                       const int* count, double* m1_out);
/* Y = M2 X for X, Y host V x p, where M2 is compute_m2(corpus, alpha0) (lda.cpp:102-123)
 * applied without forming it (the V x V matrix of the reference). */
int skc_lda_m2_apply(skc_context* ctx, int V, long long D, const long long* doc_ptr, const int* word,
                     const int* count, double alpha0, int p, const double* X, double* Y);
/* whiten(compute_m2(corpus, alpha0), k) (lda.cpp:125-143) by randomized subspace
 * iteration on the implicit M2 (block p = k + oversample rounded up to 32, `iters`
 * power steps, Gaussian start from derive_seed(seed, 0x68)) and a Rayleigh-Ritz
 * projection. Outputs: W and unwhiten V x k, singular_values k (descending eigenvalues).
 * oversample < 0 / iters < 0 select the defaults (max(16, k/4), 12). Errors follow the
 * reference: invalid rank -> SKC_INVALID_ARGUMENT, eigenvalue <= 1e-10 ->
 * SKC_NUMERICAL_ERROR "whiten: moment matrix is rank deficient at component c (...)". */
int skc_lda_whiten_corpus(skc_context* ctx, int V, long long D, const long long* doc_ptr, const int* word,
                          const int* count, double alpha0, int k, int oversample, int iters, uint64_t seed,
                          double* W, double* unwhiten, double* singular_values);
/* whiten(m2hat, k) for a dense symmetric host V x V matrix (same algorithm, DGEMM operator). */
int skc_lda_whiten_dense(skc_context* ctx, int V, const double* m2, int k, int oversample, int iters, uint64_t seed,
                         double* W, double* unwhiten, double* singular_values);

/* Document shard of sketch_whitened_m3 for multi-GPU runs: document sums over this
 * shard, normalised by the whole corpus' global_used (documents with >= 3 tokens) and
 * using its averaged M1 (global_m1, V); add_q_cubed != 0 on exactly one shard. Summing
 * the shards' data (all-reduce) gives the full sketch (the sketch is linear in the
 * per-document terms). */
int skc_sym_sketch_whitened_m3_shard(skc_sym_set* s, int V, long long D, const long long* doc_ptr, const int* word,
                                     const int* count, const double* W, double alpha0, long long global_used,
                                     const double* global_m1, int add_q_cubed, long long* used, long long* skipped);

/* Device-resident corpus (B200 extension): upload + validate + word-major transpose once,
 * then whiten and sketch without re-uploading (the reference passes Corpus& to each). */
typedef struct skc_lda_corpus skc_lda_corpus;
int skc_lda_corpus_create(skc_context* ctx, int V, long long D, const long long* doc_ptr, const int* word,
                          const int* count, skc_lda_corpus** out);
int skc_lda_corpus_destroy(skc_lda_corpus* c);
int skc_lda_corpus_info(const skc_lda_corpus* c, int* V, long long* D, long long* nnz, long long* used3);
int skc_lda_whiten_corpus_handle(skc_lda_corpus* c, double alpha0, int k, int oversample, int iters, uint64_t seed,
                                 double* W, double* unwhiten, double* singular_values);
int skc_sym_sketch_whitened_m3_corpus(skc_sym_set* s, skc_lda_corpus* c, const double* W, double alpha0,
                                      long long* used, long long* skipped);

/* recover_params(D, wm, alpha0) (lda.cpp:228-248) on ctx's device: lambda[k], A = D.A (k x k
 * row-major, column i = component i), unwhiten V x k -> Phi V x k (mu_i = 0.5 (alpha0 + 2)
 * lambda_i unwhiten A[:, i] projected onto the simplex, lda.cpp:250-271) and alpha[k]. */
int skc_lda_recover_params(skc_context* ctx, int V, int k, const double* lambda, const double* A,
                           const double* unwhiten, double alpha0, double* Phi, double* alpha);
/* heldout_likelihood(model, held) (lda.cpp:273-320) on ctx's device: Phi V x k (k <= 128),
 * held-out corpus CSR over vocabulary Vh <= V; one warp per document (500 projected-
 * gradient steps), the per-document values summed in document order. */
int skc_lda_heldout_likelihood(skc_context* ctx, int V, int k, const double* Phi, int Vh, long long D,
                               const long long* doc_ptr, const int* word, const int* count, double* ll_out,
                               long long* floored_words);

/* replicate(m).data -> host (B-major when m < 0: all replicates, B*b complex). */
int skc_sym_read_data(const skc_sym_set* s, int m, double* out_host);
/* mutable_replicate(m).data = in (bumps version, sketch.hpp:105-108); m < 0: all. */
int skc_sym_write_data(skc_sym_set* s, int m, const double* in_host);
/* Device pointer to the B*b complex data (for collectives); bump version after writes. */
int skc_sym_data_device(skc_sym_set* s, void** dev_ptr, size_t* bytes);
int skc_sym_bump_version(skc_sym_set* s);
/* sym_aux_sketches(rep(m), b, u) (sketch.cpp:412-425): s1/s2/s3 host arrays of 2*b doubles
 * (any may be NULL). */
int skc_sym_aux_sketches(const skc_sym_set* s, int m, const double* u_host, double* s1, double* s2, double* s3);
/* sketch_rank1_sym(set, m, u) (sketch.cpp:427-443): sketch of the upper-triangular
 * truncation of u^(x)3, (1/6) s1*s1*s1 + (1/2) s2*s1 + (1/3) s3 -> out 2*b doubles. */
int skc_sym_rank1_truncated(const skc_sym_set* s, int m, const double* u_host, double* out_host);
/* recover_entry(i,j,k) (sketch.cpp:363-377) */
int skc_sym_recover_entry(const skc_sym_set* s, int i, int j, int k, double* out);

/* ---- symmetric contractions: SymContractionWorkspace (contraction.hpp:14-41) */
/* Batched Ivv: out[l*n + i] = median-of-B estimate of T(I,u_l,u_l)_i
 * (contraction.cpp:128-181) for the L vectors U (L x n row-major, host). */
int skc_sym_ivv(skc_sym_set* s, const double* U_host, int L, double* out_host);
/* Batched vvv: out[l] = median-of-B estimate of T(u_l,u_l,u_l) (contraction.cpp:83-126). */
int skc_sym_vvv(skc_sym_set* s, const double* U_host, int L, double* out_host);
/* cached_transform(m) (contraction.cpp:78-81): natural-order F(data_m), 2*b doubles. */
int skc_sym_cached_transform(skc_sym_set* s, int m, double* out_host);

/* ---- fast robust tensor power method (decompose.cpp:83-115) ---------------- */
/* robust_tpm_fast(set, cfg{k, L, T_iters, seed, tol}). inits: k*L*n host array of
 * initial vectors ((c*L + tau)*n + i) or NULL to draw the reference's
 * Rng(derive_seed(seed, 0x31, c, tau)).unit_sphere(n). Outputs: lambda[k],
 * V (n x k column-major, i.e. V[c*n + i]), best_tau[k] (may be NULL). The set is
 * left deflated. SKC_DEGENERATE when a power iterate vanishes (decompose.cpp:35-40). */
int skc_sym_rtpm(skc_sym_set* s, int k, int L, int T_iters, uint64_t seed, double tol, const double* inits,
                 double* lambda, double* V, int* best_tau);
/* One RTPM component over a block of restarts (the multi-GPU building block):
 * runs T_iters normalised power steps on the L restarts U0 (L x n host), then the
 * median vvv of every final iterate. finals_out (L x n) and values_out (L) are
 * host arrays. No deflation. */
int skc_sym_rtpm_restarts(skc_sym_set* s, const double* U0_host, int L, int T_iters, double tol,
                          double* finals_out, double* values_out);

/* ---- multi-GPU: NCCL over NVLink / NVSwitch (B200 extension) ----------------
 * Replaces the reference's in-process OpenMP loops over replicates (sketch.cpp:325,
 * contraction.cpp:145) and its serial restart loop (decompose.cpp:92-112) with one
 * replica of a set per GPU and partitions that need one exchange each:
 *   dense build: equal-work i-slices of the sorted triples; pre-pass partials
 *     all-gathered (one global exponent), exact int64 accumulators all-reduced, so the
 *     sketch is bit-identical at any rank count;
 *   moment: sample blocks, per-residue partial transforms all-reduced;
 *   LDA sketch_whitened_m3: document blocks, corpus globals then data all-reduced;
 *   RTPM: restart blocks of ceil(L/R), selection values all-gathered, the first maximum
 *     over tau on every rank, the winner's vector broadcast, identical deflation.
 * A communicator spans R ranks, one context (GPU) each. Ranks live in one process
 * (skc_group_create: ncclCommInitAll over a device list, contexts returned in rank
 * order) or in one process each (rank 0 makes an id with skc_nccl_unique_id, every rank
 * passes it to skc_context_comm_init). The *_group calls are collective: every process
 * calls them with its local replicas (sets on its contexts, rank order); every replica
 * holds the same sketch before and after. Per-set input pointers may all be the same
 * host array; SKC_DEVICE inputs are per-set device pointers (each holding the whole
 * tensor / sample matrix; a rank reads only its block). */
int skc_nccl_unique_id(char* out /* 128 bytes */);
int skc_context_comm_init(skc_context* ctx, int nranks, int rank, const char* id /* 128 bytes */);
int skc_group_create(const int* devices, int ndev, skc_context** ctxs_out /* ndev */);
int skc_context_comm_info(const skc_context* ctx, int* nranks, int* rank);
/* host plumbing (no device): the i-slice bounds[nranks + 1] of a dense build and the
 * restart block [t0, t1) of a rank */
int skc_group_slices(int n, int sym, int nranks, int* bounds);
int skc_group_restart_chunk(int L, int nranks, int rank, int* t0, int* t1);
int skc_sym_accumulate_dense_group(skc_sym_set* const* sets, int nsets, const void* const* T, int dtype, int location,
                                   int assume_symmetric);
int skc_sym_accumulate_moment_group(skc_sym_set* const* sets, int nsets, const double* const* X, const double* const* w,
                                    long long N, int location);
int skc_sym_rtpm_group(skc_sym_set* const* sets, int nsets, int k, int L, int T_iters, uint64_t seed, double tol,
                       const double* inits, double* lambda, double* V, int* best_tau);
int skc_sym_sketch_whitened_m3_group(skc_sym_set* const* sets, int nsets, int V, long long D, const long long* doc_ptr,
                                     const int* word, const int* count, const double* W, double alpha0,
                                     long long* used, long long* skipped);

/* ---- asymmetric sketch set: AsymTensorSketchSet (sketch.hpp:27-82) --------- */
int skc_asym_create(skc_context* ctx, int n, uint32_t b, int B, uint64_t master_seed, skc_asym_set** out);
/* hcoef B*3*2, xcoef B*3*6 (AsymTensorSketchSet::load, sketch.cpp:276-296) */
int skc_asym_create_from_coefficients(skc_context* ctx, int n, uint32_t b, int B, uint64_t master_seed,
                                      const uint64_t* hcoef, const uint64_t* xcoef, const double* data_host,
                                      skc_asym_set** out);
int skc_asym_destroy(skc_asym_set* s);
int skc_asym_info(const skc_asym_set* s, int* n, uint32_t* b, int* B, uint64_t* master_seed, uint64_t* version);
/* bucket[3*n] (slot-major), sign[3*n] of replicate m (Replicate, sketch.hpp:29-36) */
int skc_asym_tables(const skc_asym_set* s, int m, uint32_t* bucket, double* sign);
int skc_asym_coefficients(const skc_asym_set* s, uint64_t* hcoef, uint64_t* xcoef);
/* accumulate_dense(T) (sketch.cpp:173-193) over the i-slice [i0, i1). */
int skc_asym_accumulate_dense(skc_asym_set* s, const void* T, int dtype, int location, int i0, int i1);
/* add_rank1(alpha, u, v, w) (sketch.cpp:214-222) */
int skc_asym_add_rank1(skc_asym_set* s, double alpha, const double* u, const double* v, const double* w);
/* accumulate_factored(F) (sketch.cpp:224-248): N components, a[N], U,V,W N x n
 * row-major, host arrays. */
int skc_asym_accumulate_factored(skc_asym_set* s, long long N, const double* a, const double* U,
                                 const double* V, const double* W);
/* rank1_sketch(m, u, v, w) (sketch.cpp:195-212) -> out 2*b doubles */
int skc_asym_rank1_sketch(skc_asym_set* s, int m, const double* u, const double* v, const double* w,
                          double* out_host);
int skc_asym_read_data(const skc_asym_set* s, int m, double* out_host);
int skc_asym_write_data(skc_asym_set* s, int m, const double* in_host);
int skc_asym_data_device(skc_asym_set* s, void** dev_ptr, size_t* bytes);
int skc_asym_bump_version(skc_asym_set* s);
int skc_asym_recover_entry(const skc_asym_set* s, int i, int j, int k, double* out);
/* AsymContractionWorkspace (contraction.hpp:43-77), batched over L vector pairs:
 * mode_contraction(free_mode, x_l, y_l) (contraction.cpp:248-295); Ivv(u) is
 * free_mode 0 with x = y = u; Ibc(b, c) is free_mode 0 with x = b, y = c. */
int skc_asym_mode_contraction(skc_asym_set* s, int free_mode, const double* X_host, const double* Y_host, int L,
                              double* out_host);
/* vvv(u) (contraction.cpp:209-246) */
int skc_asym_vvv(skc_asym_set* s, const double* U_host, int L, double* out_host);
int skc_asym_cached_transform(skc_asym_set* s, int m, double* out_host);

/* ---- standalone transforms: fft::forward_inplace / inverse_inplace /
 * inverse_inplace_unscaled (fft.hpp:15-20, fft.cpp:48-66) on the device of a process-wide
 * context. x: 2*b doubles (interleaved complex) transformed in place; dir -1 forward,
 * +1 inverse scaled by 1/b, +2 inverse unscaled. b must be a power of two. */
int skc_fft(double* x_host, size_t b, int dir);

/* ---- sketch file container (sketch.cpp:47-141, 264-296, 379-410, 445-449) ------ */
/* save/load and peek_sketch_mode; little-endian, magic SKCPSKT\0, version 1. Loading
 * rebuilds the tables from the stored coefficients; errors are SKC_FORMAT_ERROR. */
int skc_peek_sketch_mode(const char* path, int* mode /* 0 asym, 1 sym */);
int skc_sym_save(const skc_sym_set* s, const char* path);
int skc_sym_load(skc_context* ctx, const char* path, skc_sym_set** out);
int skc_asym_save(const skc_asym_set* s, const char* path);
int skc_asym_load(skc_context* ctx, const char* path, skc_asym_set** out);

/* ---- synthetic inputs for the benchmark configs (host generators) ---------- */
/* Planted symmetric tensor T = sum_r lambda_r v_r^(x)3 + sigma*E (BASELINE configs 0-2):
 * lambda_r ~ U[1,2], V = Q of a Gram-Schmidt QR of an n x rank N(0,1) matrix, E
 * N(0,1) drawn for i<=j<=k and mirrored. Outputs: T (n^3, fp64 or fp32 by dtype),
 * lambda[rank], V (n x rank column-major). Seeds via derive_seed(seed, 0x61..0x63). */
int skc_gen_planted_tensor(int n, int rank, double sigma, uint64_t seed, int dtype, void* T_out,
                           double* lambda_out, double* V_out);
/* Same tensor generated directly in device memory (n^3 elements of dtype at dev_out);
 * noise from a counter-based generator, so it differs from the host generator's noise. */
int skc_gen_planted_tensor_device(skc_context* ctx, int n, int rank, double sigma, uint64_t seed, int dtype,
                                  void* dev_out, double* lambda_out, double* V_out);

#ifdef __cplusplus
}
#endif
#endif /* SKETCHCP_B200_H */
