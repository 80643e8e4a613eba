// sm_100a kernels of the FFT tensor-sketch hot path.
//
//  K0  k_sym_tables / k_asym_tables   hash tables from coefficients (bit-exact integer Horner)
//  K1  k_build_prepass/main/finalize  dense sketch build: simplex (sym) or full (asym) stream,
//                                     scatter-add into smem with exact 64-bit fixed point
//                                     (two native 32-bit ATOMS.ADD + carry per contribution)
//  K4  k_spectrum                     residue-split forward FFT of every replicate
//  K3  k_sym_contract                 fused scatter -> 2x FFT -> spectrum product -> 2x IFFT -> gather
//      k_median_rows / *_vvv_finish   deterministic median over replicates (+ normalisation)
//  K2  k_sym_moment / k_asym_factored frequency-domain accumulation of rank-1 / moment sketches
//      k_freq_reduce_inverse/combine  reduce partial spectra, inverse FFT, recombine residues
//
// Reference loops replaced are cited per kernel (paths under proj/ of the reference).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>

#include "skc_fft.cuh"
#include "skc_host.hpp"
#include "skc_internal.hpp"

namespace skc {

namespace {
std::atomic<std::uint64_t> g_launches{0};
std::atomic<std::uint64_t> g_transforms{0};

inline unsigned cdiv(long long a, long long b) { return static_cast<unsigned>((a + b - 1) / b); }

// Deterministic block sum (fixed shuffle tree + fixed smem order).
template <int NT>
__device__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) {
        t = (lane < NT / 32) ? red[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    }
    return t;  // valid in thread 0
}

__device__ __forceinline__ std::uint32_t poly_eval_dev(const std::uint64_t* c, int k, std::uint32_t b,
                                                       std::uint64_t i) {
    std::uint64_t acc = 0;
    const std::uint64_t ip = i % kHashPrime;
    for (int d = k; d-- > 0;) acc = (acc * ip + c[d]) % kHashPrime;
    return static_cast<std::uint32_t>(acc % b);
}
}  // namespace

std::uint64_t launch_count() { return g_launches.load(); }
void count_launch() { g_launches.fetch_add(1); }
std::uint64_t transform_units() { return g_transforms.load(); }
void count_transforms(std::uint64_t local_ffts, int S) { g_transforms.fetch_add(local_ffts / (S > 0 ? S : 1)); }

#define SKC_LAUNCHED() count_launch()

// ============================ K0: hash tables ====================================
// sketch.cpp:24-36 (fill_sym_tables) and hashing.hpp:29-34 (PolyHash::eval)
__global__ void k_sym_tables(const std::uint64_t* __restrict__ hcoef, const std::uint64_t* __restrict__ scoef,
                             int n, std::uint32_t b, int B, std::uint32_t* b1, std::uint32_t* b2, std::uint32_t* b3,
                             std::uint8_t* sexp, std::uint32_t* packed) {
    long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= (long long)B * n) return;
    const int m = static_cast<int>(idx / n);
    const int i = static_cast<int>(idx - (long long)m * n);
    const std::uint32_t h = poly_eval_dev(hcoef + m * 6, 6, b, i);
    const std::uint32_t e = poly_eval_dev(scoef + m * 6, 6, 4u, i);
    b1[idx] = h;
    b2[idx] = static_cast<std::uint32_t>((2ull * h) % b);
    b3[idx] = static_cast<std::uint32_t>((3ull * h) % b);
    sexp[idx] = static_cast<std::uint8_t>(e);
    packed[idx] = h | (e << 30);
}

// sketch.cpp:13-22 (fill_asym_tables): h_s 2-wise into b, xi_s 6-wise Rademacher
__global__ void k_asym_tables(const std::uint64_t* __restrict__ hcoef, const std::uint64_t* __restrict__ xcoef,
                              int n, std::uint32_t b, int B, std::uint32_t* bucket, double* sign,
                              std::uint32_t* packed) {
    long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= (long long)B * 3 * n) return;
    const int ms = static_cast<int>(idx / n);  // m*3 + s
    const int i = static_cast<int>(idx - (long long)ms * n);
    const std::uint32_t h = poly_eval_dev(hcoef + ms * 2, 2, b, i);
    const std::uint32_t e = poly_eval_dev(xcoef + ms * 6, 6, 2u, i);
    bucket[idx] = h;
    sign[idx] = (e & 1u) ? -1.0 : 1.0;
    packed[idx] = h | ((e & 1u) << 31);
}

void launch_sym_tables(cudaStream_t st, const std::uint64_t* hcoef, const std::uint64_t* scoef, int n,
                       std::uint32_t b, int B, std::uint32_t* b1, std::uint32_t* b2, std::uint32_t* b3,
                       std::uint8_t* sexp, std::uint32_t* packed) {
    long long tot = (long long)B * n;
    k_sym_tables<<<cdiv(tot, 256), 256, 0, st>>>(hcoef, scoef, n, b, B, b1, b2, b3, sexp, packed);
    SKC_LAUNCHED();
}
void launch_asym_tables(cudaStream_t st, const std::uint64_t* hcoef, const std::uint64_t* xcoef, int n,
                        std::uint32_t b, int B, std::uint32_t* bucket, double* sign, std::uint32_t* packed) {
    long long tot = (long long)B * 3 * n;
    k_asym_tables<<<cdiv(tot, 256), 256, 0, st>>>(hcoef, xcoef, n, b, B, bucket, sign, packed);
    SKC_LAUNCHED();
}

// Stable rank sort of each replicate's scatter keys: perm[rank] = i ordered by
// (key & mask, i). Colliding nonzeros are then summed in ascending i by the
// segment head, so every scatter is deterministic without atomics.
__global__ void k_sort_perm(const std::uint32_t* __restrict__ keys, int n, std::uint32_t mask,
                            std::uint32_t* __restrict__ perm) {
    extern __shared__ std::uint32_t sk[];
    const std::uint32_t* kk = keys + (long long)blockIdx.x * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) sk[i] = kk[i] & mask;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const std::uint32_t key = sk[i];
        int rank = 0;
        for (int j = 0; j < n; ++j) {
            const std::uint32_t kj = sk[j];
            rank += (kj < key) || (kj == key && j < i);
        }
        perm[(long long)blockIdx.x * n + rank] = static_cast<std::uint32_t>(i);
    }
}
void launch_sort_perm(cudaStream_t st, const std::uint32_t* keys, int nrep, int n, std::uint32_t mask,
                      std::uint32_t* perm) {
    size_t smem = sizeof(std::uint32_t) * n;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_sort_perm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_sort_perm<<<nrep, 256, smem, st>>>(keys, n, mask, perm);
    SKC_LAUNCHED();
}

// ============================ K1: dense build ====================================
// Symmetric: sketch.cpp:315-345 — sorted triples i<=j<=k, weight kappa 1/3/6,
// bucket (h_i+h_j+h_k) mod b, sign root4(e_i+e_j+e_k). Asymmetric: sketch.cpp:173-193.
//
// Exact fixed point: every contribution q = round(kappa*T*2^F) is an int64 and is
// added into shared-memory (lo, hi) 32-bit limbs with two native ATOMS.ADD plus a
// carry taken from the returned old lo value. Integer addition is associative, so
// the build is bit-deterministic under any schedule; F is chosen from the L1 mass
// of the stream so that no bucket can overflow (|sum q| < 2^62).

template <typename TT, bool SYM>
__global__ void __launch_bounds__(256) k_build_prepass(const TT* __restrict__ T, int n,
                                                      const std::uint32_t* __restrict__ rowtab, int nrows,
                                                      double* __restrict__ partials, int* __restrict__ nonfinite) {
    __shared__ double red[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double acc = 0.0;
    bool bad = false;
    for (int row = blockIdx.x * 8 + warp; row < nrows; row += gridDim.x * 8) {
        const std::uint32_t ij = rowtab[row];
        const int i = static_cast<int>(ij >> 16), j = static_cast<int>(ij & 0xFFFFu);
        const TT* rp = T + ((size_t)i * n + j) * n;
        const int k0 = SYM ? j : 0;
        for (int k = k0 + lane; k < n; k += 32) {
            const double v = static_cast<double>(rp[k]);
            double kap = 1.0;
            if (SYM) kap = (i == j && j == k) ? 1.0 : ((i == j || j == k) ? 3.0 : 6.0);
            acc += kap * fabs(v);
            bad |= !isfinite(v);
        }
    }
    if (bad) atomicOr(nonfinite, 1);
    double s = block_sum<256>(acc, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void k_build_scale(const double* __restrict__ partials, int np, int* __restrict__ scale_exp) {
    __shared__ double red[8];
    double acc = 0.0;
    for (int i = threadIdx.x; i < np; i += 256) acc += partials[i];
    double s = block_sum<256>(acc, red);
    if (threadIdx.x == 0) {
        int F = 0;
        if (s > 0.0 && isfinite(s)) {
            int ex;
            frexp(s, &ex);  // s <= 2^ex
            F = 61 - ex;
            F = F > 1000 ? 1000 : (F < -1000 ? -1000 : F);
        }
        *scale_exp = F;
    }
}

__device__ __forceinline__ void add64(std::uint32_t* lo, std::uint32_t* hi, int s, long long q) {
    const std::uint32_t ql = static_cast<std::uint32_t>(q);
    const std::uint32_t qh = static_cast<std::uint32_t>(static_cast<unsigned long long>(q) >> 32);
    const std::uint32_t old = atomicAdd(lo + s, ql);
    const std::uint32_t carry = (old + ql) < old ? 1u : 0u;
    atomicAdd(hi + s, qh + carry);
}

constexpr int kBuildThreads = 1024;
constexpr int kBuildMR = 4;  // replicates handled per row pass

template <typename TT, bool SYM>
__global__ void __launch_bounds__(kBuildThreads, 1)
    k_build_main(const TT* __restrict__ T, int n, const std::uint32_t* __restrict__ packed, std::uint32_t bmask,
                 const std::uint32_t* __restrict__ rowtab, const int* __restrict__ chunk_begin, long long total_slots,
                 int slots_per_cta, int G, const int* __restrict__ scale_exp, long long* __restrict__ partials) {
    extern __shared__ std::uint32_t sacc[];
    std::uint32_t* lo = sacc;
    std::uint32_t* hi = sacc + slots_per_cta;
    const int g = blockIdx.x % G, c = blockIdx.x / G;
    const long long slot_lo = (long long)g * slots_per_cta;
    const long long slot_hi = min(slot_lo + slots_per_cta, total_slots);
    const int nslots = static_cast<int>(slot_hi - slot_lo);
    for (int s = threadIdx.x; s < 2 * slots_per_cta; s += kBuildThreads) sacc[s] = 0u;
    __syncthreads();
    if (nslots > 0) {
        const double scale = ldexp(1.0, *scale_exp);
        const long long SPR = SYM ? 2ll * (bmask + 1) : (long long)(bmask + 1);  // slots per replicate
        const int m_lo = static_cast<int>(slot_lo / SPR), m_hi = static_cast<int>((slot_hi - 1) / SPR);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int row_end = chunk_begin[c + 1];
        for (int row = chunk_begin[c] + warp; row < row_end; row += kBuildThreads / 32) {
            const std::uint32_t ij = rowtab[row];
            const int i = static_cast<int>(ij >> 16), j = static_cast<int>(ij & 0xFFFFu);
            const TT* rp = T + ((size_t)i * n + j) * n;
            const int k0 = SYM ? j : 0;
            for (int mb = m_lo; mb <= m_hi; mb += kBuildMR) {
                std::uint32_t pij[kBuildMR];
                const std::uint32_t* pk[kBuildMR];
#pragma unroll
                for (int r = 0; r < kBuildMR; ++r) {
                    const int m = min(mb + r, m_hi);
                    if (SYM) {
                        const std::uint32_t* pm = packed + (size_t)m * n;
                        pij[r] = __ldg(pm + i) + __ldg(pm + j);
                        pk[r] = pm;
                    } else {
                        const std::uint32_t* pm = packed + (size_t)m * 3 * n;
                        pij[r] = __ldg(pm + i) + __ldg(pm + n + j);
                        pk[r] = pm + 2 * n;
                    }
                }
                for (int k = k0 + lane; k < n; k += 32) {
                    const double v = static_cast<double>(rp[k]);
                    if (v == 0.0) continue;
                    double kap = 1.0;
                    if (SYM) kap = (i == j && j == k) ? 1.0 : ((i == j || j == k) ? 3.0 : 6.0);
                    const long long q = __double2ll_rn(kap * v * scale);
#pragma unroll
                    for (int r = 0; r < kBuildMR; ++r) {
                        const int m = mb + r;
                        if (m > m_hi) break;
                        const std::uint32_t p = pij[r] + __ldg(pk[r] + k);
                        long long slot;
                        if (SYM)
                            slot = (long long)m * SPR + 2ll * (p & bmask) + ((p >> 30) & 1u);
                        else
                            slot = (long long)m * SPR + (p & bmask);
                        const long long ls = slot - slot_lo;
                        if (ls < 0 || ls >= nslots) continue;
                        add64(lo, hi, static_cast<int>(ls), (p >> 31) ? -q : q);
                    }
                }
            }
        }
    }
    __syncthreads();
    long long* out = partials + (long long)c * total_slots + slot_lo;
    for (int s = threadIdx.x; s < nslots; s += kBuildThreads)
        out[s] = static_cast<long long>((static_cast<unsigned long long>(hi[s]) << 32) | lo[s]);
}

// data += (sum over chunks of partials) * 2^-F. For the symmetric set the slot
// index equals the double index into interleaved (re,im) data; asym is real-only.
template <bool SYM>
__global__ void k_build_finalize(const long long* __restrict__ partials, int C, long long total_slots,
                                 const int* __restrict__ scale_exp, double* __restrict__ data) {
    long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (s >= total_slots) return;
    unsigned long long acc = 0;
    for (int c = 0; c < C; ++c) acc += static_cast<unsigned long long>(partials[(long long)c * total_slots + s]);
    const long long q = static_cast<long long>(acc);
    if (q == 0) return;
    const double v = ldexp(static_cast<double>(q), -*scale_exp);
    if (SYM)
        data[s] += v;
    else
        data[2 * s] += v;
}

void launch_build_prepass(cudaStream_t st, const void* T, const BuildPlan& p) {
    cudaMemsetAsync(p.nonfinite, 0, sizeof(int), st);
    if (p.sym) {
        if (p.dtype == 0)
            k_build_prepass<double, true><<<kPrepassBlocks, 256, 0, st>>>((const double*)T, p.n, p.rowtab, p.nrows,
                                                                         p.prepass_partials, p.nonfinite);
        else
            k_build_prepass<float, true><<<kPrepassBlocks, 256, 0, st>>>((const float*)T, p.n, p.rowtab, p.nrows,
                                                                        p.prepass_partials, p.nonfinite);
    } else {
        if (p.dtype == 0)
            k_build_prepass<double, false><<<kPrepassBlocks, 256, 0, st>>>((const double*)T, p.n, p.rowtab, p.nrows,
                                                                          p.prepass_partials, p.nonfinite);
        else
            k_build_prepass<float, false><<<kPrepassBlocks, 256, 0, st>>>((const float*)T, p.n, p.rowtab, p.nrows,
                                                                         p.prepass_partials, p.nonfinite);
    }
    SKC_LAUNCHED();
    k_build_scale<<<1, 256, 0, st>>>(p.prepass_partials, kPrepassBlocks, p.scale_exp);
    SKC_LAUNCHED();
}

template <typename TT, bool SYM>
static void build_main_t(cudaStream_t st, const TT* T, const BuildPlan& p) {
    size_t smem = sizeof(std::uint32_t) * 2 * (size_t)p.slots_per_cta;
    cudaFuncSetAttribute(k_build_main<TT, SYM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_build_main<TT, SYM><<<p.G * p.C, kBuildThreads, smem, st>>>(T, p.n, p.packed, p.bmask, p.rowtab, p.chunk_begin,
                                                                   p.total_slots, p.slots_per_cta, p.G, p.scale_exp,
                                                                   p.partials);
    SKC_LAUNCHED();
}
void launch_build_main(cudaStream_t st, const void* T, const BuildPlan& p) {
    if (p.sym) {
        if (p.dtype == 0)
            build_main_t<double, true>(st, (const double*)T, p);
        else
            build_main_t<float, true>(st, (const float*)T, p);
    } else {
        if (p.dtype == 0)
            build_main_t<double, false>(st, (const double*)T, p);
        else
            build_main_t<float, false>(st, (const float*)T, p);
    }
}
void launch_build_finalize(cudaStream_t st, const BuildPlan& p) {
    if (p.sym)
        k_build_finalize<true><<<cdiv(p.total_slots, 256), 256, 0, st>>>(p.partials, p.C, p.total_slots, p.scale_exp,
                                                                         p.data_as_double);
    else
        k_build_finalize<false><<<cdiv(p.total_slots, 256), 256, 0, st>>>(p.partials, p.C, p.total_slots,
                                                                          p.scale_exp, p.data_as_double);
    SKC_LAUNCHED();
}

// ============================ local FFT drivers ==================================
constexpr int kFftThreads = 256;

// Forward DIF on `na` arrays of length N laid out back to back (stride padded_len(N)).
__device__ __forceinline__ void dif_arrays(double2* sm, int na, int N, const PassPlan& pl, const double2* tw,
                                           int logb) {
    const int stride = padded_len(N);
    for (int p = 0; p < pl.npass; ++p) {
        const int items = N >> pl.logr[p];
        for (int w = threadIdx.x; w < na * items; w += blockDim.x) {
            const int a = w / items;
            dif_pass_dispatch(pl.logr[p], sm + a * stride, w - a * items, pl.h[p], tw, logb);
        }
        __syncthreads();
    }
}
__device__ __forceinline__ void dit_arrays(double2* sm, int na, int N, const PassPlan& pl, const double2* tw,
                                           int logb) {
    const int stride = padded_len(N);
    for (int p = pl.npass - 1; p >= 0; --p) {
        const int items = N >> pl.logr[p];
        for (int w = threadIdx.x; w < na * items; w += blockDim.x) {
            const int a = w / items;
            dit_pass_dispatch(pl.logr[p], sm + a * stride, w - a * items, pl.h[p], tw, logb);
        }
        __syncthreads();
    }
}

// Deterministic sparse scatter of a count sketch into a residue-r local array:
// y[t mod N] += val(i) * w_b^{-r t} for t = bucket(i). perm lists indices sorted
// by (bucket mod N, i); each run of equal keys is summed by its head thread.
template <typename ValFn>
__device__ __forceinline__ void scatter_sorted(double2* y, const std::uint32_t* perm, const std::uint32_t* bucket,
                                               int n, int N, int r, std::uint32_t bmask, const double2* tw,
                                               ValFn val) {
    const std::uint32_t nmask = static_cast<std::uint32_t>(N - 1);
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        const int i = perm[q];
        const std::uint32_t t = bucket[i];
        const std::uint32_t key = t & nmask;
        if (q > 0 && (bucket[perm[q - 1]] & nmask) == key) continue;
        double2 acc = mk(0.0, 0.0);
        for (int q2 = q; q2 < n; ++q2) {
            const int i2 = (q2 == q) ? i : static_cast<int>(perm[q2]);
            const std::uint32_t t2 = (q2 == q) ? t : bucket[i2];
            if ((t2 & nmask) != key) break;
            const double2 x = val(i2);
            acc = cadd(acc, cmul(x, conj(tw[(static_cast<std::uint32_t>(r) * t2) & bmask])));
        }
        y[pad16(static_cast<int>(key))] = acc;
    }
}

__device__ __forceinline__ void zero_smem(double2* sm, int count) {
    for (int x = threadIdx.x; x < count; x += blockDim.x) sm[x] = mk(0.0, 0.0);
}

// ============================ K4: spectra ========================================
// contraction.cpp:62-72 (ensure_fresh): F(data_m) for all m, in local residue layout.
__global__ void __launch_bounds__(kFftThreads) k_spectrum(const double2* __restrict__ data, std::uint32_t b, int logb,
                                                          int N, int logN, int S, const double2* __restrict__ tw,
                                                          double2* __restrict__ spec) {
    extern __shared__ double2 sm[];
    const int r = blockIdx.x % S, m = blockIdx.x / S;
    const double2* dm = data + (size_t)m * b;
    const std::uint32_t bmask = b - 1;
    for (int tp = threadIdx.x; tp < N; tp += blockDim.x) {
        double2 y = mk(0.0, 0.0);
        for (int q = 0; q < S; ++q) {
            const std::uint32_t t = static_cast<std::uint32_t>(tp + q * N);
            y = cadd(y, cmul(dm[t], conj(tw[(static_cast<std::uint32_t>(r) * t) & bmask])));
        }
        sm[pad16(tp)] = y;
    }
    __syncthreads();
    const PassPlan pl = make_plan(N);
    dif_arrays(sm, 1, N, pl, tw, logb);
    double2* out = spec + ((size_t)m * S + r) * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) out[j] = sm[pad16(j)];
}

void launch_spectrum(cudaStream_t st, const double2* data, std::uint32_t b, int logb, int B, int N, int logN, int S,
                     const double2* tw, double2* spec) {
    size_t smem = sizeof(double2) * padded_len(N);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_spectrum, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_spectrum<<<B * S, kFftThreads, smem, st>>>(data, b, logb, N, logN, S, tw, spec);
    SKC_LAUNCHED();
    count_transforms((std::uint64_t)B * S, S);
}

// ============================ K3: symmetric contractions ==========================
// Ivv: contraction.cpp:128-181. vvv: contraction.cpp:83-126.
// One CTA per (restart l, replicate m, residue r).
__global__ void __launch_bounds__(kFftThreads) k_sym_contract(SymView v, const double* __restrict__ U, int L,
                                                              int mode, double* __restrict__ out) {
    extern __shared__ double2 sm[];
    __shared__ double red[kFftThreads / 32];
    const int N = v.N, S = v.S, n = v.n, B = v.B;
    const int r = blockIdx.x % S;
    const int m = (blockIdx.x / S) % B;
    const int l = blockIdx.x / (S * B);
    const int stride = padded_len(N);
    double2* A = sm;
    double2* Bv = sm + stride;
    const double* u = U + (size_t)l * n;
    const std::uint32_t* b1 = v.bucket1 + (size_t)m * n;
    const std::uint32_t* b2 = v.bucket2 + (size_t)m * n;
    const std::uint32_t* b3 = v.bucket3 + (size_t)m * n;
    const std::uint8_t* se = v.sexp + (size_t)m * n;
    const std::uint32_t bmask = v.b - 1;

    zero_smem(sm, 2 * stride);
    __syncthreads();
    // f1[h_i] += sigma_i u_i ; f2[2h_i] += sigma_i^2 u_i^2   (contraction.cpp:150-154)
    scatter_sorted(A, v.perm1 + (size_t)m * n, b1, n, N, r, bmask, v.tw,
                   [&](int i) { return root4_times(se[i], u[i]); });
    scatter_sorted(Bv, v.perm2 + (size_t)m * n, b2, n, N, r, bmask, v.tw, [&](int i) {
        const double ui = u[i];
        return root4_times(2u * se[i], ui * ui);
    });
    __syncthreads();
    const PassPlan pl = make_plan(N);
    dif_arrays(sm, 2, N, pl, v.tw, v.logb);
    const double2* fT = v.spec + ((size_t)m * S + r) * N;

    if (mode == 0) {
        // z1 = fT conj(f1^2 + f2), z2 = fT conj(f1)   (contraction.cpp:158-162)
        for (int j = threadIdx.x; j < N; j += blockDim.x) {
            const double2 t = fT[j];
            const double2 fu = A[pad16(j)];
            const double2 f2 = Bv[pad16(j)];
            A[pad16(j)] = cmulc(t, cadd(cmul(fu, fu), f2));
            Bv[pad16(j)] = cmulc(t, fu);
        }
        __syncthreads();
        dit_arrays(sm, 2, N, pl, v.tw, v.logb);
        const double inv_b = 1.0 / static_cast<double>(v.b);
        const std::uint32_t nmask = static_cast<std::uint32_t>(N - 1);
        double* o = out + (((size_t)l * B + m) * S + r) * n;
        const double2* dm = v.data + (size_t)m * v.b;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const unsigned e = se[i];
            const double ui = u[i];
            const std::uint32_t t1 = b1[i], t2 = b2[i];
            const double2 z1 = cmul(A[pad16(static_cast<int>(t1 & nmask))], v.tw[(static_cast<std::uint32_t>(r) * t1) & bmask]);
            const double2 z2 = cmul(Bv[pad16(static_cast<int>(t2 & nmask))], v.tw[(static_cast<std::uint32_t>(r) * t2) & bmask]);
            double val = re_rot_conj(e, z1) * (1.0 / 6.0) * inv_b;
            val += ui * re_rot_conj(2u * e, z2) * (1.0 / 3.0) * inv_b;
            if (r == 0) val += ui * ui * re_rot_conj(3u * e, dm[b3[i]]) * (1.0 / 3.0);
            o[i] = val;
        }
    } else {
        // acc1 += Re(fT conj(f1)^3), acc2 += Re(fT conj(f1) conj(f2))   (contraction.cpp:111-116)
        double acc1 = 0.0, acc2 = 0.0;
        for (int j = threadIdx.x; j < N; j += blockDim.x) {
            const double2 c1 = conj(A[pad16(j)]);
            const double2 w1 = cmul(fT[j], c1);
            acc1 += cmul(cmul(w1, c1), c1).x;
            acc2 += cmul(w1, conj(Bv[pad16(j)])).x;
        }
        const double s1 = block_sum<kFftThreads>(acc1, red);
        const double s2 = block_sum<kFftThreads>(acc2, red);
        double term3 = 0.0;
        if (r == 0) {  // contraction.cpp:117-121
            const double2* dm = v.data + (size_t)m * v.b;
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const double u3 = u[i] * u[i] * u[i];
                term3 += u3 * re_rot_conj(3u * se[i], dm[b3[i]]);
            }
        }
        const double s3 = block_sum<kFftThreads>(term3, red);
        if (threadIdx.x == 0) {
            double* o = out + (((size_t)l * B + m) * S + r) * 3;
            o[0] = s1;
            o[1] = s2;
            o[2] = s3;
        }
    }
}

void launch_sym_contract(cudaStream_t st, const SymView& v, const double* U, int L, int mode, double* out) {
    size_t smem = sizeof(double2) * 2 * padded_len(v.N);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_sym_contract, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_sym_contract<<<(unsigned)((long long)L * v.B * v.S), kFftThreads, smem, st>>>(v, U, L, mode, out);
    SKC_LAUNCHED();
    count_transforms((std::uint64_t)L * v.B * v.S * (mode == 0 ? 4 : 2), v.S);
}

// ============================ medians ============================================
// tensor.cpp:16-24: even count -> mean of the two middle order statistics.
// Rank selection (ties broken by index) returns the same order statistics.
constexpr int kMaxB = 128;

__device__ __forceinline__ double median_of(const double* est, int B) {
    const int hiR = B / 2, loR = B / 2 - 1;
    double hi = 0.0, lo = 0.0;
    for (int a = 0; a < B; ++a) {
        const double x = est[a];
        int rank = 0;
        for (int c = 0; c < B; ++c) {
            const double y = est[c];
            rank += (y < x) || (y == x && c < a);
        }
        if (rank == hiR) hi = x;
        if (rank == loR) lo = x;
    }
    return (B & 1) ? hi : 0.5 * (lo + hi);
}

// part: L x B x S x n. out (may be null): L x n medians. Unext (may be null):
// normalised medians (decompose.cpp:35-40), flags[l] set when ||.|| <= tol.
__global__ void __launch_bounds__(256) k_median_rows(const double* __restrict__ part, int B, int S, int n,
                                                      double* __restrict__ out, double* __restrict__ Unext,
                                                      double tol, int* __restrict__ flags) {
    extern __shared__ double med[];  // n
    __shared__ double red[8];
    const int l = blockIdx.x;
    double est[kMaxB];
    double ss = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        for (int m = 0; m < B; ++m) {
            const double* p = part + (((size_t)l * B + m) * S) * n + i;
            double s = p[0];
            for (int r = 1; r < S; ++r) s += p[(size_t)r * n];
            est[m] = s;
        }
        const double md = median_of(est, B);
        med[i] = md;
        if (out) out[(size_t)l * n + i] = md;
        ss += md * md;
    }
    if (Unext) {
        const double tot = block_sum<256>(ss, red);
        __shared__ double nrm_s;
        if (threadIdx.x == 0) {
            const double nrm = sqrt(tot);
            nrm_s = nrm;
            if (!(nrm > tol)) flags[l] = 1;
        }
        __syncthreads();
        const double nrm = nrm_s;
        for (int i = threadIdx.x; i < n; i += blockDim.x) Unext[(size_t)l * n + i] = med[i] / nrm;
    }
}

void launch_median_rows(cudaStream_t st, const double* part, int L, int B, int S, int n, double* out, double* Unext,
                        double tol, int* flags) {
    size_t smem = sizeof(double) * n;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_median_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_median_rows<<<L, 256, smem, st>>>(part, B, S, n, out, Unext, tol, flags);
    SKC_LAUNCHED();
}

// vvv: est_m = (acc1/6 + acc2/2)/b + term3/3  (contraction.cpp:122), median over m.
__global__ void k_sym_vvv_finish(const double* __restrict__ part, int L, int B, int S, double bd,
                                 double* __restrict__ values) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= L) return;
    double est[kMaxB];
    for (int m = 0; m < B; ++m) {
        const double* p = part + (((size_t)l * B + m) * S) * 3;
        double a1 = 0.0, a2 = 0.0;
        for (int r = 0; r < S; ++r) {
            a1 += p[r * 3 + 0];
            a2 += p[r * 3 + 1];
        }
        est[m] = (a1 / 6.0 + a2 / 2.0) / bd + p[2] / 3.0;
    }
    values[l] = median_of(est, B);
}
void launch_sym_vvv_finish(cudaStream_t st, const double* part, int L, int B, int S, std::uint32_t b,
                           double* values) {
    k_sym_vvv_finish<<<cdiv(L, 64), 64, 0, st>>>(part, L, B, S, static_cast<double>(b), values);
    SKC_LAUNCHED();
}
// asym vvv: est_m = acc/b (contraction.cpp:242)
__global__ void k_asym_vvv_finish(const double* __restrict__ part, int L, int B, int S, double bd,
                                  double* __restrict__ values) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= L) return;
    double est[kMaxB];
    for (int m = 0; m < B; ++m) {
        const double* p = part + ((size_t)l * B + m) * S;
        double a = 0.0;
        for (int r = 0; r < S; ++r) a += p[r];
        est[m] = a / bd;
    }
    values[l] = median_of(est, B);
}
void launch_asym_vvv_finish(cudaStream_t st, const double* part, int L, int B, int S, std::uint32_t b,
                            double* values) {
    k_asym_vvv_finish<<<cdiv(L, 64), 64, 0, st>>>(part, L, B, S, static_cast<double>(b), values);
    SKC_LAUNCHED();
}

// Selection step (decompose.cpp:107-115): strict '>' over tau ascending, so the
// lowest index wins ties.
__global__ void k_argmax_first(const double* __restrict__ values, int L, int* best, double* best_value) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double bv = -INFINITY;
    int bi = 0;
    for (int t = 0; t < L; ++t) {
        const double x = values[t];
        if (x > bv) {
            bv = x;
            bi = t;
        }
    }
    *best = bi;
    *best_value = bv;
}
void launch_argmax_first(cudaStream_t st, const double* values, int L, int* best, double* best_value) {
    k_argmax_first<<<1, 32, 0, st>>>(values, L, best, best_value);
    SKC_LAUNCHED();
}

// ============================ K2: frequency-domain accumulation ===================
// Symmetric moment / rank-1: acc += w * F(CS(x))^3 (sketch.cpp:353-358; lda.cpp:201-207).
__global__ void __launch_bounds__(kFftThreads) k_sym_moment(SymView v, const double* __restrict__ X,
                                                            const double* __restrict__ w, double wscale,
                                                            long long Nsamp, int chunks, double* __restrict__ acc) {
    extern __shared__ double2 sm[];
    const int N = v.N, S = v.S, n = v.n, B = v.B;
    const int r = blockIdx.x % S;
    const int m = (blockIdx.x / S) % B;
    const int ch = blockIdx.x / (S * B);
    const int stride = padded_len(N);
    double2* A = sm;
    double2* ACC = sm + stride;
    const long long per = (Nsamp + chunks - 1) / chunks;
    const long long s0 = (long long)ch * per, s1 = min(Nsamp, s0 + per);
    const std::uint32_t* b1 = v.bucket1 + (size_t)m * n;
    const std::uint8_t* se = v.sexp + (size_t)m * n;
    const std::uint32_t* perm = v.perm1 + (size_t)m * n;
    const PassPlan pl = make_plan(N);
    zero_smem(ACC, N + 8);
    for (long long s = s0; s < s1; ++s) {
        const double* x = X + (size_t)s * n;
        zero_smem(A, stride);
        __syncthreads();
        scatter_sorted(A, perm, b1, n, N, r, v.b - 1, v.tw, [&](int i) { return root4_times(se[i], x[i]); });
        __syncthreads();
        dif_arrays(A, 1, N, pl, v.tw, v.logb);
        const double ws = (w ? w[s] : 1.0) * wscale;
        for (int j = threadIdx.x; j < N; j += blockDim.x) {
            const double2 z = A[pad16(j)];
            const double2 z3 = cmul(cmul(z, z), z);
            ACC[j] = cadd(ACC[j], cscale(z3, ws));
        }
        __syncthreads();
    }
    double2* o = reinterpret_cast<double2*>(acc) + (((size_t)ch * B + m) * S + r) * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) o[j] = ACC[j];
}
void launch_sym_moment_accumulate(cudaStream_t st, const SymView& v, const double* X, const double* w, double wscale,
                                  long long Nsamp, int chunks, double* acc) {
    size_t smem = sizeof(double2) * (padded_len(v.N) + v.N + 8);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_sym_moment, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_sym_moment<<<(unsigned)((long long)chunks * v.B * v.S), kFftThreads, smem, st>>>(v, X, w, wscale, Nsamp, chunks,
                                                                                       acc);
    SKC_LAUNCHED();
    count_transforms((std::uint64_t)Nsamp * v.B * v.S, v.S);
}

// Sum the chunk partials (fixed order), inverse DIT -> tmp[m][r][t'] natural order.
__global__ void __launch_bounds__(kFftThreads) k_freq_reduce_inverse(const double2* __restrict__ acc, int chunks, int B,
                                                                     int S, int N, int logb,
                                                                     const double2* __restrict__ tw,
                                                                     double2* __restrict__ tmp) {
    extern __shared__ double2 sm[];
    const int r = blockIdx.x % S, m = blockIdx.x / S;
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
        double2 s = mk(0.0, 0.0);
        for (int c = 0; c < chunks; ++c) s = cadd(s, acc[(((size_t)c * B + m) * S + r) * N + j]);
        sm[pad16(j)] = s;
    }
    __syncthreads();
    const PassPlan pl = make_plan(N);
    dit_arrays(sm, 1, N, pl, tw, logb);
    double2* o = tmp + ((size_t)m * S + r) * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) o[j] = sm[pad16(j)];
}
void launch_freq_reduce_inverse(cudaStream_t st, const double* acc, int chunks, int B, int S, int N, int logN,
                                std::uint32_t b, int logb, const double2* tw, double2* tmp) {
    (void)logN;
    (void)b;
    size_t smem = sizeof(double2) * padded_len(N);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_freq_reduce_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_freq_reduce_inverse<<<B * S, kFftThreads, smem, st>>>(reinterpret_cast<const double2*>(acc), chunks, B, S, N,
                                                            logb, tw, tmp);
    SKC_LAUNCHED();
    count_transforms((std::uint64_t)B * S, S);
}

// dst[m][t] (+)= alpha * (1/b) * sum_r w_b^{r t} tmp[m][r][t mod N]
// (inverse_inplace scaling, fft.cpp:62-66; data += alpha*su, sketch.cpp:359).
__global__ void k_combine_residues(const double2* __restrict__ tmp, int B, int S, int N, std::uint32_t b,
                                   const double2* __restrict__ tw, double alpha, int m_only, int overwrite,
                                   double2* __restrict__ dst) {
    long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int Bm = (m_only >= 0) ? 1 : B;
    if (idx >= (long long)Bm * b) return;
    const int mm = static_cast<int>(idx / b);
    const std::uint32_t t = static_cast<std::uint32_t>(idx - (long long)mm * b);
    const int m = (m_only >= 0) ? m_only : mm;
    const std::uint32_t nmask = static_cast<std::uint32_t>(N - 1), bmask = b - 1;
    double2 s = mk(0.0, 0.0);
    const double2* tm = tmp + (size_t)m * S * N;
    for (int r = 0; r < S; ++r)
        s = cadd(s, cmul(tm[(size_t)r * N + (t & nmask)], tw[(static_cast<std::uint32_t>(r) * t) & bmask]));
    const double inv_b = 1.0 / static_cast<double>(b);
    const double2 su = cscale(s, inv_b);
    double2* d = dst + idx;
    if (overwrite)
        *d = cscale(su, alpha);
    else
        *d = cadd(*d, cscale(su, alpha));
}
void launch_combine_residues(cudaStream_t st, const double2* tmp, int B, int S, int N, std::uint32_t b,
                             const double2* tw, double alpha, int m_only, bool overwrite, double2* dst) {
    long long tot = (long long)((m_only >= 0) ? 1 : B) * b;
    k_combine_residues<<<cdiv(tot, 256), 256, 0, st>>>(tmp, B, S, N, b, tw, alpha, m_only, overwrite ? 1 : 0, dst);
    SKC_LAUNCHED();
}

// Asymmetric factored accumulation (sketch.cpp:224-248, Eq. 2):
// acc += a_c F(s1 u_c) F(s2 v_c) F(s3 w_c). m_only >= 0 restricts to one replicate.
__global__ void __launch_bounds__(kFftThreads) k_asym_factored(AsymView v, const double* __restrict__ a,
                                                               const double* __restrict__ U,
                                                               const double* __restrict__ V,
                                                               const double* __restrict__ W, long long Ncomp,
                                                               int chunks, int m_only, double* __restrict__ acc) {
    extern __shared__ double2 sm[];
    const int N = v.N, S = v.S, n = v.n;
    const int Bm = (m_only >= 0) ? 1 : v.B;
    const int r = blockIdx.x % S;
    const int mm = (blockIdx.x / S) % Bm;
    const int m = (m_only >= 0) ? m_only : mm;
    const int ch = blockIdx.x / (S * Bm);
    const int stride = padded_len(N);
    double2* ACC = sm + 3 * stride;
    const long long per = (Ncomp + chunks - 1) / chunks;
    const long long c0 = (long long)ch * per, c1 = min(Ncomp, c0 + per);
    const PassPlan pl = make_plan(N);
    zero_smem(ACC, N + 8);
    for (long long c = c0; c < c1; ++c) {
        zero_smem(sm, 3 * stride);
        __syncthreads();
        const double* vecs[3] = {U + (size_t)c * n, V + (size_t)c * n, W + (size_t)c * n};
#pragma unroll
        for (int sl = 0; sl < 3; ++sl) {
            const std::uint32_t* bk = v.bucket + ((size_t)m * 3 + sl) * n;
            const double* sg = v.sign + ((size_t)m * 3 + sl) * n;
            const double* x = vecs[sl];
            scatter_sorted(sm + sl * stride, v.perm + ((size_t)m * 3 + sl) * n, bk, n, N, r, v.b - 1, v.tw,
                           [&](int i) { return mk(sg[i] * x[i], 0.0); });
        }
        __syncthreads();
        dif_arrays(sm, 3, N, pl, v.tw, v.logb);
        const double ac = a ? a[c] : 1.0;
        for (int j = threadIdx.x; j < N; j += blockDim.x) {
            const double2 pr = cmul(sm[pad16(j)], cmul(sm[stride + pad16(j)], sm[2 * stride + pad16(j)]));
            ACC[j] = cadd(ACC[j], cscale(pr, ac));
        }
        __syncthreads();
    }
    double2* o = reinterpret_cast<double2*>(acc) + (((size_t)ch * Bm + mm) * S + r) * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) o[j] = ACC[j];
}
void launch_asym_factored_accumulate(cudaStream_t st, const AsymView& v, const double* a, const double* U,
                                     const double* V, const double* W, long long Ncomp, int chunks, int m_only,
                                     double* acc) {
    size_t smem = sizeof(double2) * (3 * padded_len(v.N) + v.N + 8);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_asym_factored, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int Bm = (m_only >= 0) ? 1 : v.B;
    k_asym_factored<<<(unsigned)((long long)chunks * Bm * v.S), kFftThreads, smem, st>>>(v, a, U, V, W, Ncomp, chunks,
                                                                                         m_only, acc);
    SKC_LAUNCHED();
    count_transforms((std::uint64_t)Ncomp * Bm * v.S * 3, v.S);
}

// ============================ K3a: asymmetric contractions ========================
// mode_contraction: contraction.cpp:248-295 (slots at :256-257).
__global__ void __launch_bounds__(kFftThreads) k_asym_mode(AsymView v, int free_mode, const double* __restrict__ X,
                                                           const double* __restrict__ Y, int L,
                                                           double* __restrict__ out) {
    extern __shared__ double2 sm[];
    const int N = v.N, S = v.S, n = v.n, B = v.B;
    const int r = blockIdx.x % S;
    const int m = (blockIdx.x / S) % B;
    const int l = blockIdx.x / (S * B);
    const int stride = padded_len(N);
    const int slot_x = free_mode == 0 ? 1 : 0;
    const int slot_y = free_mode == 2 ? 1 : 2;
    const double* x = X + (size_t)l * n;
    const double* y = Y + (size_t)l * n;
    const std::uint32_t bmask = v.b - 1;
    zero_smem(sm, 2 * stride);
    __syncthreads();
    {
        const std::uint32_t* bk = v.bucket + ((size_t)m * 3 + slot_x) * n;
        const double* sg = v.sign + ((size_t)m * 3 + slot_x) * n;
        scatter_sorted(sm, v.perm + ((size_t)m * 3 + slot_x) * n, bk, n, N, r, bmask, v.tw,
                       [&](int i) { return mk(sg[i] * x[i], 0.0); });
    }
    {
        const std::uint32_t* bk = v.bucket + ((size_t)m * 3 + slot_y) * n;
        const double* sg = v.sign + ((size_t)m * 3 + slot_y) * n;
        scatter_sorted(sm + stride, v.perm + ((size_t)m * 3 + slot_y) * n, bk, n, N, r, bmask, v.tw,
                       [&](int i) { return mk(sg[i] * y[i], 0.0); });
    }
    __syncthreads();
    const PassPlan pl = make_plan(N);
    dif_arrays(sm, 2, N, pl, v.tw, v.logb);
    const double2* fT = v.spec + ((size_t)m * S + r) * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x)
        sm[pad16(j)] = cmulc(fT[j], cmul(sm[pad16(j)], sm[stride + pad16(j)]));
    __syncthreads();
    dit_arrays(sm, 1, N, pl, v.tw, v.logb);
    const double inv_b = 1.0 / static_cast<double>(v.b);
    const std::uint32_t nmask = static_cast<std::uint32_t>(N - 1);
    const std::uint32_t* bf = v.bucket + ((size_t)m * 3 + free_mode) * n;
    const double* sf = v.sign + ((size_t)m * 3 + free_mode) * n;
    double* o = out + (((size_t)l * B + m) * S + r) * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const std::uint32_t t = bf[i];
        const double2 z = cmul(sm[pad16(static_cast<int>(t & nmask))], v.tw[(static_cast<std::uint32_t>(r) * t) & bmask]);
        o[i] = sf[i] * z.x * inv_b;
    }
}
void launch_asym_mode(cudaStream_t st, const AsymView& v, int free_mode, const double* X, const double* Y, int L,
                      double* part) {
    size_t smem = sizeof(double2) * 2 * padded_len(v.N);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_asym_mode, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_asym_mode<<<(unsigned)((long long)L * v.B * v.S), kFftThreads, smem, st>>>(v, free_mode, X, Y, L, part);
    SKC_LAUNCHED();
    count_transforms((std::uint64_t)L * v.B * v.S * 3, v.S);
}

// vvv: contraction.cpp:209-246. Partial sums of Re(fT conj(fx fy fz)) per residue.
__global__ void __launch_bounds__(kFftThreads) k_asym_vvv(AsymView v, const double* __restrict__ U, int L,
                                                          double* __restrict__ out) {
    extern __shared__ double2 sm[];
    __shared__ double red[kFftThreads / 32];
    const int N = v.N, S = v.S, n = v.n, B = v.B;
    const int r = blockIdx.x % S;
    const int m = (blockIdx.x / S) % B;
    const int l = blockIdx.x / (S * B);
    const int stride = padded_len(N);
    const double* u = U + (size_t)l * n;
    const std::uint32_t bmask = v.b - 1;
    zero_smem(sm, 3 * stride);
    __syncthreads();
#pragma unroll
    for (int sl = 0; sl < 3; ++sl) {
        const std::uint32_t* bk = v.bucket + ((size_t)m * 3 + sl) * n;
        const double* sg = v.sign + ((size_t)m * 3 + sl) * n;
        scatter_sorted(sm + sl * stride, v.perm + ((size_t)m * 3 + sl) * n, bk, n, N, r, bmask, v.tw,
                       [&](int i) { return mk(sg[i] * u[i], 0.0); });
    }
    __syncthreads();
    const PassPlan pl = make_plan(N);
    dif_arrays(sm, 3, N, pl, v.tw, v.logb);
    const double2* fT = v.spec + ((size_t)m * S + r) * N;
    double acc = 0.0;
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
        const double2 p = cmul(cmul(sm[pad16(j)], sm[stride + pad16(j)]), sm[2 * stride + pad16(j)]);
        acc += cmulc(fT[j], p).x;
    }
    const double s = block_sum<kFftThreads>(acc, red);
    if (threadIdx.x == 0) out[((size_t)l * B + m) * S + r] = s;
}
void launch_asym_vvv(cudaStream_t st, const AsymView& v, const double* U, int L, double* part) {
    size_t smem = sizeof(double2) * 3 * padded_len(v.N);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_asym_vvv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_asym_vvv<<<(unsigned)((long long)L * v.B * v.S), kFftThreads, smem, st>>>(v, U, L, part);
    SKC_LAUNCHED();
    count_transforms((std::uint64_t)L * v.B * v.S * 3, v.S);
}

// ============================ synthetic inputs ====================================
// Planted symmetric tensor on the device: sum_r lambda_r V[a,r]V[b,r]V[c,r] over the
// sorted index triple (bitwise symmetric) plus sigma * N(0,1) noise from a
// counter-based generator keyed by the sorted triple.
__device__ __forceinline__ std::uint64_t mix64(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
template <typename TT>
__global__ void k_gen_planted(int n, int rank, const double* __restrict__ lambda, const double* __restrict__ V,
                              double sigma, std::uint64_t seed, TT* __restrict__ out) {
    long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long tot = (long long)n * n * n;
    if (idx >= tot) return;
    int i = static_cast<int>(idx / ((long long)n * n));
    int j = static_cast<int>((idx / n) % n);
    int k = static_cast<int>(idx % n);
    int a = min(i, min(j, k)), c = max(i, max(j, k)), b = i + j + k - a - c;
    double s = 0.0;
    for (int r = 0; r < rank; ++r) s += lambda[r] * V[(size_t)r * n + a] * V[(size_t)r * n + b] * V[(size_t)r * n + c];
    if (sigma > 0.0) {
        const std::uint64_t key = (((std::uint64_t)a * n + b) * n + c);
        const std::uint64_t h1 = mix64(seed ^ (key * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull));
        const std::uint64_t h2 = mix64(h1 + 0x9E3779B97F4A7C15ull);
        const double u1 = (static_cast<double>(h1 >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = static_cast<double>(h2 >> 11) * 0x1.0p-53;
        s += sigma * sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    }
    out[idx] = static_cast<TT>(s);
}
void launch_gen_planted(cudaStream_t st, int n, int rank, const double* lambda, const double* V, double sigma,
                        std::uint64_t seed, int dtype, void* out) {
    long long tot = (long long)n * n * n;
    if (dtype == 0)
        k_gen_planted<double><<<cdiv(tot, 256), 256, 0, st>>>(n, rank, lambda, V, sigma, seed, (double*)out);
    else
        k_gen_planted<float><<<cdiv(tot, 256), 256, 0, st>>>(n, rank, lambda, V, sigma, seed, (float*)out);
    SKC_LAUNCHED();
}

}  // namespace skc
