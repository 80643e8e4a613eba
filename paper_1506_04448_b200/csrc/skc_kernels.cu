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
#include <cstdlib>
#include <string>

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
// replays of captured CUDA graphs count their kernels and transforms again
void count_replay(std::uint64_t launches, std::uint64_t transforms) {
    g_launches.fetch_add(launches);
    g_transforms.fetch_add(transforms);
}

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

// ============================ local FFT drivers ==================================
constexpr int kFftThreads = 256;
#ifndef SKC_FFT_MINB
#define SKC_FFT_MINB 2  // 128 registers: radix-16 passes stay in registers (minB 3 spills)
#endif

#define SKC_LOGN_SWITCH(logN, X)    \
    switch (logN) {                 \
        case 1: X(1); break;        \
        case 2: X(2); break;        \
        case 3: X(3); break;        \
        case 4: X(4); break;        \
        case 5: X(5); break;        \
        case 6: X(6); break;        \
        case 7: X(7); break;        \
        case 8: X(8); break;        \
        case 9: X(9); break;        \
        case 10: X(10); break;      \
        case 11: X(11); break;      \
        case 12: X(12); break;      \
        default: break;             \
    }

__device__ __forceinline__ void zero_smem(double2* sm, int count) {
    for (int x = threadIdx.x; x < count; x += blockDim.x) sm[x] = mk(0.0, 0.0);
}

// Deterministic sparse scatter of a count sketch into the residue-r local array:
// y[t mod N] = sum over the run of equal keys of val(i) * w_b^{-r t}. `plan` holds
// (i, t | tag) ordered by (t mod N, i); the head of each run sums it in ascending i,
// so no atomics are needed and the result does not depend on scheduling.
template <typename ValFn>
__device__ __forceinline__ void scatter_plan(double2* y, const uint2* __restrict__ plan, int n, int N, int r,
                                             std::uint32_t bmask, std::uint32_t tmask, const double2* __restrict__ tw,
                                             ValFn val) {
    const std::uint32_t nmask = static_cast<std::uint32_t>(N - 1);
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        uint2 e = plan[q];
        const std::uint32_t key = e.y & nmask;
        if (q > 0 && (plan[q - 1].y & nmask) == key) continue;
        double2 acc = mk(0.0, 0.0);
        for (int q2 = q;;) {
            const std::uint32_t t = e.y & tmask;
            acc = cadd(acc, cmul(val(e.x, e.y), conj(tw[(static_cast<std::uint32_t>(r) * t) & bmask])));
            if (++q2 >= n) break;
            e = plan[q2];
            if ((e.y & nmask) != key) break;
        }
        y[pad16(static_cast<int>(key))] = acc;
    }
}

// Two-phase deterministic scatter of up to two count sketches at once (latency-tolerant):
// phase 1 computes every contribution val(i) w_b^{-r t} independently into shared
// scratch (all loads in flight), phase 2 lets each run head sum its run in plan order.
// scratch: 2*n double2 + 2*n keys; n <= kScatterMax.
constexpr int kScatterMax = 1024;
// stwA/stwB (optional): the plan-order residue twiddles conj(w_b^{r t}) of this (m, r)
// (SymView::stw*), read coalesced instead of from the b-entry table.
template <typename ValA, typename ValB>
__device__ __forceinline__ void scatter2(double2* yA, const uint2* __restrict__ planA, ValA valA, double2* yB,
                                         const uint2* __restrict__ planB, ValB valB, int n, int N, int r,
                                         std::uint32_t bmask, std::uint32_t tmask, const double2* __restrict__ tw,
                                         double2* scr, std::uint32_t* keys, const double2* __restrict__ stwA = nullptr,
                                         const double2* __restrict__ stwB = nullptr) {
    const std::uint32_t nmask = static_cast<std::uint32_t>(N - 1);
    const int tot = yB ? 2 * n : n;
    for (int x = threadIdx.x; x < tot; x += blockDim.x) {
        const bool b = x >= n;
        const uint2 e = b ? planB[x - n] : planA[x];
        const double2 v = b ? valB(e.x, e.y) : valA(e.x, e.y);
        const std::uint32_t t = e.y & tmask;
        const double2* st = b ? stwB : stwA;
        const double2 w = st ? st[b ? x - n : x] : conj(tw[(static_cast<std::uint32_t>(r) * t) & bmask]);
        scr[x] = cmul(v, w);
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

// Scratch-free variant: every thread computes its own contribution with independent
// loads; a run head writes it (plus, rarely, its run's followers recomputed in plan
// order), non-heads write nothing. Deterministic, no extra shared memory or barrier.
template <typename ValA, typename ValB>
__device__ __forceinline__ void scatter2_direct(double2* yA, const uint2* __restrict__ planA, ValA valA, double2* yB,
                                                const uint2* __restrict__ planB, ValB valB, int n, int N, int r,
                                                std::uint32_t bmask, std::uint32_t tmask, const double2* __restrict__ tw) {
    const std::uint32_t nmask = static_cast<std::uint32_t>(N - 1);
    const int tot = yB ? 2 * n : n;
    for (int x = threadIdx.x; x < tot; x += blockDim.x) {
        const bool b = x >= n;
        const int q = b ? x - n : x;
        const uint2* plan = b ? planB : planA;
        const uint2 e = plan[q];
        const std::uint32_t key = e.y & nmask;
        const bool head = (q == 0) || ((plan[q - 1].y & nmask) != key);
        double2 acc = cmul(b ? valB(e.x, e.y) : valA(e.x, e.y), conj(tw[(static_cast<std::uint32_t>(r) * (e.y & tmask)) & bmask]));
        if (!head) continue;
        for (int q2 = q + 1; q2 < n; ++q2) {
            const uint2 f = plan[q2];
            if ((f.y & nmask) != key) break;
            acc = cadd(acc, cmul(b ? valB(f.x, f.y) : valA(f.x, f.y), conj(tw[(static_cast<std::uint32_t>(r) * (f.y & tmask)) & bmask])));
        }
        (b ? yB : yA)[pad16(static_cast<int>(key))] = acc;
    }
}

// plan[m][q] = (i, t_i | tag_i << tag_shift) for i = perm[m][q]
__global__ void k_make_plan(const std::uint32_t* __restrict__ perm, const std::uint32_t* __restrict__ bucket,
                            const std::uint8_t* __restrict__ sexp, int sexp_mult, const std::uint32_t* __restrict__ packed,
                            int n, long long total, uint2* __restrict__ plan) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= total) return;
    const long long rep = idx / n;
    const std::uint32_t i = perm[idx];
    const long long src = rep * n + i;
    std::uint32_t y = bucket[src];
    if (sexp) y |= ((static_cast<std::uint32_t>(sexp[src]) * sexp_mult) & 3u) << 28;
    if (packed) y |= packed[src] & 0x80000000u;
    plan[idx] = make_uint2(i, y);
}
void launch_make_plan(cudaStream_t st, const std::uint32_t* perm, const std::uint32_t* bucket, const std::uint8_t* sexp,
                      int sexp_mult, const std::uint32_t* packed, int nrep, int n, uint2* plan) {
    const long long tot = (long long)nrep * n;
    k_make_plan<<<cdiv(tot, 256), 256, 0, st>>>(perm, bucket, sexp, sexp_mult, packed, n, tot, plan);
    SKC_LAUNCHED();
}

// Residue twiddles of the symmetric contraction scatter/gather, per (m, r, q).
__global__ void k_sym_twiddle_tables(SymView v, double2* __restrict__ stw1, double2* __restrict__ stw2,
                                     double2* __restrict__ gtw1, double2* __restrict__ gtw2) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long tot = (long long)v.B * v.S * v.n;
    if (idx >= tot) return;
    const int q = static_cast<int>(idx % v.n);
    const int r = static_cast<int>((idx / v.n) % v.S);
    const int m = static_cast<int>(idx / ((long long)v.n * v.S));
    const std::uint32_t bmask = v.b - 1, ur = static_cast<std::uint32_t>(r);
    const size_t mq = (size_t)m * v.n + q;
    stw1[idx] = conj(v.tw[(ur * (v.plan1[mq].y & 0x0FFFFFFFu)) & bmask]);
    stw2[idx] = conj(v.tw[(ur * (v.plan2[mq].y & 0x0FFFFFFFu)) & bmask]);
    // gather weights with the sign rotation and the 1/(6b), 1/(3b) scalings folded in
    // (contraction.cpp:170-175): Re(z1 conj(sigma)) / (6b) = Re(A[h] * gtw1) etc.
    const unsigned e = v.sexp[mq];
    const double inv_b = 1.0 / static_cast<double>(v.b);
    const double2 r1 = root4_times((4u - (e & 3u)) & 3u, inv_b / 6.0);
    const double2 r2 = root4_times((4u - ((2u * e) & 3u)) & 3u, inv_b / 3.0);
    gtw1[idx] = cmul(v.tw[(ur * v.bucket1[mq]) & bmask], r1);
    gtw2[idx] = cmul(v.tw[(ur * v.bucket2[mq]) & bmask], r2);
}
void launch_sym_twiddle_tables(cudaStream_t st, const SymView& v, double2* stw1, double2* stw2, double2* gtw1,
                               double2* gtw2) {
    const long long tot = (long long)v.B * v.S * v.n;
    k_sym_twiddle_tables<<<cdiv(tot, 256), 256, 0, st>>>(v, stw1, stw2, gtw1, gtw2);
    SKC_LAUNCHED();
}

// ============================ K4: spectra ========================================
// contraction.cpp:62-72 (ensure_fresh): F(data_m) for all m, in local residue layout.
template <int LOGN>
__global__ void __launch_bounds__(kFftThreads, SKC_FFT_MINB)
    k_spectrum(const double2* __restrict__ data, std::uint32_t b, int S, const double2* __restrict__ tw,
               const double2* __restrict__ twl, double2* __restrict__ spec) {
    extern __shared__ double2 sm[];
    constexpr int N = 1 << LOGN;
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
    dif_local<LOGN>(sm, 1, twl);
    double2* out = spec + ((size_t)m * S + r) * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) out[j] = sm[pad16(j)];
}

void launch_spectrum(cudaStream_t st, const double2* data, std::uint32_t b, int logb, int B, int N, int logN, int S,
                     const double2* tw, const double2* twl, double2* spec) {
    (void)logb;
    const size_t smem = sizeof(double2) * padded_len(N);
#define L_(LG)                                                                                               \
    {                                                                                                        \
        if (smem > 48 * 1024)                                                                                \
            cudaFuncSetAttribute(k_spectrum<LG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
        k_spectrum<LG><<<B * S, kFftThreads, smem, st>>>(data, b, S, tw, twl, spec);                          \
    }
    SKC_LOGN_SWITCH(logN, L_)
#undef L_
    SKC_LAUNCHED();
    count_transforms((std::uint64_t)B * S, S);
}

// ============================ K3: symmetric contractions ==========================
// Ivv: contraction.cpp:128-181. vvv: contraction.cpp:83-126.
// One CTA per (restart block, replicate m, residue r): kLPB restarts per CTA share the
// spectrum slice F_r(T_m) (L1-resident across restarts) and amortise CTA start-up.
constexpr int kLPB = 4;
template <int LOGN, int VAR, int LR, int MINB>
__global__ void __launch_bounds__(kFftThreads, MINB)
    k_sym_contract(SymView v, const double* __restrict__ U, int L, int mode, double* __restrict__ out) {
    constexpr bool SCR = VAR == 1;
    extern __shared__ double2 sm[];
    __shared__ double red[kFftThreads / 32];
    constexpr int N = 1 << LOGN;
    constexpr int stride = N + (N >> 4) + 1;
    const int S = v.S, n = v.n, B = v.B;
    const int r = blockIdx.x % S;
    const int m = (blockIdx.x / S) % B;
    const int l0 = (blockIdx.x / (S * B)) * kLPB;
    double2* A = sm;
    double2* Bv = sm + stride;
    double2* scr = sm + 2 * stride;  // 2n (SCR only)
    std::uint32_t* keys = reinterpret_cast<std::uint32_t*>(scr + (SCR ? 2 * n : 0));
    const std::uint32_t bmask = v.b - 1;
    const double2* fT = v.spec + ((size_t)m * S + r) * N;  // re-read per restart (L1/L2 resident)
    const uint2* p1 = v.plan1 + (size_t)m * n;
    const uint2* p2 = v.plan2 + (size_t)m * n;
    const std::uint32_t* b1 = v.bucket1 + (size_t)m * n;
    const std::uint32_t* b2 = v.bucket2 + (size_t)m * n;
    const std::uint32_t* b3 = v.bucket3 + (size_t)m * n;
    const std::uint8_t* se = v.sexp + (size_t)m * n;
    const double2* dm = v.data + (size_t)m * v.b;

    for (int l = l0; l < min(L, l0 + kLPB); ++l) {
        const double* u = U + (size_t)l * n;
        zero_smem(sm, 2 * stride);
        __syncthreads();
        // f1[h_i] += sigma_i u_i ; f2[2h_i] += sigma_i^2 u_i^2   (contraction.cpp:150-154)
        auto v1 = [&](std::uint32_t i, std::uint32_t y) { return root4_times(y >> 28, u[i]); };
        auto v2 = [&](std::uint32_t i, std::uint32_t y) {
            const double ui = u[i];
            return root4_times(y >> 28, ui * ui);
        };
        if (VAR == 1) {
            scatter2(A, p1, v1, Bv, p2, v2, n, N, r, bmask, 0x0FFFFFFFu, v.tw, scr, keys);
        } else if (VAR == 2) {
            scatter2_direct(A, p1, v1, Bv, p2, v2, n, N, r, bmask, 0x0FFFFFFFu, v.tw);
        } else {
            scatter_plan(A, p1, n, N, r, bmask, 0x0FFFFFFFu, v.tw, v1);
            scatter_plan(Bv, p2, n, N, r, bmask, 0x0FFFFFFFu, v.tw, v2);
        }
        __syncthreads();
        dif_local<LOGN, LR>(sm, 2, v.twl);

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
            dit_local<LOGN, LR>(sm, 2, v.twl);
            const double inv_b = 1.0 / static_cast<double>(v.b);
            const std::uint32_t nmask = static_cast<std::uint32_t>(N - 1);
            double* o = out + (((size_t)l * B + m) * S + r) * n;
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
        __syncthreads();
    }
}

// ---- half-length f2 / z2 variant ---------------------------------------------------------
// f2 lives on even buckets 2h_i, so y_r (the residue-r local array of f2) is supported on
// even t' and its N-point DFT is periodic with period N/2: only the N/2-point DFT of the
// even subsequence is computed (Bh). In the bit-reversed local layout, full position p
// pairs with half position p >> 1. Likewise z2 is only gathered at even local positions,
// so Z2 is folded (Z[2p''] + Z[2p''+1] holds frequencies k and k + N/2) and inverted with
// an N/2-point DIT. Net: 3 of the 4 length-N transforms per restart instead of 4.
template <int LOGN, int LR, int P, int NPA = plan_npass(LOGN, LR), int NPB = plan_npass(LOGN - 1, LR)>
struct DifPair {
    __device__ __forceinline__ static void run(double2* A, double2* Bh, const double2* twl) {
        constexpr int PB = P - (NPA - NPB);
        constexpr int RA = plan_logr(LOGN, P, LR), HA = plan_h(LOGN, P, LR), IA = (1 << LOGN) >> RA;
        constexpr int RB = PB >= 0 ? plan_logr(LOGN - 1, PB, LR) : 1;
        constexpr int HB = PB >= 0 ? plan_h(LOGN - 1, PB, LR) : 1;
        constexpr int IB = PB >= 0 ? (1 << (LOGN - 1)) >> RB : 0;
        for (int w = threadIdx.x; w < IA + IB; w += blockDim.x) {
            if (w < IA)
                dif_pass_item<RA, 2 * HA == (1 << RA)>(A, w, HA, twl, LOGN);
            else
                dif_pass_item<RB, 2 * HB == (1 << RB)>(Bh, w - IA, HB, twl, LOGN);
        }
        __syncthreads();
        DifPair<LOGN, LR, P + 1, NPA, NPB>::run(A, Bh, twl);
    }
};
template <int LOGN, int LR, int NPA, int NPB>
struct DifPair<LOGN, LR, NPA, NPA, NPB> {
    __device__ __forceinline__ static void run(double2*, double2*, const double2*) {}
};
template <int LOGN, int LR, int P, int NPA = plan_npass(LOGN, LR), int NPB = plan_npass(LOGN - 1, LR)>
struct DitPair {
    __device__ __forceinline__ static void run(double2* A, double2* Bh, const double2* twl) {
        constexpr int PB = P - (NPA - NPB);
        constexpr int RA = plan_logr(LOGN, P, LR), HA = plan_h(LOGN, P, LR), IA = (1 << LOGN) >> RA;
        constexpr int RB = PB >= 0 ? plan_logr(LOGN - 1, PB, LR) : 1;
        constexpr int HB = PB >= 0 ? plan_h(LOGN - 1, PB, LR) : 1;
        constexpr int IB = PB >= 0 ? (1 << (LOGN - 1)) >> RB : 0;
        for (int w = threadIdx.x; w < IA + IB; w += blockDim.x) {
            if (w < IA)
                dit_pass_item<RA, 2 * HA == (1 << RA)>(A, w, HA, twl, LOGN);
            else
                dit_pass_item<RB, 2 * HB == (1 << RB)>(Bh, w - IA, HB, twl, LOGN);
        }
        __syncthreads();
        DitPair<LOGN, LR, P - 1, NPA, NPB>::run(A, Bh, twl);
    }
};
template <int LOGN, int LR, int NPA, int NPB>
struct DitPair<LOGN, LR, -1, NPA, NPB> {
    __device__ __forceinline__ static void run(double2*, double2*, const double2*) {}
};

#ifdef SKC_TRACE_CONTRACT
__device__ unsigned long long g_contract_phase[8];
#endif
template <int LOGN, int NT>
__device__ __forceinline__ void sym_contract_half_body(const SymView& v, const double* __restrict__ U, int L, int mode,
                                                       double* __restrict__ out) {
    extern __shared__ double2 sm[];
    __shared__ double red[NT / 32];
    constexpr int N = 1 << LOGN, NH = N / 2;
    constexpr int strideA = N + (N >> 4) + 1;
    constexpr int strideB = NH + (NH >> 4) + 1;
#ifndef SKC_CB_SC  // loads in flight per thread in the scatter / pointwise / gather phases
#define SKC_CB_SC 4
#endif
#ifndef SKC_CB_PW
#define SKC_CB_PW 3
#endif
#ifndef SKC_CB_GA
#define SKC_CB_GA 3
#endif
    constexpr int SB = SKC_CB_SC, PB = SKC_CB_PW, GB = SKC_CB_GA;
    const int S = v.S, n = v.n, B = v.B;
    const int r = blockIdx.x % S;
    const int m = (blockIdx.x / S) % B;
    const int lpb = v.lpb;
    const int l0 = (blockIdx.x / (S * B)) * lpb;
    double2* A = sm;
    double2* Bh = sm + strideA;
    // restart-invariant scatter metadata of this (m, r), built once per CTA: the complex
    // weight root4(e) conj(w_b^{r t}), the local key (f2: halved) and the index i of each
    // plan entry. Per restart only u (staged in us) changes, so a run head sums
    // wv[q] * u[idx[q]] (f2: u^2) over its run straight from shared memory.
    double2* wv = Bh + strideB;                                               // 2n
    // (local key | head << 31 | run continues << 30, index i) per plan entry: a run of equal
    // keys is summed by its head, in plan order; the flags spare the per-restart scatter the
    // neighbour reads, so an entry's loads are independent and issue together
    uint2* kx = reinterpret_cast<uint2*>(wv + 2 * n);                         // 2n
    double* us = reinterpret_cast<double*>(kx + 2 * n);                       // n
    const std::uint32_t bmask = v.b - 1;
    const std::uint32_t nmask = static_cast<std::uint32_t>(N - 1);
    const double2* fT = v.spec + ((size_t)m * S + r) * N;
    const uint2* p1 = v.plan1 + (size_t)m * n;
    const uint2* p2 = v.plan2 + (size_t)m * n;
    const std::uint32_t* b1 = v.bucket1 + (size_t)m * n;
    const std::uint32_t* b2 = v.bucket2 + (size_t)m * n;
    const std::uint32_t* b3 = v.bucket3 + (size_t)m * n;
    const std::uint8_t* se = v.sexp + (size_t)m * n;
    const double2* dm = v.data + (size_t)m * v.b;

    const size_t mr = ((size_t)m * S + r) * n;  // residue-twiddle table offset of (m, r)
#ifdef SKC_TRACE_CONTRACT
    unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tp = clock64();
#define PH(q)                                   \
    {                                           \
        const unsigned long long t_ = clock64(); \
        ph[q] += t_ - tp;                        \
        tp = t_;                                 \
    }
#else
#define PH(q)
#endif
    const bool ttab = v.stw1 != nullptr;
    for (int x = threadIdx.x; x < 2 * n; x += NT) {
        const bool hb = x >= n;
        const int q = hb ? x - n : x;
        const uint2* pl = hb ? p2 : p1;
        const uint2 e = pl[q];
        const double2 w = ttab ? (hb ? v.stw2 : v.stw1)[mr + q]
                               : conj(v.tw[(static_cast<std::uint32_t>(r) * (e.y & 0x0FFFFFFFu)) & bmask]);
        wv[x] = cmul(root4_times(e.y >> 28, 1.0), w);
        auto key_of = [&](std::uint32_t y) { return hb ? ((y & nmask) >> 1) : (y & nmask); };
        const std::uint32_t key = key_of(e.y);
        const bool head = q == 0 || key_of(pl[q - 1].y) != key;
        const bool cont = q + 1 < n && key_of(pl[q + 1].y) == key;
        kx[x] = make_uint2(key | (head ? 0x80000000u : 0u) | (cont ? 0x40000000u : 0u), e.x);
    }
    for (int l = l0; l < min(L, l0 + lpb); ++l) {
        const double* ug = U + (size_t)l * n;
        for (int x = threadIdx.x; x < n; x += NT) us[x] = ug[x];  // u staged once per restart
        zero_smem(sm, strideA + strideB);
        __syncthreads();
        PH(0)
        // deterministic scatter (contraction.cpp:150-154): the head of each run of equal
        // keys sums its run in plan order; f1 values u_i, f2 values u_i^2
        // (batches of 4 entries per thread: all their metadata loads, then the u loads, then
        // the products, so the shared-memory latencies overlap instead of chaining)
        for (int x0 = threadIdx.x; x0 < 2 * n; x0 += SB * NT) {
            uint2 k[SB];
            double2 w[SB];
            double ui[SB];
#pragma unroll
            for (int c = 0; c < SB; ++c) {
                const int x = x0 + c * NT;
                k[c] = x < 2 * n ? kx[x] : make_uint2(0u, 0u);
                w[c] = x < 2 * n ? wv[x] : mk(0.0, 0.0);
            }
#pragma unroll
            for (int c = 0; c < SB; ++c) ui[c] = (k[c].x >> 31) ? us[k[c].y] : 0.0;
#pragma unroll
            for (int c = 0; c < SB; ++c) {
                if (!(k[c].x >> 31)) continue;  // not a run head (or past the end)
                const int x = x0 + c * NT;
                const bool hb = x >= n;
                const double val = hb ? ui[c] * ui[c] : ui[c];
                double2 acc = mk(w[c].x * val, w[c].y * val);
                std::uint32_t kk = k[c].x;
                for (int x2 = x + 1; kk & 0x40000000u; ++x2) {  // the rest of the run, plan order
                    const uint2 k2 = kx[x2];
                    const double u2 = us[k2.y];
                    const double2 w2 = wv[x2];
                    const double v2 = hb ? u2 * u2 : u2;
                    acc = cadd(acc, mk(w2.x * v2, w2.y * v2));
                    kk = k2.x;
                }
                (hb ? Bh : A)[pad16(static_cast<int>(k[c].x & 0x3FFFFFFFu))] = acc;
            }
        }
        __syncthreads();
        PH(1)
        PH(2)
        DifPair<LOGN, 4, 0>::run(A, Bh, v.twl);
        PH(3)

        if (mode == 0) {
            // z1 = fT conj(f1^2 + f2) (full), Z2 = fT conj(f1) folded to N/2 (contraction.cpp:158-162)
            // (the spectrum slice comes from L2: three positions' loads are issued together)
            for (int q0 = threadIdx.x; q0 < NH; q0 += PB * NT) {
                double2 t0[PB], t1[PB];
#pragma unroll
                for (int c = 0; c < PB; ++c) {
                    const int q = q0 + c * NT;
                    t0[c] = q < NH ? fT[2 * q] : mk(0.0, 0.0);
                    t1[c] = q < NH ? fT[2 * q + 1] : mk(0.0, 0.0);
                }
#pragma unroll
                for (int c = 0; c < PB; ++c) {
                    const int q = q0 + c * NT;
                    if (q >= NH) break;
                    const int p0 = 2 * q, p1i = 2 * q + 1;
                    const double2 u0 = A[pad16(p0)], u1 = A[pad16(p1i)];
                    const double2 f2 = Bh[pad16(q)];
                    A[pad16(p0)] = cmulc(t0[c], cadd(cmul(u0, u0), f2));
                    A[pad16(p1i)] = cmulc(t1[c], cadd(cmul(u1, u1), f2));
                    Bh[pad16(q)] = cadd(cmulc(t0[c], u0), cmulc(t1[c], u1));
                }
            }
            __syncthreads();
            PH(4)
            DitPair<LOGN, 4, plan_npass(LOGN, 4) - 1>::run(A, Bh, v.twl);
            PH(5)
            const double inv_b = 1.0 / static_cast<double>(v.b);
            double* o = out + (((size_t)l * B + m) * S + r) * n;
            if (ttab) {  // folded gather weights (k_sym_twiddle_tables); three entries' loads together
                for (int i0 = threadIdx.x; i0 < n; i0 += GB * NT) {
                    std::uint32_t t1[GB], t2[GB];
                    double2 g1[GB], g2[GB];
#pragma unroll
                    for (int c = 0; c < GB; ++c) {
                        const int i = i0 + c * NT;
                        const bool ok = i < n;
                        t1[c] = ok ? b1[i] : 0u;
                        t2[c] = ok ? b2[i] : 0u;
                        g1[c] = ok ? v.gtw1[mr + i] : mk(0.0, 0.0);
                        g2[c] = ok ? v.gtw2[mr + i] : mk(0.0, 0.0);
                    }
#pragma unroll
                    for (int c = 0; c < GB; ++c) {
                        const int i = i0 + c * NT;
                        if (i >= n) break;
                        const double ui = us[i];
                        const double2 a1 = A[pad16(static_cast<int>(t1[c] & nmask))];
                        const double2 a2 = Bh[pad16(static_cast<int>((t2[c] & nmask) >> 1))];
                        double val = (a1.x * g1[c].x - a1.y * g1[c].y) + ui * (a2.x * g2[c].x - a2.y * g2[c].y);
                        if (r == 0) val += ui * ui * re_rot_conj(3u * se[i], dm[b3[i]]) * (1.0 / 3.0);
                        o[i] = val;
                    }
                }
            } else
            for (int i = threadIdx.x; i < n; i += NT) {
                const double ui = us[i];
                const std::uint32_t t1 = b1[i], t2 = b2[i];
                const double2 a1 = A[pad16(static_cast<int>(t1 & nmask))];
                const double2 a2 = Bh[pad16(static_cast<int>((t2 & nmask) >> 1))];
                double val;
                {
                    const unsigned e = se[i];
                    const double2 z1 = cmul(a1, v.tw[(static_cast<std::uint32_t>(r) * t1) & bmask]);
                    const double2 z2 = cmul(a2, v.tw[(static_cast<std::uint32_t>(r) * t2) & bmask]);
                    val = re_rot_conj(e, z1) * (1.0 / 6.0) * inv_b;
                    val += ui * re_rot_conj(2u * e, z2) * (1.0 / 3.0) * inv_b;
                }
                if (r == 0) val += ui * ui * re_rot_conj(3u * se[i], dm[b3[i]]) * (1.0 / 3.0);
                o[i] = val;
            }
        } else {
            // acc1 += Re(fT conj(f1)^3), acc2 += Re(fT conj(f1) conj(f2))   (contraction.cpp:111-116)
            double acc1 = 0.0, acc2 = 0.0;
            for (int j = threadIdx.x; j < N; j += NT) {
                const double2 c1 = conj(A[pad16(j)]);
                const double2 w1 = cmul(fT[j], c1);
                acc1 += cmul(cmul(w1, c1), c1).x;
                acc2 += cmul(w1, conj(Bh[pad16(j >> 1)])).x;
            }
            const double s1 = block_sum<NT>(acc1, red);
            const double s2 = block_sum<NT>(acc2, red);
            double term3 = 0.0;
            if (r == 0) {  // contraction.cpp:117-121
                for (int i = threadIdx.x; i < n; i += NT) {
                    const double u3 = us[i] * us[i] * us[i];
                    term3 += u3 * re_rot_conj(3u * se[i], dm[b3[i]]);
                }
            }
            const double s3 = block_sum<NT>(term3, red);
            if (threadIdx.x == 0) {
                double* o = out + (((size_t)l * B + m) * S + r) * 3;
                o[0] = s1;
                o[1] = s2;
                o[2] = s3;
            }
        }
        __syncthreads();
        PH(6)
    }
#ifdef SKC_TRACE_CONTRACT
    if (threadIdx.x == 0)
        for (int q = 0; q < 8; ++q) atomicAdd(&g_contract_phase[q], ph[q]);
#endif
#undef PH
}

template <int LOGN, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB)
    k_sym_contract_half(SymView v, const double* __restrict__ U, int L, int mode, double* __restrict__ out) {
    sym_contract_half_body<LOGN, NT>(v, U, L, mode, out);
}
// Contraction kernels (measured on B200, profiles/r01): the half-length f2/z2 kernel at
// 192 threads x 3 CTAs per SM is the default (config-1 step 0.886 ms against 1.05 for the
// full-length radix-16 kernel with scratch scatter, 0.94 for 256 x 2 CTAs, 0.97 for a
// 112-register cap). The full-length kernel (scratch or direct scatter) covers the shapes
// the half-length one does not: n above the shared-memory scatter limit, local N < 4.
template <int LG, int VAR, int LR, int MINB>
static void sym_contract_launch(cudaStream_t st, const SymView& v, const double* U, int L, int mode, double* out,
                                unsigned grid, size_t smem) {
    cudaFuncSetAttribute(k_sym_contract<LG, VAR, LR, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_sym_contract<LG, VAR, LR, MINB><<<grid, kFftThreads, smem, st>>>(v, U, L, mode, out);
}

template <int LG, int NT, int MINB>
static void sym_contract_half_launch(cudaStream_t st, const SymView& v, const double* U, int L, int mode, double* out,
                                     unsigned grid, size_t smem) {
    cudaFuncSetAttribute(k_sym_contract_half<LG, NT, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_sym_contract_half<LG, NT, MINB><<<grid, NT, smem, st>>>(v, U, L, mode, out);
}


// Restarts per CTA of the half-length contraction kernel (3 resident CTAs per SM): each
// CTA builds its (replicate, residue) scatter metadata once and then runs its restarts one
// after another, so the step's makespan is ~ ceil(CTAs / resident slots) x (restarts per
// CTA + setup), setup ~ 0.3 restart. Config 1 (16000 restart-residue tasks) is flat in this
// choice (3..13 per CTA measured 0.730..0.758 ms); config 0 (2000 tasks, ~1.2 waves at 4 per
// CTA) takes 5 per CTA, one wave (RTPM contraction time -10%).
static int contract_restarts_per_cta(int L, int per_restart_ctas) {
    static int sms[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    int& nsm = sms[dev & 63];
    if (nsm == 0) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const long long slots = 3ll * (nsm > 0 ? nsm : 148);
    int best = 4;
    double best_cost = 1e300;
    for (int lpb = 1; lpb <= 8; ++lpb) {
        const long long ctas = static_cast<long long>((L + lpb - 1) / lpb) * per_restart_ctas;
        const double cost = static_cast<double>((ctas + slots - 1) / slots) * (lpb + 0.3);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = lpb;
        }
    }
    return best;
}

void launch_sym_contract(cudaStream_t st, const SymView& v, const double* U, int L, int mode, double* out) {
    const bool scr_ok = v.n <= kScatterMax;
    if (scr_ok && v.logN >= 2) {
        SymView vv = v;
        vv.lpb = contract_restarts_per_cta(L, v.B * v.S);
        const int NH = v.N / 2;
        const size_t smem = sizeof(double2) * (padded_len(v.N) + (NH + NH / 16 + 1)) +
                            (sizeof(double2) + 2 * sizeof(std::uint32_t)) * 2 * (size_t)v.n +
                            sizeof(double) * ((size_t)v.n + 1);
        const unsigned grid = (unsigned)((long long)((L + vv.lpb - 1) / vv.lpb) * v.B * v.S);
#define LH_(LG) sym_contract_half_launch<LG, 192, 3>(st, vv, U, L, mode, out, grid, smem)
        switch (v.logN) {
            case 2: LH_(2); break;
            case 3: LH_(3); break;
            case 4: LH_(4); break;
            case 5: LH_(5); break;
            case 6: LH_(6); break;
            case 7: LH_(7); break;
            case 8: LH_(8); break;
            case 9: LH_(9); break;
            case 10: LH_(10); break;
            case 11: LH_(11); break;
            case 12: LH_(12); break;
            default: break;
        }
#undef LH_
        SKC_LAUNCHED();
        count_transforms((std::uint64_t)L * v.B * v.S * (mode == 0 ? 4 : 2), v.S);
        return;
    }
    const size_t smem = sizeof(double2) * 2 * padded_len(v.N) +
                        (scr_ok ? (sizeof(double2) + sizeof(std::uint32_t)) * 2 * (size_t)v.n : 0);
    const unsigned grid = (unsigned)((long long)((L + kLPB - 1) / kLPB) * v.B * v.S);
#define L_(LG)                                                                                         \
    {                                                                                                  \
        if (scr_ok)                                                                                    \
            sym_contract_launch<LG, 1, 4, 2>(st, v, U, L, mode, out, grid, smem);                      \
        else                                                                                           \
            sym_contract_launch<LG, 2, 4, 2>(st, v, U, L, mode, out, grid, smem);                      \
    }
    SKC_LOGN_SWITCH(v.logN, L_)
#undef L_
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

// part: L x B x S x n -> med: L x n medians over B of the residue sums (fixed order).
// Tiled form: a block takes 32 consecutive columns i of one restart l. Its 256 threads
// first sum the S residue partials of every (column, replicate) pair (coalesced over i,
// same order as k_median_cols), then rank every pair within its column (ties by index),
// so the L x n x B x S partials are read with 8x the parallelism of one thread per column.
template <int BT>
__global__ void __launch_bounds__(256) k_median_tile(const double* __restrict__ part, int L, int B, int S, int n,
                                                      double* __restrict__ med) {
    constexpr int CAP = BT > 0 ? BT : kMaxB;
    __shared__ double est[CAP][33];
    __shared__ double sel[2][32];
    const int Bn = BT > 0 ? BT : B;
    const int tiles = (n + 31) / 32;
    const int l = blockIdx.x / tiles, i0 = (blockIdx.x - l * tiles) * 32;
    const int il = threadIdx.x & 31;
    const int i = i0 + il;
    for (int m = threadIdx.x >> 5; m < Bn; m += 8) {
        double sacc = 0.0;
        if (i < n) {
            const double* p = part + (((size_t)l * Bn + m) * S) * n + i;
            sacc = p[0];
            for (int r = 1; r < S; ++r) sacc += p[(size_t)r * n];
        }
        est[m][il] = sacc;
    }
    __syncthreads();
    const int hiR = Bn / 2, loR = Bn / 2 - 1;
    for (int a = threadIdx.x >> 5; a < Bn; a += 8) {
        const double x = est[a][il];
        int rank = 0;
        for (int c = 0; c < Bn; ++c) {
            const double y = est[c][il];
            rank += (y < x) || (y == x && c < a);
        }
        if (rank == hiR) sel[1][il] = x;
        if (rank == loR) sel[0][il] = x;
    }
    __syncthreads();
    if (threadIdx.x < 32 && i < n) {
        const double hi = sel[1][il], lo = Bn > 1 ? sel[0][il] : 0.0;
        med[(size_t)l * n + i] = (Bn & 1) ? hi : 0.5 * (lo + hi);
    }
}

// Unext[l] = med[l] / ||med[l]|| (decompose.cpp:35-40), flags[l] set when ||.|| <= tol.
__global__ void __launch_bounds__(256) k_normalize_rows(const double* __restrict__ med, int n,
                                                         double* __restrict__ Unext, double tol,
                                                         int* __restrict__ flags) {
    __shared__ double red[8];
    const int l = blockIdx.x;
    const double* row = med + (size_t)l * n;
    double ss = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) ss += row[i] * row[i];
    const double tot = block_sum<256>(ss, red);
    __shared__ double nrm_s;
    if (threadIdx.x == 0) {
        const double nrm = sqrt(tot);
        nrm_s = nrm;
        if (!(nrm > tol)) flags[l] = 1;
    }
    __syncthreads();
    const double nrm = nrm_s;
    for (int i = threadIdx.x; i < n; i += blockDim.x) Unext[(size_t)l * n + i] = row[i] / nrm;
}

// out (may be null): L x n medians; Unext (may be null): normalised medians + flags.
// When out is null a library scratch buffer holds the medians (scratch: L x n).
void launch_median_rows(cudaStream_t st, const double* part, int L, int B, int S, int n, double* out, double* Unext,
                        double tol, int* flags, double* scratch) {
    double* med = out ? out : scratch;
    const unsigned grid = static_cast<unsigned>((long long)L * ((n + 31) / 32));
    switch (B) {
        case 10: k_median_tile<10><<<grid, 256, 0, st>>>(part, L, B, S, n, med); break;
        case 20: k_median_tile<20><<<grid, 256, 0, st>>>(part, L, B, S, n, med); break;
        case 40: k_median_tile<40><<<grid, 256, 0, st>>>(part, L, B, S, n, med); break;
        default: k_median_tile<0><<<grid, 256, 0, st>>>(part, L, B, S, n, med); break;
    }
    SKC_LAUNCHED();
    if (Unext) {
        k_normalize_rows<<<L, 256, 0, st>>>(med, n, Unext, tol, flags);
        SKC_LAUNCHED();
    }
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
template <int LOGN, bool SCR, int LR>
__global__ void __launch_bounds__(kFftThreads, SKC_FFT_MINB)
    k_sym_moment(SymView v, const double* __restrict__ X, const double* __restrict__ w, double wscale, long long Nsamp,
                 int chunks, double* __restrict__ acc) {
    extern __shared__ double2 sm[];
    constexpr int N = 1 << LOGN;
    constexpr int stride = N + (N >> 4) + 1;
    const int S = v.S, n = v.n, B = v.B;
    const int r = blockIdx.x % S;
    const int m = (blockIdx.x / S) % B;
    const int ch = blockIdx.x / (S * B);
    double2* A = sm;
    double2* ACC = sm + stride;
    // SCR: the sample-invariant scatter metadata of this (m, r) (weight root4(e)
    // conj(w_b^{r t}), local key, index i) is built once; per sample a run head sums
    // wv[q] x[idx[q]] over its run.
    // ACC uses the padded layout of A: the fused last DIF pass touches 16 consecutive
    // positions per thread, which the padding spreads over the banks
    double2* wv = ACC + stride;                                        // n (SCR)
    std::uint32_t* keys = reinterpret_cast<std::uint32_t*>(wv + n);   // n (SCR)
    std::uint32_t* idx = keys + n;                                     // n (SCR)
    double* xs = reinterpret_cast<double*>(idx + n);  // 2 x n (SCR): sample double buffer (2n u32: 8-byte aligned)
    const long long per = (Nsamp + chunks - 1) / chunks;
    const long long s0 = (long long)ch * per, s1 = min(Nsamp, s0 + per);
    const uint2* plan = v.plan1 + (size_t)m * n;
    const std::uint32_t bmask = v.b - 1;
    const std::uint32_t nmask = static_cast<std::uint32_t>(N - 1);
    zero_smem(ACC, stride);
    zero_smem(A, stride);
    if (SCR) {
        const double2* stw = v.stw1 ? v.stw1 + ((size_t)m * S + r) * n : nullptr;
        for (int q = threadIdx.x; q < n; q += blockDim.x) {
            const uint2 e = plan[q];
            const double2 w = stw ? stw[q] : conj(v.tw[(static_cast<std::uint32_t>(r) * (e.y & 0x0FFFFFFFu)) & bmask]);
            wv[q] = cmul(root4_times(e.y >> 28, 1.0), w);
            keys[q] = e.y & nmask;
            idx[q] = e.x;
        }
    }
    // The next sample's row is copied into the other half of xs while the current one is
    // transformed: one bulk (TMA) copy of the whole row, completing on an mbarrier per half,
    // when rows are 16-byte aligned (n even, X aligned); else per-element 8-byte cp.async.
    __shared__ __align__(8) unsigned long long mbar[2];
    const bool bulk = SCR && ((n & 1) == 0) && ((reinterpret_cast<std::uintptr_t>(X) & 15) == 0);
    const std::uint32_t mb0 = static_cast<std::uint32_t>(__cvta_generic_to_shared(&mbar[0]));
    if (bulk && threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(mb0) : "memory");
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(mb0 + 8u) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto prefetch = [&](long long smp) {
        if (!SCR || smp >= s1) return;
        const double* src = X + (size_t)smp * n;
        const int half = static_cast<int>((smp - s0) & 1);
        double* dst = xs + (size_t)half * n;
        if (bulk) {
            if (threadIdx.x == 0) {
                const std::uint32_t bytes = static_cast<std::uint32_t>(n) * 8u;
                const std::uint32_t mb = mb0 + 8u * static_cast<std::uint32_t>(half);
                const std::uint32_t da = static_cast<std::uint32_t>(__cvta_generic_to_shared(dst));
                // the half was last read by generic loads (ordered by the loop's barriers)
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(da),
                    "l"(src), "r"(bytes), "r"(mb)
                    : "memory");
            }
            return;
        }
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const std::uint32_t da = static_cast<std::uint32_t>(__cvta_generic_to_shared(dst + i));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(da), "l"(src + i) : "memory");
        }
    };
    // sample smp's row has landed in its half (parity of that half's use count)
    auto wait_row = [&](long long smp) {
        if (bulk) {
            const long long t = smp - s0;
            const std::uint32_t mb = mb0 + 8u * static_cast<std::uint32_t>(t & 1);
            const std::uint32_t par = static_cast<std::uint32_t>((t >> 1) & 1);
            std::uint32_t done = 0;
            while (!done)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                    : "=r"(done)
                    : "r"(mb), "r"(par)
                    : "memory");
        } else {
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        }
    };
    prefetch(s0);
    asm volatile("cp.async.commit_group;" ::: "memory");
    __syncthreads();
    for (long long s = s0; s < s1; ++s) {
        const double* x = X + (size_t)s * n;
        prefetch(s + 1);
        asm volatile("cp.async.commit_group;" ::: "memory");
        wait_row(s);  // this sample's row has landed
        __syncthreads();
        // A is all-zero here (initially, then re-zeroed by the accumulate pass below)
        if (SCR) {
            const double* xr = xs + (size_t)((s - s0) & 1) * n;
            for (int q = threadIdx.x; q < n; q += blockDim.x) {
                const std::uint32_t key = keys[q];
                if (q > 0 && keys[q - 1] == key) continue;
                double2 a = mk(0.0, 0.0);
                for (int q2 = q; q2 < n && keys[q2] == key; ++q2) {
                    const double xi = xr[idx[q2]];
                    const double2 wq = wv[q2];
                    a = cadd(a, mk(wq.x * xi, wq.y * xi));
                }
                A[pad16(static_cast<int>(key))] = a;
            }
        } else {
            auto vx = [&](std::uint32_t i, std::uint32_t y) { return root4_times(y >> 28, x[i]); };
            scatter_plan(A, plan, n, N, r, bmask, 0x0FFFFFFFu, v.tw, vx);
        }
        __syncthreads();
        const double ws = (w ? w[s] : 1.0) * wscale;
        // the last DIF pass feeds the cube-accumulate directly (no extra pass over A)
        dif_local_epilogue<LOGN, LR>(A, v.twl, [&](int j, double2 z) {
            A[pad16(j)] = mk(0.0, 0.0);  // ready for the next sample's scatter
            const double2 z3 = cmul(cmul(z, z), z);
            ACC[pad16(j)] = cadd(ACC[pad16(j)], cscale(z3, ws));
        });
        __syncthreads();
    }
    double2* o = reinterpret_cast<double2*>(acc) + (((size_t)ch * B + m) * S + r) * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) o[j] = ACC[pad16(j)];
}
// Paired-sample form of k_sym_moment for local length 2048 (the b >= 2^11 shapes: configs 3
// and 4). Two samples go through the transform together and the accumulators live in
// registers:
//   - the passes run 16 x 16 x 8 (the same radix-2 stage sequence as the 8 x 16 x 16 plan, so
//     the same bit-reversed layout): the two radix-16 passes have 2 x 128 items for the 256
//     threads (one sample left half of them idle), and the closing radix-8 pass gives thread
//     t the 8 consecutive outputs [8t, 8t + 8) of every sample, so the cube-accumulate adds
//     into 8 complex registers instead of a read-modify-write of a shared-memory array;
//   - the freed array holds the second sample: same shared-memory footprint, 2 CTAs per SM,
//     half the barriers per sample;
//   - both rows of a pair arrive by ONE bulk (TMA) copy (rows s, s + 1 are contiguous in X)
//     into a single buffer, issued once the scatter has consumed the previous pair.
template <int LOGN>
__global__ void __launch_bounds__((1 << LOGN) / 8, 2)
    k_sym_moment_pair(SymView v, const double* __restrict__ X, const double* __restrict__ w, double wscale,
                      long long Nsamp, int chunks, double* __restrict__ acc) {
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
    double2* wv = A1 + stride;                                         // n
    // (local key | head << 31 | run continues << 30, index i): see sym_contract_half_body
    uint2* kx = reinterpret_cast<uint2*>(wv + n);                      // n
    double* xs = reinterpret_cast<double*>(kx + n);                    // 2 x n: the pair's rows
    const long long per = (Nsamp + chunks - 1) / chunks;
    const long long s0 = (long long)ch * per, s1 = min(Nsamp, s0 + per);
    const uint2* plan = v.plan1 + (size_t)m * n;
    const std::uint32_t bmask = v.b - 1;
    const std::uint32_t nmask = static_cast<std::uint32_t>(N - 1);
    // Scatter order. The plan lists the entries by local key, equal keys adjacent (a run is
    // summed in plan order, sketch.cpp:353-356). Entries are regrouped by their rank in the
    // run: rank 0 (one per occupied position, ~79% of the entries at n = 1000) sorted by the
    // sample index i, then rank 1 sorted by i, then the deeper ranks in plan order. Phase 1 of a
    // scatter writes the rank-0 products (distinct positions, the sample read almost
    // contiguously instead of at random), phase 2 adds the rank-1 products and walks what is
    // left of the run: the same additions in the same order as a head walking its run.
    //   kx.x = local key | position of the run's rank-2 entry << 12 | run continues << 30
    __shared__ int s_cls[3];  // class sizes: rank 0, rank 1, rank >= 2
    {
        double2* twv = A0;                                                 // n (plan order)
        uint2* tkx = reinterpret_cast<uint2*>(A0 + n);                     // n: (key | min(rank, 2) << 12 | cont << 30, i)
        unsigned short* inv = reinterpret_cast<unsigned short*>(A1);       // n: plan position of index i
        unsigned short* dst = inv + n + (n & 1);                           // n: final position of plan entry q
        const double2* stw = v.stw1 ? v.stw1 + ((size_t)m * S + r) * n : nullptr;
        for (int q = threadIdx.x; q < n; q += NT) {
            const uint2 e = plan[q];
            const double2 tw = stw ? stw[q] : conj(v.tw[(static_cast<std::uint32_t>(r) * (e.y & 0x0FFFFFFFu)) & bmask]);
            twv[q] = cmul(root4_times(e.y >> 28, 1.0), tw);
            const std::uint32_t key = e.y & nmask;
            int rk = 0;
            while (rk < 2 && q - rk - 1 >= 0 && (plan[q - rk - 1].y & nmask) == key) ++rk;
            const bool cont = q + 1 < n && (plan[q + 1].y & nmask) == key;
            tkx[q] = make_uint2(key | (static_cast<std::uint32_t>(rk) << 12) | (cont ? 0x40000000u : 0u), e.x);
            inv[e.x] = static_cast<unsigned short>(q);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            const std::uint32_t lt = (1u << lane) - 1u;
            int c0 = 0, c1 = 0, c2 = 0;
            for (int base = 0; base < n; base += 32) {  // class sizes
                const int q = base + lane;
                const int rk = q < n ? static_cast<int>((tkx[q].x >> 12) & 3u) : -1;
                c0 += __popc(__ballot_sync(0xffffffffu, rk == 0));
                c1 += __popc(__ballot_sync(0xffffffffu, rk == 1));
            }
            const int b1 = c0, b2 = c0 + c1;
            c0 = 0;
            c1 = 0;
            for (int base = 0; base < n; base += 32) {
                const int i = base + lane;  // ranks 0 and 1 in index order
                const int qi = i < n ? static_cast<int>(inv[i]) : 0;
                const int rki = i < n ? static_cast<int>((tkx[qi].x >> 12) & 3u) : -1;
                const std::uint32_t m0 = __ballot_sync(0xffffffffu, rki == 0), m1 = __ballot_sync(0xffffffffu, rki == 1);
                if (rki == 0) dst[qi] = static_cast<unsigned short>(c0 + __popc(m0 & lt));
                if (rki == 1) dst[qi] = static_cast<unsigned short>(b1 + c1 + __popc(m1 & lt));
                c0 += __popc(m0);
                c1 += __popc(m1);
                const int q = base + lane;  // deeper ranks in plan order
                const int rkq = q < n ? static_cast<int>((tkx[q].x >> 12) & 3u) : -1;
                const std::uint32_t m2 = __ballot_sync(0xffffffffu, rkq == 2);
                if (rkq == 2) dst[q] = static_cast<unsigned short>(b2 + c2 + __popc(m2 & lt));
                c2 += __popc(m2);
            }
            if (lane == 0) {
                s_cls[0] = b1;
                s_cls[1] = b2 - b1;
                s_cls[2] = c2;
            }
        }
        __syncthreads();
        for (int q = threadIdx.x; q < n; q += NT) {
            const uint2 t = tkx[q];
            const int d = dst[q];
            const std::uint32_t nxt = (t.x & 0x40000000u) ? static_cast<std::uint32_t>(dst[q + 1]) : 0u;
            wv[d] = twv[q];
            kx[d] = make_uint2((t.x & 0x40000FFFu) | (nxt << 12), t.y);
        }
        __syncthreads();
        zero_smem(A0, 2 * stride);
    }
    __shared__ __align__(8) unsigned long long mbar;
    const bool bulk = ((n & 1) == 0) && ((reinterpret_cast<std::uintptr_t>(X) & 15) == 0);
    const std::uint32_t mb = static_cast<std::uint32_t>(__cvta_generic_to_shared(&mbar));
    if (bulk && threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(mb) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // rows [smp, smp + cnt) -> xs (thread 0; the buffer's previous readers are behind a barrier)
    auto prefetch = [&](long long smp) {
        if (!bulk || smp >= s1 || threadIdx.x != 0) return;
        const std::uint32_t bytes = static_cast<std::uint32_t>(min(2ll, s1 - smp)) * static_cast<std::uint32_t>(n) * 8u;
        const std::uint32_t da = static_cast<std::uint32_t>(__cvta_generic_to_shared(xs));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(da),
                     "l"(X + (size_t)smp * n), "r"(bytes), "r"(mb)
                     : "memory");
    };
    double2 accr[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) accr[q] = mk(0.0, 0.0);
    const int wi = static_cast<int>((threadIdx.x & ~15u) | ((threadIdx.x & 7u) << 1) | ((threadIdx.x >> 3) & 1u));
    prefetch(s0);
    std::uint32_t par = 0;
    for (long long s = s0; s < s1; s += 2) {
        const int cnt = static_cast<int>(min(2ll, s1 - s));
        if (bulk) {
            std::uint32_t done = 0;
            while (!done)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                    : "=r"(done)
                    : "r"(mb), "r"(par)
                    : "memory");
            par ^= 1u;
        } else {
            for (int i = threadIdx.x; i < cnt * n; i += NT) xs[i] = X[(size_t)s * n + i];
            __syncthreads();
        }
        // A0, A1 are all-zero here (initially, then re-zeroed by the closing pass).
        const double* xs1 = cnt > 1 ? xs + n : xs;
        const int R0 = s_cls[0], R1 = s_cls[1];
        // phase 1: rank-0 entries (4 per thread at a time: metadata, then the sample, then the products)
        for (int e0 = threadIdx.x; e0 < R0; e0 += 4 * NT) {
            uint2 k[4];
            double2 wq[4];
            double x0[4], x1[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int e = min(e0 + c * NT, R0 - 1);
                k[c] = kx[e];
                wq[c] = wv[e];
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                x0[c] = xs[k[c].y];
                x1[c] = xs1[k[c].y];
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if (e0 + c * NT >= R0) break;
                const int pj = pad16(static_cast<int>(k[c].x & 0xFFFu));
                A0[pj] = mk(wq[c].x * x0[c], wq[c].y * x0[c]);
                if (cnt > 1) A1[pj] = mk(wq[c].x * x1[c], wq[c].y * x1[c]);
            }
        }
        __syncthreads();
        // phase 2: rank-1 entries add to their position, then the rest of the run in plan order
        for (int e = R0 + threadIdx.x; e < R0 + R1; e += NT) {
            uint2 k = kx[e];
            double2 wq = wv[e];
            const int pj = pad16(static_cast<int>(k.x & 0xFFFu));
            double2 a0 = A0[pj], a1 = cnt > 1 ? A1[pj] : mk(0.0, 0.0);
            for (;;) {
                const double y0 = xs[k.y], y1 = xs1[k.y];
                a0 = cadd(a0, mk(wq.x * y0, wq.y * y0));
                a1 = cadd(a1, mk(wq.x * y1, wq.y * y1));
                if (!(k.x & 0x40000000u)) break;
                const int e2 = static_cast<int>((k.x >> 12) & 0xFFFu);  // the run's next entry
                k = kx[e2];
                wq = wv[e2];
            }
            A0[pj] = a0;
            if (cnt > 1) A1[pj] = a1;
        }
        __syncthreads();
        prefetch(s + 2);  // xs is consumed: the next pair lands during the passes
        // radix-16 passes: half-sizes N/2, N/32, ... down to 64 (2 x N/16 items)
        constexpr int NP16 = (LOGN - 3) / 4;
#pragma unroll
        for (int pz = 0; pz < NP16; ++pz) {
            const int h = (N >> 1) >> (4 * pz);
            for (int it = threadIdx.x; it < cnt * (N / 16); it += NT) {
                const int a = it / (N / 16);
                dif_pass_item<4>(a ? A1 : A0, it - a * (N / 16), h, v.twl, LOGN);
            }
            __syncthreads();
        }
        // closing radix-8 pass (half-size 4): a thread holds the 8 consecutive outputs of item wi
        // of each sample. Item w starts at padded position 8w + w/2, i.e. bank group (w/2) mod 8,
        // so the 8 lanes of a quarter-warp take items 2l + p (l = lane & 7): distinct groups
        // (items 8q .. 8q + 7 in lane order would collide two by two)
#pragma unroll 1
        for (int c = 0; c < cnt; ++c) {
            double2* A = c ? A1 : A0;
            const double ws = (w ? w[s + c] : 1.0) * wscale;
            double2 z[8];
            int base, g;
            dif_item_core<3, true>(A, wi, 4, v.twl, LOGN, z, base, g);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                A[pad16(base + q * g)] = mk(0.0, 0.0);  // ready for the next pair's scatter
                const double2 z3 = cmul(cmul(z[q], z[q]), z[q]);
                accr[q] = cadd(accr[q], cscale(z3, ws));
            }
        }
        __syncthreads();
    }
    double2* o = reinterpret_cast<double2*>(acc) + (((size_t)ch * B + m) * S + r) * N;
#pragma unroll
    for (int q = 0; q < 8; ++q) o[8 * wi + q] = accr[q];
}
size_t moment_pair_smem(int N, int n) {
    return sizeof(double2) * 2 * static_cast<size_t>(padded_len(N)) +
           (sizeof(double2) + sizeof(uint2)) * static_cast<size_t>(n) + 2 * sizeof(double) * static_cast<size_t>(n);
}

template <int LR>
static void moment_launch(cudaStream_t st, const SymView& v, const double* X, const double* w, double wscale,
                          long long Nsamp, int chunks, double* acc, bool scr, size_t smem, unsigned grid) {
#define L_(LG)                                                                                                         \
    {                                                                                                                  \
        if (scr) {                                                                                                     \
            cudaFuncSetAttribute(k_sym_moment<LG, true, LR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
            k_sym_moment<LG, true, LR><<<grid, kFftThreads, smem, st>>>(v, X, w, wscale, Nsamp, chunks, acc);          \
        } else {                                                                                                       \
            cudaFuncSetAttribute(k_sym_moment<LG, false, LR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
            k_sym_moment<LG, false, LR><<<grid, kFftThreads, smem, st>>>(v, X, w, wscale, Nsamp, chunks, acc);         \
        }                                                                                                              \
    }
    SKC_LOGN_SWITCH(v.logN, L_)
#undef L_
}
void launch_sym_moment_accumulate(cudaStream_t st, const SymView& v, const double* X, const double* w, double wscale,
                                  long long Nsamp, int chunks, double* acc) {
    const bool scr = v.n <= kScatterMax;
    const unsigned grid = (unsigned)((long long)chunks * v.B * v.S);
    if (scr && v.logN == 11) {  // local length 2048: paired samples, register accumulators
        const size_t smem2 = moment_pair_smem(v.N, v.n);
        cudaFuncSetAttribute(k_sym_moment_pair<11>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
        k_sym_moment_pair<11><<<grid, 256, smem2, st>>>(v, X, w, wscale, Nsamp, chunks, acc);
        SKC_LAUNCHED();
        count_transforms((std::uint64_t)Nsamp * v.B * v.S, v.S);
        return;
    }
    const size_t smem = sizeof(double2) * (2 * padded_len(v.N)) +
                        (scr ? (sizeof(double2) + 2 * sizeof(std::uint32_t) + 2 * sizeof(double)) * (size_t)v.n + 8 : 0);
    moment_launch<4>(st, v, X, w, wscale, Nsamp, chunks, acc, scr, smem, grid);  // radix-16 local passes
    SKC_LAUNCHED();
    count_transforms((std::uint64_t)Nsamp * v.B * v.S, v.S);
}

// Sum the chunk partials (fixed order), inverse DIT -> tmp[m][r][t'] natural order.
template <int LOGN>
__global__ void __launch_bounds__(kFftThreads, SKC_FFT_MINB)
    k_freq_reduce_inverse(const double2* __restrict__ acc, int chunks, int B, int S, const double2* __restrict__ twl,
                          double2* __restrict__ tmp) {
    extern __shared__ double2 sm[];
    constexpr int N = 1 << LOGN;
    const int r = blockIdx.x % S, m = blockIdx.x / S;
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
        double2 s = mk(0.0, 0.0);
        for (int c = 0; c < chunks; ++c) s = cadd(s, acc[(((size_t)c * B + m) * S + r) * N + j]);
        sm[pad16(j)] = s;
    }
    __syncthreads();
    dit_local<LOGN>(sm, 1, twl);
    double2* o = tmp + ((size_t)m * S + r) * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) o[j] = sm[pad16(j)];
}
void launch_freq_reduce_inverse(cudaStream_t st, const double* acc, int chunks, int B, int S, int N, int logN,
                                std::uint32_t b, int logb, const double2* twl, double2* tmp) {
    (void)b;
    (void)logb;
    const size_t smem = sizeof(double2) * padded_len(N);
#define L_(LG)                                                                                                    \
    {                                                                                                             \
        if (smem > 48 * 1024)                                                                                     \
            cudaFuncSetAttribute(k_freq_reduce_inverse<LG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        k_freq_reduce_inverse<LG><<<B * S, kFftThreads, smem, st>>>(reinterpret_cast<const double2*>(acc), chunks, B, S, \
                                                                    twl, tmp);                                   \
    }
    SKC_LOGN_SWITCH(logN, L_)
#undef L_
    SKC_LAUNCHED();
    count_transforms((std::uint64_t)B * S, S);
}

// dst[m][t] (+)= alpha * (1/b) * sum_r w_b^{r t} tmp[m][r][t mod N]
// (inverse_inplace scaling, fft.cpp:62-66; data += alpha*su, sketch.cpp:359).
__global__ void k_combine_residues(const double2* __restrict__ tmp, int B, int S, int N, std::uint32_t b,
                                   const double2* __restrict__ tw, double alpha, int m_only, int overwrite, int scaled,
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
    const double2 su = scaled ? cscale(s, inv_b) : s;
    double2* d = dst + idx;
    if (overwrite)
        *d = cscale(su, alpha);
    else
        *d = cadd(*d, cscale(su, alpha));
}
void launch_combine_residues(cudaStream_t st, const double2* tmp, int B, int S, int N, std::uint32_t b,
                             const double2* tw, double alpha, int m_only, bool overwrite, double2* dst, bool scaled) {
    long long tot = (long long)((m_only >= 0) ? 1 : B) * b;
    k_combine_residues<<<cdiv(tot, 256), 256, 0, st>>>(tmp, B, S, N, b, tw, alpha, m_only, overwrite ? 1 : 0,
                                                       scaled ? 1 : 0, dst);
    SKC_LAUNCHED();
}

// Asymmetric factored accumulation (sketch.cpp:224-248, Eq. 2):
// acc += a_c F(s1 u_c) F(s2 v_c) F(s3 w_c). m_only >= 0 restricts to one replicate.
template <int LOGN>
__global__ void __launch_bounds__(kFftThreads, 1)
    k_asym_factored(AsymView v, const double* __restrict__ a, const double* __restrict__ U,
                    const double* __restrict__ V, const double* __restrict__ W, long long Ncomp, int chunks,
                    int m_only, double* __restrict__ acc) {
    extern __shared__ double2 sm[];
    constexpr int N = 1 << LOGN;
    constexpr int stride = N + (N >> 4) + 1;
    const int S = v.S, n = v.n;
    const int Bm = (m_only >= 0) ? 1 : v.B;
    const int r = blockIdx.x % S;
    const int mm = (blockIdx.x / S) % Bm;
    const int m = (m_only >= 0) ? m_only : mm;
    const int ch = blockIdx.x / (S * Bm);
    double2* ACC = sm + 3 * stride;
    const long long per = (Ncomp + chunks - 1) / chunks;
    const long long c0 = (long long)ch * per, c1 = min(Ncomp, c0 + per);
    zero_smem(ACC, N + 8);
    for (long long c = c0; c < c1; ++c) {
        zero_smem(sm, 3 * stride);
        __syncthreads();
        const double* vecs[3] = {U + (size_t)c * n, V + (size_t)c * n, W + (size_t)c * n};
#pragma unroll
        for (int sl = 0; sl < 3; ++sl) {
            const double* x = vecs[sl];
            scatter_plan(sm + sl * stride, v.plan + ((size_t)m * 3 + sl) * n, n, N, r, v.b - 1, 0x7FFFFFFFu, v.tw,
                         [&](std::uint32_t i, std::uint32_t y) { return mk((y >> 31) ? -x[i] : x[i], 0.0); });
        }
        __syncthreads();
        dif_local<LOGN>(sm, 3, v.twl);
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
    const size_t smem = sizeof(double2) * (3 * padded_len(v.N) + v.N + 8);
    const int Bm = (m_only >= 0) ? 1 : v.B;
    const unsigned grid = (unsigned)((long long)chunks * Bm * v.S);
#define L_(LG)                                                                                                   \
    {                                                                                                            \
        if (smem > 48 * 1024)                                                                                    \
            cudaFuncSetAttribute(k_asym_factored<LG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
        k_asym_factored<LG><<<grid, kFftThreads, smem, st>>>(v, a, U, V, W, Ncomp, chunks, m_only, acc);         \
    }
    SKC_LOGN_SWITCH(v.logN, L_)
#undef L_
    SKC_LAUNCHED();
    count_transforms((std::uint64_t)Ncomp * Bm * v.S * 3, v.S);
}

// ============================ K3a: asymmetric contractions ========================
// mode_contraction: contraction.cpp:248-295 (slots at :256-257).
template <int LOGN>
__global__ void __launch_bounds__(kFftThreads, SKC_FFT_MINB)
    k_asym_mode(AsymView v, int free_mode, const double* __restrict__ X, const double* __restrict__ Y, int L,
                double* __restrict__ out) {
    extern __shared__ double2 sm[];
    constexpr int N = 1 << LOGN;
    constexpr int stride = N + (N >> 4) + 1;
    const int S = v.S, n = v.n, B = v.B;
    const int r = blockIdx.x % S;
    const int m = (blockIdx.x / S) % B;
    const int l = blockIdx.x / (S * B);
    const int slot_x = free_mode == 0 ? 1 : 0;
    const int slot_y = free_mode == 2 ? 1 : 2;
    const double* x = X + (size_t)l * n;
    const double* y = Y + (size_t)l * n;
    const std::uint32_t bmask = v.b - 1;
    zero_smem(sm, 2 * stride);
    __syncthreads();
    scatter_plan(sm, v.plan + ((size_t)m * 3 + slot_x) * n, n, N, r, bmask, 0x7FFFFFFFu, v.tw,
                 [&](std::uint32_t i, std::uint32_t tg) { return mk((tg >> 31) ? -x[i] : x[i], 0.0); });
    scatter_plan(sm + stride, v.plan + ((size_t)m * 3 + slot_y) * n, n, N, r, bmask, 0x7FFFFFFFu, v.tw,
                 [&](std::uint32_t i, std::uint32_t tg) { return mk((tg >> 31) ? -y[i] : y[i], 0.0); });
    __syncthreads();
    dif_local<LOGN>(sm, 2, v.twl);
    const double2* fT = v.spec + ((size_t)m * S + r) * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x)
        sm[pad16(j)] = cmulc(fT[j], cmul(sm[pad16(j)], sm[stride + pad16(j)]));
    __syncthreads();
    dit_local<LOGN>(sm, 1, v.twl);
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
    const size_t smem = sizeof(double2) * 2 * padded_len(v.N);
    const unsigned grid = (unsigned)((long long)L * v.B * v.S);
#define L_(LG)                                                                                               \
    {                                                                                                        \
        if (smem > 48 * 1024)                                                                                \
            cudaFuncSetAttribute(k_asym_mode<LG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
        k_asym_mode<LG><<<grid, kFftThreads, smem, st>>>(v, free_mode, X, Y, L, part);                       \
    }
    SKC_LOGN_SWITCH(v.logN, L_)
#undef L_
    SKC_LAUNCHED();
    count_transforms((std::uint64_t)L * v.B * v.S * 3, v.S);
}

// vvv: contraction.cpp:209-246. Partial sums of Re(fT conj(fx fy fz)) per residue.
template <int LOGN>
__global__ void __launch_bounds__(kFftThreads, 2)
    k_asym_vvv(AsymView v, const double* __restrict__ U, int L, double* __restrict__ out) {
    extern __shared__ double2 sm[];
    __shared__ double red[kFftThreads / 32];
    constexpr int N = 1 << LOGN;
    constexpr int stride = N + (N >> 4) + 1;
    const int S = v.S, n = v.n, B = v.B;
    const int r = blockIdx.x % S;
    const int m = (blockIdx.x / S) % B;
    const int l = blockIdx.x / (S * B);
    const double* u = U + (size_t)l * n;
    const std::uint32_t bmask = v.b - 1;
    zero_smem(sm, 3 * stride);
    __syncthreads();
#pragma unroll
    for (int sl = 0; sl < 3; ++sl)
        scatter_plan(sm + sl * stride, v.plan + ((size_t)m * 3 + sl) * n, n, N, r, bmask, 0x7FFFFFFFu, v.tw,
                     [&](std::uint32_t i, std::uint32_t tg) { return mk((tg >> 31) ? -u[i] : u[i], 0.0); });
    __syncthreads();
    dif_local<LOGN>(sm, 3, v.twl);
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
    const size_t smem = sizeof(double2) * 3 * padded_len(v.N);
    const unsigned grid = (unsigned)((long long)L * v.B * v.S);
#define L_(LG)                                                                                              \
    {                                                                                                       \
        if (smem > 48 * 1024)                                                                               \
            cudaFuncSetAttribute(k_asym_vvv<LG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
        k_asym_vvv<LG><<<grid, kFftThreads, smem, st>>>(v, U, L, part);                                     \
    }
    SKC_LOGN_SWITCH(v.logN, L_)
#undef L_
    SKC_LAUNCHED();
    count_transforms((std::uint64_t)L * v.B * v.S * 3, v.S);
}

// ============================ sym_aux_sketches / sketch_rank1_sym ===================
// sketch.cpp:412-425: s1[h] += sigma u, s2[2h] += sigma^2 u^2, s3[3h] += sigma^3 u^3,
// accumulated in ascending i by one thread (exact reference order; a test hook).
__global__ void k_sym_aux(const std::uint32_t* __restrict__ b1, const std::uint32_t* __restrict__ b2,
                          const std::uint32_t* __restrict__ b3, const std::uint8_t* __restrict__ se,
                          const double* __restrict__ u, int n, std::uint32_t b, double2* __restrict__ out) {
    double2* s1 = out;
    double2* s2 = out + b;
    double2* s3 = out + 2 * (size_t)b;
    for (std::uint32_t t = threadIdx.x; t < 3 * b; t += blockDim.x) out[t] = mk(0.0, 0.0);
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int i = 0; i < n; ++i) {
        const double ui = u[i];
        const unsigned e = se[i];
        s1[b1[i]] = cadd(s1[b1[i]], root4_times(e, ui));
        s2[b2[i]] = cadd(s2[b2[i]], root4_times(2u * e, ui * ui));
        s3[b3[i]] = cadd(s3[b3[i]], root4_times(3u * e, ui * ui * ui));
    }
}
void launch_sym_aux(cudaStream_t st, const SymView& v, int m, const double* u, double2* out) {
    const size_t off = (size_t)m * v.n;
    k_sym_aux<<<1, 256, 0, st>>>(v.bucket1 + off, v.bucket2 + off, v.bucket3 + off, v.sexp + off, u, v.n, v.b, out);
    SKC_LAUNCHED();
}
// sketch.cpp:438-439: acc = f1 (f1 f1 / 6 + f2 / 2) on the local spectra of [s1; s2]
__global__ void k_rank1_trunc_product(const double2* __restrict__ spec2, long long len, double2* __restrict__ acc) {
    const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (j >= len) return;
    const double2 f1 = spec2[j], f2 = spec2[len + j];
    acc[j] = cmul(f1, cadd(cscale(cmul(f1, f1), 1.0 / 6.0), cscale(f2, 0.5)));
}
void launch_rank1_trunc_product(cudaStream_t st, const double2* spec2, long long len, double2* acc) {
    k_rank1_trunc_product<<<cdiv(len, 256), 256, 0, st>>>(spec2, len, acc);
    SKC_LAUNCHED();
}
// out += s3 / 3 (sketch.cpp:441)
__global__ void k_add_third(const double2* __restrict__ s3, std::uint32_t b, double2* __restrict__ out) {
    const std::uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= b) return;
    out[t] = cadd(out[t], cscale(s3[t], 1.0 / 3.0));
}
void launch_add_third(cudaStream_t st, const double2* s3, std::uint32_t b, double2* out) {
    k_add_third<<<cdiv(b, 256), 256, 0, st>>>(s3, b, out);
    SKC_LAUNCHED();
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

#ifdef SKC_TRACE_CONTRACT
// experiment build only: per-phase cycle sums of k_sym_contract_half (thread 0 per CTA)
extern "C" int skc_debug_contract_phases(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, skc::g_contract_phase, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {};
        cudaMemcpyToSymbol(skc::g_contract_phase, z, sizeof(z));
    }
    return 0;
}
#endif
