// Residue-split, in-shared-memory radix-16 FFT used by every sketch kernel.
//
// A length-b transform (b = S * N, N = "local length") is split into S independent
// CTA-local transforms of length N, one per frequency residue r in [0, S):
//
//   forward   F[r + S*f2] = sum_{t'} ( sum_{t = t' mod N} x[t] w_b^{-r t} ) w_N^{-f2 t'}
//   inverse   z[t]        = sum_r w_b^{r t} v_r[t mod N],
//             v_r[t']     = sum_{f2} Z[r + S*f2] w_N^{f2 t'}
//
// Sketch inputs are sparse (n nonzeros: count sketches of n-vectors) and contraction
// outputs are read at n positions only, so the split needs no cross-CTA exchange:
// the prologue scatters the n nonzeros with their residue twiddle and the epilogue
// gathers n outputs. The local transform is an in-place decimation-in-frequency
// (forward, natural -> bit-reversed order) and its mirror decimation-in-time
// (inverse, bit-reversed -> natural); spectra are stored in that bit-reversed
// local order, so no reorder pass is ever needed (pointwise products do not care).
//
// Everything here is __host__ __device__ so tests can emulate a CTA on the CPU
// (tests/cpu_emulation/) and check the index algebra against the oracle FFT.
// Semantics follow the reference wrapper proj/src/fft.cpp:48-77 (FFTW_FORWARD sign,
// unnormalised forward, inverse unscaled unless the caller scales by 1/b).
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define SKC_HD __host__ __device__ __forceinline__
#else
#define SKC_HD inline
#include <cmath>
struct double2 {
    double x, y;
};
#endif

namespace skc {

SKC_HD double2 mk(double x, double y) {
    double2 r;
    r.x = x;
    r.y = y;
    return r;
}
SKC_HD double2 cadd(double2 a, double2 b) { return mk(a.x + b.x, a.y + b.y); }
SKC_HD double2 csub(double2 a, double2 b) { return mk(a.x - b.x, a.y - b.y); }
SKC_HD double2 cmul(double2 a, double2 b) { return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
SKC_HD double2 conj(double2 a) { return mk(a.x, -a.y); }
SKC_HD double2 cscale(double2 a, double s) { return mk(a.x * s, a.y * s); }
// a * conj(b)
SKC_HD double2 cmulc(double2 a, double2 b) { return mk(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y); }

// omega^e with omega = i (complex4 signs, proj/src/sketch.cpp:38-45): e mod 4.
SKC_HD double2 root4_times(unsigned e, double v) {
    switch (e & 3u) {
        case 0: return mk(v, 0.0);
        case 1: return mk(0.0, v);
        case 2: return mk(-v, 0.0);
        default: return mk(0.0, -v);
    }
}
// Re(omega^{-e} z) (proj/src/contraction.cpp:40-47)
SKC_HD double re_rot_conj(unsigned e, double2 z) {
    switch (e & 3u) {
        case 0: return z.x;
        case 1: return z.y;
        case 2: return -z.x;
        default: return -z.y;
    }
}

// Padded shared-memory index: one pad slot per 16 complex values keeps the
// radix-16 passes free of bank conflicts for 16-byte elements.
SKC_HD int pad16(int x) { return x + (x >> 4); }
SKC_HD int padded_len(int N) { return N + (N >> 4) + 1; }

SKC_HD int ilog2(unsigned x) {
    int r = 0;
    while ((1u << r) < x) ++r;
    return r;
}

// Constant roots w_M^{-q} for M in {2,4,8,16}, q < M/2 (forward sign).
SKC_HD double2 const_root(int M, int q) {
    // cos/sin of 2*pi*q/16 for q = 0..7
    const double c16[8] = {1.0,
                           0.92387953251128675613,
                           0.70710678118654752440,
                           0.38268343236508977173,
                           0.0,
                           -0.38268343236508977173,
                           -0.70710678118654752440,
                           -0.92387953251128675613};
    const double s16[8] = {0.0,
                           0.38268343236508977173,
                           0.70710678118654752440,
                           0.92387953251128675613,
                           1.0,
                           0.92387953251128675613,
                           0.70710678118654752440,
                           0.38268343236508977173};
    int idx = q * (16 / M);
    return mk(c16[idx], -s16[idx]);
}

// d * w_M^{-q} (forward sign; CONJ: d * w_M^{+q}) for a compile-time root: the multiples of
// pi/4 need no multiplication (or one scaling by sqrt(1/2)). Used by the passes whose stage
// twiddle is 1 (element spacing 1: the last DIF pass, the first DIT pass), where every
// butterfly factor is such a constant.
SKC_HD double2 cmul_root(double2 d, int M, int q, bool cj) {
    const int idx = q * (16 / M);  // angle 2 pi idx / 16, idx in [0, 8)
    const double c = 0.70710678118654752440;
    switch (idx) {
        case 0: return d;
        case 4: return cj ? mk(-d.y, d.x) : mk(d.y, -d.x);
        case 2: return cj ? mk(c * (d.x - d.y), c * (d.x + d.y)) : mk(c * (d.x + d.y), c * (d.y - d.x));
        case 6: return cj ? mk(-c * (d.x + d.y), c * (d.x - d.y)) : mk(c * (d.y - d.x), -c * (d.x + d.y));
        default: {
            const double2 r = const_root(M, q);
            return cmul(d, cj ? conj(r) : r);
        }
    }
}

// Pass plan for a local length N = 2^p: the first pass takes radix 2^(p mod 4)
// (if nonzero), every later pass radix 16. Pass j starts at half-size h_j.
struct PassPlan {
    int npass;
    int logr[8];  // log2 radix of pass j
    int h[8];     // half-size at the start of pass j
};

SKC_HD PassPlan make_plan(int N) {
    PassPlan pl;
    pl.npass = 0;
    int p = ilog2(static_cast<unsigned>(N));
    int h = N >> 1;
    int first = p % 4;
    if (first == 0 && p > 0) first = 4;
    int rem = p;
    int lr = first;
    while (rem > 0) {
        pl.logr[pl.npass] = lr;
        pl.h[pl.npass] = h;
        pl.npass++;
        h >>= lr;
        rem -= lr;
        lr = 4;
    }
    return pl;
}

// One forward (DIF) pass on item w of array x (length N, padded smem layout).
// tw: table of w_b^k = (cos 2 pi k / b, sin 2 pi k / b), k in [0, b).
// logb_over: log2(b) used to index tw for stage twiddles w_{2hs}^{-pos}.
// Core of a DIF pass item: loads the item's R inputs, runs the butterflies and leaves the
// outputs in v (output q belongs at position base + q * g).
// UNIT: the pass has element spacing 1 (2h = R), so pos = 0 and every stage twiddle is 1.
template <int LOGR, bool UNIT = false>
SKC_HD void dif_item_core(double2* x, int w, int h, const double2* tw, int logb, double2 (&v)[1 << LOGR], int& base,
                          int& g) {
    constexpr int R = 1 << LOGR;
    g = (2 * h) >> LOGR;  // element spacing
    const int block = w / g;
    const int pos = w - block * g;
    base = block * 2 * h + pos;
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = x[pad16(base + q * g)];
    if (UNIT) {
#pragma unroll
        for (int s = 0; s < LOGR; ++s) {
            const int Hq = R >> (s + 1);
#pragma unroll
            for (int q = 0; q < R; ++q) {
                if (q & Hq) continue;
                const double2 a = v[q], c = v[q + Hq];
                v[q] = cadd(a, c);
                v[q + Hq] = cmul_root(csub(a, c), R >> s, q & (Hq - 1), false);
            }
        }
        return;
    }
    // stage twiddles: w_{2h}^{-pos} from the table, then w_{2hs}^{-pos} = (w_{2h}^{-pos})^(2^s)
    // by repeated squaring (one table read per item instead of LOGR)
    double2 W = conj(tw[static_cast<unsigned>(pos) << (logb - ilog2(static_cast<unsigned>(2 * h)))]);
#pragma unroll
    for (int s = 0; s < LOGR; ++s) {
        const int Hq = R >> (s + 1);
        if (s > 0) W = cmul(W, W);
#pragma unroll
        for (int q = 0; q < R; ++q) {
            if (q & Hq) continue;
            const int qp = q & (Hq - 1);  // position inside the (R>>s)-block, lower half
            double2 a = v[q], c = v[q + Hq];
            v[q] = cadd(a, c);
            double2 d = csub(a, c);
            double2 tw2 = (qp == 0) ? W : cmul(W, const_root(R >> s, qp));
            v[q + Hq] = cmul(d, tw2);
        }
    }
}
template <int LOGR, bool UNIT = false>
SKC_HD void dif_pass_item(double2* x, int w, int h, const double2* tw, int logb) {
    constexpr int R = 1 << LOGR;
    double2 v[R];
    int base, g;
    dif_item_core<LOGR, UNIT>(x, w, h, tw, logb, v, base, g);
#pragma unroll
    for (int q = 0; q < R; ++q) x[pad16(base + q * g)] = v[q];
}

// Mirror inverse (DIT) pass: unscaled, conjugate twiddles.
template <int LOGR, bool UNIT = false>
SKC_HD void dit_pass_item(double2* x, int w, int h, const double2* tw, int logb) {
    constexpr int R = 1 << LOGR;
    const int g = (2 * h) >> LOGR;
    const int block = w / g;
    const int pos = w - block * g;
    const int base = block * 2 * h + pos;
    double2 v[R];
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = x[pad16(base + q * g)];
    if (UNIT) {  // element spacing 1: every stage twiddle is 1
#pragma unroll
        for (int s = LOGR - 1; s >= 0; --s) {
            const int Hq = R >> (s + 1);
#pragma unroll
            for (int q = 0; q < R; ++q) {
                if (q & Hq) continue;
                const double2 a = v[q];
                const double2 c = cmul_root(v[q + Hq], R >> s, q & (Hq - 1), true);
                v[q] = cadd(a, c);
                v[q + Hq] = csub(a, c);
            }
        }
    } else {
        // stage twiddles w_{2hs}^{pos}, s = 0..LOGR-1, by repeated squaring of w_{2h}^{pos}
        double2 Ws[LOGR];
        Ws[0] = tw[static_cast<unsigned>(pos) << (logb - ilog2(static_cast<unsigned>(2 * h)))];
#pragma unroll
        for (int s = 1; s < LOGR; ++s) Ws[s] = cmul(Ws[s - 1], Ws[s - 1]);
#pragma unroll
        for (int s = LOGR - 1; s >= 0; --s) {
            const int Hq = R >> (s + 1);
            const double2 W = Ws[s];
#pragma unroll
            for (int q = 0; q < R; ++q) {
                if (q & Hq) continue;
                const int qp = q & (Hq - 1);
                double2 tw2 = (qp == 0) ? W : cmul(W, conj(const_root(R >> s, qp)));
                double2 a = v[q];
                double2 c = cmul(v[q + Hq], tw2);
                v[q] = cadd(a, c);
                v[q + Hq] = csub(a, c);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) x[pad16(base + q * g)] = v[q];
}

SKC_HD void dif_pass_dispatch(int logr, double2* x, int w, int h, const double2* tw, int logb) {
    const bool unit = (2 * h) == (1 << logr);  // element spacing 1
    switch (logr) {
        case 1: unit ? dif_pass_item<1, true>(x, w, h, tw, logb) : dif_pass_item<1>(x, w, h, tw, logb); break;
        case 2: unit ? dif_pass_item<2, true>(x, w, h, tw, logb) : dif_pass_item<2>(x, w, h, tw, logb); break;
        case 3: unit ? dif_pass_item<3, true>(x, w, h, tw, logb) : dif_pass_item<3>(x, w, h, tw, logb); break;
        default: unit ? dif_pass_item<4, true>(x, w, h, tw, logb) : dif_pass_item<4>(x, w, h, tw, logb); break;
    }
}
SKC_HD void dit_pass_dispatch(int logr, double2* x, int w, int h, const double2* tw, int logb) {
    const bool unit = (2 * h) == (1 << logr);
    switch (logr) {
        case 1: unit ? dit_pass_item<1, true>(x, w, h, tw, logb) : dit_pass_item<1>(x, w, h, tw, logb); break;
        case 2: unit ? dit_pass_item<2, true>(x, w, h, tw, logb) : dit_pass_item<2>(x, w, h, tw, logb); break;
        case 3: unit ? dit_pass_item<3, true>(x, w, h, tw, logb) : dit_pass_item<3>(x, w, h, tw, logb); break;
        default: unit ? dit_pass_item<4, true>(x, w, h, tw, logb) : dit_pass_item<4>(x, w, h, tw, logb); break;
    }
}

// ---- compile-time pass plans ----------------------------------------------------------
// Max radix 2^LR per pass (LR = 4: radix-16, the make_plan decomposition; LR = 3:
// radix-8, fewer registers per thread at the cost of one more pass over shared memory).
constexpr int plan_first(int logN, int LR = 4) { return (logN % LR) ? (logN % LR) : LR; }
constexpr int plan_npass(int logN, int LR = 4) { return logN == 0 ? 0 : 1 + (logN - plan_first(logN, LR)) / LR; }
constexpr int plan_logr(int logN, int p, int LR = 4) { return p == 0 ? plan_first(logN, LR) : LR; }
constexpr int plan_h(int logN, int p, int LR = 4) {
    int h = (1 << logN) >> 1;
    for (int q = 0; q < p; ++q) h >>= plan_logr(logN, q, LR);
    return h;
}

#ifdef __CUDACC__
// Forward DIF over `na` back-to-back padded arrays of length 2^LOGN. `twl` is the local
// table w_N^k (k < N): stage twiddles are twl[pos << (LOGN - log2(2 hs))], contiguous,
// so a CTA's whole twiddle working set is N*16 bytes.
template <int LOGN, int LR, int P, int NP = plan_npass(LOGN, LR)>
struct DifPasses {
    __device__ __forceinline__ static void run(double2* sm, int na, const double2* twl) {
        constexpr int R_ = plan_logr(LOGN, P, LR);
        constexpr int H = plan_h(LOGN, P, LR);
        constexpr int items = (1 << LOGN) >> R_;
        constexpr int stride = (1 << LOGN) + ((1 << LOGN) >> 4) + 1;
        for (int w = threadIdx.x; w < na * items; w += blockDim.x) {
            const int a = w / items;
            dif_pass_item<R_, 2 * H == (1 << R_)>(sm + a * stride, w - a * items, H, twl, LOGN);
        }
        __syncthreads();
        DifPasses<LOGN, LR, P + 1, NP>::run(sm, na, twl);
    }
};
template <int LOGN, int LR, int NP>
struct DifPasses<LOGN, LR, NP, NP> {
    __device__ __forceinline__ static void run(double2*, int, const double2*) {}
};
// Mirror inverse (DIT, unscaled), passes in reverse order.
template <int LOGN, int LR, int P>
struct DitPasses {
    __device__ __forceinline__ static void run(double2* sm, int na, const double2* twl) {
        constexpr int R_ = plan_logr(LOGN, P, LR);
        constexpr int H = plan_h(LOGN, P, LR);
        constexpr int items = (1 << LOGN) >> R_;
        constexpr int stride = (1 << LOGN) + ((1 << LOGN) >> 4) + 1;
        for (int w = threadIdx.x; w < na * items; w += blockDim.x) {
            const int a = w / items;
            dit_pass_item<R_, 2 * H == (1 << R_)>(sm + a * stride, w - a * items, H, twl, LOGN);
        }
        __syncthreads();
        DitPasses<LOGN, LR, P - 1>::run(sm, na, twl);
    }
};
template <int LOGN, int LR>
struct DitPasses<LOGN, LR, -1> {
    __device__ __forceinline__ static void run(double2*, int, const double2*) {}
};
template <int LOGN, int LR = 4>
__device__ __forceinline__ void dif_local(double2* sm, int na, const double2* twl) {
    DifPasses<LOGN, LR, 0>::run(sm, na, twl);
}
// DIF of one padded array whose last pass hands every output (local position j, value)
// to epi instead of storing it, so a pointwise epilogue (e.g. the moment cube-accumulate)
// needs no extra pass over shared memory; epi owns A[pad16(j)] (each j is visited once).
// The caller synchronises afterwards.
template <int LOGN, int LR, typename Epi>
__device__ __forceinline__ void dif_local_epilogue(double2* A, const double2* twl, Epi epi) {
    constexpr int NP = plan_npass(LOGN, LR);
    DifPasses<LOGN, LR, 0, NP - 1>::run(A, 1, twl);
    constexpr int R_ = plan_logr(LOGN, NP - 1, LR);
    constexpr int H = plan_h(LOGN, NP - 1, LR);
    constexpr int items = (1 << LOGN) >> R_;
    for (int w = threadIdx.x; w < items; w += blockDim.x) {
        double2 v[1 << R_];
        int base, g;
        dif_item_core<R_, 2 * H == (1 << R_)>(A, w, H, twl, LOGN, v, base, g);
#pragma unroll
        for (int q = 0; q < (1 << R_); ++q) epi(base + q * g, v[q]);
    }
}
template <int LOGN, int LR = 4>
__device__ __forceinline__ void dit_local(double2* sm, int na, const double2* twl) {
    DitPasses<LOGN, LR, plan_npass(LOGN, LR) - 1>::run(sm, na, twl);
}
#endif

// Bit reversal of j over `bits` bits: local spectrum slot j holds frequency
// f = r + S * bitrev(j).
SKC_HD unsigned bitrev(unsigned j, int bits) {
    unsigned r = 0;
    for (int i = 0; i < bits; ++i) {
        r = (r << 1) | (j & 1u);
        j >>= 1;
    }
    return r;
}

}  // namespace skc
