// K1: dense tensor-sketch build on sm_100a.
//
// Replaces the reference hot loops
//   symmetric  proj/src/sketch.cpp:315-345 — sorted triples i<=j<=k, weight kappa 1/3/6,
//              bucket (h_i+h_j+h_k) mod b, sign root4(e_i+e_j+e_k);
//   asymmetric proj/src/sketch.cpp:173-193 — all (i,j,k), bucket (h1_i+h2_j+h3_k) mod b,
//              sign xi1 xi2 xi3.
//
// Layout of the work. The B x b complex sketch set (5.2 MB at config 1) does not fit one
// SM's shared memory and each tensor entry lands in B random buckets. The default
// kernel (k_build_cls) cuts the slot space into classes: a window is one (replicate,
// parity, bucket residue) class, and for every row (i, j) the entries that land in it are
// one contiguous run of a per-window class list of the k indices, so each (entry,
// replicate) pair is evaluated exactly once. One persistent 1024-thread CTA per SM holds
// one window; rows are handed out dynamically from per-window counters and CTAs migrate
// between windows, so the SMs finish together and all windows sweep the rows in the same
// order (their gathers of the same rows hit L2). The older contiguous-slot-range kernel
// (k_build_flat: every CTA evaluates every entry against the 1-2 replicates its range
// overlaps) remains for small asymmetric builds and for shapes outside the class-list
// limits (b > 2^22, or n beyond the packed list words).
//
// Accumulation is exact 64-bit fixed point: q = round(kappa*T*2^F) is split into two
// 32-bit limbs added with native ATOMS.ADD (shared fp64 atomics are CAS loops on
// sm_100a); the carry out of the low limb is taken from the returned old value, so the
// sum is exact mod 2^64 under any interleaving and the build is bit-deterministic.
// F = min(61 - ceil(log2(sum kappa|T|)), 50 - ceil(log2(max kappa|T|))) from a
// deterministic pre-pass bounds every bucket sum by 2^62 and every single |q| by 2^50.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include "skc_host.hpp"
#include "skc_internal.hpp"

namespace skc {

namespace {
// Launch with programmatic stream serialization when pdl is set: the kernel may begin
// before its predecessor finishes and must griddepcontrol.wait before reading its output.
template <typename... KA, typename... Args>
void pdl_launch(void (*kern)(KA...), unsigned grid, unsigned block, size_t smem, cudaStream_t st, bool pdl,
                Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KA>(args)...);
}
inline unsigned cdiv(long long a, long long b) { return static_cast<unsigned>((a + b - 1) / b); }

template <int NT>
__device__ double block_sum_b(double v, double* red) {
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
    return t;
}
}  // namespace

// Block reduction of the pre-pass statistics into partials segment k at [k * grid + blk]:
// 0 the kappa|T| sum (fixed shuffle/block order), 1 its maximum, 2 the sum of squares
// (fixed order), 3 the smallest nonzero kappa|T|. 2 and 3 feed the main pass's resolution
// check (cta_scale_exp).
template <int NT>
__device__ void prepass_block_stats(double sum, double mx, double sq, double mn, double* red, double* partials) {
    constexpr int W = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double s = block_sum_b<NT>(sum, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
    const double q = block_sum_b<NT>(sq, red);
    if (threadIdx.x == 0) partials[2 * gridDim.x + blockIdx.x] = q;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    __syncthreads();
    if (lane == 0) {
        red[warp] = mx;
        red[W + warp] = mn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0, l = INFINITY;
        for (int w = 0; w < W; ++w) {
            m = fmax(m, red[w]);
            l = fmin(l, red[W + w]);
        }
        partials[gridDim.x + blockIdx.x] = m;
        partials[3 * gridDim.x + blockIdx.x] = l;
    }
}

// ---- pre-pass ---------------------------------------------------------------------
// One warp per row segment T[i][j][k0:n]. Every mode computes the row's L1 mass
// sum kappa|T| in a fixed order, the block max of kappa|T| and the non-finite flag; the
// per-block partials (L1 at [blk], max at [gridDim + blk]) give the global exponent.
//   kQuant: writes the packed fixed-point stream qbuf[rowoff + e] = round(kappa T 2^Frow),
//           Frow = 61 - ceil(log2 rowL1), for the contiguous-window kernels (they rescale
//           q >> (Frow - F));
//   kRaw:   writes the row segment as is (packed, element type TT) for the class-list
//           kernel when T is not device-resident (pinned host memory read over the bus);
//   kNone:  no writes (the class-list kernel gathers from a device-resident T).
enum PrepassMode { kQuant = 0, kRaw = 1, kNone = 2 };
template <typename TT, bool SYM, int NTQ, int MODE>
__global__ void __launch_bounds__(NTQ) k_build_quantize(const TT* __restrict__ T, int n,
                                                       const std::uint32_t* __restrict__ rowtab,
                                                       const long long* __restrict__ rowoff, int nrows,
                                                       long long* __restrict__ qbuf, short* __restrict__ rowF,
                                                       double* __restrict__ partials, int* __restrict__ nonfinite,
                                                       bool vec16, double band_lo, double band_hi) {
    constexpr int W = NTQ / 32;
    extern __shared__ double stage[];  // W warps x n: each element of T is read exactly once
    __shared__ double red[2 * W];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* st = stage + (size_t)warp * n;
    double blk = 0.0, bmax = 0.0, bsq = 0.0, bmn = INFINITY;
    bool bad = false;
    TT* xraw = reinterpret_cast<TT*>(qbuf);  // kRaw output
    // 16-byte path: the first 128-vector block of the warp's next row is loaded before the
    // current row's reduction and stores, so each warp keeps a row's reads in flight.
    // EPV elements per 16-byte vector (2 fp64, 4 fp32).
    constexpr int EPV = 16 / static_cast<int>(sizeof(TT));
    const bool v16 = vec16;
    auto row_geom = [&](int r, const double2*& tp, int& npair, int& off) {
        const std::uint32_t ijr = rowtab[r];
        const int ir = static_cast<int>(ijr >> 16), jr = static_cast<int>(ijr & 0xFFFFu);
        const int k0r = SYM ? jr : 0;
        const size_t e0 = ((size_t)ir * n + jr) * n + k0r;
        const size_t ea = e0 & ~static_cast<size_t>(EPV - 1);
        npair = static_cast<int>((e0 + (n - k0r) - ea + EPV - 1) / EPV);
        tp = reinterpret_cast<const double2*>(T + ea);
        off = static_cast<int>(e0 - ea);
    };
    // element h of a 16-byte vector
    auto elem = [](const double2& v, int h) -> double {
        if constexpr (sizeof(TT) == 8) {
            return h ? v.y : v.x;
        } else {
            const unsigned long long w = static_cast<unsigned long long>(__double_as_longlong((h >> 1) ? v.y : v.x));
            return static_cast<double>(__int_as_float(static_cast<int>((h & 1) ? (w >> 32) : (w & 0xFFFFFFFFull))));
        }
    };
    auto load_first = [&](int r, double2 (&v)[4]) {
        const double2* tp;
        int npair, off;
        row_geom(r, tp, npair, off);
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = (lane + 32 * u < npair) ? tp[lane + 32 * u] : make_double2(0.0, 0.0);
    };
    double2 pv[4];
    if (v16 && blockIdx.x * W + warp < nrows) load_first(blockIdx.x * W + warp, pv);
    for (int row = blockIdx.x * W + warp; row < nrows; row += gridDim.x * W) {
        const std::uint32_t ij = rowtab[row];
        const int i = static_cast<int>(ij >> 16), j = static_cast<int>(ij & 0xFFFFu);
        const TT* rp = T + ((size_t)i * n + j) * n;
        const int k0 = SYM ? j : 0;
        const double kdiag = SYM ? ((i == j) ? 1.0 : 3.0) : 1.0;
        const double koff = SYM ? ((i == j) ? 3.0 : 6.0) : 1.0;
        double a0 = 0.0;
        TT* xo = MODE == kRaw ? xraw + rowoff[row] : nullptr;
        if (v16) {
            // 16-byte loads from a 16-byte aligned base covering the row segment: T may be
            // pinned host memory read in place over PCIe, where wider requests carry less
            // header overhead per byte. 4 vector loads in flight per lane.
            const double2* tp;
            int npair, off;  // off < EPV: leading elements to skip
            row_geom(row, tp, npair, off);
            double2 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = pv[u];
            if (row + gridDim.x * W < nrows) load_first(row + gridDim.x * W, pv);
            for (int pb = lane; pb < npair; pb += 128) {
                if (pb != lane) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) v[u] = (pb + 32 * u < npair) ? tp[pb + 32 * u] : make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int q = EPV * (pb + 32 * u) - off;  // row-relative index of element 0 of v[u]
#pragma unroll
                    for (int h = 0; h < EPV; ++h) {
                        const int kk = q + h;
                        if (kk >= 0 && kk < n - k0) {
                            const double x = elem(v[u], h);
                            const int k = k0 + kk;
                            const double kv0 = ((SYM && k == j) ? kdiag : koff) * x;
                            // magnitude band [band_lo, band_hi) of kappa |T| (HDR builds; else all)
                            const bool keep = fabs(kv0) >= band_lo && fabs(kv0) < band_hi;
                            const double kv = keep ? kv0 : 0.0;
                            if (MODE == kQuant) st[kk] = kv;
                            if (MODE == kRaw) xo[kk] = keep ? static_cast<TT>(x) : TT(0);
                            a0 += fabs(kv);
                            bmax = fmax(bmax, fabs(kv));
                            bsq += kv * kv;
                            if (kv != 0.0) bmn = fmin(bmn, fabs(kv));
                            bad |= !isfinite(x);
                        }
                    }
                }
            }
        } else {
            // 4 loads in flight per lane
            for (int kb = k0 + lane; kb < n; kb += 128) {
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = (kb + 32 * u < n) ? static_cast<double>(rp[kb + 32 * u]) : 0.0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = kb + 32 * u;
                    if (k < n) {
                        const double kv0 = ((SYM && k == j) ? kdiag : koff) * v[u];
                        const bool keep = fabs(kv0) >= band_lo && fabs(kv0) < band_hi;
                        const double kv = keep ? kv0 : 0.0;
                        if (MODE == kQuant) st[k - k0] = kv;
                        if (MODE == kRaw) xo[k - k0] = keep ? rp[k] : TT(0);
                        a0 += fabs(kv);
                        bmax = fmax(bmax, fabs(kv));
                        bsq += kv * kv;
                        if (kv != 0.0) bmn = fmin(bmn, fabs(kv));
                        bad |= !isfinite(v[u]);
                    }
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a0 = __shfl_sync(0xffffffffu, a0, 0);  // lane 0's sum for every lane (xor trees may differ in the last bit)
        if (MODE == kQuant) {
            int F = 0;
            if (a0 > 0.0 && isfinite(a0)) {
                int ex;
                frexp(a0, &ex);
                F = 61 - ex;
                F = F > 1000 ? 1000 : (F < -1000 ? -1000 : F);
            }
            const double scale = ldexp(1.0, F);
            __syncwarp();
            long long* qo = qbuf + rowoff[row] - k0;
            for (int k = k0 + lane; k < n; k += 32) {
                const double kv = st[k - k0];
                qo[k] = isfinite(kv) ? __double2ll_rn(kv * scale) : 0ll;
            }
            __syncwarp();
            if (lane == 0) rowF[row] = static_cast<short>(F);
        }
        blk += (lane == 0) ? a0 : 0.0;
    }
    if (bad) atomicOr(nonfinite, 1);
    prepass_block_stats<NTQ>(blk, bmax, bsq, bmn, red, partials);
}

// Lean sums-only pre-pass (default for device-resident class-list builds). Each lane
// keeps its own kappa-weighted L1 sum, maximum, sum of squares and smallest nonzero magnitude
// across all the rows its warp visits; one block reduction at the end. kappa is constant
// along a row except on its k = j entry (6 / 3 off the diagonal rows, 3 / 1 on them), so a
// lane accumulates the row unweighted -- per entry one widening, one add, one fma, a float
// (or double) max and an integer min of the magnitude bits -- and applies the row's kappa
// once; lane 0 peels the k = j entry. (The previous form weighted every entry: 34 warp
// instructions per 32 entries, issue- and conversion-bound at 2.6 TB/s on fp32 input.)
// Rows are dealt to warps in grid-strided pairs with all of a pair's loads issued before any
// is consumed. Non-finite entries surface as a non-finite lane sum.
__device__ __forceinline__ float mag(float x) { return fabsf(x); }
__device__ __forceinline__ double mag(double x) { return fabs(x); }
__device__ __forceinline__ float max_of(float a, float b) { return fmaxf(a, b); }  // NaN: the sum carries it
__device__ __forceinline__ double max_of(double a, double b) { return fmax(a, b); }
template <typename TT>
struct MagBits;  // magnitude bits as an unsigned integer: orders like the magnitude itself
template <>
struct MagBits<float> {
    using U = std::uint32_t;
    static __device__ __forceinline__ U of(float a) { return __float_as_uint(a); }
    static __device__ __forceinline__ double back(U u) { return static_cast<double>(__uint_as_float(u)); }
};
template <>
struct MagBits<double> {  // the high word (exponent and 20 mantissa bits): rounds the minimum down
    using U = std::uint32_t;
    static __device__ __forceinline__ U of(double a) { return static_cast<U>(__double2hiint(a)); }
    static __device__ __forceinline__ double back(U u) { return __hiloint2double(static_cast<int>(u), 0); }
};
#ifndef SKC_SUMS_MINB  // experiment builds only
#define SKC_SUMS_MINB 5
#endif
#ifndef SKC_SUMS_U32
#define SKC_SUMS_U32 4
#endif
template <typename TT, bool SYM>
__global__ void __launch_bounds__(256, SKC_SUMS_MINB) k_build_sums_lean(const TT* __restrict__ T, int n,
                                                            const std::uint32_t* __restrict__ rowtab, int nrows,
                                                            double* __restrict__ partials, int* __restrict__ nonfinite) {
    constexpr int W = 8, U = sizeof(TT) == 4 ? SKC_SUMS_U32 : 4;  // (8 fp32 loads per lane and row measured no faster: sums_ab.sh)
    using MB = MagBits<TT>;
    using UB = typename MB::U;
    __shared__ double red[2 * W];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double acc = 0.0, mx = 0.0, sq = 0.0;
    float mn = INFINITY;  // smallest nonzero kappa|T|, rounded down (a register less than fp64)
    const int stride = gridDim.x * W;
    const int row0 = blockIdx.x * W + warp;
    std::uint32_t nij[2];  // the next pair's (i, j) words, fetched one step ahead
#pragma unroll
    for (int h = 0; h < 2; ++h) nij[h] = row0 + h * stride < nrows ? __ldg(rowtab + row0 + h * stride) : 0u;
    // one entry of weight w into the lane totals
    auto fold = [&](double w, double d, TT m, UB nz) {
        acc = fma(w, d, acc);
        mx = fmax(mx, w * static_cast<double>(m));
        if (nz != ~UB(0)) mn = fminf(mn, __double2float_rd(w * MB::back(nz + 1)));
    };
    for (int row = row0; row < nrows; row += 2 * stride) {
        const TT* rp[2];
        int k0[2];
        bool dg[2];
        TT v[2][U];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int rw = row + h * stride;
            const bool ok = rw < nrows;
            const std::uint32_t ij = nij[h];
            nij[h] = rw + 2 * stride < nrows ? __ldg(rowtab + rw + 2 * stride) : 0u;
            const int i = static_cast<int>(ij >> 16), j = static_cast<int>(ij & 0xFFFFu);
            k0[h] = ok ? (SYM ? j : 0) : n;
            rp[h] = T + ((size_t)i * n + j) * n;
            dg[h] = i == j;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = k0[h] + lane + 32 * u;
                v[h][u] = k < n ? __ldg(rp[h] + k) : TT(0);
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            // kappa: 6 (3 if i = j) off the k = j entry, 3 (1 if i = j) on it
            const double wr = !SYM ? 1.0 : (dg[h] ? 3.0 : 6.0);
            if (SYM && lane == 0 && k0[h] < n) {  // the k = j entry, peeled
                const TT a0 = mag(v[h][0]);
                const double d0 = static_cast<double>(a0), w0 = dg[h] ? 1.0 : 3.0;
                fold(w0, d0, a0, MB::of(a0) - 1);
                sq = fma(w0 * d0, w0 * d0, sq);
                v[h][0] = TT(0);
            }
            double rs = 0.0, rq = 0.0;  // the row's unweighted sum and sum of squares (this lane)
            TT rm = TT(0);               // ... maximum
            UB rn = ~UB(0);              // ... smallest nonzero magnitude bits - 1 (zero wraps to the top)
            for (int kb = k0[h] + lane;; kb += 32 * U) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const TT a = mag(v[h][u]);
                    const double d = static_cast<double>(a);
                    rs += d;
                    rq = fma(d, d, rq);
                    rm = max_of(rm, a);
                    const UB nb = MB::of(a) - 1;
                    rn = nb < rn ? nb : rn;
                }
                if (kb + 32 * U >= n) break;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = kb + 32 * U + 32 * u;
                    v[h][u] = k < n ? __ldg(rp[h] + k) : TT(0);
                }
            }
            fold(wr, rs, rm, rn);
            sq = fma(wr * wr, rq, sq);
            // (a NaN entry drops out of the maximum: rs carries it into acc)
        }
    }
    // (no flag write: the main pass derives it from these partials)
    prepass_block_stats<256>(acc, mx, sq, static_cast<double>(mn), red, partials);
}

// Exponent histogram of kappa|T| over the build's rows (HDR builds only): one warp per row,
// shared-memory bins, one global add per non-empty bin and block.
template <typename TT, bool SYM>
__global__ void __launch_bounds__(256) k_build_exp_hist(const TT* __restrict__ T, int n,
                                                         const std::uint32_t* __restrict__ rowtab, int nrows,
                                                         unsigned long long* __restrict__ hist) {
    __shared__ unsigned int sh[kExpBins];
    for (int x = threadIdx.x; x < kExpBins; x += 256) sh[x] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int row = blockIdx.x * 8 + warp; row < nrows; row += gridDim.x * 8) {
        const std::uint32_t ij = rowtab[row];
        const int i = static_cast<int>(ij >> 16), j = static_cast<int>(ij & 0xFFFFu);
        const int k0 = SYM ? j : 0;
        const TT* rp = T + ((size_t)i * n + j) * n;
        for (int k = k0 + lane; k < n; k += 32) {
            const double w = !SYM ? 1.0 : (k == k0 ? (i == j ? 1.0 : 3.0) : (i == j ? 3.0 : 6.0));
            const double a = w * fabs(static_cast<double>(rp[k]));
            if (a > 0.0 && isfinite(a)) atomicAdd(&sh[ilogb(a) + kExpBias], 1u);
        }
    }
    __syncthreads();
    for (int x = threadIdx.x; x < kExpBins; x += 256)
        if (sh[x]) atomicAdd(hist + x, static_cast<unsigned long long>(sh[x]));
}
void launch_build_exp_hist(cudaStream_t st, const void* T, const BuildPlan& p, unsigned long long* hist) {
    const unsigned grid = 4u * 148u;
    if (p.sym) {
        if (p.dtype == 0) k_build_exp_hist<double, true><<<grid, 256, 0, st>>>((const double*)T, p.n, p.rowtab, p.nrows, hist);
        else k_build_exp_hist<float, true><<<grid, 256, 0, st>>>((const float*)T, p.n, p.rowtab, p.nrows, hist);
    } else {
        if (p.dtype == 0) k_build_exp_hist<double, false><<<grid, 256, 0, st>>>((const double*)T, p.n, p.rowtab, p.nrows, hist);
        else k_build_exp_hist<float, false><<<grid, 256, 0, st>>>((const float*)T, p.n, p.rowtab, p.nrows, hist);
    }
    count_launch();
}

// Default: kPrepassBlocks x 256 threads over all SMs (HBM-bound). Pipelined zero-copy
// builds use p.prepass_blocks x 1024-thread blocks on a few SMs (PCIe-bound), leaving the
// rest to the concurrent main pass of the previous chunk.
void launch_build_prepass(cudaStream_t st, const void* T, const BuildPlan& p) {
    if (p.reset_nonfinite && p.xsrc_mode != 1) cudaMemsetAsync(p.nonfinite, 0, sizeof(int), st);
    const bool wide = p.prepass_threads == 1024;
    const int blocks = p.prepass_blocks;
    const bool vec16 = (reinterpret_cast<std::uintptr_t>(T) & 15) == 0;
    const int mode = p.xsrc_mode == 0 ? kQuant : p.xsrc_mode == 1 ? kNone : kRaw;
#define QUANT_M(TT, SY, MD)                                                                                           \
    {                                                                                                                 \
        if (wide) {                                                                                                   \
            const size_t smem = MD == kQuant ? sizeof(double) * 32 * (size_t)p.n : 0;                                 \
            if (smem > 48 * 1024)                                                                                     \
                cudaFuncSetAttribute(k_build_quantize<TT, SY, 1024, MD>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                     (int)smem);                                                                      \
            k_build_quantize<TT, SY, 1024, MD><<<blocks, 1024, smem, st>>>((const TT*)T, p.n, p.rowtab, p.rowoff,    \
                                                                           p.nrows, p.qbuf, p.rowF,                  \
                                                                           p.prepass_partials, p.nonfinite, vec16,   \
                                                                           p.band_lo, p.band_hi);                    \
        } else {                                                                                                      \
            const size_t smem = MD == kQuant ? sizeof(double) * 8 * (size_t)p.n : 0;                                  \
            if (smem > 48 * 1024)                                                                                     \
                cudaFuncSetAttribute(k_build_quantize<TT, SY, 256, MD>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                     (int)smem);                                                                      \
            k_build_quantize<TT, SY, 256, MD><<<blocks, 256, smem, st>>>((const TT*)T, p.n, p.rowtab, p.rowoff,      \
                                                                         p.nrows, p.qbuf, p.rowF,                    \
                                                                         p.prepass_partials, p.nonfinite, vec16,     \
                                                                         p.band_lo, p.band_hi);                      \
        }                                                                                                             \
    }
#define QUANT(TT, SY)                                                                                 \
    {                                                                                                 \
        if (mode == kQuant) QUANT_M(TT, SY, kQuant)                                                   \
        else if (mode == kRaw) QUANT_M(TT, SY, kRaw)                                                  \
        else k_build_sums_lean<TT, SY><<<blocks, 256, 0, st>>>(                                       \
            (const TT*)T, p.n, p.rowtab, p.nrows, p.prepass_partials, p.nonfinite);                   \
    }
    if (p.sym) {
        if (p.dtype == 0) QUANT(double, true)
        else QUANT(float, true)
    } else {
        if (p.dtype == 0) QUANT(double, false)
        else QUANT(float, false)
    }
#undef QUANT
#undef QUANT_M
    count_launch();
}

// ---- main pass -----------------------------------------------------------------------

// Exact 64-bit add of (ql, qh) into the limb pair (lo at addr_lo, hi at addr_hi). The
// limbs live in separate planes (4-byte stride: random slots spread over all 32 banks).
// The carry out of the low limb comes from the returned old value (add.cc / addc).
// Branch-free: callers redirect out-of-window contributions to a per-lane trash pair,
// which costs two extra ATOMS but no divergence or reconvergence barriers.
__device__ __forceinline__ void add64(std::uint32_t addr_lo, std::uint32_t addr_hi, std::uint32_t ql,
                                      std::uint32_t qh) {
    asm volatile(
        "{\n\t.reg .u32 old, c;\n\t"
        "atom.shared.add.u32 old, [%0], %2;\n\t"
        "add.cc.u32 c, old, %2;\n\t"
        "addc.u32 c, %3, 0;\n\t"
        "red.shared.add.u32 [%1], c;\n\t}" ::"r"(addr_lo),
        "r"(addr_hi), "r"(ql), "r"(qh));
}

// Same add with the limb addresses formed inside the asm block from an opaque window
// base (the compiler otherwise re-derives the shared-window base per use).
__device__ __forceinline__ void add64_idx(std::uint32_t idx, std::uint32_t sbase, std::uint32_t hioff, std::uint32_t ql,
                                          std::uint32_t qh) {
    asm volatile(
        "{\n\t.reg .u32 al, ah, old, c;\n\t"
        "mad.lo.u32 al, %0, 4, %1;\n\t"
        "add.u32 ah, al, %2;\n\t"
        "atom.shared.add.u32 old, [al], %3;\n\t"
        "add.cc.u32 c, old, %3;\n\t"
        "addc.u32 c, %4, 0;\n\t"
        "red.shared.add.u32 [ah], c;\n\t}" ::"r"(idx),
        "r"(sbase), "r"(hioff), "r"(ql), "r"(qh));
}
__device__ __forceinline__ std::uint32_t lds_u32(std::uint32_t addr) {
    std::uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
template <typename T>
__device__ __forceinline__ T pin(T v) {  // opaque copy: keeps a kernel constant in a register
    asm volatile("mov.b32 %0, %0;" : "+r"(v));
    return v;
}

struct BuildArgs {
    int n, B, G, nrows;
    std::uint32_t bmask;
    long long total_slots;
    int slots_per_cta;
    const std::uint32_t* rowtab;
    const long long* rowoff;
    const short* rowF;
    const long long* qbuf;
    const std::uint32_t* packed;
    const double* partials;        // pre-pass partials: nseg x [np L1 sums, np maxima of kappa|T|]
    int np, nseg;                  // nseg > 1: all-gathered partials of nseg ranks
    const void* xsrc;              // class-list kernel: T itself (xmode 1) or its packed row copy (xmode 2)
    int xmode;
    int* scale_out;                // global exponent F, written by CTA 0 for the finalize
    int* nonfinite_out;            // lean pre-pass: CTA 0 stores the flag from the partials (no memset)
    int* ovf_out;                  // one-limb windows: set when a limb overflowed (zero on entry)
    int sym_even_F;                // symmetric one-limb / two-limb class-list builds: F even (see cta_scale_exp)
    int* next_row;                 // G row (or tile) counters, then G per-window CTA counts (class-list
                                   // kernel); zero on entry, the finalize re-zeroes all 2G
    int lock_rows;                 // class-list kernel: a CTA leaves a window this many rows ahead of a
                                   // window with fewer CTAs (windows sweep the rows together: L2 reuse)
    int qbits;                     // max |q| exponent: 50 (two limbs) or 22 (one limb, fp32 input)
    long long total_entries;       // entries of the whole build (all ranks): the mean of kappa|T|
    double entries_per_slot;       // total_entries / slots per replicate (bucket thickness)
    double rho_max;                // resolution bound (see cta_scale_exp)

    unsigned long long* acc;       // total_slots exact accumulators (zero on entry; the finalize re-zeroes them)
};

// Global exponent F = min(61 - ceil(log2(sum kappa|T|)), 50 - ceil(log2(max kappa|T|))):
// every bucket sum of q stays below 2^62 and every single |q| below 2^50, so the class-list
// kernel can round kappa*T*2^F to an integer with one fma against 1.5*2^52. Every CTA
// sums the pre-pass partials in the same fixed order (lane-strided, then a fixed shuffle
// tree read from lane 0), so all CTAs agree; CTA 0 publishes F.
__shared__ int s_hdr;  // set by cta_scale_exp: this build adds nothing (resolution check)
__device__ int cta_scale_exp(const BuildArgs& a) {
    __shared__ int sF;
    if (threadIdx.x < 32) {
        double acc = 0.0, mx = 0.0, sq = 0.0, mn = INFINITY;
        for (int x = threadIdx.x; x < a.np * a.nseg; x += 32) {
            const int sg = x / a.np, id = x - sg * a.np;
            const double* seg = a.partials + 4ll * sg * a.np;
            acc += seg[id];
            mx = fmax(mx, seg[a.np + id]);
            sq += seg[2 * a.np + id];
            mn = fmin(mn, seg[3 * a.np + id]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            acc += __shfl_xor_sync(0xffffffffu, acc, o);
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            sq += __shfl_xor_sync(0xffffffffu, sq, o);
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        }
        if (threadIdx.x == 0) {
            int F = 0;
            if (acc > 0.0 && isfinite(acc)) {
                int ex, exm;
                frexp(acc, &ex);  // acc <= 2^ex
                frexp(mx, &exm);  // mx <= 2^exm
                F = min(61 - ex, a.qbits - exm);
                F = F > 1000 ? 1000 : (F < -1000 ? -1000 : F);
                // symmetric class-list builds take F even: the exponent field of the scale
                // kappa * 2^F = 1.5 * 2^(F+2) is then odd, so kappa 6 -> 3 (i = j rows) is one
                // XOR of its low bit (the row word carries that bit)
                if (a.sym_even_F) F &= ~1;
            }
            // Resolution check: the fixed-point step 2^-F relative to the mean kappa|T| bounds
            // the relative error of every bucket (it is ~0.6 x that ratio, the sqrt(count)
            // of the rounding walk cancelling against the bucket's own growth). Above rho_max
            // (one limb: 2^-17, two limbs: 2^-33, i.e. entries spanning more magnitudes than
            // one fixed-point scale keeps to the contract) nothing is added: the host redoes
            // the build with two limbs (flag 1) or in magnitude bands (flag 2).
            // Buckets are sums of ~c = entries_per_slot terms (Poisson). When they are thin
            // (c < 8: a bucket may be one or two entries) or the mass sits in few entries
            // (N_eff = (sum)^2 / sum of squares; c N_eff / N < 4: some buckets likely hold
            // none of the heavy entries; light tails have N_eff / N ~ 2/pi), a bucket may
            // hold only small entries, so the step is measured against the smallest nonzero
            // one; otherwise against the mean.
            int hdr = 0;
            if (acc > 0.0 && isfinite(acc) && isfinite(sq)) {
                const double N = static_cast<double>(a.total_entries);
                const double neff = (acc / sqrt(sq)) * (acc / sqrt(sq));
                const bool thin = a.entries_per_slot < 8.0 || a.entries_per_slot * neff < 4.0 * N;
                const double rho = thin ? ldexp(1.0, -F) / mn : ldexp(N, -F) / acc;
                if (rho > a.rho_max) hdr = a.qbits < 50 ? 1 : 2;
            }
            sF = F;
            s_hdr = hdr;
            if (blockIdx.x == 0) {
                *a.scale_out = F;
                // a non-finite entry makes its lane's (non-negative) sum, hence acc, non-finite
                if (a.nonfinite_out) *a.nonfinite_out = isfinite(acc) ? 0 : 1;
                if (hdr) atomicOr(a.ovf_out, hdr);
            }
        }
    }
    __syncthreads();
    return sF;
}

// Flat-chunk variant of the persistent build (default). A warp grabs a chunk of up to 16
// consecutive rows, stages their metadata (relative start, k offset, exponent shift,
// row-pair hash words) in its slice of shared memory, and then streams the chunk's
// entries as one contiguous run of qbuf: lane e handles entries e, e+32, ... regardless
// of row boundaries, advancing its row cursor when it crosses one. Short rows no longer
// leave lanes idle, the 128-entry loads are independent of row bookkeeping (the next
// block is prefetched before the current one is processed), and the per-row work is a
// few shared-memory reads per crossing lane.
constexpr int kFlatRows = 16;
__host__ __device__ constexpr int flat_meta_words(int rmax) { return (kFlatRows + 1) + 2 * kFlatRows + rmax * kFlatRows; }

template <bool SYM, int RMAX>
__global__ void __launch_bounds__(1024, 1) k_build_flat(BuildArgs a) {
    constexpr int NT = 1024;
    extern __shared__ std::uint32_t sacc[];
    __shared__ int s_next_g;
    const int spc = a.slots_per_cta;
    const int plane = spc + 32;
    std::uint32_t* ptab = sacc + 2 * plane;
    std::uint32_t* pij_tab = ptab + RMAX * a.n;
    const int n = a.n, nrows = a.nrows;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // per-warp chunk metadata
    std::uint32_t* wm = pij_tab + RMAX * 2 * n + warp * flat_meta_words(RMAX);
    std::uint32_t* m_start = wm;                       // kFlatRows + 1 (relative starts, last = E)
    int* m_kofs = reinterpret_cast<int*>(wm + kFlatRows + 1);
    int* m_d = m_kofs + kFlatRows;
    std::uint32_t* m_pij = reinterpret_cast<std::uint32_t*>(m_d + kFlatRows);  // RMAX x kFlatRows
    const long long spr = SYM ? 2ll * (a.bmask + 1) : static_cast<long long>(a.bmask + 1);
    const int prow = SYM ? n : 3 * n;
    const int F = cta_scale_exp(a);
    if (s_hdr) return;
    std::uint32_t sbase = static_cast<std::uint32_t>(__cvta_generic_to_shared(sacc));
    asm volatile("mov.b32 %0, %0;" : "+r"(sbase));  // keep in a register (no per-use S2UR/ULEA)
    const std::uint32_t hioff = 4u * static_cast<std::uint32_t>(plane);
    const std::uint32_t trash_idx = static_cast<std::uint32_t>(spc + lane);

    int g = static_cast<int>((static_cast<long long>(blockIdx.x) * a.G) / gridDim.x);
    while (g >= 0) {
        const long long slot_lo = (long long)g * spc;
        const long long slot_hi = min(slot_lo + spc, a.total_slots);
        const int nslots = static_cast<int>(slot_hi - slot_lo);
        const int m_lo = static_cast<int>(slot_lo / spr);
        const int R = static_cast<int>((slot_hi - 1) / spr) - m_lo + 1;
        for (int s = threadIdx.x; s < 2 * plane; s += NT) sacc[s] = 0u;
        // SYM: tables in the doubled form 2h | e<<30 (from h | e<<30): the sum q of a row-pair
        // word and a k word carries 2*(bucket sum) in bits 1.. and the exponent mod 4 in bits
        // 30-31, so the slot 2*bucket + parity is one funnel of q and q >> 30 and the sign is
        // q's sign bit (b <= 2^27 keeps the bucket carries below bit 30).
        auto cv = [](std::uint32_t x) { return SYM ? (((x & 0x3FFFFFFFu) << 1) | (x & 0xC0000000u)) : x; };
        for (int x = threadIdx.x; x < RMAX * n; x += NT) {
            const int r = x / n, k = x - r * n;
            const std::uint32_t* pm = a.packed + (size_t)(m_lo + min(r, R - 1)) * prow;
            ptab[x] = cv(pm[(SYM ? 0 : 2 * n) + k]);
            pij_tab[r * 2 * n + k] = cv(pm[k]);
            pij_tab[r * 2 * n + n + k] = cv(pm[(SYM ? 0 : n) + k]);
        }
        __syncthreads();
        std::uint32_t base[RMAX];
#pragma unroll
        for (int r = 0; r < RMAX; ++r) base[r] = pin(static_cast<std::uint32_t>((long long)(m_lo + r) * spr - slot_lo));
        const std::uint32_t nsl = pin(static_cast<std::uint32_t>(nslots));
        const std::uint32_t bmask = pin(a.bmask);
        const std::uint32_t m1 = pin(2u * a.bmask);  // SYM: 2*bucket mask in the doubled form
        const std::uint32_t n4 = pin(4u * static_cast<std::uint32_t>(n));
        const std::uint32_t ptab_s = pin(sbase + 4u * static_cast<std::uint32_t>(2 * plane));

        int c0 = 0;
        if (lane == 0) c0 = atomicAdd(a.next_row + g, kFlatRows);
        c0 = __shfl_sync(0xffffffffu, c0, 0);
        while (c0 < nrows) {
            int cn = 0;  // next grab, one chunk ahead
            if (lane == 0) cn = atomicAdd(a.next_row + g, kFlatRows);
            const int nr = min(kFlatRows, nrows - c0);
            // stage the chunk's row metadata (lane l -> row c0 + l)
            long long off = 0;
            int len = 0;
            if (lane < nr) {
                const int row = c0 + lane;
                const std::uint32_t ij = __ldg(a.rowtab + row);
                off = __ldg(a.rowoff + row);
                const int i = static_cast<int>(ij >> 16), j = static_cast<int>(ij & 0xFFFFu);
                len = SYM ? n - j : n;
                m_d[lane] = static_cast<int>(__ldg(a.rowF + row)) - F;
#pragma unroll
                for (int r = 0; r < RMAX; ++r) m_pij[r * kFlatRows + lane] = pij_tab[r * 2 * n + i] + pij_tab[r * 2 * n + n + j];
                m_kofs[lane] = SYM ? j : 0;  // relative start subtracted below
            }
            const long long off0 = __shfl_sync(0xffffffffu, off, 0);
            const int rel = static_cast<int>(off - off0);
            const int E = __shfl_sync(0xffffffffu, rel + len, nr - 1);
            if (lane < nr) {
                m_start[lane] = static_cast<std::uint32_t>(rel);
                m_kofs[lane] -= rel;
            }
            if (lane == 0) m_start[nr] = static_cast<std::uint32_t>(E);
            __syncwarp();
            const long long* qch = a.qbuf + off0;
            int t = 0;
            int cur_end = static_cast<int>(m_start[1]);
            int kofs = m_kofs[0], d = m_d[0];
            std::uint32_t pij[RMAX];
#pragma unroll
            for (int r = 0; r < RMAX; ++r) pij[r] = m_pij[r * kFlatRows];
            auto load4 = [&](long long (&q)[4], int eb) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = eb + lane + 32 * u;
                    q[u] = (e < E) ? __ldg(qch + e) : 0ll;
                }
            };
            auto process = [&](const long long (&qc)[4], int eb) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = eb + lane + 32 * u;
                    if (eb + 32 * u >= E) break;  // warp-uniform
                    if (e < E) {
                        while (e >= cur_end) {  // crossed into the next row of the chunk
                            ++t;
                            cur_end = static_cast<int>(m_start[t + 1]);
                            kofs = m_kofs[t];
                            d = m_d[t];
#pragma unroll
                            for (int r = 0; r < RMAX; ++r) pij[r] = m_pij[r * kFlatRows + t];
                        }
                        const std::uint32_t kaddr = ptab_s + 4u * static_cast<std::uint32_t>(e + kofs);
                        // zero entries add nothing (sketch.cpp:337 skips them)
                        const unsigned long long qq = static_cast<unsigned long long>(qc[u] >> d);
                        const unsigned long long nq = 0ull - qq;
                        const std::uint32_t ql = static_cast<std::uint32_t>(qq), qh = static_cast<std::uint32_t>(qq >> 32);
                        const std::uint32_t nql = static_cast<std::uint32_t>(nq), nqh = static_cast<std::uint32_t>(nq >> 32);
#pragma unroll
                        for (int r = 0; r < RMAX; ++r) {
                            if (r < R) {  // CTA-uniform
                                const std::uint32_t p = pij[r] + lds_u32(kaddr + static_cast<std::uint32_t>(r) * n4);
                                const std::uint32_t s = base[r] + (SYM ? ((p & m1) | ((p >> 30) & ~m1)) : (p & bmask));
                                const bool neg = static_cast<int>(p) < 0;
                                add64_idx(s < nsl ? s : trash_idx, sbase, hioff, neg ? nql : ql, neg ? nqh : qh);
                            }
                        }
                    }
                }
            };
            // ping-pong over 128-entry blocks: the next block's loads are in flight while the
            // current one is processed, with no register copies between iterations
            long long qa[4], qb[4];
            load4(qa, 0);
            for (int eb = 0; eb < E; eb += 256) {
                load4(qb, eb + 128);
                process(qa, eb);
                if (eb + 128 >= E) break;
                load4(qa, eb + 256);
                process(qb, eb + 128);
            }
            __syncwarp();  // metadata slice reused by the next chunk
            c0 = __shfl_sync(0xffffffffu, cn, 0);
        }
        __syncthreads();
        unsigned long long* out = a.acc + slot_lo;
        for (int s = threadIdx.x; s < nslots; s += NT) {
            const unsigned long long v = (static_cast<unsigned long long>(sacc[plane + s]) << 32) | sacc[s];
            if (v) atomicAdd(out + s, v);
        }
        if (threadIdx.x == 0) {
            int best = -1, left = 0;
            for (int tt = 0; tt < a.G; ++tt) {
                const int l = nrows - *((volatile int*)(a.next_row + tt));
                if (l > left) {
                    left = l;
                    best = tt;
                }
            }
            s_next_g = best;
        }
        __syncthreads();
        g = s_next_g;
    }
}

// ---- class-list build (symmetric sets, default when a window fits) -----------------------
// A window ("type") is one (replicate m, parity P, bucket residue r mod 2^TB) class of the
// slot space: the b/2^TB buckets t = r (mod 2^TB) of replicate m in the real (P = 0) or
// imaginary (P = 1) plane. The destination of entry (i, j, k) under replicate m has
// bucket (c_ij + h_k) mod b and parity (e_ij + e_k) & 1, so for a fixed row (i, j) the
// entries that land in the window are exactly those k in one class of the k index set:
// e_k & 1 = P ^ (e_ij & 1) and h_k = r - c_ij (mod 2^TB). Each window keeps its k indices
// grouped by class (stable, so ascending k within a class) with a suffix table giving the
// first list position with k >= j. The rows' in-window entries are then one contiguous run
// of the class list, gathered from the row in qbuf: every (entry, replicate) pair is
// evaluated once, in the one window it lands in (no out-of-window evaluations, no trash
// atomics), against ~2.2 evaluations per pair for the contiguous-slot windows above.
constexpr int kClsRows = 32;  // rows per grab
__host__ __device__ constexpr int cls_sfx_words(int C, int n) { return (C * (n + 1) + 1) / 2; }

// Window limbs (plus 32 dummy slots per plane), class list, hash words, suffix tables and
// the 32 warps' row tables (one int4 per row of a grab).
size_t cls_smem_bytes(std::uint32_t b, int tbits, int n, bool sym, bool one_limb) {
    const int C = (sym ? 2 : 1) << tbits;
    const size_t W = static_cast<size_t>(b) >> tbits;
    const size_t fixed = (sizeof(std::uint32_t) * ((one_limb ? 1 : 2) * (W + 32) + 3 * (size_t)n + cls_sfx_words(C, n)) + 15) &
                         ~size_t(15);
    return fixed + 32 * kClsRows * sizeof(int4);
}

// One-limb add for fp32 inputs (|q| < 2^22): the window keeps each slot's exact sum
// mod 2^32 biased by 2^30, u = v + 2^30, so the centred value v starts at 0 and a pass's
// partial sums (~sqrt(count) * |q|) stay far from the edges. The flush adds
// v = int32(u - 2^30) to the slot's 64-bit accumulator, so without an overflow the
// accumulator holds the exact sum, as with two limbs.
constexpr std::uint32_t kLimbBias = 0x40000000u;
// Overflow guard, conservative and branch-free, one OR per add: bit 31 of the returned old
// limb u is set exactly when the state before the add was outside [-2^30, 2^30) (as long
// as |v| < 2^30 + 2^31, which holds below). An add that starts inside ends inside
// (-2^30 - 2^22, 2^30 + 2^22), which the flush decodes exactly, so no add can overflow
// without an earlier or the same add being flagged. The window pass reports the flag and
// the host then discards the build (the finalize adds nothing) and repeats it exactly with
// two limbs. Ordinary data (|v| needs ~2^8 same-signed full-scale adds to one slot) never
// takes that path.
__device__ __forceinline__ void add32_at(std::uint32_t addr, std::int32_t q, std::uint32_t& ovf) {
    std::uint32_t old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(static_cast<std::uint32_t>(q)));
    ovf |= old;
}
__device__ __forceinline__ void add32_idx(std::uint32_t idx, std::uint32_t sbase, std::int32_t q, std::uint32_t& ovf) {
    add32_at(sbase + 4u * idx, q, ovf);
}
// Exact 64-bit add at a precomputed low-limb byte address (the high limb is hioff above).
__device__ __forceinline__ void add64_at(std::uint32_t al, std::uint32_t hioff, std::uint32_t ql, std::uint32_t qh) {
    asm volatile(
        "{\n\t.reg .u32 ah, old, c;\n\t"
        "add.u32 ah, %0, %1;\n\t"
        "atom.shared.add.u32 old, [%0], %2;\n\t"
        "add.cc.u32 c, old, %2;\n\t"
        "addc.u32 c, %3, 0;\n\t"
        "red.shared.add.u32 [ah], c;\n\t}" ::"r"(al),
        "r"(hioff), "r"(ql), "r"(qh));
}
// Entries are read straight from T (device-resident: xmode 1) or from the pre-pass's packed
// row copy (xmode 2), element type XT, and rounded to q = round(kappa * T * 2^F) by one fma
// against 1.5 * 2^52 (fp64 input, two limbs, |q| < 2^50) or 1.5 * 2^23 (fp32 input, one
// limb, |q| < 2^22): exact single rounding either way. The scale's sign bit carries the
// complex4 sign, so the add needs no separate negation. kappa is per row (6 or 3 sym; 1
// asym); the k = j entry of a sym row, whose kappa is 3 (or 1), gets its correction
// (-3 or -2) added once per row when the row's metadata is built.
//
// A warp grabs 32 rows of its window and walks their in-window runs as one flat entry
// range: a warp-level scan of the run lengths gives each row's end, lane e takes entries
// e, e+32, ... across row boundaries with a row cursor over one int4 of row metadata per row
// (end entry, list position - entry index, source offset, row word), reads the list word,
// gathers the entry from the row and adds it. Four 32-entry blocks are fetched before
// their adds, ping-pong (measured against a per-row 32-entry slab table: config 1
// 0.449 vs 0.501 ms, config 2 2.60 vs 2.69 ms, bit-identical; microbench/walk_ab.sh).
template <bool SYM, int TB, typename XT, bool L1>
__global__ void __launch_bounds__(1024, 1) k_build_cls(BuildArgs a) {
    constexpr int NT = 1024, C = (SYM ? 2 : 1) << TB, NPL = L1 ? 1 : 2;  // limb planes in the window
    constexpr std::uint32_t tmask = (1u << TB) - 1u;
    extern __shared__ __align__(16) std::uint32_t sm[];
    __shared__ int s_next_g;
    __shared__ int s_leave;  // set by warp 0: the CTA moves to window s_next_g after the grabs in flight
    __shared__ int s_cend[C];
    __shared__ int s_wcnt[C * 32];  // per-(class, 32-k segment) counts, then their scan
    const int n = a.n, nrows = a.nrows;
    int* const ncta = a.next_row + a.G;  // CTAs working on each window
    const int W = static_cast<int>((a.bmask + 1u) >> TB);  // slots per window
    const int WP = W + 32;  // plane stride: slots W + lane are inactive lanes' private dummy slots
    // n list words grouped by class: h_k | k << KS | e_k << 30 (KS = log2 b + 2 clears the
    // 3-term bucket sum; the host checks that k fits below bit 30)
    std::uint32_t* lst = sm + NPL * WP;
    std::uint32_t* pw = reinterpret_cast<std::uint32_t*>(lst + n);  // sym n: h | e << 30; asym 2n: modes 1, 2
    unsigned short* sfx = reinterpret_cast<unsigned short*>(pw + 2 * n);  // C x (n + 1)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // per-warp row table of the current grab: one int4 per row
    int4* meta = reinterpret_cast<int4*>(
                     sm + ((static_cast<size_t>(NPL * WP + 3 * n + cls_sfx_words(C, n)) + 3) & ~static_cast<size_t>(3))) +
                 warp * kClsRows;
    // F comes from the pre-pass partials: read after griddepcontrol.wait, which the first
    // window's prologue (zeroing, hash words, class lists) runs ahead of (PDL launch)
    int F = 0;
    bool have_F = false;
    std::uint32_t sbase = static_cast<std::uint32_t>(__cvta_generic_to_shared(sm));
    asm volatile("mov.b32 %0, %0;" : "+r"(sbase));
    const std::uint32_t hioff = pin(4u * static_cast<std::uint32_t>(WP));
    const std::uint32_t bmask = pin(a.bmask);
    const std::uint32_t lst_s = pin(sbase + 4u * NPL * static_cast<std::uint32_t>(WP));
    const int KS = __popc(a.bmask) + 2;
    const std::uint32_t kmask = pin((1u << (30 - KS)) - 1u);
    const std::uint32_t wmask = pin(~(kmask << KS));
    const XT* __restrict__ xsrc = static_cast<const XT*>(a.xsrc);
    // high word of kappa * 2^F (fp64; the float bits for one limb): sym kappa 6 = 1.5 * 2^2
    // (kappa 3 is one exponent step less); asym kappa 1
    constexpr int EXS = L1 ? 23 : 20;          // exponent field position
    constexpr int EXB = L1 ? 127 : 1023;       // exponent bias
    std::uint32_t sc_hi0 = 0;
    std::uint32_t ovf = 0;  // one-limb overflow indicator (sign bit)
    constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
    constexpr long long kMagicBits = 0x4338000000000000ll;
    // exact round(x * sc): |x * sc| < 2^50, one rounding in the fma
    auto to_fixed = [](double x, std::uint32_t schi) -> long long {
        const double sc = __hiloint2double(static_cast<int>(schi), 0);
        return __double_as_longlong(fma(x, sc, kMagic)) - kMagicBits;
    };
    // exact round(x * sc) in fp32: |x * sc| < 2^22, one rounding in the fma against 1.5 * 2^23
    auto to_fixed32 = [](float x, std::uint32_t scbits) -> std::int32_t {
        return __float_as_int(__fmaf_rn(x, __int_as_float(static_cast<int>(scbits)), 12582912.0f)) - 0x4B400000;
    };

    int g = static_cast<int>((static_cast<long long>(blockIdx.x) * a.G) / gridDim.x);
    if (threadIdx.x == 0) atomicAdd(ncta + g, 1);
    while (g >= 0) {
        const int m = g / C, P = SYM ? (g >> TB) & 1 : 0, r = g & static_cast<int>(tmask);
        if (threadIdx.x == 0) s_leave = 0;
        for (int s = threadIdx.x; s < NPL * WP; s += NT) sm[s] = L1 ? kLimbBias : 0u;
        unsigned long long* gacc = a.acc + static_cast<long long>(g) * W;  // this window's accumulators
        // asym packed words are h | neg << 31 for modes 1..3 (B x 3 x n): the list holds
        // mode 3, the row pair word is mode 1 (i) + mode 2 (j); bit 31 of a sum is the sign
        for (int k = threadIdx.x; k < (SYM ? n : 2 * n); k += NT) pw[k] = a.packed[(size_t)m * (SYM ? n : 3 * n) + k];
        __syncthreads();
        const std::uint32_t* lw_src = SYM ? pw : a.packed + (size_t)m * 3 * n + 2 * n;
        auto cls_of = [&](std::uint32_t w) {
            return static_cast<int>(SYM ? ((((w >> 30) & 1u) << TB) | (w & tmask)) : (w & tmask));
        };
        const std::uint32_t lt = (1u << lane) - 1u;
        if (n <= 32 * 32) {
            // stable class grouping of k and the suffix tables, one 32-k segment per warp:
            // per-segment class counts, a class-major scan over the segments, then each
            // warp places its k's (3 barriers instead of one warp walking all of n)
            const int k = warp * 32 + lane;
            const std::uint32_t w = k < n ? lw_src[k] : 0u;
            const int c = k < n ? cls_of(w) : -1;
            std::uint32_t mk[C];
#pragma unroll
            for (int cc = 0; cc < C; ++cc) mk[cc] = __ballot_sync(0xffffffffu, c == cc);
#pragma unroll
            for (int cc = 0; cc < C; ++cc)
                if (lane == cc) s_wcnt[cc * 32 + warp] = __popc(mk[cc]);
            __syncthreads();
            if (warp == 0) {  // exclusive scan over (class, segment) in class-major order
                int base = 0;
                for (int cc = 0; cc < C; ++cc) {
                    const int v = s_wcnt[cc * 32 + lane];
                    int incl = v;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int t = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += t;
                    }
                    s_wcnt[cc * 32 + lane] = base + incl - v;
                    base += __shfl_sync(0xffffffffu, incl, 31);
                    if (lane == 0) s_cend[cc] = base;
                }
            }
            __syncthreads();
            if (warp * 32 < n) {
#pragma unroll
                for (int cc = 0; cc < C; ++cc) {
                    const int pos = s_wcnt[cc * 32 + warp] + __popc(mk[cc] & lt);
                    if (k < n) sfx[cc * (n + 1) + k] = static_cast<unsigned short>(pos);
                    if (c == cc) lst[pos] = w | (static_cast<std::uint32_t>(k) << KS);
                }
            }
            if (threadIdx.x < C) sfx[threadIdx.x * (n + 1) + n] = static_cast<unsigned short>(s_cend[threadIdx.x]);
        } else if (warp == 0) {  // large n: one warp walks the k segments in order
            int cnt = 0;  // lane c: size of class c
            for (int base = 0; base < n; base += 32) {
                const int k = base + lane;
                const int c = k < n ? cls_of(lw_src[k]) : -1;
#pragma unroll
                for (int cc = 0; cc < C; ++cc) {
                    const int pc = __popc(__ballot_sync(0xffffffffu, c == cc));
                    if (lane == cc) cnt += pc;
                }
            }
            int run = cnt;  // exclusive scan over the class lanes
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, run, o);
                if (lane >= o) run += v;
            }
            run -= cnt;  // lane c: start of class c
            if (lane < C) s_cend[lane] = run + cnt;
            for (int base = 0; base < n; base += 32) {
                const int k = base + lane;
                const std::uint32_t w = k < n ? lw_src[k] : 0u;
                const int c = k < n ? cls_of(w) : -1;
#pragma unroll
                for (int cc = 0; cc < C; ++cc) {
                    const std::uint32_t mk = __ballot_sync(0xffffffffu, c == cc);
                    const int rc = __shfl_sync(0xffffffffu, run, cc);
                    const int pos = rc + __popc(mk & lt);
                    if (k < n) sfx[cc * (n + 1) + k] = static_cast<unsigned short>(pos);
                    if (c == cc) lst[pos] = w | (static_cast<std::uint32_t>(k) << KS);
                    if (lane == cc) run += __popc(mk);
                }
            }
            if (lane < C) sfx[lane * (n + 1) + n] = static_cast<unsigned short>(run);
        }
        __syncthreads();
        if (!have_F) {  // block-uniform
            asm volatile("griddepcontrol.wait;" ::: "memory");
            F = cta_scale_exp(a);
            sc_hi0 = pin(SYM ? ((static_cast<std::uint32_t>(EXB + F + 2) << EXS) | (1u << (EXS - 1)))
                             : (static_cast<std::uint32_t>(EXB + F) << EXS));
            have_F = true;
            asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        }
        if (s_hdr) break;  // block-uniform: the build is redone (two limbs / bands)

        constexpr int R = kClsRows;
        int c0 = 0;
        if (lane == 0) c0 = atomicAdd(a.next_row + g, R);
        c0 = __shfl_sync(0xffffffffu, c0, 0);
        int grabs = 0;
        while (c0 < nrows) {
            // Lockstep: every 4th grab warp 0 compares this window's cursor with the others.
            // A window worked by more CTAs runs ahead; once it leads a window with fewer CTAs
            // by lock_rows, one CTA moves there (the counts swap, so the lead shrinks again).
            // All windows then stay within ~lock_rows of each other and every row is fetched
            // from HBM about once for all of them.
            if (warp == 0 && (++grabs & 3) == 0 && *((volatile int*)&s_leave) == 0) {
                const int mine = *((volatile int*)(a.next_row + g));
                const int cmine = *((volatile int*)(ncta + g));
                int best = INT_MAX, bt = -1;
                for (int tt = lane; tt < a.G; tt += 32) {
                    const int cur = *((volatile int*)(a.next_row + tt));
                    const int ct = *((volatile int*)(ncta + tt));
                    if (ct < cmine && mine - cur > a.lock_rows && cur < best) {
                        best = cur;
                        bt = tt;
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const int ob = __shfl_xor_sync(0xffffffffu, best, o), ot = __shfl_xor_sync(0xffffffffu, bt, o);
                    if (ob < best || (ob == best && ot > bt)) {
                        best = ob;
                        bt = ot;
                    }
                }
                if (bt >= 0 && mine < nrows) {
                    if (lane == 0) {
                        const int old = atomicSub(ncta + g, 1);
                        if (old > *((volatile int*)(ncta + bt))) {
                            atomicAdd(ncta + bt, 1);
                            s_next_g = bt;
                            __threadfence_block();
                            s_leave = 1;
                        } else {
                            atomicAdd(ncta + g, 1);  // another CTA of this window moved first
                        }
                    }
                }
            }
            int cn = INT_MAX;  // next grab, one grab ahead (none once the CTA is leaving)
            if (lane == 0 && *((volatile int*)&s_leave) == 0) cn = atomicAdd(a.next_row + g, R);
            const int nr = min(R, nrows - c0);
            long long off = 0;  // source element index of (i, j, 0)
            int cnt = 0, pos0 = 0;
            std::uint32_t pwd = 0;
            if (lane < nr) {
                const int row = c0 + lane;
                const std::uint32_t ij = __ldg(a.rowtab + row);
                const int i = static_cast<int>(ij >> 16);
                const int j = static_cast<int>(ij & 0xFFFFu);
                off = a.xmode == 1 ? (static_cast<long long>(i) * n + j) * n : __ldg(a.rowoff + row) - (SYM ? j : 0);
                const std::uint32_t pij = pw[i] + pw[(SYM ? 0 : n) + j];
                const int cl = SYM ? static_cast<int>(((((pij >> 30) & 1u) ^ static_cast<std::uint32_t>(P)) << TB) |
                                                      ((static_cast<std::uint32_t>(r) - pij) & tmask))
                                   : static_cast<int>((static_cast<std::uint32_t>(r) - pij) & tmask);
                pos0 = sfx[cl * (n + 1) + (SYM ? j : 0)];
                cnt = s_cend[cl] - pos0;
                const bool ii = SYM && i == j;
                // bucket sums < 3b <= 3 * 2^21 stay below bit 23; bit 23 marks i = j (kappa 3)
                pwd = pij + (ii ? (1u << 23) : 0u);
                if (SYM && cnt > 0) {
                    // k = j: kappa 3 (i < j) or 1 (i = j) where the row walk applies 6 or 3
                    const std::uint32_t lw0 = lst[pos0];
                    if (static_cast<int>((lw0 >> KS) & kmask) == j) {
                        const std::uint32_t p0 = pij + (lw0 & wmask);
                        // -3 * 2^F = -1.5 * 2^(F+1);  -2 * 2^F = -1.0 * 2^(F+1)
                        const std::uint32_t hi =
                            ((static_cast<std::uint32_t>(EXB + F + 1) << EXS) | (ii ? 0u : (1u << (EXS - 1)))) ^
                            0x80000000u ^ (p0 & 0x80000000u);
                        if (L1) {
                            add32_idx((p0 & bmask) >> TB, sbase, to_fixed32(static_cast<float>(xsrc[off + j]), hi),
                                      ovf);
                        } else {
                            const unsigned long long qd =
                                static_cast<unsigned long long>(to_fixed(static_cast<double>(xsrc[off + j]), hi));
                            add64_idx((p0 & bmask) >> TB, sbase, hioff, static_cast<std::uint32_t>(qd),
                                      static_cast<std::uint32_t>(qd >> 32));
                        }
                    }
                }
            }
            // flat walk: the grab's in-window runs are one contiguous entry range; lane e
            // takes entries e, e+32, ... across row boundaries with a row cursor over one
            // int4 per row (end entry, list position - entry index, source offset, row word)
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const long long off0 = __shfl_sync(0xffffffffu, off, 0);
            const int E = __shfl_sync(0xffffffffu, incl, 31);
            // .y: byte address of the row's list run, minus 4 x its first entry index
            if (lane < nr)
                meta[lane] = make_int4(incl, static_cast<int>(lst_s + 4u * static_cast<std::uint32_t>(pos0 - (incl - cnt))),
                                       static_cast<int>(off - off0), static_cast<int>(pwd));
            __syncwarp();
            const XT* qch = xsrc + off0;
            asm volatile("mov.b64 %0, %0;" : "+l"(qch));
            int t = 0;
            int4 cur = meta[0];
            auto fetch = [&](XT& x, std::uint32_t& pv, int e) {
                if (e >= cur.x) {  // crossed into a later row of the grab
                    cur = meta[++t];
                    while (e >= cur.x) cur = meta[++t];
                }
                const std::uint32_t lw = lds_u32(static_cast<std::uint32_t>(cur.y) + 4u * static_cast<std::uint32_t>(e));
                x = __ldg(qch + static_cast<std::uint32_t>(cur.z + static_cast<int>((lw >> KS) & kmask)));
                pv = static_cast<std::uint32_t>(cur.w) + (lw & wmask);
            };
            // lanes past the grab's end add 0 into their private dummy slot W + lane
            auto load4 = [&](XT (&x)[4], std::uint32_t (&pv)[4], bool (&ac)[4], int eb) {
                if (eb + 128 <= E) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        fetch(x[u], pv[u], eb + lane + 32 * u);
                        ac[u] = true;
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int e = eb + lane + 32 * u;
                        x[u] = XT(0);
                        pv[u] = 0u;
                        ac[u] = e < E;
                        if (ac[u]) fetch(x[u], pv[u], e);
                    }
                }
            };
            // byte address of the entry's low limb: window slot (p & bmask) >> TB
            auto slot_addr = [&](std::uint32_t pv) -> std::uint32_t {
                const std::uint32_t x = pv & (bmask & ~tmask);
                if constexpr (TB <= 2) return sbase + (x << (2 - TB));
                else return sbase + (x >> (TB - 2));
            };
            auto add_one = [&](XT x, std::uint32_t pv, std::uint32_t addr, bool act) {
                // kappa * 2^F with the complex4 sign (bit 31 of p) in its sign bit
                if (L1) {
                    // fp32 scale: the sign (bit 31) and the i = j halving (bit 23, the low
                    // exponent bit) in one LOP3
                    const std::uint32_t hi = sc_hi0 ^ (pv & (SYM ? 0x80800000u : 0x80000000u));
                    const std::int32_t q = to_fixed32(static_cast<float>(x), hi);
                    add32_at(addr, act ? q : 0, ovf);
                } else {
                    // fp64 scale high word: exponent low bit at 20 (F even: halving = XOR)
                    const std::uint32_t hi = (SYM ? sc_hi0 ^ ((pv >> 3) & (1u << 20)) : sc_hi0) ^ (pv & 0x80000000u);
                    const long long v = act ? to_fixed(static_cast<double>(x), hi) : 0ll;
                    add64_at(addr, hioff, static_cast<std::uint32_t>(v),
                             static_cast<std::uint32_t>(static_cast<unsigned long long>(v) >> 32));
                }
            };
            // full 128-entry blocks: no bound checks
            auto process_full = [&](const XT (&x)[4], const std::uint32_t (&pv)[4]) {
#pragma unroll
                for (int u = 0; u < 4; ++u) add_one(x[u], pv[u], slot_addr(pv[u]), true);
            };
            // the grab's last block: lanes past the end add 0 into their private dummy slot
            auto process_tail = [&](const XT (&x)[4], const std::uint32_t (&pv)[4], const bool (&ac)[4], int eb) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (eb + 32 * u >= E) break;  // warp-uniform
                    add_one(x[u], pv[u], ac[u] ? slot_addr(pv[u]) : sbase + 4u * static_cast<std::uint32_t>(W + lane), ac[u]);
                }
            };
            auto process = [&](const XT (&x)[4], const std::uint32_t (&pv)[4], const bool (&ac)[4], int eb) {
                if (eb + 128 <= E) process_full(x, pv);
                else process_tail(x, pv, ac, eb);
            };
            XT xa[4], xb[4];
            std::uint32_t pa[4], pb[4];
            bool aa[4], ab[4];
            load4(xa, pa, aa, 0);
            for (int eb = 0; eb < E; eb += 256) {
                load4(xb, pb, ab, eb + 128);
                process(xa, pa, aa, eb);
                if (eb + 128 >= E) break;
                load4(xa, pa, aa, eb + 256);
                process(xb, pb, ab, eb + 128);
            }
            __syncwarp();  // the row table is rewritten by the next grab
            c0 = __shfl_sync(0xffffffffu, cn, 0);
        }
        if (L1 && __any_sync(0xffffffffu, static_cast<std::int32_t>(ovf) < 0) && lane == 0) atomicOr(a.ovf_out, 1);
        __syncthreads();
        // flush into the window-major exact accumulators acc[g * W + s]: consecutive
        // threads add consecutive 8-byte words (coalesced RED.64; integer adds commute, so
        // the sketch stays bit-deterministic)
        for (int s = threadIdx.x; s < W; s += NT) {
            const unsigned long long v =
                L1 ? static_cast<unsigned long long>(static_cast<long long>(static_cast<std::int32_t>(sm[s] - kLimbBias)))
                   : (static_cast<unsigned long long>(sm[WP + s]) << 32) | sm[s];
            if (v) atomicAdd(gacc + s, v);
        }
        if (threadIdx.x == 0 && s_leave == 0) {  // rows exhausted: the window with the most rows left
            int best = -1, left = 0;
            for (int tt = 0; tt < a.G; ++tt) {
                const int l = nrows - *((volatile int*)(a.next_row + tt));
                if (l > left) {
                    left = l;
                    best = tt;
                }
            }
            atomicSub(ncta + g, 1);
            if (best >= 0) atomicAdd(ncta + best, 1);
            s_next_g = best;
        }
        __syncthreads();
        g = s_next_g;
        __syncthreads();  // s_leave is reset at the top of the next window
    }
    if (!have_F) {  // (a CTA that took no window) still orders itself after the pre-pass and
                    // derives F, so CTA 0 always publishes scale_exp / nonfinite for the finalize
        asm volatile("griddepcontrol.wait;" ::: "memory");
        F = cta_scale_exp(a);
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
}

template <bool SYM, int TB, typename XT, bool L1>
static void cls_launch2(cudaStream_t st, const BuildPlan& p, const BuildArgs& a, size_t smem) {
    cudaFuncSetAttribute(k_build_cls<SYM, TB, XT, L1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    pdl_launch(k_build_cls<SYM, TB, XT, L1>, p.P, 1024, smem, st, p.pdl, a);
}
// fp64 input: two limbs (|q| < 2^50, the fp64 tolerance); fp32 input: one biased limb with
// the rare carry (|q| < 2^22: resolution 2^-22 of max kappa|T|, against the 1e-4 fp32
// contract), half the window bytes, so half the bucket classes and half the gathers per entry
template <int TB>
static void cls_launch(cudaStream_t st, const BuildPlan& p, const BuildArgs& a) {
    const size_t smem = cls_smem_bytes(p.bmask + 1u, TB, p.n, p.sym, p.one_limb);
    if (p.sym) {
        if (p.dtype == 0) cls_launch2<true, TB, double, false>(st, p, a, smem);
        else if (p.one_limb) cls_launch2<true, TB, float, true>(st, p, a, smem);
        else cls_launch2<true, TB, float, false>(st, p, a, smem);
    } else {
        if (p.dtype == 0) cls_launch2<false, TB, double, false>(st, p, a, smem);
        else if (p.one_limb) cls_launch2<false, TB, float, true>(st, p, a, smem);
        else cls_launch2<false, TB, float, false>(st, p, a, smem);
    }
    count_launch();
}

template <bool SYM, int RMAX>
static void build_launch(cudaStream_t st, const BuildPlan& p, const BuildArgs& a) {
    const size_t smem = build_smem_bytes(p.slots_per_cta, RMAX, p.n);
    cudaFuncSetAttribute(k_build_flat<SYM, RMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_build_flat<SYM, RMAX><<<p.P, 1024, smem, st>>>(a);
    count_launch();
}

template <bool SYM>
static void build_dispatch(cudaStream_t st, const BuildPlan& p, const BuildArgs& a) {
    if (p.R <= 1)
        build_launch<SYM, 1>(st, p, a);
    else if (p.R <= 2)
        build_launch<SYM, 2>(st, p, a);
    else if (p.R <= 4)
        build_launch<SYM, 4>(st, p, a);
    else if (p.R <= 8)
        build_launch<SYM, 8>(st, p, a);
    else
        build_launch<SYM, 16>(st, p, a);
}

size_t build_smem_bytes(long long slots_per_cta, int R, int n) {
    const int rm = R <= 1 ? 1 : R <= 2 ? 2 : R <= 4 ? 4 : R <= 8 ? 8 : 16;
    return sizeof(std::uint32_t) *
           (2 * ((size_t)slots_per_cta + 32) + 3 * (size_t)rm * n + 32 * (size_t)flat_meta_words(rm));
}

void launch_build_main(cudaStream_t st, const void* T, const BuildPlan& p) {
    BuildArgs a;
    a.n = p.n;
    a.B = p.B;
    a.G = p.G;
    a.nrows = p.nrows;
    a.bmask = p.bmask;
    a.total_slots = p.total_slots;
    a.slots_per_cta = p.slots_per_cta;
    a.rowtab = p.rowtab;
    a.rowoff = p.rowoff;
    a.rowF = p.rowF;
    a.qbuf = p.qbuf;
    a.packed = p.packed;
    a.partials = p.prepass_partials;
    a.np = p.prepass_blocks;
    a.nseg = p.nseg;
    a.xsrc = p.xsrc_mode == 1 ? T : static_cast<const void*>(p.qbuf);
    a.xmode = p.xsrc_mode;
    a.scale_out = p.scale_exp;
    a.nonfinite_out = p.xsrc_mode == 1 ? p.nonfinite : nullptr;
    a.ovf_out = p.ovf;
    a.sym_even_F = (p.cls_bits >= 0 && p.sym) ? 1 : 0;
    a.next_row = p.next_row;
    a.lock_rows = p.lock_rows;
    a.acc = p.acc;
    a.qbits = (p.cls_bits >= 0 && p.one_limb) ? 22 : 50;
    a.total_entries = p.total_entries;
    a.entries_per_slot = static_cast<double>(p.total_entries) / (p.sym ? 2.0 * (p.bmask + 1.0) : (p.bmask + 1.0));
    a.rho_max = p.rho_max > 0 ? p.rho_max : (a.qbits < 50 ? 0x1p-17 : 0x1p-33);

    if (p.cls_bits >= 0) {
        switch (p.cls_bits) {
            case 0: cls_launch<0>(st, p, a); break;
            case 1: cls_launch<1>(st, p, a); break;
            case 2: cls_launch<2>(st, p, a); break;
            default: cls_launch<3>(st, p, a); break;
        }
    } else if (p.sym)
        build_dispatch<true>(st, p, a);
    else
        build_dispatch<false>(st, p, a);
}

// ---- finalize --------------------------------------------------------------------------
// data += acc * 2^-F, skipped when the pre-pass flagged a non-finite entry (the caller then
// reports the error with the set untouched). For the symmetric set the slot index is the
// double index into interleaved (re, im) data; the asymmetric set is real-only. The
// accumulators and the row counters are re-zeroed here for the next build (no memsets).
// The one-limb overflow flag lives kOvfOffset ints after the non-finite flag.
constexpr int kOvfOffset = 2;
__device__ __forceinline__ double pow2_neg(int F) {  // 2^-F exactly, |F| <= 1000
    return __longlong_as_double(static_cast<long long>(1023 - F) << 52);
}
// Data slot of accumulator index ai: the contiguous-window kernels keep data order; the
// class-list kernel keeps window-major order ai = g * W + t (tb >= 0: bucket-class bits),
// window g = (replicate m, [parity P,] residue r), bucket (t << tb) | r. The finalize walks
// ai (coalesced accumulator reads) and scatters into the interleaved data.
__device__ __forceinline__ long long data_index(long long ai, int tb, bool sym, std::uint32_t bmask) {
    if (tb < 0) return ai;
    const int logb = __popc(bmask);
    const int logW = logb - tb, logC = tb + (sym ? 1 : 0);
    const long long g = ai >> logW, t = ai & ((1ll << logW) - 1);
    const long long m = g >> logC, rem = g & ((1ll << logC) - 1);
    const long long r = rem & ((1ll << tb) - 1), P = sym ? rem >> tb : 0;
    const long long bucket = (t << tb) | r;
    return sym ? (m << (logb + 1)) + 2 * bucket + P : (m << logb) + bucket;
}
template <bool SYM>
__global__ void k_build_finalize(unsigned long long* __restrict__ acc, long long total_slots,
                                 const int* __restrict__ scale_exp, const int* __restrict__ nonfinite,
                                 double* __restrict__ data, int* __restrict__ counters, int ncounters, int tb,
                                 std::uint32_t bmask) {
    // 4 slots per thread (strided by the grid) so each thread has independent loads in flight
    const long long base = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // main pass complete (PDL launch)
    if (base < ncounters) counters[base] = 0;
    const bool bad = (nonfinite[0] | nonfinite[kOvfOffset]) != 0;
    const double sc = pow2_neg(*scale_exp);
    long long q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const long long s = base + u * stride;
        q[u] = s < total_slots ? static_cast<long long>(acc[s]) : 0ll;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const long long s = base + u * stride;
        if (q[u] == 0) continue;
        acc[s] = 0ull;
        if (bad) continue;
        const double v = static_cast<double>(q[u]) * sc;  // == ldexp(double(q), -F)
        const long long d = data_index(s, tb, SYM, bmask);
        if (SYM)
            data[d] += v;
        else
            data[2 * d] += v;
    }
}

// Symmetric class-list builds with one window per (replicate, parity) (tb = 0): the real
// and imaginary windows of replicate m are acc[2m*b + t] and acc[(2m+1)*b + t], so a
// thread takes both and updates the complex data[m*b + t] with one 16-byte load and
// store (the generic walk writes every other double). Same arithmetic as
// k_build_finalize: a zero accumulator leaves its component untouched.
__global__ void k_build_finalize_sym_pair(unsigned long long* __restrict__ acc, long long pairs, int logb,
                                          const int* __restrict__ scale_exp, const int* __restrict__ nonfinite,
                                          double2* __restrict__ data, int* __restrict__ counters, int ncounters) {
    const long long base = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // main pass complete (PDL launch)
    if (base < ncounters) counters[base] = 0;
    const bool bad = (nonfinite[0] | nonfinite[kOvfOffset]) != 0;
    const double sc = pow2_neg(*scale_exp);
    const long long bm = (1ll << logb) - 1;
    long long q0[2], q1[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const long long x = base + u * stride;
        const long long a0 = ((x >> logb) << (logb + 1)) | (x & bm);  // (2m) * b + t
        q0[u] = x < pairs ? static_cast<long long>(acc[a0]) : 0ll;
        q1[u] = x < pairs ? static_cast<long long>(acc[a0 + (bm + 1)]) : 0ll;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        if ((q0[u] | q1[u]) == 0) continue;
        const long long x = base + u * stride;
        const long long a0 = ((x >> logb) << (logb + 1)) | (x & bm);
        if (q0[u]) acc[a0] = 0ull;
        if (q1[u]) acc[a0 + (bm + 1)] = 0ull;
        if (bad) continue;
        double2 d = data[x];
        if (q0[u]) d.x += static_cast<double>(q0[u]) * sc;
        if (q1[u]) d.y += static_cast<double>(q1[u]) * sc;
        data[x] = d;
    }
}

// Pipelined builds: K chunk accumulators with their own exponents, summed in chunk order.
template <bool SYM>
__global__ void k_build_finalize_multi(unsigned long long* __restrict__ acc, int K, long long total_slots,
                                       const int* __restrict__ scale_exps, const int* __restrict__ nonfinite,
                                       double* __restrict__ data, int* __restrict__ counters, int ncounters, int tb,
                                       std::uint32_t bmask) {
    const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (s < ncounters) counters[s] = 0;
    if (s >= total_slots) return;
    const bool bad = (nonfinite[0] | nonfinite[kOvfOffset]) != 0;
    double v = 0.0;
    bool any = false;
    for (int c = 0; c < K; ++c) {
        const long long q = static_cast<long long>(acc[(long long)c * total_slots + s]);
        if (q) {
            acc[(long long)c * total_slots + s] = 0ull;
            v += static_cast<double>(q) * pow2_neg(scale_exps[c]);
            any = true;
        }
    }
    if (!any || bad) return;
    const long long d = data_index(s, tb, SYM, bmask);
    if (SYM)
        data[d] += v;
    else
        data[2 * d] += v;
}
void launch_build_finalize_multi(cudaStream_t st, const BuildPlan& p, int K, const int* scale_exps, int* counters,
                                 int ncounters) {
    const unsigned grid = cdiv(std::max<long long>(p.total_slots, ncounters), 256);
    if (p.sym)
        k_build_finalize_multi<true><<<grid, 256, 0, st>>>(p.acc, K, p.total_slots, scale_exps, p.nonfinite,
                                                           p.data_as_double, counters, ncounters, p.cls_bits, p.bmask);
    else
        k_build_finalize_multi<false><<<grid, 256, 0, st>>>(p.acc, K, p.total_slots, scale_exps, p.nonfinite,
                                                            p.data_as_double, counters, ncounters, p.cls_bits, p.bmask);
    count_launch();
}

void launch_build_finalize(cudaStream_t st, const BuildPlan& p) {
    const unsigned grid = cdiv(std::max<long long>((p.total_slots + 3) / 4, 2 * p.G), 256);
    const bool pdl = p.pdl && p.cls_bits >= 0;  // only the class-list main pass triggers early
    if (p.sym && p.cls_bits == 0) {
        const long long pairs = p.total_slots / 2;  // B x b complex entries
        const int logb = __builtin_ctz(p.bmask + 1u);
        const unsigned g2 = cdiv(std::max<long long>((pairs + 1) / 2, 2 * p.G), 256);
        pdl_launch(k_build_finalize_sym_pair, g2, 256, 0, st, pdl, p.acc, pairs, logb, p.scale_exp, p.nonfinite,
                   reinterpret_cast<double2*>(p.data_as_double), p.next_row, 2 * p.G);
    } else if (p.sym)
        pdl_launch(k_build_finalize<true>, grid, 256, 0, st, pdl, p.acc, p.total_slots, p.scale_exp, p.nonfinite,
                   p.data_as_double, p.next_row, 2 * p.G, p.cls_bits, p.bmask);
    else
        pdl_launch(k_build_finalize<false>, grid, 256, 0, st, pdl, p.acc, p.total_slots, p.scale_exp, p.nonfinite,
                   p.data_as_double, p.next_row, 2 * p.G, p.cls_bits, p.bmask);
    count_launch();
}

}  // namespace skc
