// K1: dense tensor-sketch build on sm_100a.
//
// Replaces the reference hot loops
//   symmetric  proj/src/sketch.cpp:315-345 — sorted triples i<=j<=k, weight kappa 1/3/6,
//              bucket (h_i+h_j+h_k) mod b, sign root4(e_i+e_j+e_k);
//   asymmetric proj/src/sketch.cpp:173-193 — all (i,j,k), bucket (h1_i+h2_j+h3_k) mod b,
//              sign xi1 xi2 xi3.
//
// Layout of the work. The B x b complex sketch set (5.2 MB at config 1) does not fit one
// SM's shared memory and each tensor entry lands in B random buckets, so the slot space
// (replicate, bucket, re/im) is cut into G contiguous ranges of ~29K slots (~227 KB of
// limbs) and the sorted-triple rows into C chunks, G*C ~= #SMs. CTA (g, c) streams the
// rows of chunk c with coalesced loads (a warp per row segment, a lane per k),
// converts each entry to fixed point once, and evaluates it against the 1-2 replicates
// its range overlaps; in-range contributions go to shared memory. The measured
// alternative that enumerated only owned contributions through per-class suffix
// tables executed 3x more instructions (profiles/).
//
// Accumulation is exact 64-bit fixed point: q = round(kappa*T*2^F) is split into two
// 32-bit limbs added with native ATOMS.ADD (shared fp64 atomics are CAS loops on
// sm_100a); the carry out of the low limb is taken from the returned old value, so the
// sum is exact mod 2^64 under any interleaving and the build is bit-deterministic.
// F = 61 - ceil(log2(sum kappa|T|)) from a deterministic pre-pass bounds every bucket.
#include <cuda_runtime.h>

#include "skc_host.hpp"
#include "skc_internal.hpp"

namespace skc {

namespace {
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

// ---- quantize pass ----------------------------------------------------------------
// One warp per row: reads the row segment twice (the second read hits L1), computes
// the row's L1 mass sum kappa|T| in a fixed order, and writes the packed fixed-point
// stream qbuf[rowoff + e] = round(kappa T 2^Frow) with Frow = 61 - ceil(log2 rowL1).
// The main pass rescales q >> (Frow - F) to the global exponent F, so T is read from
// HBM once per build. Per-block L1 partials are summed in a fixed order (deterministic).
template <typename TT, bool SYM>
__global__ void __launch_bounds__(256) k_build_quantize(const TT* __restrict__ T, int n,
                                                       const std::uint32_t* __restrict__ rowtab,
                                                       const long long* __restrict__ rowoff, int nrows,
                                                       long long* __restrict__ qbuf, short* __restrict__ rowF,
                                                       double* __restrict__ partials, int* __restrict__ nonfinite) {
    extern __shared__ double stage[];  // 8 warps x n: each element of T is read exactly once
    __shared__ double red[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* st = stage + (size_t)warp * n;
    double blk = 0.0;
    bool bad = false;
    for (int row = blockIdx.x * 8 + warp; row < nrows; row += gridDim.x * 8) {
        const std::uint32_t ij = rowtab[row];
        const int i = static_cast<int>(ij >> 16), j = static_cast<int>(ij & 0xFFFFu);
        const TT* rp = T + ((size_t)i * n + j) * n;
        const int k0 = SYM ? j : 0;
        const double kdiag = SYM ? ((i == j) ? 1.0 : 3.0) : 1.0;
        const double koff = SYM ? ((i == j) ? 3.0 : 6.0) : 1.0;
        double a0 = 0.0;
        // 4 loads in flight per lane (T may be host memory read over PCIe)
        for (int kb = k0 + lane; kb < n; kb += 128) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = (kb + 32 * u < n) ? static_cast<double>(rp[kb + 32 * u]) : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = kb + 32 * u;
                if (k < n) {
                    const double kv = ((SYM && k == j) ? kdiag : koff) * v[u];
                    st[k - k0] = kv;
                    a0 += fabs(kv);
                    bad |= !isfinite(v[u]);
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a0 += __shfl_xor_sync(0xffffffffu, a0, o);
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
        blk += (lane == 0) ? a0 : 0.0;
    }
    if (bad) atomicOr(nonfinite, 1);
    const double s = block_sum_b<256>(blk, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// Global exponent F = 61 - ceil(log2(sum kappa|T|)): every bucket sum of q stays below 2^62.
__global__ void k_build_scale(const double* __restrict__ partials, int np, int* __restrict__ scale_exp) {
    __shared__ double red[8];
    double acc = 0.0;
    for (int i = threadIdx.x; i < np; i += 256) acc += partials[i];
    const double s = block_sum_b<256>(acc, red);
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

void launch_build_prepass(cudaStream_t st, const void* T, const BuildPlan& p) {
    cudaMemsetAsync(p.nonfinite, 0, sizeof(int), st);
#define QUANT(TT, SY)                                                                                             \
    {                                                                                                             \
        const size_t smem = sizeof(double) * 8 * (size_t)p.n;                                                     \
        if (smem > 48 * 1024)                                                                                     \
            cudaFuncSetAttribute(k_build_quantize<TT, SY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        k_build_quantize<TT, SY><<<kPrepassBlocks, 256, smem, st>>>((const TT*)T, p.n, p.rowtab, p.rowoff, p.nrows,  \
                                                                   p.qbuf, p.rowF, p.prepass_partials, p.nonfinite); \
    }
    if (p.sym) {
        if (p.dtype == 0) QUANT(double, true)
        else QUANT(float, true)
    } else {
        if (p.dtype == 0) QUANT(double, false)
        else QUANT(float, false)
    }
#undef QUANT
    count_launch();
    k_build_scale<<<1, 256, 0, st>>>(p.prepass_partials, kPrepassBlocks, p.scale_exp);
    count_launch();
}

// ---- main pass -----------------------------------------------------------------------
constexpr int kBuildThreads = 1024;

__device__ __forceinline__ std::uint32_t atom_add_shared(std::uint32_t addr, std::uint32_t v) {
    std::uint32_t old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void red_add_shared(std::uint32_t addr, std::uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// Exact 64-bit add into an interleaved (lo, hi) limb pair at addr, addr+4: the carry
// out of lo is recovered from the returned old value.
__device__ __forceinline__ void add64(std::uint32_t addr, long long q) {
    const std::uint32_t ql = static_cast<std::uint32_t>(q);
    const std::uint32_t qh = static_cast<std::uint32_t>(static_cast<unsigned long long>(q) >> 32);
    const std::uint32_t old = atom_add_shared(addr, ql);
    const std::uint32_t carry = static_cast<std::uint32_t>((static_cast<unsigned long long>(old) + ql) >> 32);
    red_add_shared(addr + 4u, qh + carry);
}

struct BuildArgs {
    int n, B;
    std::uint32_t bmask;
    long long total_slots;
    int slots_per_cta, G;
    const std::uint32_t* rowtab;
    const long long* rowoff;
    const short* rowF;
    const long long* qbuf;
    const int* chunk_begin;
    const std::uint32_t* packed;
    const int* scale_exp;
    long long* partials;  // C x total_slots (natural slot order)
};

// CTA (g, c): contiguous slot range g of the B x (2b | b) slot space, rows of chunk c.
// Every streamed entry is evaluated against the (1..RMAX) replicates the range
// overlaps; in-range contributions go to the shared-memory limbs.
template <bool SYM, int RMAX>
__global__ void __launch_bounds__(kBuildThreads, 1) k_build_range(BuildArgs a) {
    extern __shared__ std::uint32_t sacc[];
    const int g = blockIdx.x % a.G, c = blockIdx.x / a.G;
    const long long slot_lo = (long long)g * a.slots_per_cta;
    const long long slot_hi = min(slot_lo + a.slots_per_cta, a.total_slots);
    const int nslots = static_cast<int>(slot_hi - slot_lo);
    const int n = a.n;
    const long long spr = SYM ? 2ll * (a.bmask + 1) : static_cast<long long>(a.bmask + 1);
    const int m_lo = static_cast<int>(slot_lo / spr);
    const int R = static_cast<int>((slot_hi - 1) / spr) - m_lo + 1;
    std::uint32_t* lo = sacc;
    std::uint32_t* ptab = sacc + 2 * a.slots_per_cta;  // RMAX x n (streamed-mode hashes)
    std::uint32_t* pij_tab = ptab + RMAX * n;          // RMAX x 2n (row-pair hashes)
    for (int s = threadIdx.x; s < 2 * a.slots_per_cta; s += kBuildThreads) lo[s] = 0u;
    const int prow = SYM ? n : 3 * n;
    for (int x = threadIdx.x; x < RMAX * n; x += kBuildThreads) {
        const int r = x / n, k = x - r * n;
        const std::uint32_t* pm = a.packed + (size_t)(m_lo + min(r, R - 1)) * prow;
        ptab[x] = pm[(SYM ? 0 : 2 * n) + k];
        pij_tab[r * 2 * n + k] = pm[k];
        pij_tab[r * 2 * n + n + k] = pm[(SYM ? 0 : n) + k];
    }
    __syncthreads();
    const int F = *a.scale_exp;
    const std::uint32_t sbase = static_cast<std::uint32_t>(__cvta_generic_to_shared(sacc));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int row_end = a.chunk_begin[c + 1];
    int base[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) base[r] = static_cast<int>((long long)(m_lo + r) * spr - slot_lo);

    for (int row = a.chunk_begin[c] + warp; row < row_end; row += kBuildThreads / 32) {
        const std::uint32_t ij = __ldg(a.rowtab + row);
        const int i = static_cast<int>(ij >> 16), j = static_cast<int>(ij & 0xFFFFu);
        const int k0 = SYM ? j : 0;
        const long long* qrow = a.qbuf + __ldg(a.rowoff + row) - k0;
        const int d = static_cast<int>(__ldg(a.rowF + row)) - F;  // >= 0
        std::uint32_t pij[RMAX];
#pragma unroll
        for (int r = 0; r < RMAX; ++r) pij[r] = pij_tab[r * 2 * n + i] + pij_tab[r * 2 * n + n + j];
        // 4 independent loads in flight per lane before any use (latency hiding)
        for (int kb = k0 + lane; kb < n; kb += 128) {
            long long qv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) qv[u] = (kb + 32 * u < n) ? __ldg(qrow + kb + 32 * u) : 0ll;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = kb + 32 * u;
                if (k >= n) break;
                const long long q = qv[u] >> d;  // zero entries add nothing (sketch.cpp:337 skips them)
                const long long nq = -q;
#pragma unroll
                for (int r = 0; r < RMAX; ++r) {
                    if (r < R) {
                        const std::uint32_t p = pij[r] + ptab[r * n + k];
                        const int s = base[r] + (SYM ? static_cast<int>(((p & a.bmask) << 1) | ((p >> 30) & 1u))
                                                     : static_cast<int>(p & a.bmask));
                        if (static_cast<unsigned>(s) < static_cast<unsigned>(nslots))
                            add64(sbase + 8u * static_cast<std::uint32_t>(s), (p >> 31) ? nq : q);
                    }
                }
            }
        }
    }
    __syncthreads();
    long long* out = a.partials + (long long)c * a.total_slots + slot_lo;
    const unsigned long long* limbs = reinterpret_cast<const unsigned long long*>(sacc);  // (lo, hi) pairs
    for (int s = threadIdx.x; s < nslots; s += kBuildThreads) out[s] = static_cast<long long>(limbs[s]);
}

template <bool SYM, int RMAX>
static void build_launch(cudaStream_t st, const BuildPlan& p, const BuildArgs& a) {
    const size_t smem = sizeof(std::uint32_t) * (2 * (size_t)p.slots_per_cta + 3 * (size_t)RMAX * p.n);
    cudaFuncSetAttribute(k_build_range<SYM, RMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_build_range<SYM, RMAX><<<p.G * p.C, kBuildThreads, smem, st>>>(a);
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
    int rm = R <= 1 ? 1 : R <= 2 ? 2 : R <= 4 ? 4 : R <= 8 ? 8 : 16;
    return sizeof(std::uint32_t) * (2 * (size_t)slots_per_cta + 3 * (size_t)rm * n);
}

void launch_build_main(cudaStream_t st, const void* T, const BuildPlan& p) {
    (void)T;
    BuildArgs a;
    a.n = p.n;
    a.B = p.B;
    a.bmask = p.bmask;
    a.total_slots = p.total_slots;
    a.slots_per_cta = p.slots_per_cta;
    a.G = p.G;
    a.rowtab = p.rowtab;
    a.rowoff = p.rowoff;
    a.rowF = p.rowF;
    a.qbuf = p.qbuf;
    a.chunk_begin = p.chunk_begin;
    a.packed = p.packed;
    a.scale_exp = p.scale_exp;
    a.partials = p.partials;
    if (p.sym)
        build_dispatch<true>(st, p, a);
    else
        build_dispatch<false>(st, p, a);
}

// ---- finalize --------------------------------------------------------------------------
// data += (sum over chunks of partials) * 2^-F. For the symmetric set the slot index is
// the double index into interleaved (re, im) data; the asymmetric set is real-only.
template <bool SYM>
__global__ void k_build_finalize(const long long* __restrict__ partials, int C, long long total_slots,
                                 const int* __restrict__ scale_exp, double* __restrict__ data) {
    const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
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

void launch_build_finalize(cudaStream_t st, const BuildPlan& p) {
    if (p.sym)
        k_build_finalize<true><<<cdiv(p.total_slots, 256), 256, 0, st>>>(p.partials, p.C, p.total_slots, p.scale_exp,
                                                                         p.data_as_double);
    else
        k_build_finalize<false><<<cdiv(p.total_slots, 256), 256, 0, st>>>(p.partials, p.C, p.total_slots,
                                                                          p.scale_exp, p.data_as_double);
    count_launch();
}

}  // namespace skc
