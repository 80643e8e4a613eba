// Dense sketch builds (sketch.cpp accumulate_dense): input staging and the
// quantize / scatter / finalize orchestration of skc_build.cu.
#include "skc_abi_impl.hpp"

namespace skcabi {

// ---- dense build orchestration ------------------------------------------------------
// Device-visible view of the input tensor. Device pointers are used as is. Pinned
// (page-locked, UVA-mapped) host memory is read in place by the quantize pass, so only
// the bytes the build reads cross the bus. Pageable host memory is staged, copying only
// the row blocks the build reads (sym: T[i][i:n][:], asym: T[i0:i1]) unless the full
// tensor is needed by the symmetry check.
const void* stage_tensor(skc_context* ctx, const void* T, int n, int dtype, int location, bool sym, int i0, int i1,
                         bool need_full, size_t* h2d_bytes, bool* zero_copy) {
    if (h2d_bytes) *h2d_bytes = 0;
    if (zero_copy) *zero_copy = false;
    if (location == SKC_DEVICE) return T;
    const size_t es = dtype == SKC_F64 ? 8 : 4;
    const size_t n2 = static_cast<size_t>(n) * n;
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, T) == cudaSuccess && attr.type == cudaMemoryTypeHost &&
        attr.devicePointer != nullptr) {
        if (zero_copy) *zero_copy = true;
        return attr.devicePointer;
    }
    cudaGetLastError();  // clear a failed attribute query on pageable memory
    ctx->tensor_stage.alloc(n2 * n * es);
    unsigned char* dst = ctx->tensor_stage.p;
    const unsigned char* src = static_cast<const unsigned char*>(T);
    size_t moved = 0;
    if (need_full) {
        CK(cudaMemcpyAsync(dst, src, n2 * n * es, cudaMemcpyHostToDevice, ctx->stream));
        moved = n2 * n * es;
    } else if (sym) {
        for (int i = i0; i < i1; ++i) {
            const size_t off = (static_cast<size_t>(i) * n + i) * n * es, len = static_cast<size_t>(n - i) * n * es;
            CK(cudaMemcpyAsync(dst + off, src + off, len, cudaMemcpyHostToDevice, ctx->stream));
            moved += len;
        }
    } else {
        const size_t off = static_cast<size_t>(i0) * n2 * es, len = static_cast<size_t>(i1 - i0) * n2 * es;
        CK(cudaMemcpyAsync(dst + off, src + off, len, cudaMemcpyHostToDevice, ctx->stream));
        moved = len;
    }
    if (h2d_bytes) *h2d_bytes = moved;
    return dst;
}

// The exact accumulators and row counters are zero between builds: the finalize re-zeroes
// what the build used. A fresh allocation (or a build that failed before its finalize was
// enqueued) is cleared here.
void ensure_build_scratch_clean(skc_context* ctx) {
    if (ctx->build_scratch_clean && ctx->build_acc.p == ctx->build_acc_clean_p &&
        ctx->build_ints.p == ctx->build_ints_clean_p && ctx->build_acc.count == ctx->build_acc_clean_n &&
        ctx->build_ints.count == ctx->build_ints_clean_n)
        return;
    CK(cudaMemsetAsync(ctx->build_acc.p, 0, ctx->build_acc.count * sizeof(unsigned long long), ctx->stream));
    CK(cudaMemsetAsync(ctx->build_ints.p, 0, ctx->build_ints.count * sizeof(int), ctx->stream));
    ctx->build_acc_clean_p = ctx->build_acc.p;
    ctx->build_ints_clean_p = ctx->build_ints.p;
    ctx->build_acc_clean_n = ctx->build_acc.count;
    ctx->build_ints_clean_n = ctx->build_ints.count;
    ctx->build_scratch_clean = true;
}

#ifndef SKC_LOCK_MB  // experiment builds (microbench/lock_ab.sh) compile other spreads; 0: off
#define SKC_LOCK_MB 12
#endif
constexpr double kLockMB = SKC_LOCK_MB;
#ifndef SKC_SUMS_MINB  // resident blocks per SM of the lean sums pre-pass (skc_build.cu)
#define SKC_SUMS_MINB 5
#endif
constexpr int kSumsBlocksPerSM = SKC_SUMS_MINB;

// Scratch and launch plan of one dense build of rows [i0, i1) on ctx (no launches). The
// plan depends only on the shape (n, b, B, dtype, sym, limbs), so replicas of a set on
// several devices get the same accumulator layout, and an empty row range still yields a
// valid plan (nrows 0).
skc_context::RowTab& prepare_dense_build(skc_context* ctx, int n, int dtype, bool sym, int i0, int i1, int B,
                                         std::uint32_t b, const std::uint32_t* packed, double2* data, bool zero_copy,
                                         bool two_limb, BuildPlan& p) {
    skc_context::RowTab& rt = ctx->rowtab(n, i0, std::max(i0, i1), sym);
    const long long total_slots = static_cast<long long>(B) * (sym ? 2ll * b : static_cast<long long>(b));
    // slots per CTA limited by shared memory (limbs + per-replicate hash tables)
    int G = 1;
    for (;; ++G) {
        long long spc = ((total_slots + G - 1) / G + 31) / 32 * 32;
        const long long spr0 = sym ? 2ll * b : static_cast<long long>(b);
        int Rg = 1;
        for (int g = 0; g < G; ++g) {
            const long long lo = g * spc, hi = std::min(lo + spc, total_slots);
            if (hi > lo) Rg = std::max(Rg, static_cast<int>((hi - 1) / spr0 - lo / spr0 + 1));
        }
        if (Rg <= 16 && build_smem_bytes(spc, Rg, n) <= static_cast<size_t>(ctx->smem_optin - 1024)) break;
        if (G > 4096) fail(kInvalidArgument, "accumulate_dense: sketch set too large for the dense build");
    }
    long long spc = (total_slots + G - 1) / G;
    spc = (spc + 31) / 32 * 32;
    // Dense builds take the class-list kernel when a (replicate, [parity,] bucket class)
    // window fits: the fewest bucket-class bits t <= 3 whose window + tables fit.
    int cls_bits = -1;
    // (class lists pack k above the 3-term bucket sum: n <= 2^(28 - log2 b))
    int logb = 0;
    while ((1u << logb) < b) ++logb;
    // (small asymmetric builds are flush/setup-bound with few windows: C0's asym build
    // measured 93 us on the contiguous-window kernel against 113 us here)
    const bool small_asym = !sym && rt.cum.back() < (4ll << 20);
    // fp32 input: one biased limb per slot, unless a previous attempt overflowed a limb
    const bool one_limb = dtype == SKC_F32 && !two_limb;
    if (!small_asym && b <= (1u << 21) && b >= 64 &&
        static_cast<long long>(n - 1) < (1ll << (28 - logb))) {
        for (int t = 0; t <= 3; ++t)
            if (cls_smem_bytes(b, t, n, sym, one_limb) <= static_cast<size_t>(ctx->smem_optin - 4096)) {
                cls_bits = t;
                break;
            }
    }
    if (cls_bits >= 0) G = B * ((sym ? 2 : 1) << cls_bits);
    const long long spr = sym ? 2ll * b : static_cast<long long>(b);
    int R = 1;
    std::vector<int> Rg(G, 1);
    for (int g = 0; g < G; ++g) {
        const long long lo = g * spc, hi = std::min(lo + spc, total_slots);
        if (hi > lo) Rg[g] = static_cast<int>((hi - 1) / spr - lo / spr + 1);
        R = std::max(R, Rg[g]);
    }
    require(R <= 16, "accumulate_dense: slot range spans too many replicates");
    const long long tot = rt.cum.back();
    const int P = std::max(1, ctx->sms);  // one persistent CTA per SM, rows handed out dynamically
    ctx->build_ints.alloc(2 * static_cast<size_t>(G));
    ctx->build_acc.alloc(static_cast<size_t>(total_slots));
    ctx->qbuf.alloc(static_cast<size_t>(std::max<long long>(1, tot)));
    ctx->rowF.alloc(static_cast<size_t>(std::max(1, rt.nrows)));
    ctx->prepass.alloc(4 * kPrepassBlocks);  // sums, maxima, sums of squares, minima
    ctx->ints.alloc(16);

    p = BuildPlan();
    p.n = n;
    p.sym = sym;
    p.dtype = dtype;
    p.rowtab = rt.rows.p;
    p.nrows = rt.nrows;
    p.P = P;
    p.G = G;
    p.next_row = ctx->build_ints.p;
    p.acc = ctx->build_acc.p;
    // the flat kernel's doubled SYM tables need bucket sums below bit 30: b <= 2^27
    if (cls_bits < 0 && sym && b > (1u << 27))
        fail(kInvalidArgument, "accumulate_dense: symmetric dense builds support b <= 2^27");
    p.cls_bits = cls_bits;
    p.one_limb = cls_bits >= 0 && one_limb;
    // class-list builds read T in place when it is device-resident (row offsets relative to
    // a 32-row chunk fit in 32 bits for n <= 30000), else a packed raw copy of the rows
    p.xsrc_mode = cls_bits < 0 ? 0 : ((!zero_copy && n <= 30000) ? 1 : 2);
    p.total_slots = total_slots;
    p.slots_per_cta = static_cast<int>(spc);
    p.R = R;
    p.bmask = b - 1;
    p.B = B;
    p.packed = packed;
    p.rowoff = rt.offs.p;
    p.qbuf = ctx->qbuf.p;
    p.rowF = ctx->rowF.p;
    p.prepass_partials = ctx->prepass.p;
    p.scale_exp = ctx->ints.p;
    p.nonfinite = ctx->ints.p + 1;
    p.ovf = ctx->ints.p + 3;  // nonfinite + kOvfOffset
    if (!ctx->build_ovf_clean) {
        CK(cudaMemsetAsync(p.ovf, 0, sizeof(int), ctx->stream));
        ctx->build_ovf_clean = true;
    }
    p.data_as_double = reinterpret_cast<double*>(data);
    if (p.xsrc_mode == 1)  // device-resident class-list build: sums-only pre-pass, one wave of 5 blocks/SM
        p.prepass_blocks = std::min(kPrepassBlocks, std::max(1, ctx->sms) * kSumsBlocksPerSM);
    p.total_entries = tot;
    // Lockstep of the class-list windows: every window sweeps all rows, so the rows are read
    // from HBM once only while the windows' cursors stay within what L2 holds. ~12 MB of
    // rows (the two L2 partitions mirror each other's lines: ~60 MB usable); off when the
    // whole stream fits.
    {
        const double es = dtype == SKC_F32 ? 4.0 : 8.0;
        const double bytes = static_cast<double>(tot) * es;
        // (only with >= 3 CTAs per window: at 148 CTAs over 80 windows the moves cost 0.4-2.4%
        // more than the L2 hits return, and over 160 windows CTAs would chase empty windows:
        // 1.49 against 0.88 ms, microbench/lock_many_windows.py)
        if (kLockMB > 0 && cls_bits >= 0 && rt.nrows > 0 && bytes > 48e6 && P >= 3 * G)
            p.lock_rows = std::max(256, static_cast<int>(kLockMB * 1e6 / (bytes / rt.nrows)));
    }
    return rt;
}

// High-dynamic-range builds (the resolution check of the main pass flagged the tensor):
// entries are split by the magnitude of kappa|T| into bands of at most 16 binades (from the
// exponent histogram, empty ranges skipped), and each band is built with its own exponent
// from its own sums: the raw-copy (class-list) or fixed-point (contiguous-window) pre-pass
// writes the band's entries and zeros elsewhere, then the main pass and the finalize add
// that band's sketch to the data. Within a band max/min kappa|T| < 2^16, so every bucket
// keeps <= ~2^-34 of its own magnitude; the fp64 reference sum (sketch.cpp:340) keeps
// ~2^-52 of its terms' magnitude. Exact per band, bands added in fp64 (one rounding each).
void run_dense_build_banded(skc_context* ctx, const void* Tdev, int n, int dtype, bool sym, int i0, int i1, int B,
                            std::uint32_t b, const std::uint32_t* packed, double2* data, bool zero_copy) {
    BuildPlan p;
    skc_context::RowTab& rt = prepare_dense_build(ctx, n, dtype, sym, i0, i1, B, b, packed, data, zero_copy, true, p);
    if (rt.nrows == 0) return;
    DevBuf<unsigned long long> hist;
    hist.alloc(kExpBins);
    CK(cudaMemsetAsync(hist.p, 0, sizeof(unsigned long long) * kExpBins, ctx->stream));
    launch_build_exp_hist(ctx->stream, Tdev, p, hist.p);
    ctx->check_launch();
    std::vector<unsigned long long> h(kExpBins);
    CK(cudaMemcpyAsync(h.data(), hist.p, sizeof(unsigned long long) * kExpBins, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    for (int e = kExpBins - 1; e >= 0;) {
        while (e >= 0 && h[e] == 0) --e;
        if (e < 0) break;
        const int top = e, bot = std::max(0, top - 15);
        e = bot - 1;
        BuildPlan q = p;
        q.band_lo = std::ldexp(1.0, bot - kExpBias);
        q.band_hi = std::ldexp(1.0, top - kExpBias + 1);
        q.rho_max = INFINITY;
        q.xsrc_mode = q.cls_bits >= 0 ? 2 : 0;  // the pre-pass writes the band's (masked) copy
        q.prepass_blocks = kPrepassBlocks;
        q.pdl = false;
        ensure_build_scratch_clean(ctx);
        ctx->build_scratch_clean = false;
        CK(cudaMemsetAsync(q.nonfinite, 0, sizeof(int), ctx->stream));
        {
            SKC_PROF(ctx, "build_prepass");
            launch_build_prepass(ctx->stream, Tdev, q);
        }
        {
            SKC_PROF(ctx, "build_main");
            launch_build_main(ctx->stream, Tdev, q);
        }
        {
            SKC_PROF(ctx, "build_finalize");
            launch_build_finalize(ctx->stream, q);
        }
        ctx->build_scratch_clean = true;
        ctx->check_launch();
    }
    ++ctx->build_banded;
}

void run_dense_build(skc_context* ctx, const void* Tdev, int n, int dtype, bool sym, int i0, int i1, int B,
                     std::uint32_t b, const std::uint32_t* packed, double2* data, bool zero_copy, bool two_limb) {
    if (i0 >= i1) return;
    BuildPlan p;
    skc_context::RowTab& rt = prepare_dense_build(ctx, n, dtype, sym, i0, i1, B, b, packed, data, zero_copy, two_limb, p);
    if (rt.nrows == 0) return;
    const long long total_slots = p.total_slots;
    const long long tot = rt.cum.back();
    const int G = p.G;
    // Zero-copy host input: the quantize pass is bus-bound, so the rows are cut into K
    // chunks and chunk c+1 is read over PCIe (a few SMs, wide blocks) while the main pass
    // of chunk c runs on the other SMs (second stream). Each chunk keeps its own exponent
    // and exact accumulator; the finalize sums the K chunk sketches in order.
    // (the raw-copy pre-pass of class-list builds stages nothing in shared memory; the
    // fixed-point pre-pass of the contiguous-window kernels stages 32 rows)
    const int K = (zero_copy && rt.nrows >= 4096 &&
                   (p.xsrc_mode == 2 || sizeof(double) * 32 * (size_t)n <= (size_t)ctx->smem_optin - 1024))
                      ? 4
                      : 1;
    if (K > 1) {
        const int qsms = 16;  // SMs given to the bus-bound quantize pass
        p.P = std::max(1, ctx->sms - qsms);
        p.prepass_threads = 1024;
        p.prepass_blocks = qsms;
        p.prepass_warps = 32;
        ctx->build_acc.alloc(static_cast<size_t>(K) * total_slots);
        ctx->build_ints.alloc(2 * static_cast<size_t>(K) * G);
        ctx->ints.alloc(16);
        ctx->prepass.alloc(4 * static_cast<size_t>(K) * qsms);
        ensure_build_scratch_clean(ctx);
        ctx->build_scratch_clean = false;
        if (!ctx->stream2) CK(cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking));
        if (!ctx->ev_q[0])
            for (int c = 0; c < 5; ++c) CK(cudaEventCreateWithFlags(&ctx->ev_q[c], cudaEventDisableTiming));
        // decreasing chunk sizes: chunk c's main pass (~0.4x the bus time of its rows) hides
        // under chunk c+1's bus reads, and the exposed tail (last main pass) stays short
        static const double kFrac4[5] = {0.0, 0.42, 0.72, 0.90, 1.0};
        std::vector<int> rb(K + 1, 0);
        for (int c = 1; c < K; ++c) {
            const long long target = (K == 4) ? static_cast<long long>(static_cast<double>(tot) * kFrac4[c]) : tot * c / K;
            rb[c] = static_cast<int>(std::lower_bound(rt.cum.begin(), rt.cum.end(), target) - rt.cum.begin());
            rb[c] = std::min(std::max(rb[c], rb[c - 1]), rt.nrows);
        }
        rb[K] = rt.nrows;
        CK(cudaMemsetAsync(p.nonfinite, 0, sizeof(int), ctx->stream));
        {
            SKC_PROF(ctx, "build_pipelined");
            for (int c = 0; c < K; ++c) {
                BuildPlan pc = p;
                pc.rowtab = rt.rows.p + rb[c];
                pc.rowoff = rt.offs.p + rb[c];
                pc.rowF = ctx->rowF.p + rb[c];
                pc.nrows = rb[c + 1] - rb[c];
                pc.total_entries = rt.cum[rb[c + 1]] - rt.cum[rb[c]];
                pc.prepass_partials = ctx->prepass.p + 4 * static_cast<size_t>(c) * qsms;
                pc.scale_exp = ctx->ints.p + 4 + c;
                pc.reset_nonfinite = false;
                pc.acc = ctx->build_acc.p + static_cast<size_t>(c) * total_slots;
                pc.next_row = ctx->build_ints.p + 2 * static_cast<size_t>(c) * G;
                if (pc.nrows > 0) launch_build_prepass(ctx->stream, Tdev, pc);
                CK(cudaEventRecord(ctx->ev_q[c], ctx->stream));
                CK(cudaStreamWaitEvent(ctx->stream2, ctx->ev_q[c], 0));
                if (pc.nrows > 0) {
                    launch_build_main(ctx->stream2, Tdev, pc);
                }  // (an empty chunk's accumulator stays zero)
            }
            CK(cudaEventRecord(ctx->ev_q[K], ctx->stream2));
            CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_q[K], 0));
            BuildPlan pf = p;
            pf.acc = ctx->build_acc.p;
            launch_build_finalize_multi(ctx->stream, pf, K, ctx->ints.p + 4, ctx->build_ints.p, 2 * K * G);
            ctx->build_scratch_clean = true;
        }
        ctx->check_launch();
    } else {
        ensure_build_scratch_clean(ctx);
        ctx->build_scratch_clean = false;
        p.pdl = true;
        {
            SKC_PROF(ctx, "build_prepass");
            launch_build_prepass(ctx->stream, Tdev, p);
        }
        ctx->check_launch();
        {
            SKC_PROF(ctx, "build_main");
            launch_build_main(ctx->stream, Tdev, p);
        }
        ctx->check_launch();
        {
            SKC_PROF(ctx, "build_finalize");
            launch_build_finalize(ctx->stream, p);  // device-side no-op when nonfinite
            ctx->build_scratch_clean = true;
        }
        ctx->check_launch();
    }
    int* flag = ctx->pinned_ints();  // pinned: a direct DMA, not a staged pageable copy
    CK(cudaMemcpyAsync(flag, p.nonfinite, 3 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    const int nonfinite = flag[0], overflow = flag[2] & 1, hdr = flag[2] & 2;
    // Fixed-point accumulation cannot carry NaN/Inf the way the reference's
    // floating-point sum would; reject instead of producing a wrong sketch.
    if (nonfinite) {
        if (overflow) {
            CK(cudaMemsetAsync(p.ovf, 0, sizeof(int), ctx->stream));
            ctx->sync();
        }
        fail(kInvalidArgument, "accumulate_dense: tensor has a non-finite entry");
    }
    if (hdr) {  // beyond one fixed-point scale: the finalize added nothing; redo in magnitude bands
        CK(cudaMemsetAsync(p.ovf, 0, sizeof(int), ctx->stream));
        run_dense_build_banded(ctx, Tdev, n, dtype, sym, i0, i1, B, b, packed, data, zero_copy);
        return;
    }
    if (overflow) {  // a one-limb window overflowed: the finalize added nothing; redo exactly
        CK(cudaMemsetAsync(p.ovf, 0, sizeof(int), ctx->stream));
        ++ctx->build_two_limb_retries;
        run_dense_build(ctx, Tdev, n, dtype, sym, i0, i1, B, b, packed, data, zero_copy, true);
    }
}

}  // namespace skcabi
