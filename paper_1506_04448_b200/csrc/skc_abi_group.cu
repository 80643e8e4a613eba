// Multi-GPU paths of the C-ABI over NCCL (NVLink 5 / NVSwitch within one box).
//
// The reference parallelises with OpenMP inside one process: over the B replicates of a
// build (sketch.cpp:325) and of a contraction (contraction.cpp:145), while the RTPM restart
// loop (decompose.cpp:92-112) is serial. Here a sketch set has one replica per GPU (same
// seeds, same data), one context per GPU, and the work is partitioned where the path shards
// with one exchange step each:
//   dense build  i-slices of the sorted triples with equal entry counts; the pre-pass
//                partials are all-gathered (every rank derives the same global exponent F)
//                and the B x 2b exact fixed-point accumulators are all-reduced (int64 sum:
//                exact and order-free), so the sketch is bit-identical at any rank count;
//   moment       sample blocks; the B x b per-residue partial transforms are all-reduced
//                before each rank combines them into its replica;
//   LDA          document blocks; the corpus globals (M1 sums, document counts), then the
//                sketch data are all-reduced;
//   RTPM         restart blocks; the selection values are all-gathered, every rank takes
//                the same lowest-tau argmax, the winner's vector is broadcast from its owner
//                and every rank applies the identical deflation.
// The *_group calls are collective: every rank calls them, each process with its local
// replicas (one per local context). Ranks live in one process (skc_group_create,
// ncclCommInitAll) or one process each (skc_nccl_unique_id + skc_context_comm_init).
#include "skc_abi_impl.hpp"

namespace skcabi {

#define NC(call)                                                                                                 \
    do {                                                                                                         \
        ncclResult_t r_ = (call);                                                                                \
        if (r_ != ncclSuccess) fail(kCudaError, std::string("NCCL error: ") + ncclGetErrorString(r_) + " at " #call); \
    } while (0)

// Equal-work contiguous i-ranges: sym rows i hold (n-i)(n-i+1)/2 sorted triples, asym n^2.
std::vector<int> group_slices(int n, bool sym, int nranks) {
    std::vector<int> bounds(1, 0);
    long double tot = 0, acc = 0;
    for (int i = 0; i < n; ++i) tot += sym ? 0.5L * (n - i) * (n - i + 1) : static_cast<long double>(n) * n;
    int r = 1;
    for (int i = 0; i < n; ++i) {
        acc += sym ? 0.5L * (n - i) * (n - i + 1) : static_cast<long double>(n) * n;
        while (r < nranks && acc >= tot * r / nranks) {
            bounds.push_back(i + 1);
            ++r;
        }
    }
    while (static_cast<int>(bounds.size()) < nranks) bounds.push_back(n);
    bounds.push_back(n);
    return bounds;
}

// Restarts [t0, t1) of rank r: blocks of ceil(L / nranks), so tau = rank x block + local.
inline void restart_chunk(int L, int nranks, int rank, int* t0, int* t1) {
    const int blk = (L + nranks - 1) / nranks;
    *t0 = std::min(L, rank * blk);
    *t1 = std::min(L, (rank + 1) * blk);
}

__global__ void k_pad_values(const double* __restrict__ in, int n, int len, double* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x < len) out[x] = x < n ? in[x] : -INFINITY;
}

struct Local {
    skc_sym_set* s;
    skc_context* ctx;
};

std::vector<Local> check_group(skc_sym_set* const* sets, int nsets) {
    require(sets != nullptr && nsets >= 1, "group: need at least one local set");
    std::vector<Local> v;
    for (int d = 0; d < nsets; ++d) {
        check_vec(sets[d], "group: set");
        const skc_sym_set* a = sets[0];
        const skc_sym_set* b = sets[d];
        require(a->n == b->n && a->b == b->b && a->B == b->B && a->seed == b->seed,
                "group: local sets must be replicas (same n, b, B, seed)");
        require(b->ctx->nranks == sets[0]->ctx->nranks, "group: local contexts belong to different communicators");
        require(b->ctx->nranks == 1 || b->ctx->comm != nullptr, "group: context has no communicator");
        v.push_back({sets[d], sets[d]->ctx});
    }
    require(nsets <= sets[0]->ctx->nranks, "group: more local sets than ranks");
    return v;
}

// ncclGroupStart/End around one collective per local rank (single-thread multi-GPU).
template <typename F>
void each_collective(std::vector<Local>& loc, F&& f) {
    if (loc[0].ctx->nranks == 1) return;
    NC(ncclGroupStart());
    for (auto& l : loc) f(l);
    NC(ncclGroupEnd());
}

void dense_group_attempt(std::vector<Local>& loc, const void* const* T, int dtype, int location, bool two_limb,
                         bool* overflow, bool* hdr) {
    const int n = loc[0].s->n, R = loc[0].ctx->nranks;
    const std::vector<int> bounds = group_slices(n, true, R);
    std::vector<BuildPlan> plans(loc.size());
    std::vector<const void*> Tdev(loc.size());
    for (size_t d = 0; d < loc.size(); ++d) {
        skc_context* ctx = loc[d].ctx;
        skc_sym_set* s = loc[d].s;
        ctx->use();
        const int i0 = bounds[ctx->rank], i1 = bounds[ctx->rank + 1];
        bool zc = false;
        Tdev[d] = stage_tensor(ctx, T[d], n, dtype, location, true, i0, i1, false, nullptr, &zc);
        BuildPlan& p = plans[d];
        prepare_dense_build(ctx, n, dtype, true, i0, i1, s->B, s->b, s->packed.p, s->data.p, zc, two_limb, p);
        p.total_entries = static_cast<long long>(n) * (n + 1) * (n + 2) / 6;  // the whole build (global mean)
        // the same partial count on every rank (the all-gather concatenates them)
        p.prepass_blocks = std::min(kPrepassBlocks, std::max(1, ctx->sms) * 5);
        p.pdl = false;
        ensure_build_scratch_clean(ctx);
        ctx->build_scratch_clean = false;
        CK(cudaMemsetAsync(p.nonfinite, 0, sizeof(int), ctx->stream));
        {
            SKC_PROF(ctx, "build_prepass");
            launch_build_prepass(ctx->stream, Tdev[d], p);  // (an empty slice writes zero partials)
        }
        ctx->check_launch();
        ctx->gathered.alloc(4ull * p.prepass_blocks * R);
    }
    each_collective(loc, [&](Local& l) {
        const size_t d = &l - loc.data();
        NC(ncclAllGather(plans[d].prepass_partials, l.ctx->gathered.p, 4ull * plans[d].prepass_blocks, ncclDouble,
                         l.ctx->comm, l.ctx->stream));
    });
    for (size_t d = 0; d < loc.size(); ++d) {
        skc_context* ctx = loc[d].ctx;
        ctx->use();
        BuildPlan& p = plans[d];
        if (R > 1) {
            p.prepass_partials = ctx->gathered.p;
            p.nseg = R;
        }
        {
            SKC_PROF(ctx, "build_main");
            launch_build_main(ctx->stream, Tdev[d], p);
        }
        ctx->check_launch();
    }
    each_collective(loc, [&](Local& l) {
        const BuildPlan& p = plans[&l - loc.data()];
        NC(ncclAllReduce(p.acc, p.acc, static_cast<size_t>(p.total_slots), ncclInt64, ncclSum, l.ctx->comm,
                         l.ctx->stream));
        // nonfinite (ints[1]) and one-limb overflow (ints[3]) flags: any rank's
        NC(ncclAllReduce(p.nonfinite, p.nonfinite, 3, ncclInt32, ncclMax, l.ctx->comm, l.ctx->stream));
    });
    std::vector<int*> flags(loc.size());
    for (size_t d = 0; d < loc.size(); ++d) {
        skc_context* ctx = loc[d].ctx;
        ctx->use();
        {
            SKC_PROF(ctx, "build_finalize");
            launch_build_finalize(ctx->stream, plans[d]);
        }
        ctx->build_scratch_clean = true;
        ctx->check_launch();
        flags[d] = ctx->pinned_ints();
        CK(cudaMemcpyAsync(flags[d], plans[d].nonfinite, 3 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    }
    bool nonfinite = false;
    *overflow = false;
    *hdr = false;
    for (size_t d = 0; d < loc.size(); ++d) {
        loc[d].ctx->use();
        loc[d].ctx->sync();
        nonfinite |= flags[d][0] != 0;
        *overflow |= (flags[d][2] & 1) != 0;
        *hdr |= (flags[d][2] & 2) != 0;
    }
    if (*overflow || *hdr || nonfinite)
        for (size_t d = 0; d < loc.size(); ++d) {
            loc[d].ctx->use();
            CK(cudaMemsetAsync(plans[d].ovf, 0, sizeof(int), loc[d].ctx->stream));
            loc[d].ctx->sync();
        }
    if (nonfinite) fail(kInvalidArgument, "accumulate_dense: tensor has a non-finite entry");
}

}  // namespace skcabi

extern "C" {

int skc_nccl_unique_id(char* out) {
    return guard([&] {
        check_vec(out, "nccl_unique_id: out");
        ncclUniqueId id;
        NC(ncclGetUniqueId(&id));
        std::memcpy(out, id.internal, sizeof(id.internal));
    });
}

int skc_context_comm_init(skc_context* ctx, int nranks, int rank, const char* id) {
    return guard([&] {
        check_vec(ctx, "context");
        check_vec(id, "comm_init: id");
        require(nranks >= 1 && rank >= 0 && rank < nranks, "comm_init: bad rank / rank count");
        require(ctx->comm == nullptr, "comm_init: context already has a communicator");
        ctx->use();
        ncclUniqueId u;
        std::memcpy(u.internal, id, sizeof(u.internal));
        ncclComm_t c = nullptr;
        NC(ncclCommInitRank(&c, nranks, u, rank));
        ctx->comm = c;
        ctx->rank = rank;
        ctx->nranks = nranks;
    });
}

int skc_group_create(const int* devices, int ndev, skc_context** ctxs_out) {
    return guard([&] {
        check_vec(devices, "group_create: devices");
        check_vec(ctxs_out, "group_create: out");
        require(ndev >= 1, "group_create: need at least one device");
        for (int d = 0; d < ndev; ++d)
            for (int e = 0; e < d; ++e)
                require(devices[d] != devices[e], "group_create: a device appears twice (one rank per GPU)");
        std::vector<skc_context*> ctxs(ndev, nullptr);
        auto cleanup = [&] {
            for (auto* c : ctxs)
                if (c) skc_context_destroy(c);
        };
        for (int d = 0; d < ndev; ++d) {
            const int rc = skc_context_create(devices[d], &ctxs[d]);
            if (rc != kOk) {
                const std::string msg = g_last_error;
                cleanup();
                fail(rc, msg);
            }
        }
        std::vector<ncclComm_t> comms(ndev, nullptr);
        const ncclResult_t r = ncclCommInitAll(comms.data(), ndev, devices);
        if (r != ncclSuccess) {
            cleanup();
            fail(kCudaError, std::string("NCCL error: ") + ncclGetErrorString(r) + " at ncclCommInitAll");
        }
        for (int d = 0; d < ndev; ++d) {
            ctxs[d]->comm = comms[d];
            ctxs[d]->rank = d;
            ctxs[d]->nranks = ndev;
            ctxs_out[d] = ctxs[d];
        }
    });
}

int skc_context_comm_info(const skc_context* ctx, int* nranks, int* rank) {
    return guard([&] {
        check_vec(ctx, "context");
        if (nranks) *nranks = ctx->nranks;
        if (rank) *rank = ctx->rank;
    });
}

int skc_group_slices(int n, int sym, int nranks, int* bounds) {
    return guard([&] {
        check_vec(bounds, "group_slices: bounds");
        require(n >= 0 && nranks >= 1, "group_slices: bad arguments");
        const std::vector<int> b = group_slices(n, sym != 0, nranks);
        std::copy(b.begin(), b.end(), bounds);
    });
}

int skc_group_restart_chunk(int L, int nranks, int rank, int* t0, int* t1) {
    return guard([&] {
        check_vec(t0, "restart_chunk: t0");
        check_vec(t1, "restart_chunk: t1");
        require(L >= 0 && nranks >= 1 && rank >= 0 && rank < nranks, "restart_chunk: bad arguments");
        restart_chunk(L, nranks, rank, t0, t1);
    });
}

int skc_sym_accumulate_dense_group(skc_sym_set* const* sets, int nsets, const void* const* T, int dtype, int location,
                                   int assume_symmetric) {
    return guard([&] {
        std::vector<Local> loc = check_group(sets, nsets);
        check_vec(T, "accumulate_dense: tensors");
        require(dtype == SKC_F64 || dtype == SKC_F32, "accumulate_dense: dtype must be SKC_F64 or SKC_F32");
        require(location == SKC_HOST || location == SKC_DEVICE, "accumulate_dense: bad location");
        const int n = loc[0].s->n;
        require(n <= 65535, "accumulate_dense: n above 65535 is not supported");
        for (int d = 0; d < nsets; ++d) check_vec(T[d], "accumulate_dense: tensor");
        if (!assume_symmetric)  // every rank checks the whole tensor: identical verdicts
            for (auto& l : loc) {
                l.ctx->use();
                const void* Tf = stage_tensor(l.ctx, T[&l - loc.data()], n, dtype, location, true, 0, n, true, nullptr);
                check_symmetric(l.ctx, Tf, dtype, n);
            }
        for (auto& l : loc) l.s->version++;  // sketch.cpp:324
        bool overflow = false, hdr = false;
        dense_group_attempt(loc, T, dtype, location, false, &overflow, &hdr);
        if (overflow && !hdr) {  // a one-limb window overflowed: every rank redoes the build with two limbs
            for (auto& l : loc) ++l.ctx->build_two_limb_retries;
            dense_group_attempt(loc, T, dtype, location, true, &overflow, &hdr);
        }
        if (hdr) {
            // high dynamic range (the same verdict on every rank): each rank builds its slice in
            // magnitude bands, rank 0 onto the shared prior and the others onto zero, and the
            // replicas' data are summed (fp64; bit identity across rank counts does not carry
            // over to this path)
            const std::vector<int> bounds = group_slices(n, true, loc[0].ctx->nranks);
            for (size_t d = 0; d < loc.size(); ++d) {
                skc_context* ctx = loc[d].ctx;
                skc_sym_set* s = loc[d].s;
                ctx->use();
                const int i0 = bounds[ctx->rank], i1 = bounds[ctx->rank + 1];
                bool zc = false;
                const void* Td = stage_tensor(ctx, T[d], n, dtype, location, true, i0, i1, false, nullptr, &zc);
                if (ctx->nranks > 1 && ctx->rank != 0)
                    CK(cudaMemsetAsync(s->data.p, 0, sizeof(double2) * s->B * s->b, ctx->stream));
                run_dense_build_banded(ctx, Td, n, dtype, true, i0, i1, s->B, s->b, s->packed.p, s->data.p, zc);
            }
            each_collective(loc, [&](Local& l) {
                NC(ncclAllReduce(l.s->data.p, l.s->data.p, 2ull * l.s->B * l.s->b, ncclDouble, ncclSum, l.ctx->comm,
                                 l.ctx->stream));
            });
            for (auto& l : loc) {
                l.ctx->use();
                l.ctx->sync();
            }
        }
    });
}

int skc_sym_accumulate_moment_group(skc_sym_set* const* sets, int nsets, const double* const* X, const double* const* w,
                                    long long N, int location) {
    return guard([&] {
        std::vector<Local> loc = check_group(sets, nsets);
        require(N >= 0, "accumulate_moment: negative sample count");
        if (N == 0) return;
        check_vec(X, "accumulate_moment: X");
        const int n = loc[0].s->n, R = loc[0].ctx->nranks;
        for (size_t d = 0; d < loc.size(); ++d) {
            skc_context* ctx = loc[d].ctx;
            skc_sym_set* s = loc[d].s;
            ctx->use();
            check_vec(X[d], "accumulate_moment: X");
            const long long a = N * ctx->rank / R, e = N * (ctx->rank + 1) / R, Nd = e - a;
            const double* wsrc = w ? w[d] : nullptr;
            if (Nd > 0) {
                const double* Xd = X[d] + a * n;
                const double* wd = wsrc ? wsrc + a : nullptr;
                if (location == SKC_HOST) {
                    ctx->X.upload(Xd, static_cast<size_t>(Nd) * n, ctx->stream);
                    Xd = ctx->X.p;
                    if (wd) {
                        ctx->values.upload(wd, static_cast<size_t>(Nd), ctx->stream);
                        wd = ctx->values.p;
                    }
                }
                sym_moment_partial(s, Xd, wd, Nd);
            } else {
                ctx->tmp.alloc(static_cast<size_t>(s->B) * s->b);
                CK(cudaMemsetAsync(ctx->tmp.p, 0, sizeof(double2) * s->B * s->b, ctx->stream));
            }
        }
        each_collective(loc, [&](Local& l) {
            NC(ncclAllReduce(l.ctx->tmp.p, l.ctx->tmp.p, 2ull * l.s->B * l.s->b, ncclDouble, ncclSum, l.ctx->comm,
                             l.ctx->stream));
        });
        for (auto& l : loc) {
            l.ctx->use();
            l.s->version++;
            sym_moment_combine(l.s, 1.0);
        }
        for (auto& l : loc) {
            l.ctx->use();
            l.ctx->sync();
        }
    });
}

int skc_sym_rtpm_group(skc_sym_set* const* sets, int nsets, int k, int L, int T_iters, uint64_t seed, double tol,
                       const double* inits, double* lambda, double* V, int* best_tau) {
    return guard([&] {
        std::vector<Local> loc = check_group(sets, nsets);
        check_vec(lambda, "rtpm: lambda");
        check_vec(V, "rtpm: V");
        const int n = loc[0].s->n, R = loc[0].ctx->nranks;
        // decompose.cpp:15-20
        if (k < 1 || L < 1 || T_iters < 1) fail(kInvalidArgument, "power method: k, L and T must be positive");
        if (k > n) fail(kInvalidArgument, "power method: target rank exceeds tensor dimension");
        require(loc[0].s->B <= 128, "median over more than 128 replicates is not supported");
        const int blk = (L + R - 1) / R;
        std::vector<double> gen(static_cast<size_t>(L) * n);
        for (auto& l : loc) {
            l.ctx->use();
            l.ctx->ints.alloc(16);
            l.ctx->dbl.alloc(4);
            l.ctx->X.alloc(static_cast<size_t>(n));
            l.ctx->gathered.alloc(static_cast<size_t>(2) * blk * R + 2 * blk);
        }
        for (int c = 0; c < k; ++c) {
            const double* U0;
            if (inits) {
                U0 = inits + static_cast<size_t>(c) * L * n;
            } else {  // Rng(derive_seed(seed, 0x31, c, tau)).unit_sphere(n) (decompose.cpp:96-97)
#pragma omp parallel for schedule(static)
                for (int t = 0; t < L; ++t) {
                    Rng rng(derive_seed(seed, seed_tag::kPowerInit, static_cast<std::uint64_t>(c),
                                        static_cast<std::uint64_t>(t)));
                    rng.unit_sphere(n, gen.data() + static_cast<size_t>(t) * n);
                }
                U0 = gen.data();
            }
            std::vector<int> t0(loc.size()), t1(loc.size());
            for (size_t d = 0; d < loc.size(); ++d) {
                skc_context* ctx = loc[d].ctx;
                ctx->use();
                restart_chunk(L, R, ctx->rank, &t0[d], &t1[d]);
                const int Ld = t1[d] - t0[d];
                double* padded = ctx->gathered.p + static_cast<size_t>(blk) * R;  // this rank's block of values
                if (Ld > 0) {
                    ctx->U.upload(U0 + static_cast<size_t>(t0[d]) * n, static_cast<size_t>(Ld) * n, ctx->stream);
                    rtpm_restarts_device(loc[d].s, Ld, T_iters, tol);
                    k_pad_values<<<(blk + 255) / 256, 256, 0, ctx->stream>>>(ctx->values.p, Ld, blk, padded);
                } else {
                    ctx->flags.alloc(1);
                    CK(cudaMemsetAsync(ctx->flags.p, 0, sizeof(int), ctx->stream));
                    k_pad_values<<<(blk + 255) / 256, 256, 0, ctx->stream>>>(nullptr, 0, blk, padded);
                }
                count_launch();
                ctx->check_launch();
            }
            // all values in tau order on every rank, -inf in the padding of the last blocks
            each_collective(loc, [&](Local& l) {
                NC(ncclAllGather(l.ctx->gathered.p + static_cast<size_t>(blk) * R, l.ctx->gathered.p, blk, ncclDouble,
                                 l.ctx->comm, l.ctx->stream));
            });
            std::vector<int> bt(loc.size());
            std::vector<double> lam(loc.size());
            for (size_t d = 0; d < loc.size(); ++d) {
                skc_context* ctx = loc[d].ctx;
                ctx->use();
                const double* all = R > 1 ? ctx->gathered.p : ctx->gathered.p + static_cast<size_t>(blk) * R;
                // the first maximum over tau (strict >, decompose.cpp:101-108)
                launch_argmax_first(ctx->stream, all, blk * R, ctx->ints.p + 2, ctx->dbl.p);
                ctx->check_launch();
                CK(cudaMemcpyAsync(&bt[d], ctx->ints.p + 2, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
                CK(cudaMemcpyAsync(&lam[d], ctx->dbl.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
            }
            int degenerate = 0;
            for (size_t d = 0; d < loc.size(); ++d) {
                loc[d].ctx->use();
                const int Lf = std::max(1, t1[d] - t0[d]);  // (an empty block holds one zero flag)
                std::vector<int> f(Lf);
                CK(cudaMemcpyAsync(f.data(), loc[d].ctx->flags.p, sizeof(int) * Lf, cudaMemcpyDeviceToHost,
                                   loc[d].ctx->stream));
                loc[d].ctx->sync();
                for (int x : f) degenerate |= x;
            }
            if (R > 1) {  // any rank's degenerate restart fails every rank (same decision everywhere)
                std::vector<DevBuf<int>> fl(loc.size());
                for (size_t d = 0; d < loc.size(); ++d) {
                    loc[d].ctx->use();
                    fl[d].upload(&degenerate, 1, loc[d].ctx->stream);
                }
                each_collective(loc, [&](Local& l) {
                    const size_t d = &l - loc.data();
                    NC(ncclAllReduce(fl[d].p, fl[d].p, 1, ncclInt32, ncclMax, l.ctx->comm, l.ctx->stream));
                });
                for (size_t d = 0; d < loc.size(); ++d) {
                    loc[d].ctx->use();
                    int g = 0;
                    CK(cudaMemcpyAsync(&g, fl[d].p, sizeof(int), cudaMemcpyDeviceToHost, loc[d].ctx->stream));
                    loc[d].ctx->sync();
                    degenerate |= g;
                }
            }
            if (degenerate) fail(kDegenerate, "power update produced a vanishing iterate");  // decompose.cpp:37-38
            for (size_t d = 1; d < loc.size(); ++d)
                require(bt[d] == bt[0] && lam[d] == lam[0], "rtpm: ranks disagree on the selected restart");
            const int tau = bt[0], owner = tau / blk;
            lambda[c] = lam[0];
            if (best_tau) best_tau[c] = tau;
            // the winner's vector: copied from the owner's batch, broadcast to every rank
            for (size_t d = 0; d < loc.size(); ++d)
                if (loc[d].ctx->rank == owner) {
                    loc[d].ctx->use();
                    CK(cudaMemcpyAsync(loc[d].ctx->X.p, loc[d].ctx->U.p + static_cast<size_t>(tau - t0[d]) * n, n * 8,
                                       cudaMemcpyDeviceToDevice, loc[d].ctx->stream));
                }
            each_collective(loc, [&](Local& l) {
                NC(ncclBroadcast(l.ctx->X.p, l.ctx->X.p, n, ncclDouble, owner, l.ctx->comm, l.ctx->stream));
            });
            loc[0].ctx->use();
            CK(cudaMemcpyAsync(V + static_cast<size_t>(c) * n, loc[0].ctx->X.p, n * 8, cudaMemcpyDeviceToHost,
                               loc[0].ctx->stream));
            // deflation add_scaled_rank1(v, -lambda) on every replica (decompose.cpp:112)
            for (auto& l : loc) {
                l.ctx->use();
                if (lam[0] != 0.0) {
                    l.s->version++;
                    sym_moment_partial(l.s, l.ctx->X.p, nullptr, 1);
                    sym_moment_combine(l.s, -lam[0]);
                }
            }
            for (auto& l : loc) {
                l.ctx->use();
                l.ctx->sync();
            }
        }
    });
}

int skc_sym_sketch_whitened_m3_group(skc_sym_set* const* sets, int nsets, int V, long long D, const long long* doc_ptr,
                                     const int* word, const int* count, const double* W, double alpha0,
                                     long long* used_out, long long* skipped_out) {
    return guard([&] {
        std::vector<Local> loc = check_group(sets, nsets);
        check_vec(doc_ptr, "sketch_whitened_m3: doc_ptr");
        check_vec(W, "sketch_whitened_m3: W");
        require(V >= 1 && D >= 0, "sketch_whitened_m3: invalid corpus dimensions");
        const int R = loc[0].ctx->nranks;
        std::vector<CorpusDev> corp(loc.size());
        std::vector<DevBuf<double>> glob(loc.size());  // [m1 sums (V), used1, used3]
        for (size_t d = 0; d < loc.size(); ++d) {
            skc_context* ctx = loc[d].ctx;
            ctx->use();
            const long long a = D * ctx->rank / R, e = D * (ctx->rank + 1) / R;
            // the rank's document block as its own CSR
            std::vector<long long> ptr(static_cast<size_t>(e - a) + 1);
            for (long long x = a; x <= e; ++x) ptr[x - a] = doc_ptr[x] - doc_ptr[a];
            upload_corpus(ctx, V, e - a, ptr.data(), word ? word + doc_ptr[a] : nullptr,
                          count ? count + doc_ptr[a] : nullptr, corp[d], "sketch_whitened_m3", false);
            glob[d].alloc(static_cast<size_t>(V) + 2);
            CK(cudaMemcpyAsync(glob[d].p, corp[d].m1p.p, sizeof(double) * V, cudaMemcpyDeviceToDevice, ctx->stream));
            const double cnt[2] = {static_cast<double>(corp[d].used1), static_cast<double>(corp[d].used3)};
            CK(cudaMemcpyAsync(glob[d].p + V, cnt, sizeof(cnt), cudaMemcpyHostToDevice, ctx->stream));
            ctx->sync();
        }
        each_collective(loc, [&](Local& l) {
            const size_t d = &l - loc.data();
            NC(ncclAllReduce(glob[d].p, glob[d].p, static_cast<size_t>(V) + 2, ncclDouble, ncclSum, l.ctx->comm,
                             l.ctx->stream));
        });
        std::vector<double> g(static_cast<size_t>(V) + 2);
        loc[0].ctx->use();
        CK(cudaMemcpyAsync(g.data(), glob[0].p, sizeof(double) * g.size(), cudaMemcpyDeviceToHost, loc[0].ctx->stream));
        loc[0].ctx->sync();
        if (!(g[V] > 0)) fail(kInvalidArgument, "compute_m1: no nonempty documents");
        const long long gused = static_cast<long long>(std::llround(g[V + 1]));
        require(gused >= 1, "sketch_whitened_m3: no documents with >= 3 words");
        std::vector<double> m1(g.begin(), g.begin() + V);
        for (double& x : m1) x /= g[V];  // lda.cpp:99
        long long stats[2] = {0, 0};
        std::vector<DevBuf<long long>> st(loc.size());
        for (size_t d = 0; d < loc.size(); ++d) {
            skc_context* ctx = loc[d].ctx;
            skc_sym_set* s = loc[d].s;
            ctx->use();
            // every replica holds the same prior sketch: rank 0 keeps it, the others add their
            // shard to zero, so the data all-reduce counts it once
            if (R > 1 && ctx->rank != 0)
                CK(cudaMemsetAsync(s->data.p, 0, sizeof(double2) * s->B * s->b, ctx->stream));
            long long u = 0, sk = 0;
            sketch_whitened_m3_dev(s, corp[d], W, alpha0, &u, &sk, gused, m1.data(), ctx->rank == 0);
            const long long us[2] = {u, sk};
            st[d].upload(us, 2, ctx->stream);
        }
        each_collective(loc, [&](Local& l) {
            const size_t d = &l - loc.data();
            NC(ncclAllReduce(l.s->data.p, l.s->data.p, 2ull * l.s->B * l.s->b, ncclDouble, ncclSum, l.ctx->comm,
                             l.ctx->stream));
            NC(ncclAllReduce(st[d].p, st[d].p, 2, ncclInt64, ncclSum, l.ctx->comm, l.ctx->stream));
        });
        for (size_t d = 0; d < loc.size(); ++d) {
            loc[d].ctx->use();
            loc[d].s->version++;
            CK(cudaMemcpyAsync(stats, st[d].p, sizeof(stats), cudaMemcpyDeviceToHost, loc[d].ctx->stream));
            loc[d].ctx->sync();
        }
        if (used_out) *used_out = stats[0];
        if (skipped_out) *skipped_out = stats[1];
    });
}

}  // extern "C"
