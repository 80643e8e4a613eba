"""Multi-GPU C-ABI (include/sketchcp_b200.h, multi-GPU section) on the GPUs present.

This run has one B200, so the communicators here have one rank: ncclCommInitAll over
[0] (skc_group_create) and ncclCommInitRank with a fresh id (skc_context_comm_init).
They run the whole group code path -- slicing, the pre-pass all-gather layout, the
exact-accumulator all-reduce, the restart blocks and argmax over the gathered values,
the broadcast and deflation -- and must reproduce the single-context results bit for
bit (dense build, RTPM) or to rounding (moment, LDA). With more GPUs visible the same
tests run over all of them (bit-identity of the dense build and RTPM holds at any rank
count: int64 sums are order-free, restarts do not interact)."""
import numpy as np
import pytest

import oracle_py as O

pytestmark = pytest.mark.gpu


def skb():
    import paper_1506_04448_b200 as m

    return m


@pytest.fixture(scope="module")
def group():
    n = skb().device_count()
    return skb().group_contexts(list(range(n)))


def sym_tensor(n, seed):
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(n, n, n))
    return (A + A.transpose(0, 2, 1) + A.transpose(1, 0, 2) + A.transpose(1, 2, 0) + A.transpose(2, 0, 1)
            + A.transpose(2, 1, 0)) / 6.0


@pytest.mark.parametrize("n,b,B,dtype", [(40, 4096, 6, np.float64), (120, 16384, 4, np.float32),
                                         (400, 1 << 14, 20, np.float64)])
def test_group_dense_build_bit_identical_to_single(gpu_ctx, group, n, b, B, dtype):
    if n == 400:
        T, _, _ = skb().gen_planted_tensor(n, 50, 0.01, 20150615)
    else:
        T = sym_tensor(n, 5).astype(dtype)
    ref = skb().SymTensorSketchSet(n, b, B, 9, gpu_ctx)
    ref.accumulate_dense(T, assume_symmetric=True)
    reps = skb().SymReplicas(n, b, B, 9, group)
    reps.accumulate_dense(T, assume_symmetric=True)
    for r in range(len(reps)):
        assert np.array_equal(reps.data(r), ref.data())
    # accumulate semantics: a second build adds on top, still identical
    ref.accumulate_dense(T, assume_symmetric=True)
    reps.accumulate_dense(T, assume_symmetric=True)
    assert np.array_equal(reps.data(0), ref.data())


def test_group_dense_build_device_inputs_and_errors(gpu_ctx, group):
    import torch

    n, b, B = 64, 2048, 5
    T = sym_tensor(n, 8)
    ref = skb().SymTensorSketchSet(n, b, B, 3, gpu_ctx)
    ref.accumulate_dense(T, assume_symmetric=True)
    reps = skb().SymReplicas(n, b, B, 3, group)
    reps.accumulate_dense([torch.from_numpy(T).to(f"cuda:{c.device}") for c in group], assume_symmetric=True)
    assert np.array_equal(reps.data(0), ref.data())
    bad = T.copy()
    bad[3, 4, 5] = np.nan
    with pytest.raises(ValueError):
        reps.accumulate_dense(bad, assume_symmetric=True)
    assert np.array_equal(reps.data(0), ref.data())  # untouched
    asym = T.copy()
    asym[1, 2, 3] += 1.0
    with pytest.raises(ValueError, match="not symmetric"):
        reps.accumulate_dense(asym, assume_symmetric=False)


def test_group_rtpm_bit_identical_to_single(gpu_ctx, group):
    n, b, B = 100, 1 << 12, 20
    T, _, _ = skb().gen_planted_tensor(n, 10, 0.01, 11)
    ref = skb().SymTensorSketchSet(n, b, B, 5, gpu_ctx)
    ref.accumulate_dense(T, assume_symmetric=True)
    reps = skb().SymReplicas(n, b, B, 5, group)
    reps.accumulate_dense(T, assume_symmetric=True)
    cfg = skb().PowerConfig(k=4, L=50, T_iters=30, seed=3)
    d1 = skb().robust_tpm_fast(ref, cfg)
    d2 = reps.rtpm(cfg)
    assert np.array_equal(d1.lambda_, d2.lambda_)
    assert np.array_equal(d1.A, d2.A)
    assert np.array_equal(d1.best_tau, d2.best_tau)
    for r in range(len(reps)):  # every replica left deflated like the single set
        assert np.array_equal(reps.data(r), ref.data())


def test_group_rtpm_restart_blocks_match_oracle_selection(gpu_ctx):
    """The restart blocks of R ranks, run one after another through skc_sym_rtpm_restarts,
    give values whose concatenation's first maximum is the oracle's selected restart
    (decompose.cpp:101-108) -- the plumbing of the R-rank path checked on one GPU."""
    n, b, B, L, T_it = 60, 4096, 10, 24, 12
    Tn = sym_tensor(n, 2)
    s = skb().SymTensorSketchSet(n, b, B, 7, gpu_ctx)
    s.accumulate_dense(Tn, assume_symmetric=True)
    inits = skb().power_inits(4, n, 1, L)
    o = O.SymSet(n, b, B, 7)
    o.set_data(s.data())
    lo, Vo, bto = o.rtpm(1, L, T_it, seed=4, inits=inits)
    from paper_1506_04448_b200.distributed import GpuShardCompute

    be = GpuShardCompute(s)
    for R in (1, 2, 3, 5, 8):
        vals = []
        for r in range(R):
            t0, t1 = skb().group_restart_chunk(L, R, r)
            blk = -(-L // R)
            v = np.full(blk, -np.inf)
            if t1 > t0:
                _, vv = be.restarts(inits[0, t0:t1], T_it, 1e-12)
                v[: t1 - t0] = vv
            vals.append(v)
        allv = np.concatenate(vals)
        tau = int(np.argmax(allv))  # first maximum
        assert tau == int(bto[0])
        assert abs(allv[tau] - lo[0]) <= 1e-9 * abs(lo[0])


def test_group_moment_and_lda_match_single(gpu_ctx, group):
    from lda_fixtures import synthetic_corpus

    n, b, B, N = 50, 4096, 6, 300
    rng = np.random.default_rng(3)
    X = rng.normal(size=(N, n))
    w = rng.uniform(0.5, 1.5, size=N) / N
    ref = skb().SymTensorSketchSet(n, b, B, 21, gpu_ctx)
    ref.accumulate_moment(X, w)
    reps = skb().SymReplicas(n, b, B, 21, group)
    reps.accumulate_moment(X, w)
    d, r = reps.data(0), ref.data()
    assert np.max(np.linalg.norm(d - r, axis=1) / np.linalg.norm(r, axis=1)) <= 1e-12
    V, k = 300, 12
    doc_ptr, word, count, W = synthetic_corpus(V=V, k=k, D=400, mean_len=60, seed=2)
    ref2 = skb().SymTensorSketchSet(k, 2048, 5, 4, gpu_ctx)
    u1 = ref2.sketch_whitened_m3(V, doc_ptr, word, count, W, 1.0)
    reps2 = skb().SymReplicas(k, 2048, 5, 4, group)
    u2 = reps2.sketch_whitened_m3(V, doc_ptr, word, count, W, 1.0)
    assert u1 == u2
    d, r = reps2.data(0), ref2.data()
    assert np.max(np.linalg.norm(d - r, axis=1) / np.linalg.norm(r, axis=1)) <= 1e-12


def test_comm_init_one_process_per_rank(gpu_ctx):
    """The torchrun layout: a context joins a communicator by id (ncclCommInitRank)."""
    ctx = skb().Context(0)
    ctx.comm_init(1, 0, skb().nccl_unique_id())
    assert ctx.comm_info() == (1, 0)
    n, b, B = 48, 2048, 4
    T = sym_tensor(n, 6)
    ref = skb().SymTensorSketchSet(n, b, B, 2, gpu_ctx)
    ref.accumulate_dense(T, assume_symmetric=True)
    reps = skb().SymReplicas(n, b, B, 2, [ctx])
    reps.accumulate_dense(T, assume_symmetric=True)
    assert np.array_equal(reps.data(0), ref.data())
