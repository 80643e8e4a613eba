"""GPU parity of the sm_100a path against the CPU oracle, through the C-ABI.

Tolerances (BASELINE.json north_star): hash tables bit-exact; sketches
per-replicate ||d||_2/||s||_2 <= 1e-9 (fp64 input) and <= 1e-4 (fp32 input);
contraction vectors ||d||_inf/||v||_inf <= 1e-9; RTPM (lambda_k, v_k) relative
<= 1e-9 after sign/permutation alignment.
"""
import json
import pathlib

import numpy as np
import pytest

import oracle_py as O

pytestmark = pytest.mark.gpu

SKETCH_TOL = 1e-9
SKETCH_TOL_F32 = 1e-4
VEC_TOL = 1e-9
GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"


def skb():
    import paper_1506_04448_b200 as m

    return m


def sym_tensor(n, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(n, n, n)) * scale
    return sum(A.transpose(p) for p in [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]) / 6


def rel_per_replicate(got, ref):
    num = np.linalg.norm(got - ref, axis=-1)
    den = np.maximum(np.linalg.norm(ref, axis=-1), 1e-300)
    return float(np.max(num / den))


def vec_rel(got, ref):
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))


# ---------------------------------------------------------------- tables
@pytest.mark.parametrize("n,b,B,seed", [(7, 16, 3, 1), (100, 4096, 20, 0), (257, 2, 2, 99), (33, 1 << 16, 4, 2**63 + 5)])
def test_sym_tables_bit_exact(gpu_ctx, n, b, B, seed):
    s = skb().SymTensorSketchSet(n, b, B, seed, gpu_ctx)
    o = O.SymSet(n, b, B, seed)
    hc, sc = s.coefficients()
    for m in range(B):
        b1, b2, b3, se = s.tables(m)
        ob1, ob2, ob3, ose, ohc, osc = o.tables(m)
        assert np.array_equal(b1, ob1) and np.array_equal(b2, ob2) and np.array_equal(b3, ob3)
        assert np.array_equal(se, ose)
        assert np.array_equal(hc[m], ohc) and np.array_equal(sc[m], osc)


@pytest.mark.parametrize("n,b,B,seed", [(7, 16, 3, 1), (100, 4096, 20, 0), (50, 2, 2, 5)])
def test_asym_tables_bit_exact(gpu_ctx, n, b, B, seed):
    s = skb().AsymTensorSketchSet(n, b, B, seed, gpu_ctx)
    o = O.AsymSet(n, b, B, seed)
    hc, xc = s.coefficients()
    for m in range(B):
        bk, sg = s.tables(m)
        obk, osg, ohc, oxc = o.tables(m)
        assert np.array_equal(bk, obk) and np.array_equal(sg, osg)
        assert np.array_equal(hc[m], ohc) and np.array_equal(xc[m], oxc)


# ---------------------------------------------------------------- dense builds
@pytest.mark.parametrize("n,b,B", [(12, 64, 3), (40, 1024, 5), (64, 4096, 20), (30, 16384, 4), (9, 2, 3), (1, 8, 2)])
def test_sym_dense_build_matches_oracle(gpu_ctx, n, b, B):
    T = sym_tensor(n, n + b)
    s = skb().SymTensorSketchSet(n, b, B, 11, gpu_ctx)
    o = O.SymSet(n, b, B, 11)
    s.accumulate_dense(T, assume_symmetric=True)
    o.accumulate_dense(T, assume_symmetric=True)
    assert rel_per_replicate(s.data(), o.data()) <= SKETCH_TOL
    assert s.version() == 1


@pytest.mark.parametrize("n,b,B,seed", [(40, 1024, 5, 1), (64, 4096, 20, 2), (36, 1 << 16, 3, 3), (17, 64, 4, 4),
                                        (120, 16384, 6, 5), (20, 1 << 15, 2, 6), (24, 1 << 17, 2, 7)])
def test_dense_builds_across_bucket_class_bits_match_oracle(gpu_ctx, n, b, B, seed):
    """Symmetric and asymmetric fp64 builds with 0-3 bucket-class bits (b = 2^6 .. 2^17)
    against the oracle (sketch.cpp:173-193, 315-345)."""
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(n, n, n))
    T = sum(A.transpose(p) for p in [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]) / 6
    s = skb().SymTensorSketchSet(n, b, B, seed, gpu_ctx)
    s.accumulate_dense(T, assume_symmetric=True)
    o = O.SymSet(n, b, B, seed)
    o.accumulate_dense(T, True)
    assert rel_per_replicate(s.data(), o.data()) <= SKETCH_TOL
    a = skb().AsymTensorSketchSet(n, b, B, seed, gpu_ctx)
    a.accumulate_dense(A)
    oa = O.AsymSet(n, b, B, seed)
    oa.accumulate_dense(A)
    assert rel_per_replicate(a.data(), oa.data()) <= SKETCH_TOL


def test_f32_one_limb_build_large_n_matches_oracle(gpu_ctx):
    """n > 1024 (the one-warp class-table path), fp32 device-generated input: the one-limb
    accumulator (|q| < 2^26 with the rare carry into the 64-bit accumulator) against the
    oracle's fp64 sums of the same fp32 entries. Contract: 1e-4 (fp32); the one-limb
    resolution (2^-21 of max kappa|T|: |q| < 2^22, F even) gives ~1e-6 relative for
    Gaussian-like entries (max/rms ~ 6), asserted at 1e-5."""
    import torch

    n, b, B, seed = 1100, 1 << 12, 2, 8
    Td = torch.empty(n ** 3, dtype=torch.float32, device="cuda")
    skb().gen_planted_tensor_device(gpu_ctx, n, 4, 0.01, seed, Td.data_ptr(), dtype=np.float32)
    s = skb().SymTensorSketchSet(n, b, B, seed, gpu_ctx)
    s.accumulate_dense(Td, assume_symmetric=True)
    Th = Td.cpu().numpy().reshape(n, n, n)
    del Td
    o = O.SymSet(n, b, B, seed)
    O.lib().orc_set_num_threads(B)
    o.accumulate_dense_slice(Th, 0, n)
    err = rel_per_replicate(s.data(), o.data())
    assert err <= SKETCH_TOL_F32 and err <= 1e-5, err


def test_f32_one_limb_overflow_falls_back_to_two_limbs(gpu_ctx):
    """An fp32 tensor whose entries all carry the same complex4 sign under replicate 0
    (nonzero only where (e_i + e_j + e_k) mod 4 == 0) drives every real-plane slot of
    that replicate up by same-signed full-scale adds, thousands per slot per window pass:
    the one-limb windows overflow, the build is discarded and repeated with two limbs, and
    the sketch still matches the oracle."""
    import torch

    n, b, B, seed = 700, 64, 1, 3
    o = O.SymSet(n, b, B, seed)
    e = o.tables(0)[3].astype(np.int64)
    T = (((e[:, None, None] + e[None, :, None] + e[None, None, :]) % 4) == 0).astype(np.float32)
    Td = torch.from_numpy(T).cuda().reshape(-1)
    s = skb().SymTensorSketchSet(n, b, B, seed, gpu_ctx)
    before = gpu_ctx.build_retries()
    s.accumulate_dense(Td, assume_symmetric=True)
    assert gpu_ctx.build_retries() == before + 1
    o.accumulate_dense_slice(T, 0, n)
    assert rel_per_replicate(s.data(), o.data()) <= 1e-12  # integer-valued: exact


def test_device_input_ordered_after_torch_stream(gpu_ctx):
    """A device tensor still being produced by in-flight torch kernels on torch's current
    stream: the library stream waits on it (skc_context_wait_stream), so the
    sketch equals the one of the finished tensor."""
    import torch

    n, b, B = 96, 4096, 4
    T = sym_tensor(n, 21)
    ref = skb().SymTensorSketchSet(n, b, B, 5, gpu_ctx)
    ref.accumulate_dense(T, assume_symmetric=True)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        big = torch.randn(4096, 4096, device="cuda")
        for _ in range(20):  # keep the stream busy, then produce the input on it
            big = big @ big * 1e-3
        # H2D copy and an elementwise kernel queued behind the matmuls on the side stream
        Td = torch.from_numpy(T).to("cuda", non_blocking=True).reshape(-1) + 0.0
        s = skb().SymTensorSketchSet(n, b, B, 5, gpu_ctx)
        s.accumulate_dense(Td, assume_symmetric=True)
    assert np.array_equal(s.data(), ref.data())


def test_sym_dense_build_is_deterministic(gpu_ctx):
    T = sym_tensor(48, 3)
    outs = []
    for _ in range(2):
        s = skb().SymTensorSketchSet(48, 2048, 6, 7, gpu_ctx)
        s.accumulate_dense(T, assume_symmetric=True)
        outs.append(s.data())
    assert np.array_equal(outs[0], outs[1])


def test_sym_dense_build_f32_input(gpu_ctx):
    T = sym_tensor(36, 4).astype(np.float32)
    s = skb().SymTensorSketchSet(36, 1 << 16, 3, 5, gpu_ctx)
    o = O.SymSet(36, 1 << 16, 3, 5)
    s.accumulate_dense(T, assume_symmetric=True)
    o.accumulate_dense(T.astype(np.float64), assume_symmetric=True)
    assert rel_per_replicate(s.data(), o.data()) <= SKETCH_TOL_F32


def test_sym_dense_slices_sum_to_whole(gpu_ctx):
    n = 30
    T = sym_tensor(n, 8)
    whole = skb().SymTensorSketchSet(n, 512, 4, 3, gpu_ctx)
    whole.accumulate_dense(T, assume_symmetric=True)
    parts = skb().SymTensorSketchSet(n, 512, 4, 3, gpu_ctx)
    for i0, i1 in [(0, 5), (5, 17), (17, 30)]:
        parts.accumulate_dense(T, assume_symmetric=True, i0=i0, i1=i1)
    assert rel_per_replicate(parts.data(), whole.data()) <= 1e-12


def test_sym_dense_device_tensor_and_accumulate(gpu_ctx):
    import torch

    n = 20
    T = sym_tensor(n, 9)
    s = skb().SymTensorSketchSet(n, 256, 3, 1, gpu_ctx)
    o = O.SymSet(n, 256, 3, 1)
    Td = torch.from_numpy(T).cuda()
    s.accumulate_dense(Td, assume_symmetric=True)
    s.accumulate_dense(Td, assume_symmetric=True)  # accumulates (+=)
    o.accumulate_dense(T, True)
    o.accumulate_dense(T, True)
    assert rel_per_replicate(s.data(), o.data()) <= SKETCH_TOL


def test_sym_dense_pinned_and_pageable_host_inputs(gpu_ctx):
    """Pinned host tensors are read in place over the bus, pageable ones staged by row
    blocks; both must give the device-resident result (and the oracle's)."""
    import torch

    n = 33
    T = sym_tensor(n, 12)
    pinned = torch.from_numpy(T.copy()).pin_memory().numpy()
    ref = O.SymSet(n, 1024, 4, 9)
    ref.accumulate_dense(T, True)
    for src in (T, pinned):
        s = skb().SymTensorSketchSet(n, 1024, 4, 9, gpu_ctx)
        s.accumulate_dense(src, assume_symmetric=True)
        assert rel_per_replicate(s.data(), ref.data()) <= SKETCH_TOL
    sl = skb().SymTensorSketchSet(n, 1024, 4, 9, gpu_ctx)
    sl.accumulate_dense(pinned, assume_symmetric=True, i0=0, i1=10)
    sl.accumulate_dense(T, assume_symmetric=True, i0=10, i1=n)
    assert rel_per_replicate(sl.data(), ref.data()) <= SKETCH_TOL


@pytest.mark.parametrize("sym", [True, False])
def test_dense_pinned_pipelined_build(gpu_ctx, sym):
    """Large enough pinned inputs take the chunked zero-copy pipeline (bus-bound quantize
    of chunk c+1 overlapping the main pass of chunk c, per-chunk exponents); the result
    must match the oracle and the device-resident build, including a NaN rejection that
    leaves the set untouched."""
    import torch

    n = 140 if sym else 48  # sym: 9870 rows; asym: 2304 rows -> also the unpipelined branch
    T = sym_tensor(n, 31)
    pinned = torch.from_numpy(T.copy()).pin_memory().numpy()
    if sym:
        ref = O.SymSet(n, 2048, 6, 4)
        ref.accumulate_dense(T, True)
        s = skb().SymTensorSketchSet(n, 2048, 6, 4, gpu_ctx)
        d = skb().SymTensorSketchSet(n, 2048, 6, 4, gpu_ctx)
        s.accumulate_dense(pinned, assume_symmetric=True)
        d.accumulate_dense(torch.from_numpy(T).cuda(), assume_symmetric=True)
    else:
        ref = O.AsymSet(n, 2048, 6, 4)
        ref.accumulate_dense(T)
        s = skb().AsymTensorSketchSet(n, 2048, 6, 4, gpu_ctx)
        d = skb().AsymTensorSketchSet(n, 2048, 6, 4, gpu_ctx)
        s.accumulate_dense(pinned)
        d.accumulate_dense(torch.from_numpy(T).cuda())
    assert rel_per_replicate(s.data(), ref.data()) <= SKETCH_TOL
    # per-chunk exponents (pinned) vs the global one (device): both exact fixed point at
    # resolutions ~2^-61 of their L1 mass, so they differ only by that rounding
    assert rel_per_replicate(s.data(), d.data()) <= 1e-12
    bad = pinned.copy()
    bad[n - 1, n - 1, n - 1] = np.nan
    bad = torch.from_numpy(bad).pin_memory().numpy()
    before = s.data().copy()
    with pytest.raises(ValueError):
        if sym:
            s.accumulate_dense(bad, assume_symmetric=True)
        else:
            s.accumulate_dense(bad)
    assert np.array_equal(s.data(), before)


def test_sym_dense_symmetry_check_message(gpu_ctx):
    n = 6
    T = sym_tensor(n, 1)
    T[1, 3, 2] += 0.5
    s = skb().SymTensorSketchSet(n, 64, 2, 1, gpu_ctx)
    o = O.SymSet(n, 64, 2, 1)
    with pytest.raises(ValueError) as e:
        s.accumulate_dense(T)
    with pytest.raises(O.OracleError) as eo:
        o.accumulate_dense(T)
    assert str(e.value) == str(eo.value)
    assert s.version() == 0


def test_sym_zero_and_single_entry(gpu_ctx):
    n = 10
    s = skb().SymTensorSketchSet(n, 128, 5, 3, gpu_ctx)
    s.accumulate_dense(np.zeros((n, n, n)), assume_symmetric=True)
    assert not np.any(s.data())
    T = np.zeros((n, n, n))
    for p in [(1, 2, 3), (1, 3, 2), (2, 1, 3), (2, 3, 1), (3, 1, 2), (3, 2, 1)]:
        T[p] = 6.0
    s.accumulate_dense(T, assume_symmetric=True)
    assert s.recover_entry(1, 2, 3) == pytest.approx(6.0, abs=1e-12)
    o = O.SymSet(n, 128, 5, 3)
    o.accumulate_dense(T, True)
    assert s.recover_entry(3, 1, 2) == o.recover_entry(3, 1, 2)


def test_nonfinite_input_rejected(gpu_ctx):
    n = 5
    T = sym_tensor(n, 2)
    T[0, 0, 0] = np.nan
    s = skb().SymTensorSketchSet(n, 64, 2, 1, gpu_ctx)
    with pytest.raises(ValueError):
        s.accumulate_dense(T, assume_symmetric=True)


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_nonfinite_device_tensor_rejected_then_next_build_clean(gpu_ctx, bad):
    """Device-resident builds derive the non-finite flag from the sums pre-pass partials
    (no per-call reset): a rejected build leaves the set untouched and the next valid
    build on the same context succeeds and matches the oracle."""
    import torch

    n = 37
    T = sym_tensor(n, 5)
    ref = O.SymSet(n, 1024, 4, 3)
    ref.accumulate_dense(T, True)
    s = skb().SymTensorSketchSet(n, 1024, 4, 3, gpu_ctx)
    Tb = T.copy()
    for idx in [(3, 7, 20), (7, 20, 3), (20, 3, 7), (3, 20, 7), (7, 3, 20), (20, 7, 3)]:
        Tb[idx] = bad
    before = s.data().copy()
    with pytest.raises(ValueError):
        s.accumulate_dense(torch.from_numpy(Tb).cuda(), assume_symmetric=True)
    assert np.array_equal(s.data(), before)
    s.accumulate_dense(torch.from_numpy(T).cuda(), assume_symmetric=True)
    assert rel_per_replicate(s.data(), ref.data()) <= SKETCH_TOL
    # asymmetric set, large enough for the class-list build (and its lean pre-pass)
    na = 170
    Ta = np.random.default_rng(8).standard_normal((na, na, na))
    aref = O.AsymSet(na, 2048, 2, 5)
    aref.accumulate_dense(Ta)
    a = skb().AsymTensorSketchSet(na, 2048, 2, 5, gpu_ctx)
    Tab = Ta.copy()
    Tab[na - 1, 0, na // 2] = bad
    with pytest.raises(ValueError):
        a.accumulate_dense(torch.from_numpy(Tab).cuda())
    assert not np.any(a.data())
    a.accumulate_dense(torch.from_numpy(Ta).cuda())
    assert rel_per_replicate(a.data(), aref.data()) <= SKETCH_TOL


@pytest.mark.parametrize("n,b,B", [(10, 64, 3), (24, 4096, 6), (16, 1 << 15, 2)])
def test_asym_dense_build_matches_oracle(gpu_ctx, n, b, B):
    T = np.random.default_rng(n).normal(size=(n, n, n))
    s = skb().AsymTensorSketchSet(n, b, B, 17, gpu_ctx)
    o = O.AsymSet(n, b, B, 17)
    s.accumulate_dense(T)
    o.accumulate_dense(T)
    assert rel_per_replicate(s.data(), o.data()) <= SKETCH_TOL
    for (i, j, k) in [(0, 1, 2), (n - 1, 0, n - 1)]:
        assert s.recover_entry(i, j, k) == pytest.approx(o.recover_entry(i, j, k), abs=1e-12)


# ---------------------------------------------------------------- spectra & contractions
@pytest.mark.parametrize("n,b,B", [(12, 64, 3), (50, 4096, 8), (40, 16384, 4), (8, 2, 2), (9, 8, 3)])
def test_sym_contractions_match_oracle(gpu_ctx, n, b, B):
    T = sym_tensor(n, b + n)
    s = skb().SymTensorSketchSet(n, b, B, 23, gpu_ctx)
    o = O.SymSet(n, b, B, 23)
    s.accumulate_dense(T, True)
    o.accumulate_dense(T, True)
    ws = skb().SymContractionWorkspace(s)
    for m in range(B):
        ref = o.cached_transform(m)
        assert np.max(np.abs(ws.cached_transform(m) - ref)) <= 1e-12 * max(np.max(np.abs(ref)), 1e-300)
    rng = np.random.default_rng(5)
    U = rng.normal(size=(7, n))
    U /= np.linalg.norm(U, axis=1, keepdims=True)
    got = ws.Ivv(U)
    for l in range(U.shape[0]):
        assert vec_rel(got[l], o.ivv(U[l])) <= VEC_TOL
    gv = ws.vvv(U)
    for l in range(U.shape[0]):
        ov = o.vvv(U[l])
        assert abs(gv[l] - ov) <= VEC_TOL * max(abs(ov), np.max(np.abs(T)))


def test_sym_golden_fixture(gpu_ctx):
    g = json.loads((GOLDEN / "oracle_golden.json").read_text())["sym_small"]
    n, b, B = g["n"], g["b"], g["B"]
    s = skb().SymTensorSketchSet(n, b, B, g["seed"], gpu_ctx)
    s.accumulate_dense(np.array(g["T"]).reshape(n, n, n))
    ref = (np.array(g["data_re"]) + 1j * np.array(g["data_im"])).reshape(B, b)
    assert rel_per_replicate(s.data(), ref) <= SKETCH_TOL
    ws = skb().SymContractionWorkspace(s)
    assert vec_rel(ws.Ivv(np.array(g["u"])), np.array(g["ivv"])) <= VEC_TOL
    assert abs(ws.vvv(np.array(g["u"])) - g["vvv"]) <= 1e-9 * abs(g["vvv"])


def test_cached_transform_refreshes_on_mutation(gpu_ctx):
    n, b, B = 10, 256, 3
    s = skb().SymTensorSketchSet(n, b, B, 1, gpu_ctx)
    s.accumulate_dense(sym_tensor(n, 1), True)
    ws = skb().SymContractionWorkspace(s)
    f0 = ws.cached_transform(1)
    d = s.data()
    d[1] *= 2
    s.set_data(None, d)
    assert np.allclose(ws.cached_transform(1), 2 * f0, rtol=0, atol=1e-12 * np.max(np.abs(f0)))


# ---------------------------------------------------------------- rank-1 / moment
@pytest.mark.parametrize("n,b,B", [(9, 64, 3), (100, 4096, 20), (50, 16384, 4)])
def test_add_scaled_rank1_matches_oracle(gpu_ctx, n, b, B):
    T = sym_tensor(n, 2)
    u = np.random.default_rng(3).normal(size=n)
    s = skb().SymTensorSketchSet(n, b, B, 4, gpu_ctx)
    o = O.SymSet(n, b, B, 4)
    s.accumulate_dense(T, True)
    o.accumulate_dense(T, True)
    s.add_scaled_rank1(u, -1.75)
    o.add_scaled_rank1(u, -1.75)
    assert rel_per_replicate(s.data(), o.data()) <= SKETCH_TOL
    v0 = s.version()
    s.add_scaled_rank1(u, 0.0)  # alpha == 0 is a no-op (sketch.cpp:349)
    assert s.version() == v0


def test_moment_equals_sum_of_rank1(gpu_ctx):
    n, b, B, N = 12, 512, 4, 37
    rng = np.random.default_rng(8)
    X = rng.normal(size=(N, n))
    w = rng.uniform(size=N)
    s = skb().SymTensorSketchSet(n, b, B, 9, gpu_ctx)
    s.accumulate_moment(X, w)
    o = O.SymSet(n, b, B, 9)
    for i in range(N):
        o.add_scaled_rank1(X[i], w[i])
    assert rel_per_replicate(s.data(), o.data()) <= SKETCH_TOL
    d = O.SymSet(n, b, B, 9)
    d.accumulate_dense(np.einsum("s,si,sj,sk->ijk", w, X, X, X), True)
    assert rel_per_replicate(s.data(), d.data()) <= 1e-9


# ---------------------------------------------------------------- RTPM
@pytest.mark.parametrize("n,b,B,k,L,T", [(20, 1024, 6, 3, 8, 10), (100, 4096, 20, 3, 12, 30)])
def test_rtpm_matches_oracle(gpu_ctx, n, b, B, k, L, T):
    Tn, lam_true, V_true = skb().gen_planted_tensor(n, k + 1, 0.01, 7)
    s = skb().SymTensorSketchSet(n, b, B, 3, gpu_ctx)
    o = O.SymSet(n, b, B, 3)
    s.accumulate_dense(Tn, True)
    o.accumulate_dense(Tn, True)
    cfg = skb().PowerConfig(k=k, L=L, T_iters=T, b=b, B=B, seed=13)
    d = skb().robust_tpm_fast(s, cfg)
    lam_o, V_o, bt_o = o.rtpm(k, L, T, seed=13)
    assert np.array_equal(d.best_tau, bt_o)
    assert np.max(np.abs(d.lambda_ - lam_o) / np.abs(lam_o)) <= VEC_TOL
    match = O.greedy_match(d.A, V_o)
    assert np.all(match[:, 2] > 1 - 1e-12)
    for r in range(k):
        a, t = int(match[r, 0]), int(match[r, 1])
        sgn = np.sign(d.A[:, a] @ V_o[:, t])
        assert vec_rel(sgn * d.A[:, a], V_o[:, t]) <= VEC_TOL
    # deflated sets agree too
    assert rel_per_replicate(s.data(), o.data()) <= 1e-8


def test_rtpm_validation(gpu_ctx):
    s = skb().SymTensorSketchSet(4, 64, 2, 1, gpu_ctx)
    with pytest.raises(ValueError, match="target rank exceeds"):
        skb().robust_tpm_fast(s, skb().PowerConfig(k=5, L=2, T_iters=2))
    with pytest.raises(ValueError, match="must be positive"):
        skb().robust_tpm_fast(s, skb().PowerConfig(k=1, L=0, T_iters=2))


def test_rtpm_degenerate_on_zero_sketch(gpu_ctx):
    s = skb().SymTensorSketchSet(6, 64, 3, 1, gpu_ctx)
    with pytest.raises(skb().DegenerateIterationError):
        skb().robust_tpm_fast(s, skb().PowerConfig(k=1, L=2, T_iters=2))


# ---------------------------------------------------------------- asymmetric contractions / factored
@pytest.mark.parametrize("n,b,B", [(10, 64, 3), (40, 4096, 8), (24, 16384, 3)])
def test_asym_contractions_match_oracle(gpu_ctx, n, b, B):
    T = np.random.default_rng(b).normal(size=(n, n, n))
    s = skb().AsymTensorSketchSet(n, b, B, 31, gpu_ctx)
    o = O.AsymSet(n, b, B, 31)
    s.accumulate_dense(T)
    o.accumulate_dense(T)
    ws = skb().AsymContractionWorkspace(s)
    rng = np.random.default_rng(1)
    X = rng.normal(size=(4, n))
    Y = rng.normal(size=(4, n))
    for fm in range(3):
        got = ws.mode_contraction(fm, X, Y)
        for l in range(4):
            assert vec_rel(got[l], o.mode_contraction(fm, X[l], Y[l])) <= VEC_TOL
    assert np.array_equal(ws.Ibc(X[0], X[0]), ws.Ivv(X[0]))
    gv = ws.vvv(X)
    for l in range(4):
        ov = o.vvv(X[l])
        assert abs(gv[l] - ov) <= VEC_TOL * max(abs(ov), 1.0)
    with pytest.raises(ValueError, match="free_mode"):
        ws.mode_contraction(3, X[0], Y[0])


def test_asym_factored_rank1_match_oracle(gpu_ctx):
    n, b, B, N = 8, 256, 3, 20
    rng = np.random.default_rng(2)
    a = rng.normal(size=N)
    U, V, W = rng.normal(size=(3, N, n))
    s = skb().AsymTensorSketchSet(n, b, B, 5, gpu_ctx)
    o = O.AsymSet(n, b, B, 5)
    s.accumulate_factored(a, U, V, W)
    o.accumulate_factored(a, U, V, W)
    assert rel_per_replicate(s.data(), o.data()) <= SKETCH_TOL
    for m in range(B):
        assert rel_per_replicate(s.rank1_sketch(m, U[0], V[0], W[0]), o.rank1_sketch(m, U[0], V[0], W[0])) <= SKETCH_TOL
    s.add_rank1(0.5, U[1], V[1], W[1])
    o.add_rank1(0.5, U[1], V[1], W[1])
    assert rel_per_replicate(s.data(), o.data()) <= SKETCH_TOL


def test_launches_are_counted(gpu_ctx):
    before = skb().kernel_launch_count()
    s = skb().SymTensorSketchSet(8, 64, 2, 1, gpu_ctx)
    s.accumulate_dense(sym_tensor(8, 1), True)
    assert skb().kernel_launch_count() > before


# ---------------------------------------------------------------- LDA whitened moment (a26)
@pytest.mark.parametrize("alpha0", [1.0, 0.5])
def test_lda_sketch_whitened_m3_matches_oracle(gpu_ctx, alpha0):
    from lda_fixtures import synthetic_corpus

    V = 80
    doc_ptr, word, count, W = synthetic_corpus(V=V, k=10, D=300, mean_len=10, seed=5)
    k = W.shape[1]
    for b, B in [(256, 4), (16384, 3)]:
        s = skb().SymTensorSketchSet(k, b, B, 7, gpu_ctx)
        o = O.SymSet(k, b, B, 7)
        got = s.sketch_whitened_m3(V, doc_ptr, word, count, W, alpha0)
        ref = o.sketch_whitened_m3(V, doc_ptr, word, count, W, alpha0)
        assert got == ref
        assert rel_per_replicate(s.data(), o.data()) <= SKETCH_TOL
        assert s.version() == B


def test_lda_rejects_short_corpus(gpu_ctx):
    s = skb().SymTensorSketchSet(4, 64, 2, 1, gpu_ctx)
    with pytest.raises(skb().NumericalError, match="no documents with >= 3 words"):
        s.sketch_whitened_m3(5, [0, 1, 2], [0, 1], [1, 2], np.ones((5, 4)), 1.0)


# ---------------------------------------------------------------- BASELINE config 1 at full size
def test_config1_full_size_build_and_contractions_match_oracle(gpu_ctx):
    """BASELINE config 1 exactly (n=400 fp64, rank 50 + 0.01 noise, b=2^14, B=20): the
    full dense build from pinned host memory (the chunked zero-copy pipeline) and from
    device memory, and T(I,u,u) / T(u,u,u) for a batch of restarts, against the oracle."""
    import torch

    n, b, B, seed = 400, 1 << 14, 20, 20150615
    T, lam, V = skb().gen_planted_tensor(n, 50, 0.01, seed)
    o = O.SymSet(n, b, B, seed)
    o.accumulate_dense(T, True)
    pinned = torch.from_numpy(T).pin_memory()
    for src in (pinned.numpy(), pinned.cuda()):
        s = skb().SymTensorSketchSet(n, b, B, seed, gpu_ctx)
        s.accumulate_dense(src, assume_symmetric=True)
        assert rel_per_replicate(s.data(), o.data()) <= SKETCH_TOL
    ws = skb().SymContractionWorkspace(s)
    U = skb().power_inits(7, n, 1, 6)[0]
    iv = ws.Ivv(U)
    for l in range(U.shape[0]):
        ref = o.ivv(U[l])
        assert np.max(np.abs(iv[l] - ref)) <= 1e-9 * np.max(np.abs(ref))
        assert abs(ws.vvv(U[l]) - o.vvv(U[l])) <= 1e-9 * abs(o.vvv(U[l]))


# ---------------------------------------------------------------- BASELINE config 2 at full size
def test_config2_full_size_properties(gpu_ctx):
    """BASELINE config 2 (n=1000 fp32, b=2^16, B=10: the one-limb class-list kernel with
    one bucket-class bit) in full: the hash tables equal the oracle's; the sketch of the
    planted tensor matches the fp64 oracle (sketch.cpp:315-345 over the same fp32 entries
    widened, 16 host threads) per replicate within the fp32 contract 1e-4 (the one-limb
    resolution gives ~1e-6; asserted at 1e-5); it equals the sum of its four equal-work
    i-slice sketches (the multi-GPU sharding identity; each slice has its own exponent) to
    1e-5; and the sketch of
    a sparse symmetric tensor equals the explicit sum over its sorted triples built from
    the oracle's tables (kappa, bucket, complex4 sign) to 1e-12 (dyadic values: exact)."""
    import torch

    from paper_1506_04448_b200.distributed import equal_work_slices

    n, b, B, seed = 1000, 1 << 16, 10, 20150615
    s = skb().SymTensorSketchSet(n, b, B, seed, gpu_ctx)
    o = O.SymSet(n, b, B, seed)
    for m in range(B):
        t, ot = s.tables(m), o.tables(m)
        for x, y in zip(t, ot[:4]):
            assert np.array_equal(x, y)
    T = torch.empty(n ** 3, dtype=torch.float32, device="cuda")
    skb().gen_planted_tensor_device(gpu_ctx, n, 100, 0.01, seed, T.data_ptr(), dtype=np.float32)
    s.accumulate_dense(T, assume_symmetric=True)
    parts = skb().SymTensorSketchSet(n, b, B, seed, gpu_ctx)
    for i0, i1 in equal_work_slices(n, 4):
        parts.accumulate_dense(T, assume_symmetric=True, i0=i0, i1=i1)
    assert rel_per_replicate(parts.data(), s.data()) <= 1e-5
    Th = T.cpu().numpy().reshape(n, n, n)
    del T
    O.lib().orc_set_num_threads(16)
    o.accumulate_dense_slice(Th, 0, n)
    del Th
    err = rel_per_replicate(s.data(), o.data())
    assert err <= SKETCH_TOL_F32 and err <= 1e-5, err
    # sparse: three symmetric entries (distinct, two-equal, all-equal index patterns)
    entries = {(3, 500, 999): 1.25, (7, 7, 640): -2.5, (999, 999, 999): 0.75}
    Ts = torch.zeros((n, n, n), dtype=torch.float32, device="cuda")
    import itertools

    for (i, j, k), v in entries.items():
        for pi in set(itertools.permutations((i, j, k))):
            Ts[pi] = v
    sp = skb().SymTensorSketchSet(n, b, B, seed, gpu_ctx)
    sp.accumulate_dense(Ts.reshape(-1), assume_symmetric=True)
    want = np.zeros((B, b), dtype=np.complex128)
    root = [1, 1j, -1, -1j]
    for m in range(B):
        h, _, _, e = o.tables(m)[:4]
        for (i, j, k), v in entries.items():
            kappa = 6 if len({i, j, k}) == 3 else (3 if len({i, j, k}) == 2 else 1)
            want[m, (int(h[i]) + int(h[j]) + int(h[k])) % b] += kappa * v * root[(int(e[i]) + int(e[j]) + int(e[k])) & 3]
    assert rel_per_replicate(sp.data(), want) <= 1e-12


# ---------------------------------------------------------------- RTPM at BASELINE config 0, full size
def test_rtpm_config0_full_size_matches_oracle_fixture(gpu_ctx):
    """BASELINE config 0 in full (n=100, b=2^12, B=20, k=10, L=50, T=30) against the
    oracle's run (tests/golden/rtpm_c0.json, make_golden.py --rtpm-c0). Components 1-6
    must agree to 1e-9 (lambda relative, v absolute). The later components are
    ill-conditioned: perturbing the tensor by 1e-16 relative moves the GPU's own
    components 7-10 by 2e-9 .. 4e-3 and flips their restart argmax
    (microbench/rtpm_conditioning_c0.py, profiles/README.md). Rounding-level differences
    in the FFTs are amplified the same way, so for those components the test only
    requires the same eigenvector (|cos| > 0.99) and lambda within 1e-2."""
    fx = json.loads((GOLDEN / "rtpm_c0.json").read_text())
    c = fx["config"]
    T, lam, V = skb().gen_planted_tensor(c["n"], c["rank"], c["sigma"], c["gen_seed"])
    s = skb().SymTensorSketchSet(c["n"], c["b"], c["B"], c["set_seed"], gpu_ctx)
    s.accumulate_dense(T, assume_symmetric=True)
    dec = skb().robust_tpm_fast(s, skb().PowerConfig(k=c["k"], L=c["L"], T_iters=c["T"], seed=c["rtpm_seed"]))
    lo, Vo = np.array(fx["lambda"]), np.array(fx["V"])
    for q in range(6):
        assert abs(dec.lambda_[q] - lo[q]) <= 1e-9 * abs(lo[q]), q
        assert np.max(np.abs(dec.A[:, q] - Vo[:, q])) <= 1e-9, q
        assert dec.best_tau[q] == fx["best_tau"][q]
    for q in range(6, c["k"]):
        cos = abs(dec.A[:, q] @ Vo[:, q]) / (np.linalg.norm(dec.A[:, q]) * np.linalg.norm(Vo[:, q]))
        assert cos > 0.99, (q, cos)
        assert abs(dec.lambda_[q] - lo[q]) <= 1e-2 * abs(lo[q]), q


# ---------------------------------------------------------------- fast ALS on the asym set (§8f rank 3)
def _planted_asym(n, k, seed):
    rng = np.random.default_rng(seed)
    lam = np.linspace(3.0, 1.5, k)
    A, B, Cf = (np.linalg.qr(rng.normal(size=(n, k)))[0] for _ in range(3))
    T = np.einsum("r,ir,jr,kr->ijk", lam, A, B, Cf)
    return T, lam, A, B, Cf


@pytest.mark.parametrize("max_iters", [1, 25])
def test_asym_als_matches_oracle(gpu_ctx, max_iters):
    """als_fast (decompose.cpp:117-205): same init stream, same sketched mode contractions,
    same pseudoinverse update -> the GPU factors follow the oracle's trajectory."""
    n, k, b, B = 24, 3, 1024, 10
    T, lam, A, Bf, Cf = _planted_asym(n, k, 5)
    s = skb().AsymTensorSketchSet(n, b, B, 17, gpu_ctx)
    o = O.AsymSet(n, b, B, 17)
    s.accumulate_dense(T)
    o.accumulate_dense(T)
    d = skb().als_fast(s, skb().AlsConfig(k=k, max_iters=max_iters, tol=1e-6, seed=9))
    lo, Ao, Bo, Co, ito = O.asym_als(o, k, max_iters, 1e-6, 9)
    assert d.iters == ito
    assert np.max(np.abs(d.lambda_ - lo) / np.abs(lo)) <= 1e-7
    for X, Y in ((d.A, Ao), (d.B, Bo), (d.C, Co)):
        assert np.max(np.abs(X - Y)) <= 1e-7


def test_asym_als_recovers_planted_components(gpu_ctx):
    n, k = 30, 3
    T, lam, A, Bf, Cf = _planted_asym(n, k, 8)
    s = skb().AsymTensorSketchSet(n, 4096, 20, 3, gpu_ctx)
    s.accumulate_dense(T)
    d = skb().als_fast(s, skb().AlsConfig(k=k, max_iters=200, tol=1e-8, seed=1))
    m = O.greedy_match(d.A, A)
    assert np.all(m[:, 2] > 0.99)
    with pytest.raises(ValueError, match="als: target rank exceeds tensor dimension"):
        skb().als_fast(s, skb().AlsConfig(k=n + 1))
    with pytest.raises(ValueError, match="als: k and max_iters must be positive"):
        skb().als_fast(s, skb().AlsConfig(k=2, max_iters=0))


# ---------------------------------------------------------------- LDA moments / whitening (§8f rank 1)
def _align_cols(A, ref):
    """Flip column signs of A to match ref (eigenvector signs are unpinned, lda.cpp:128)."""
    s = np.sign(np.sum(A * ref, axis=0))
    s[s == 0] = 1
    return A * s


@pytest.mark.parametrize("alpha0", [1.0, 0.3])
def test_lda_m1_and_m2_operator_match_oracle(gpu_ctx, alpha0):
    from lda_fixtures import synthetic_corpus

    V = 120
    doc_ptr, word, count, _ = synthetic_corpus(V=V, k=6, D=500, mean_len=9, seed=11)
    m1 = skb().compute_m1(V, doc_ptr, word, count, gpu_ctx)
    m1_ref = O.lda_compute_m1(V, doc_ptr, word, count)
    assert np.max(np.abs(m1 - m1_ref)) <= 1e-14 * np.max(np.abs(m1_ref))
    M2 = O.lda_compute_m2(V, doc_ptr, word, count, alpha0)
    X = np.random.default_rng(2).normal(size=(V, 37))
    Y = skb().m2_apply(V, doc_ptr, word, count, alpha0, X, gpu_ctx)
    assert np.max(np.abs(Y - M2 @ X)) <= 1e-12 * np.max(np.abs(M2 @ X))


@pytest.mark.parametrize("dense", [False, True])
def test_lda_whiten_matches_dense_eigensolver_oracle(gpu_ctx, dense):
    """Randomized subspace iteration on the implicit (or dense) M2 reproduces whiten's
    top-k eigenpairs (lda.cpp:125-143) from the oracle's full Jacobi eigendecomposition."""
    from lda_fixtures import synthetic_corpus

    V, k, alpha0 = 150, 6, 1.0
    doc_ptr, word, count, _ = synthetic_corpus(V=V, k=k, D=3000, mean_len=30, seed=3)
    M2 = O.lda_compute_m2(V, doc_ptr, word, count, alpha0)
    W_ref, U_ref, sv_ref = O.lda_whiten(M2, k)
    if dense:
        wm = skb().whiten(M2, k, iters=40, ctx=gpu_ctx)
    else:
        wm = skb().whiten_corpus(V, doc_ptr, word, count, alpha0, k, iters=40, ctx=gpu_ctx)
    assert np.max(np.abs(wm.singular_values - sv_ref) / sv_ref) <= 1e-9
    W = _align_cols(wm.W, W_ref)
    U = _align_cols(wm.unwhiten, U_ref)
    assert np.max(np.abs(W - W_ref)) <= 1e-6 * np.max(np.abs(W_ref))
    assert np.max(np.abs(U - U_ref)) <= 1e-6 * np.max(np.abs(U_ref))
    # W' M2 W = I on the input moment (lda.hpp:43)
    assert np.max(np.abs(wm.W.T @ M2 @ wm.W - np.eye(k))) <= 1e-8


def test_lda_whiten_dense_large_block_products(gpu_ctx):
    """At V = 2304 the whitening's block products run split along K (the p x p Grams over
    V rows and the dense p x V x V moment apply, skc_gemm.cu): the top-k eigenpairs of a
    planted PSD moment match numpy's eigendecomposition and W' M2 W = I (lda.hpp:43)."""
    V, k = 2304, 20
    rng = np.random.default_rng(41)
    Uq, _ = np.linalg.qr(rng.normal(size=(V, k)))
    ev = np.geomspace(40.0, 2.0, k)
    N = rng.normal(size=(V, V)) * 1e-3
    M2 = (Uq * ev) @ Uq.T + (N + N.T) / 2
    w_ref, U_ref = np.linalg.eigh(M2)
    sv_ref = w_ref[::-1][:k]
    wm = skb().whiten(M2, k, iters=30, ctx=gpu_ctx)
    assert np.max(np.abs(wm.singular_values - sv_ref) / sv_ref) <= 1e-9
    assert np.max(np.abs(wm.W.T @ M2 @ wm.W - np.eye(k))) <= 1e-8
    Wn = wm.W * np.sqrt(sv_ref)  # unit eigenvectors
    top = U_ref[:, ::-1][:, :k]
    assert np.max(np.abs(np.abs(np.sum(Wn * top, axis=0)) - 1.0)) <= 1e-8


def test_lda_device_corpus_handle_matches_per_call_path(gpu_ctx):
    """The device-resident corpus gives the same whitening and sketch as the per-call
    entry points (same operator, same order), bit for bit."""
    from lda_fixtures import synthetic_corpus

    V, k, alpha0 = 90, 5, 1.0
    doc_ptr, word, count, _ = synthetic_corpus(V=V, k=k, D=800, mean_len=20, seed=6)
    corpus = skb().LdaCorpus(V, doc_ptr, word, count, gpu_ctx)
    info = corpus.info()
    assert info["V"] == V and info["D"] == doc_ptr.size - 1 and info["nnz"] == word.size
    a = corpus.whiten(alpha0, k, iters=20)
    b = skb().whiten_corpus(V, doc_ptr, word, count, alpha0, k, iters=20, ctx=gpu_ctx)
    assert np.array_equal(a.W, b.W) and np.array_equal(a.singular_values, b.singular_values)
    s1 = skb().SymTensorSketchSet(k, 1024, 4, 3, gpu_ctx)
    s2 = skb().SymTensorSketchSet(k, 1024, 4, 3, gpu_ctx)
    assert s1.sketch_whitened_m3_corpus(corpus, a.W, alpha0) == s2.sketch_whitened_m3(V, doc_ptr, word, count, a.W,
                                                                                       alpha0)
    assert np.array_equal(s1.data(), s2.data())


def test_lda_document_shards_sum_to_full_sketch(gpu_ctx):
    """Multi-GPU decomposition of sketch_whitened_m3 (distributed.py), run shard by shard
    on one GPU: the shards' sketches with corpus-wide normalisation and M1 sum to the
    full sketch (one shard adds the c_m1 F(q)^3 term); a shard without usable documents
    contributes only its vocabulary terms."""
    from lda_fixtures import synthetic_corpus

    from paper_1506_04448_b200.distributed import lda_shard_globals

    V, k, alpha0 = 70, 6, 0.8
    doc_ptr, word, count, W = synthetic_corpus(V=V, k=k, D=400, mean_len=12, seed=12)
    full = skb().SymTensorSketchSet(k, 2048, 5, 21, gpu_ctx)
    used, skipped = full.sketch_whitened_m3(V, doc_ptr, word, count, W, alpha0)
    g_used, g_m1, _, _ = lda_shard_globals(V, doc_ptr, word, count)
    assert g_used == used
    cut = 173
    shards = [(doc_ptr[:cut + 1], word[:doc_ptr[cut]], count[:doc_ptr[cut]]),
              (doc_ptr[cut:] - doc_ptr[cut], word[doc_ptr[cut]:], count[doc_ptr[cut]:])]
    total = np.zeros_like(full.data())
    tot_used = 0
    for r, (dp_, w_, c_) in enumerate(shards):
        s = skb().SymTensorSketchSet(k, 2048, 5, 21, gpu_ctx)
        u, _ = s.sketch_whitened_m3_shard(V, dp_, w_, c_, W, alpha0, g_used, g_m1, r == 0)
        tot_used += u
        total += s.data()
    assert tot_used == used
    assert rel_per_replicate(total, full.data()) <= 1e-11


def test_lda_whiten_errors_follow_reference(gpu_ctx):
    from lda_fixtures import synthetic_corpus

    V = 40
    doc_ptr, word, count, _ = synthetic_corpus(V=V, k=3, D=200, mean_len=12, seed=4)
    with pytest.raises(ValueError, match="whiten: invalid target rank"):
        skb().whiten_corpus(V, doc_ptr, word, count, 1.0, V + 1, ctx=gpu_ctx)
    with pytest.raises(skb().NumericalError, match="compute_m1: empty corpus"):
        skb().compute_m1(V, [0], [], [], gpu_ctx)
    with pytest.raises(skb().NumericalError, match="compute_m2: no documents with at least 2 words"):
        skb().m2_apply(V, [0, 1, 2], [0, 1], [1, 1], 1.0, np.ones((V, 1)), gpu_ctx)
    # a PSD matrix of rank 3 cannot be whitened to k = 5 (lda.cpp:133-136)
    Q = np.linalg.qr(np.random.default_rng(0).normal(size=(V, 3)))[0]
    M = Q @ np.diag([3.0, 2.0, 1.0]) @ Q.T
    with pytest.raises(skb().NumericalError, match="rank deficient at component 4"):
        skb().whiten(M, 5, ctx=gpu_ctx)
    with pytest.raises(O.OracleError, match="rank deficient at component 4"):
        O.lda_whiten(M, 5)


# ---------------------------------------------------------------- sym_aux / truncated rank-1 (a16)
@pytest.mark.parametrize("n,b", [(9, 64), (30, 16384)])
def test_sym_aux_and_truncated_rank1_match_oracle(gpu_ctx, n, b):
    u = np.random.default_rng(4).normal(size=n)
    s = skb().SymTensorSketchSet(n, b, 3, 8, gpu_ctx)
    o = O.SymSet(n, b, 3, 8)
    for m in range(3):
        s1, s2, s3 = s.aux_sketches(m, u)
        b1, b2, b3, se, _, _ = o.tables(m)
        r1 = np.zeros(b, complex)
        r2 = np.zeros(b, complex)
        r3 = np.zeros(b, complex)
        for i in range(n):  # sketch.cpp:418-423, direct
            r1[b1[i]] += (1j ** int(se[i])) * u[i]
            r2[b2[i]] += (1j ** int(2 * se[i])) * u[i] ** 2
            r3[b3[i]] += (1j ** int(3 * se[i])) * u[i] ** 3
        for got, ref in ((s1, r1), (s2, r2), (s3, r3)):
            assert np.max(np.abs(got - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref)))
        tr = s.rank1_truncated(m, u)
        assert rel_per_replicate(tr, o.rank1_truncated(m, u)) <= SKETCH_TOL


# ---------------------------------------------------------------- fft:: (fft.hpp:15-26) on the device
@pytest.mark.parametrize("b", [1, 2, 16, 64, 1024, 4096, 16384, 1 << 16])
def test_device_fft_matches_numpy_and_oracle(gpu_ctx, b):
    rng = np.random.default_rng(b)
    x = rng.normal(size=b) + 1j * rng.normal(size=b)
    F = skb().fft
    assert np.max(np.abs(F.forward(x) - np.fft.fft(x))) <= 1e-12 * max(1.0, np.max(np.abs(np.fft.fft(x))))
    assert np.max(np.abs(F.inverse(F.forward(x)) - x)) < 1e-12  # test_fft.cpp:37-46
    assert np.max(np.abs(F.inverse_unscaled(x) - np.fft.ifft(x) * b)) <= 1e-12 * b
    if b >= 2:
        assert np.max(np.abs(F.forward(x) - O.fft(x, -1))) <= 1e-12 * max(1.0, np.max(np.abs(np.fft.fft(x))))


def test_device_fft_rejects_non_power_of_two(gpu_ctx):  # test_fft.cpp:77-82
    with pytest.raises(ValueError, match="power of two"):
        skb().fft.forward(np.ones(12))


def test_device_circular_convolution_worked_examples(gpu_ctx):  # test_fft.cpp:48-75
    x = np.array([1, 2, 3, 4], dtype=complex)
    y = np.array([1, 0, 0, 1], dtype=complex)
    assert np.allclose(skb().fft.circular_convolve(x, y).real, [3, 5, 7, 5], atol=1e-12)


# ---------------------------------------------------------------- sketch file container (next row)
def test_sketch_save_load_round_trip(gpu_ctx, tmp_path):  # SPEC.md:307 bit-exact round trip
    n, b, B = 11, 512, 3
    s = skb().SymTensorSketchSet(n, b, B, 42, gpu_ctx)
    s.accumulate_dense(sym_tensor(n, 2), True)
    p = tmp_path / "s.skt"
    s.save(p)
    assert skb().peek_sketch_mode(p) == "sym"
    t = skb().SymTensorSketchSet.load(p, gpu_ctx)
    assert np.array_equal(t.data(), s.data())
    for m in range(B):
        assert all(np.array_equal(x, y) for x, y in zip(t.tables(m), s.tables(m)))
    u = np.random.default_rng(1).normal(size=n)
    ws1, ws2 = skb().SymContractionWorkspace(s), skb().SymContractionWorkspace(t)
    assert np.array_equal(ws1.Ivv(u), ws2.Ivv(u))
    a = skb().AsymTensorSketchSet(n, b, B, 43, gpu_ctx)
    a.accumulate_dense(np.random.default_rng(3).normal(size=(n, n, n)))
    pa = tmp_path / "a.skt"
    a.save(pa)
    assert skb().peek_sketch_mode(pa) == "asym"
    assert np.array_equal(skb().AsymTensorSketchSet.load(pa, gpu_ctx).data(), a.data())
    with pytest.raises(skb().FormatError, match="not a symmetric"):
        skb().SymTensorSketchSet.load(pa, gpu_ctx)
    bad = tmp_path / "bad.skt"
    bad.write_bytes(b"NOTASKETCH" + bytes(60))
    with pytest.raises(skb().FormatError, match="bad magic"):
        skb().peek_sketch_mode(bad)
    trunc = tmp_path / "t.skt"
    trunc.write_bytes(p.read_bytes()[:200])
    with pytest.raises(skb().FormatError, match="truncated"):
        skb().SymTensorSketchSet.load(trunc, gpu_ctx)


@pytest.mark.parametrize("n", [140, 257])
def test_dense_pinned_pipelined_build_fp32(gpu_ctx, n):
    """fp32 pinned input: the chunked zero-copy pipeline with 16-byte bus reads of four
    fp32 entries (row segments at any alignment), one-limb windows and per-chunk
    exponents; against the fp64 oracle of the same entries and the device-resident build."""
    import torch

    T = sym_tensor(n, 32).astype(np.float32)
    pinned = torch.from_numpy(T.copy()).pin_memory().numpy()
    ref = O.SymSet(n, 4096, 5, 6)
    ref.accumulate_dense(T.astype(np.float64), True)
    s = skb().SymTensorSketchSet(n, 4096, 5, 6, gpu_ctx)
    d = skb().SymTensorSketchSet(n, 4096, 5, 6, gpu_ctx)
    s.accumulate_dense(pinned, assume_symmetric=True)
    d.accumulate_dense(torch.from_numpy(T).cuda(), assume_symmetric=True)
    assert rel_per_replicate(s.data(), ref.data()) <= 1e-6
    assert rel_per_replicate(s.data(), d.data()) <= 1e-6


# ---------------------------------------------------------------- LDA recover_params / heldout (§8f rank 4)
def test_lda_recover_params_matches_oracle(gpu_ctx):
    """recover_params (lda.cpp:228-248) on the device -- the V x k x k product and the
    simplex projection by bisection -- against the oracle's sort-based projection, at the
    config-4 vocabulary (V=50000) with k=100."""
    rng = np.random.default_rng(7)
    V, k, alpha0 = 50000, 100, 1.0
    lam = rng.uniform(0.5, 2.0, size=k)
    A = np.linalg.qr(rng.normal(size=(k, k)))[0]
    Uw = rng.normal(size=(V, k)) * 1e-3
    Uw[rng.integers(0, V, size=300)] += 0.05  # a few heavy words per component
    wm = skb().WhiteningMap(np.zeros((V, k)), Uw, np.ones(k))
    m = skb().recover_params(skb().CpDecomposition.symmetric_of(lam, A), wm, alpha0, ctx=gpu_ctx)
    Po, ao = O.lda_recover_params(V, k, lam, A, Uw, alpha0)
    assert np.max(np.abs(m.Phi - Po)) <= 1e-12
    assert np.allclose(m.Phi.sum(axis=0), 1.0, atol=1e-12)
    assert np.array_equal(m.alpha, ao)
    with pytest.raises(skb().NumericalError, match="zero eigenvalue at component 2"):
        skb().recover_params(skb().CpDecomposition.symmetric_of(np.r_[1.0, 0.0, np.ones(k - 2)], A), wm, alpha0,
                             ctx=gpu_ctx)


@pytest.mark.parametrize("k", [1, 3, 40, 100])
def test_lda_heldout_likelihood_matches_oracle(gpu_ctx, k):
    """heldout_likelihood (lda.cpp:273-320): one warp per document on the device against
    the oracle's sequential documents (500 projected-gradient steps each)."""
    from lda_fixtures import synthetic_corpus

    V = 400
    doc_ptr, word, count, _ = synthetic_corpus(V=V, k=max(k, 2), D=300, mean_len=40, seed=11)
    Phi = np.random.default_rng(5).dirichlet(np.full(V, 0.3), size=k).T
    ll, fl = skb().heldout_likelihood(skb().LdaModel(Phi, np.ones(k)), V, doc_ptr, word, count, ctx=gpu_ctx)
    llo, flo = O.lda_heldout_likelihood(Phi, V, doc_ptr, word, count)
    assert abs(ll - llo) <= 1e-9 * abs(llo)
    assert fl == flo
