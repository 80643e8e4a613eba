"""High-dynamic-range dense builds (fixed-point resolution is global).

One exact fixed-point scale per build keeps every bucket to ~0.6 x 2^-F / mean(kappa|T|)
of its own magnitude. The main pass checks that ratio; beyond 2^-33 (2^-17 for one-limb
fp32 windows) it adds nothing and the host redoes the build in magnitude bands of at most
16 binades, each with its own exponent (skc_abi_build.cu run_dense_build_banded). The
error of every bucket is compared with the oracle's fp64 sum (sketch.cpp:315-345) relative
to that bucket's absolute mass A_t = sum over its terms of kappa|T_ijk|, the scale of the
reference's own rounding."""
import itertools

import numpy as np
import pytest

import oracle_py as O

pytestmark = pytest.mark.gpu


def skb():
    import paper_1506_04448_b200 as m

    return m


def from_triples(n, val):
    """Symmetric tensor from one value per sorted triple."""
    T = np.zeros((n, n, n))
    for (i, j, k), v in val.items():
        for p in set(itertools.permutations((i, j, k))):
            T[p] = v
    return T


def bucket_mass(n, b, B, seed, T):
    """A[m, slot, parity] = sum of kappa|T_ijk| over the sorted triples landing there."""
    o = O.SymSet(n, b, B, seed)
    A = np.zeros((B, b, 2))
    ii, jj, kk = np.array([t for t in itertools.combinations_with_replacement(range(n), 3)]).T
    kap = np.where((ii == jj) & (jj == kk), 1.0, np.where((ii == jj) | (jj == kk), 3.0, 6.0))
    mag = kap * np.abs(T[ii, jj, kk])
    for m in range(B):
        h, _, _, e = o.tables(m)[:4]
        h = np.asarray(h, dtype=np.int64)
        e = np.asarray(e, dtype=np.int64)
        slot = (h[ii] + h[jj] + h[kk]) % b
        par = (e[ii] + e[jj] + e[kk]) & 1
        np.add.at(A[m], (slot, par), mag)
    return A


def per_bucket_error(got, ref, A):
    d = np.stack([np.abs(got.real - ref.real), np.abs(got.imag - ref.imag)], axis=-1)
    mask = A > 0
    return float(np.max(d[mask] / A[mask]))


def hdr_tensor(n, seed, span):
    rng = np.random.default_rng(seed)
    val = {t: rng.choice([-1.0, 1.0]) * 10.0 ** rng.uniform(-span, 0)
           for t in itertools.combinations_with_replacement(range(n), 3)}
    return from_triples(n, val)


@pytest.mark.parametrize("kind", ["log_uniform_1e12", "spike_1e12"])
def test_hdr_fp64_per_bucket_error_vs_oracle(gpu_ctx, kind):
    n, b, B, seed = 36, 2048, 4, 17
    if kind == "spike_1e12":
        rng = np.random.default_rng(3)
        val = {t: rng.normal() for t in itertools.combinations_with_replacement(range(n), 3)}
        val[(2, 5, 30)] = 3.0e12
        T = from_triples(n, val)
    else:
        T = hdr_tensor(n, 4, 12)
    A = bucket_mass(n, b, B, seed, T)
    o = O.SymSet(n, b, B, seed)
    o.accumulate_dense(T, True)
    before = gpu_ctx.build_banded()
    s = skb().SymTensorSketchSet(n, b, B, seed, gpu_ctx)
    s.accumulate_dense(T, assume_symmetric=True)
    assert gpu_ctx.build_banded() == before + 1  # the resolution check sent it to the banded path
    err = per_bucket_error(s.data(), o.data(), A)
    assert err <= 1e-10, err
    # pinned host input (raw-copy pre-pass) takes the same route
    import torch

    pinned = torch.from_numpy(T.copy()).pin_memory().numpy()
    p = skb().SymTensorSketchSet(n, b, B, seed, gpu_ctx)
    p.accumulate_dense(pinned, assume_symmetric=True)
    assert per_bucket_error(p.data(), o.data(), A) <= 1e-10


def test_hdr_fp32_goes_to_two_limbs_or_bands(gpu_ctx):
    """fp32 entries spanning 1e6: too wide for one 32-bit limb per slot, so the build is
    redone (two limbs or bands) and every bucket still meets the fp64 oracle of the same
    fp32 entries."""
    import torch

    n, b, B, seed = 40, 4096, 5, 23
    T = hdr_tensor(n, 9, 6).astype(np.float32)
    A = bucket_mass(n, b, B, seed, T.astype(np.float64))
    o = O.SymSet(n, b, B, seed)
    o.accumulate_dense(T.astype(np.float64), True)
    r0, b0 = gpu_ctx.build_retries(), gpu_ctx.build_banded()
    s = skb().SymTensorSketchSet(n, b, B, seed, gpu_ctx)
    s.accumulate_dense(torch.from_numpy(T).cuda(), assume_symmetric=True)
    assert gpu_ctx.build_retries() + gpu_ctx.build_banded() > r0 + b0
    assert per_bucket_error(s.data(), o.data(), A) <= 1e-10


def test_ordinary_tensors_keep_the_single_scale_fast_path(gpu_ctx):
    """The BASELINE generators (planted rank + Gaussian noise) stay on one exact scale: no
    retry, no bands -- config 0's shape (n=100, b=2^12: ~21 entries per slot) included."""
    import torch

    r0, b0 = gpu_ctx.build_retries(), gpu_ctx.build_banded()
    T0, _, _ = skb().gen_planted_tensor(100, 10, 0.01, 11)
    skb().SymTensorSketchSet(100, 1 << 12, 20, 5, gpu_ctx).accumulate_dense(T0, assume_symmetric=True)
    for n, dt in ((120, np.float64), (160, np.float32)):
        T, _, _ = skb().gen_planted_tensor(n, 5, 0.01, 7, dtype=dt)
        s = skb().SymTensorSketchSet(n, 4096, 4, 3, gpu_ctx)
        s.accumulate_dense(torch.from_numpy(np.asarray(T)).cuda(), assume_symmetric=True)
    assert gpu_ctx.build_retries() == r0 and gpu_ctx.build_banded() == b0


@pytest.mark.parametrize("n,b", [(20, 1024), (48, 4096)])
def test_hdr_asym_per_bucket_error_vs_oracle(gpu_ctx, n, b):
    """Asymmetric builds (sketch.cpp:173-193) with entries spanning 1e12: the small build
    takes the contiguous-window kernel (fixed-point pre-pass, banded), the larger the
    class-list kernel; every bucket within 1e-10 of its mass either way."""
    B, seed = 4, 29
    rng = np.random.default_rng(n)
    T = rng.choice([-1.0, 1.0], size=(n, n, n)) * 10.0 ** rng.uniform(-12, 0, size=(n, n, n))
    o = O.AsymSet(n, b, B, seed)
    o.accumulate_dense(T)
    A = np.zeros((B, b))
    ii, jj, kk = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    for m in range(B):
        bk = np.asarray(o.tables(m)[0], dtype=np.int64)
        slot = (bk[0][ii] + bk[1][jj] + bk[2][kk]) % b
        np.add.at(A[m], slot.ravel(), np.abs(T).ravel())
    before = gpu_ctx.build_banded()
    s = skb().AsymTensorSketchSet(n, b, B, seed, gpu_ctx)
    s.accumulate_dense(T)
    # thin buckets (~8 entries per slot at n=20) and heavy tails (at n=48, ~27 entries per
    # slot but only ~2 of them carry the mass) go to bands
    assert gpu_ctx.build_banded() == before + 1
    got, ref = s.data(), o.data()
    mask = A > 0
    err = np.max(np.abs(got.real - ref.real)[mask] / A[mask])
    assert err <= 1e-10, err
