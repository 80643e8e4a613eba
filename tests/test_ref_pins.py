"""The oracle restatement (oracle/sketchcp_oracle.cpp) pinned to the reference itself:
proj/src compiled verbatim into oracle/_ref (against compat/Eigen and an fftw3.h
stand-in, oracle/Makefile `ref`), same inputs through both. Integer work (seeds, hash
tables, unit-sphere draws) must be bit-exact; floating-point results agree to the stated
tolerances (the FFT stand-in and the oracle's FFT are separate implementations of the same
transform). Skipped where oracle/_ref was not built (no /root/reference)."""
import numpy as np
import pytest

import oracle_py as O
import ref_py as R

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (no /root/reference)")


def sym_tensor(n, seed):
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(n, n, n))
    return (A + A.transpose(0, 2, 1) + A.transpose(1, 0, 2) + A.transpose(1, 2, 0) + A.transpose(2, 0, 1)
            + A.transpose(2, 1, 0)) / 6.0


def rel(a, b):
    return float(np.max(np.linalg.norm(a - b, axis=-1) / np.maximum(np.linalg.norm(b, axis=-1), 1e-300)))


def test_seeds_unit_sphere_and_sym_tables_bit_exact():
    for args in [(0, 0x21, 0, 0), (42, 0x22, 5, 0), (2**63 + 17, 0x11, 3, 2), (7, 0x31, 9, 49)]:
        assert R.lib().ref_derive_seed(*args) == O.derive_seed(*args)
    for seed in (1, 99, 2**40 + 3):
        assert np.array_equal(R.unit_sphere(seed, 37), O.unit_sphere(seed, 37))
    for n, b, B, seed in [(30, 1024, 4, 3), (101, 4096, 3, 20150615)]:
        r, o = R.SymSet(n, b, B, seed), O.SymSet(n, b, B, seed)
        for m in range(B):
            for x, y in zip(r.tables(m), o.tables(m)[:4]):
                assert np.array_equal(np.asarray(x, dtype=np.int64), np.asarray(y, dtype=np.int64))


def test_fft_semantics_agree():
    rng = np.random.default_rng(1)
    for b in (2, 8, 1024, 1 << 14):
        x = rng.normal(size=b) + 1j * rng.normal(size=b)
        fr, fo = R.fft(x, -1), O.fft(x, -1)
        assert np.max(np.abs(fr - fo)) <= 1e-12 * np.max(np.abs(fo))
        assert np.max(np.abs(R.fft(fr, 1) - x)) <= 1e-12 * np.max(np.abs(x))


@pytest.mark.parametrize("n,b,B,seed", [(24, 1024, 5, 7), (50, 4096, 8, 3)])
def test_sym_build_contractions_rank1_match_reference(n, b, B, seed):
    T = sym_tensor(n, seed)
    r, o = R.SymSet(n, b, B, seed), O.SymSet(n, b, B, seed)
    r.accumulate_dense(T, assume_symmetric=False)  # also runs the reference's symmetry check
    o.accumulate_dense(T, False)
    assert rel(o.data(), r.data()) <= 1e-13  # same sorted-triple loop (sketch.cpp:315-345)
    u = np.random.default_rng(seed + 1).normal(size=n)
    r.add_scaled_rank1(u, -0.7)
    o.add_scaled_rank1(u, -0.7)
    assert rel(o.data(), r.data()) <= 1e-12
    v = np.random.default_rng(seed + 2).normal(size=n)
    iv_r, iv_o = r.ivv(v), o.ivv(v)
    assert np.max(np.abs(iv_r - iv_o)) <= 1e-12 * np.max(np.abs(iv_r))
    assert abs(r.vvv(v) - o.vvv(v)) <= 1e-12 * abs(r.vvv(v))
    for (i, j, k) in [(0, 1, 2), (3, 3, 5), (n - 1, n - 1, n - 1)]:
        assert abs(r.recover_entry(i, j, k) - o.recover_entry(i, j, k)) <= 1e-10


def test_robust_tpm_fast_matches_reference():
    """decompose.cpp:83-115 itself (Rng inits, T normalised Ivv steps, strict > selection,
    add_scaled_rank1 deflation) against the oracle on a planted rank-3 tensor."""
    n, b, B = 30, 2048, 10
    rng = np.random.default_rng(5)
    Q = np.linalg.qr(rng.normal(size=(n, 3)))[0]
    T = np.einsum("r,ir,jr,kr->ijk", np.array([3.0, 2.0, 1.5]), Q, Q, Q)
    r, o = R.SymSet(n, b, B, 9), O.SymSet(n, b, B, 9)
    r.accumulate_dense(T, True)
    o.accumulate_dense(T, True)
    lr, Vr = r.rtpm(3, 10, 15, seed=4)
    lo, Vo, _ = o.rtpm(3, 10, 15, seed=4)
    assert np.max(np.abs(lr - lo) / np.abs(lr)) <= 1e-9
    assert np.max(np.abs(Vr - Vo)) <= 1e-9
    assert rel(o.data(), r.data()) <= 1e-12  # both left deflated


def test_asym_build_and_contractions_match_reference():
    n, b, B = 20, 1024, 6
    T = np.random.default_rng(2).normal(size=(n, n, n))
    r, o = R.AsymSet(n, b, B, 13), O.AsymSet(n, b, B, 13)
    r.accumulate_dense(T)
    o.accumulate_dense(T)
    assert rel(o.data(), r.data()) <= 1e-13
    x, y = np.random.default_rng(3).normal(size=(2, n))
    assert abs(r.vvv(x) - o.vvv(x)) <= 1e-12 * abs(r.vvv(x))
    for mode in (0, 1, 2):
        a, c = r.mode_contraction(mode, x, y), o.mode_contraction(mode, x, y)
        assert np.max(np.abs(a - c)) <= 1e-12 * np.max(np.abs(a))
