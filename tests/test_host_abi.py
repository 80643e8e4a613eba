"""CPU-only checks of the product library: it loads, exports every symbol the
C-ABI header declares, and its host-side (bit-exact) helpers agree with the
oracle. No device compute happens here."""
import pathlib
import re
import subprocess

import numpy as np
import pytest

import oracle_py as O

ROOT = pathlib.Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "sketchcp_b200.h"


def _declared():
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"\b(skc_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_1506_04448_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (skc_[a-z0-9_]+)", out))
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing
    # and the ctypes table covers them all
    assert set(_declared()) <= set(_lib.SIGNATURES)


def test_library_is_sm100a():
    from paper_1506_04448_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_derive_seed_matches_oracle():
    import paper_1506_04448_b200 as skb

    for args in [(0, 0x21, 0, 0), (42, 0x22, 5, 0), (2**63 + 17, 0x11, 3, 2), (7, 0x31, 9, 49)]:
        assert skb.derive_seed(*args) == O.derive_seed(*args)


def test_unit_sphere_and_power_inits_bit_exact():
    import paper_1506_04448_b200 as skb

    for seed in (1, 99, 2**40 + 3):
        assert np.array_equal(skb.unit_sphere(seed, 37), O.unit_sphere(seed, 37))
    inits = skb.power_inits(seed=5, n=11, k=3, L=4)
    for c in range(3):
        for t in range(4):
            assert np.array_equal(inits[c, t], O.unit_sphere(O.derive_seed(5, 0x31, c, t), 11))


def test_poly_coefficients_and_eval_bit_exact():
    import ctypes as C

    from paper_1506_04448_b200 import _lib

    for k, b, seed in [(6, 1024, 42), (2, 16, 7), (6, 4, 1234)]:
        out = np.empty(k, dtype=np.uint64)
        _lib.check(_lib.lib.skc_poly_coefficients(k, seed, out.ctypes.data_as(C.POINTER(C.c_uint64))))
        assert np.array_equal(out, O.polyhash_from_seed(k, b, seed))
        for i in range(50):
            v = _lib.lib.skc_poly_eval(out.ctypes.data_as(C.POINTER(C.c_uint64)), k, b, i)
            assert v == O.polyhash_eval(out, b, [i])[0]


def test_planted_generator_deterministic_and_symmetric():
    import paper_1506_04448_b200 as skb

    T1, lam1, V1 = skb.gen_planted_tensor(9, 3, 0.01, 7)
    T2, lam2, V2 = skb.gen_planted_tensor(9, 3, 0.01, 7)
    assert np.array_equal(T1, T2) and np.array_equal(lam1, lam2)
    assert np.all((lam1 >= 1) & (lam1 <= 2))
    assert np.allclose(V1.T @ V1, np.eye(3), atol=1e-12)
    for p in [(0, 2, 1), (1, 0, 2), (2, 1, 0)]:
        assert np.array_equal(T1, T1.transpose(p))
    assert O.lib().orc_first_asymmetric_triple(O.dp(T1), 9, 0.0, (O.C.c_int * 3)()) == 0


def test_no_gpu_means_loud_failure():
    """Without a device the library must fail (no silent CPU fallback)."""
    import paper_1506_04448_b200 as skb

    if skb.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(skb.CudaError):
        skb.Context(0)


# ---- LDA recover_params / heldout_likelihood (lda.cpp:228-320): the oracle pinned to an --
# independent numpy restatement (the device path is checked against the oracle in
# tests/test_gpu_parity.py)
def _np_project_to_simplex(y):
    u = np.sort(y)[::-1]
    css = np.cumsum(u)
    t = (css - 1.0) / np.arange(1, y.size + 1)
    ok = np.nonzero(u - t > 0)[0]
    if ok.size == 0:
        return np.full(y.size, 1.0 / y.size)
    return np.maximum(y - t[ok[-1]], 0.0)


def test_oracle_lda_recover_params_matches_restatement():
    rng = np.random.default_rng(1)
    V, k, alpha0 = 30, 4, 0.8
    lam = rng.uniform(0.5, 2.0, size=k)
    A = np.linalg.qr(rng.normal(size=(k, k)))[0]
    Uw = rng.normal(size=(V, k))
    Phi, alpha = O.lda_recover_params(V, k, lam, A, Uw, alpha0)
    for i in range(k):
        mu = 0.5 * (alpha0 + 2.0) * lam[i] * (Uw @ A[:, i])
        assert np.allclose(Phi[:, i], _np_project_to_simplex(mu), rtol=0, atol=1e-14)
        assert np.isclose(alpha[i], 4 * alpha0 * (alpha0 + 1) / ((alpha0 + 2) ** 2 * lam[i] ** 2), rtol=1e-15)
    with pytest.raises(O.OracleError, match="zero eigenvalue at component 2"):
        O.lda_recover_params(V, k, np.array([1.0, 0.0, 1.0, 1.0]), A, Uw, alpha0)


def test_oracle_lda_heldout_likelihood_matches_restatement():
    from lda_fixtures import synthetic_corpus

    V, k = 25, 3
    doc_ptr, word, count, _ = synthetic_corpus(V=V, k=k, D=30, mean_len=10, seed=8)
    Phi = np.random.default_rng(3).dirichlet(np.full(V, 0.5), size=k).T
    ll, fl = O.lda_heldout_likelihood(Phi, V, doc_ptr, word, count)
    gram = Phi.T @ Phi
    step = 1.0 / np.linalg.eigvalsh(gram).max()
    tot_ll, used, floored = 0.0, 0, 0
    for d in range(doc_ptr.size - 1):
        ws = word[doc_ptr[d]:doc_ptr[d + 1]]
        cs = count[doc_ptr[d]:doc_ptr[d + 1]].astype(float)
        m = cs.sum()
        if m < 1:
            continue
        used += 1
        phi_tw = (cs / m) @ Phi[ws]
        pi = np.full(k, 1.0 / k)
        for _ in range(500):
            nxt = _np_project_to_simplex(pi - step * (gram @ pi - phi_tw))
            moved = np.linalg.norm(nxt - pi)
            pi = nxt
            if moved <= 1e-8:
                break
        p = Phi[ws] @ pi
        floored += int(np.sum(p < 1e-12))
        p = np.maximum(p, 1e-12)
        tot_ll += float(cs @ np.log(p)) / m
    assert abs(ll - tot_ll / used) <= 1e-10 * abs(tot_ll / used)
    assert fl == floored


def test_group_slices_and_restart_chunks():
    """Host plumbing of the multi-GPU C-ABI (no device): equal-work i-slices cover [0, n)
    in order and agree with distributed.equal_work_slices; restart blocks of
    ceil(L / R) partition [0, L) in tau order."""
    import paper_1506_04448_b200 as skb
    from paper_1506_04448_b200.distributed import equal_work_slices

    for n in (1, 5, 100, 400, 1000):
        for world in (1, 2, 3, 4, 8):
            sl = skb.group_slices(n, world)
            assert sl[0][0] == 0 and sl[-1][1] == n
            assert all(a[1] == b[0] and a[0] <= a[1] for a, b in zip(sl, sl[1:]))
            assert sl == [tuple(x) for x in equal_work_slices(n, world)]
            if n >= 100:
                work = [sum((n - i) * (n - i + 1) // 2 for i in range(a, b)) for a, b in sl]
                assert max(work) - min(work) <= (n * (n + 1) // 2) * 2  # within ~one row pair of slices
    for L in (1, 7, 50, 100):
        for world in (1, 2, 3, 8, 13):
            ch = [skb.group_restart_chunk(L, world, r) for r in range(world)]
            blk = -(-L // world)
            assert ch[0][0] == 0 and ch[-1][1] == L
            for r, (a, b) in enumerate(ch):
                assert a == min(L, r * blk) and b == min(L, (r + 1) * blk)
