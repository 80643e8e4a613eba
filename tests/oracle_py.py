"""ctypes wrapper of the CPU oracle (oracle/_build/liboracle.so).

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may use this module.
"""
from __future__ import annotations

import ctypes as C
import pathlib
import subprocess

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
ORACLE_DIR = ROOT / "oracle"
ORACLE_LIB = ORACLE_DIR / "_build" / "liboracle.so"


def build_oracle() -> pathlib.Path:
    src = ORACLE_DIR / "sketchcp_oracle.cpp"
    if not ORACLE_LIB.exists() or ORACLE_LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(ORACLE_DIR)], check=True)
    return ORACLE_LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(str(build_oracle()))
        _setup(_lib)
    return _lib


d_p = C.POINTER(C.c_double)
u64_p = C.POINTER(C.c_uint64)
u32_p = C.POINTER(C.c_uint32)
u8_p = C.POINTER(C.c_uint8)
i_p = C.POINTER(C.c_int)
ll_p = C.POINTER(C.c_longlong)
vp = C.c_void_p


def _setup(L):
    sig = {
        "orc_last_error": (C.c_char_p, []),
        "orc_num_threads": (C.c_int, []),
        "orc_set_num_threads": (None, [C.c_int]),
        "orc_derive_seed": (C.c_uint64, [C.c_uint64] * 4),
        "orc_sym_accumulate_dense_slice": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int]),
        "orc_gen_planted_slice": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int, C.c_int, vp,
                                            d_p, d_p]),
        "orc_rng_u64": (None, [C.c_uint64, C.c_int, u64_p]),
        "orc_lda_recover_params": (C.c_int, [C.c_int, C.c_int, d_p, d_p, d_p, C.c_double, d_p, d_p]),
        "orc_lda_heldout_likelihood": (C.c_int, [C.c_int, C.c_int, d_p, C.c_int, C.c_longlong, ll_p, i_p, i_p, d_p,
                                                 ll_p]),
        "orc_rng_gaussian": (None, [C.c_uint64, C.c_int, d_p]),
        "orc_rng_unit_sphere": (None, [C.c_uint64, C.c_int, d_p]),
        "orc_polyhash_from_seed": (C.c_int, [C.c_int, C.c_uint32, C.c_uint64, u64_p]),
        "orc_polyhash_eval": (C.c_int, [u64_p, C.c_int, C.c_uint32, u64_p, C.c_int, u32_p]),
        "orc_symmetric_bucket": (C.c_int, [u64_p, C.c_int, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, u32_p]),
        "orc_fft": (C.c_int, [d_p, C.c_size_t, C.c_int]),
        "orc_circular_convolve": (C.c_int, [d_p, d_p, C.c_size_t, C.c_size_t, d_p]),
        "orc_transform_count": (C.c_uint64, []),
        "orc_median": (C.c_double, [d_p, C.c_int]),
        "orc_sym_create": (C.c_int, [C.c_int, C.c_uint32, C.c_int, C.c_uint64, C.POINTER(vp)]),
        "orc_sym_destroy": (None, [vp]),
        "orc_sym_version": (C.c_uint64, [vp]),
        "orc_sym_tables": (C.c_int, [vp, C.c_int, u32_p, u32_p, u32_p, u8_p, u64_p, u64_p]),
        "orc_sym_accumulate_dense": (C.c_int, [vp, d_p, C.c_int]),
        "orc_sym_add_scaled_rank1": (C.c_int, [vp, d_p, C.c_double]),
        "orc_sym_get_data": (C.c_int, [vp, d_p]),
        "orc_sym_set_data": (C.c_int, [vp, d_p]),
        "orc_sym_recover_entry": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, d_p]),
        "orc_sym_rank1_truncated": (C.c_int, [vp, C.c_int, d_p, d_p]),
        "orc_sym_ivv": (C.c_int, [vp, d_p, d_p]),
        "orc_sym_vvv": (C.c_int, [vp, d_p, d_p]),
        "orc_sym_ivv_batch": (C.c_int, [vp, C.c_int, d_p, d_p]),
        "orc_sym_vvv_batch": (C.c_int, [vp, C.c_int, d_p, d_p]),
        "orc_sym_cached_transform": (C.c_int, [vp, C.c_int, d_p]),
        "orc_sym_rtpm": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_double, d_p, d_p, d_p, i_p]),
        "orc_lda_sketch_whitened_m3": (C.c_int, [vp, C.c_int, C.c_int, ll_p, i_p, i_p, d_p, C.c_double, ll_p, ll_p]),
        "orc_asym_create": (C.c_int, [C.c_int, C.c_uint32, C.c_int, C.c_uint64, C.POINTER(vp)]),
        "orc_asym_destroy": (None, [vp]),
        "orc_asym_tables": (C.c_int, [vp, C.c_int, u32_p, d_p, u64_p, u64_p]),
        "orc_asym_accumulate_dense": (C.c_int, [vp, d_p]),
        "orc_asym_add_rank1": (C.c_int, [vp, C.c_double, d_p, d_p, d_p]),
        "orc_asym_accumulate_factored": (C.c_int, [vp, C.c_int, d_p, d_p, d_p, d_p]),
        "orc_asym_rank1_sketch": (C.c_int, [vp, C.c_int, d_p, d_p, d_p, d_p]),
        "orc_asym_get_data": (C.c_int, [vp, d_p]),
        "orc_asym_recover_entry": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, d_p]),
        "orc_asym_vvv": (C.c_int, [vp, d_p, d_p]),
        "orc_asym_mode_contraction": (C.c_int, [vp, C.c_int, d_p, d_p, d_p]),
        "orc_contract_vvv_exact": (C.c_double, [d_p, C.c_int, d_p]),
        "orc_contract_Ivv_exact": (None, [d_p, C.c_int, d_p, d_p, d_p]),
        "orc_first_asymmetric_triple": (C.c_int, [d_p, C.c_int, C.c_double, i_p]),
        "orc_greedy_match": (C.c_int, [d_p, C.c_int, d_p, C.c_int, C.c_int, d_p]),
        "orc_asym_als": (C.c_int, [vp, C.c_int, C.c_int, C.c_double, C.c_uint64, d_p, d_p, d_p, d_p, i_p]),
        "orc_pinv_spectral": (C.c_int, [C.c_int, d_p, d_p]),
        "orc_lda_compute_m1": (C.c_int, [C.c_int, C.c_int, ll_p, i_p, i_p, d_p]),
        "orc_lda_compute_m2": (C.c_int, [C.c_int, C.c_int, ll_p, i_p, i_p, C.c_double, d_p]),
        "orc_sym_eigen": (C.c_int, [C.c_int, d_p, d_p, d_p]),
        "orc_lda_whiten": (C.c_int, [C.c_int, d_p, C.c_int, d_p, d_p, d_p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _chk(code):
    if code != 0:
        raise OracleError(code, lib().orc_last_error().decode())


def dp(a):
    return a.ctypes.data_as(d_p)


def f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def derive_seed(master, tag, i0=0, i1=0):
    return int(lib().orc_derive_seed(master, tag, i0, i1))


def rng_u64(seed, count):
    out = np.empty(count, dtype=np.uint64)
    lib().orc_rng_u64(seed, count, out.ctypes.data_as(u64_p))
    return out


def unit_sphere(seed, n):
    out = np.empty(n)
    lib().orc_rng_unit_sphere(seed, n, dp(out))
    return out


def polyhash_from_seed(k, b, seed):
    out = np.empty(k, dtype=np.uint64)
    _chk(lib().orc_polyhash_from_seed(k, b, seed, out.ctypes.data_as(u64_p)))
    return out


def polyhash_eval(coeffs, b, idx):
    c = np.ascontiguousarray(coeffs, dtype=np.uint64)
    i = np.ascontiguousarray(idx, dtype=np.uint64)
    out = np.empty(i.size, dtype=np.uint32)
    _chk(lib().orc_polyhash_eval(c.ctypes.data_as(u64_p), c.size, b, i.ctypes.data_as(u64_p), i.size,
                                 out.ctypes.data_as(u32_p)))
    return out


def symmetric_bucket(coeffs, b, i, j, k):
    c = np.ascontiguousarray(coeffs, dtype=np.uint64)
    out = C.c_uint32()
    _chk(lib().orc_symmetric_bucket(c.ctypes.data_as(u64_p), c.size, b, i, j, k, C.byref(out)))
    return out.value


def fft(x, direction):
    """direction: -1 forward, +1 inverse (scaled), +2 inverse unscaled."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.complex128)).copy()
    _chk(lib().orc_fft(a.ctypes.data_as(d_p), a.size, direction))
    return a


def circular_convolve(x, y):
    a = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    c = np.ascontiguousarray(np.asarray(y, dtype=np.complex128))
    out = np.empty(max(a.size, c.size), dtype=np.complex128)
    _chk(lib().orc_circular_convolve(a.ctypes.data_as(d_p), c.ctypes.data_as(d_p), a.size, c.size,
                                     out.ctypes.data_as(d_p)))
    return out


def transform_count():
    return int(lib().orc_transform_count())


def median(v):
    a = f64(v).copy()
    return float(lib().orc_median(dp(a), a.size))


class SymSet:
    def __init__(self, n, b, B, seed):
        h = vp()
        _chk(lib().orc_sym_create(n, b, B, seed, C.byref(h)))
        self.h, self.n, self.b, self.B = h, n, b, B

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_sym_destroy(self.h)

    def version(self):
        return int(lib().orc_sym_version(self.h))

    def tables(self, m):
        n = self.n
        b1, b2, b3 = (np.empty(n, dtype=np.uint32) for _ in range(3))
        se = np.empty(n, dtype=np.uint8)
        hc = np.empty(6, dtype=np.uint64)
        sc = np.empty(6, dtype=np.uint64)
        _chk(lib().orc_sym_tables(self.h, m, b1.ctypes.data_as(u32_p), b2.ctypes.data_as(u32_p),
                                  b3.ctypes.data_as(u32_p), se.ctypes.data_as(u8_p), hc.ctypes.data_as(u64_p),
                                  sc.ctypes.data_as(u64_p)))
        return b1, b2, b3, se, hc, sc

    def accumulate_dense(self, T, assume_symmetric=False):
        T = f64(T)
        _chk(lib().orc_sym_accumulate_dense(self.h, dp(T), int(bool(assume_symmetric))))

    def accumulate_dense_slice(self, T, i0, i1):
        """Rows i in [i0, i1) of sketch.cpp:315-345; T holds those rows (float64 or float32)."""
        a = np.ascontiguousarray(T)
        if a.dtype not in (np.float64, np.float32):
            a = a.astype(np.float64)
        if a.size != (i1 - i0) * self.n * self.n:
            raise ValueError("accumulate_dense_slice: T must hold (i1 - i0) * n^2 entries")
        _chk(lib().orc_sym_accumulate_dense_slice(self.h, a.ctypes.data_as(vp), int(a.dtype == np.float32),
                                                  int(i0), int(i1)))

    def add_scaled_rank1(self, u, alpha):
        _chk(lib().orc_sym_add_scaled_rank1(self.h, dp(f64(u)), float(alpha)))

    def data(self):
        out = np.empty((self.B, self.b), dtype=np.complex128)
        _chk(lib().orc_sym_get_data(self.h, out.ctypes.data_as(d_p)))
        return out

    def set_data(self, d):
        a = np.ascontiguousarray(np.asarray(d, dtype=np.complex128).reshape(self.B, self.b))
        _chk(lib().orc_sym_set_data(self.h, a.ctypes.data_as(d_p)))

    def recover_entry(self, i, j, k):
        out = C.c_double()
        _chk(lib().orc_sym_recover_entry(self.h, i, j, k, C.byref(out)))
        return out.value

    def rank1_truncated(self, m, u):
        out = np.empty(self.b, dtype=np.complex128)
        _chk(lib().orc_sym_rank1_truncated(self.h, m, dp(f64(u)), out.ctypes.data_as(d_p)))
        return out

    def ivv(self, u):
        out = np.empty(self.n)
        _chk(lib().orc_sym_ivv(self.h, dp(f64(u)), dp(out)))
        return out

    def vvv(self, u):
        out = C.c_double()
        _chk(lib().orc_sym_vvv(self.h, dp(f64(u)), C.byref(out)))
        return out.value

    def ivv_batch(self, U):
        """ivv of each row of U (L x n), restarts on the oracle's threads."""
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.empty_like(U)
        _chk(lib().orc_sym_ivv_batch(self.h, U.shape[0], dp(U), dp(out)))
        return out

    def vvv_batch(self, U):
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.empty(U.shape[0])
        _chk(lib().orc_sym_vvv_batch(self.h, U.shape[0], dp(U), dp(out)))
        return out

    def cached_transform(self, m):
        out = np.empty(self.b, dtype=np.complex128)
        _chk(lib().orc_sym_cached_transform(self.h, m, out.ctypes.data_as(d_p)))
        return out

    def rtpm(self, k, L, T, seed=0, tol=1e-12, inits=None):
        lam = np.empty(k)
        V = np.empty((k, self.n))
        bt = (C.c_int * k)()
        ip = None if inits is None else dp(f64(inits))
        _chk(lib().orc_sym_rtpm(self.h, k, L, T, seed, tol, ip, dp(lam), dp(V), bt))
        return lam, V.T.copy(), np.array(bt[:])

    def sketch_whitened_m3(self, V, doc_ptr, word, count, W, alpha0):
        dpn = np.ascontiguousarray(doc_ptr, dtype=np.int64)
        wd = np.ascontiguousarray(word, dtype=np.int32)
        ct = np.ascontiguousarray(count, dtype=np.int32)
        Wm = f64(W)
        used, skipped = C.c_longlong(), C.c_longlong()
        _chk(lib().orc_lda_sketch_whitened_m3(self.h, V, dpn.size - 1, dpn.ctypes.data_as(ll_p), wd.ctypes.data_as(i_p),
                                              ct.ctypes.data_as(i_p), dp(Wm), float(alpha0), C.byref(used),
                                              C.byref(skipped)))
        return used.value, skipped.value


class AsymSet:
    def __init__(self, n, b, B, seed):
        h = vp()
        _chk(lib().orc_asym_create(n, b, B, seed, C.byref(h)))
        self.h, self.n, self.b, self.B = h, n, b, B

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_asym_destroy(self.h)

    def tables(self, m):
        n = self.n
        bk = np.empty(3 * n, dtype=np.uint32)
        sg = np.empty(3 * n)
        hc = np.empty(6, dtype=np.uint64)
        xc = np.empty(18, dtype=np.uint64)
        _chk(lib().orc_asym_tables(self.h, m, bk.ctypes.data_as(u32_p), dp(sg), hc.ctypes.data_as(u64_p),
                                   xc.ctypes.data_as(u64_p)))
        return bk.reshape(3, n), sg.reshape(3, n), hc.reshape(3, 2), xc.reshape(3, 6)

    def accumulate_dense(self, T):
        _chk(lib().orc_asym_accumulate_dense(self.h, dp(f64(T))))

    def add_rank1(self, alpha, u, v, w):
        _chk(lib().orc_asym_add_rank1(self.h, float(alpha), dp(f64(u)), dp(f64(v)), dp(f64(w))))

    def accumulate_factored(self, a, U, V, W):
        a = f64(a)
        _chk(lib().orc_asym_accumulate_factored(self.h, a.size, dp(a), dp(f64(U)), dp(f64(V)), dp(f64(W))))

    def rank1_sketch(self, m, u, v, w):
        out = np.empty(self.b, dtype=np.complex128)
        _chk(lib().orc_asym_rank1_sketch(self.h, m, dp(f64(u)), dp(f64(v)), dp(f64(w)), out.ctypes.data_as(d_p)))
        return out

    def data(self):
        out = np.empty((self.B, self.b), dtype=np.complex128)
        _chk(lib().orc_asym_get_data(self.h, out.ctypes.data_as(d_p)))
        return out

    def recover_entry(self, i, j, k):
        out = C.c_double()
        _chk(lib().orc_asym_recover_entry(self.h, i, j, k, C.byref(out)))
        return out.value

    def vvv(self, u):
        out = C.c_double()
        _chk(lib().orc_asym_vvv(self.h, dp(f64(u)), C.byref(out)))
        return out.value

    def mode_contraction(self, free_mode, x, y):
        out = np.empty(self.n)
        _chk(lib().orc_asym_mode_contraction(self.h, free_mode, dp(f64(x)), dp(f64(y)), dp(out)))
        return out


def contract_vvv_exact(T, u):
    T = f64(T)
    return float(lib().orc_contract_vvv_exact(dp(T), T.shape[0], dp(f64(u))))


def contract_Ivv_exact(T, u, v):
    T = f64(T)
    out = np.empty(T.shape[0])
    lib().orc_contract_Ivv_exact(dp(T), T.shape[0], dp(f64(u)), dp(f64(v)), dp(out))
    return out


def asym_als(aset, k, max_iters=1000, tol=1e-6, seed=0):
    """decompose.cpp:117-205 als_fast on an oracle AsymSet -> (lambda, A, B, C, iters); factors n x k."""
    n = aset.n
    lam = np.zeros(k)
    A, B, Cm = (np.zeros((k, n)) for _ in range(3))  # column-major n x k == k x n row-major
    it = C.c_int()
    _chk(lib().orc_asym_als(aset.h, k, max_iters, tol, seed, dp(lam), dp(A), dp(B), dp(Cm), C.byref(it)))
    return lam, A.T.copy(), B.T.copy(), Cm.T.copy(), it.value


def pinv_spectral(G):
    G = f64(G)
    k = G.shape[0]
    P = np.zeros((k, k))
    _chk(lib().orc_pinv_spectral(k, dp(G), dp(P)))
    return P


def _corpus(doc_ptr, word, count):
    dpn = np.ascontiguousarray(doc_ptr, dtype=np.int64)
    wd = np.ascontiguousarray(word, dtype=np.int32)
    ct = np.ascontiguousarray(count, dtype=np.int32)
    return dpn, wd, ct


def lda_compute_m1(V, doc_ptr, word, count):
    """lda.cpp:88-100"""
    dpn, wd, ct = _corpus(doc_ptr, word, count)
    out = np.zeros(V)
    _chk(lib().orc_lda_compute_m1(V, dpn.size - 1, dpn.ctypes.data_as(ll_p), wd.ctypes.data_as(i_p),
                                  ct.ctypes.data_as(i_p), dp(out)))
    return out


def lda_compute_m2(V, doc_ptr, word, count, alpha0):
    """lda.cpp:102-123 (dense V x V)"""
    dpn, wd, ct = _corpus(doc_ptr, word, count)
    out = np.zeros((V, V))
    _chk(lib().orc_lda_compute_m2(V, dpn.size - 1, dpn.ctypes.data_as(ll_p), wd.ctypes.data_as(i_p),
                                  ct.ctypes.data_as(i_p), float(alpha0), dp(out)))
    return out


def sym_eigen(A):
    """Jacobi eigensolver (ascending), stand-in for Eigen::SelfAdjointEigenSolver."""
    A = f64(A)
    n = A.shape[0]
    ev, U = np.zeros(n), np.zeros((n, n))
    _chk(lib().orc_sym_eigen(n, dp(A), dp(ev), dp(U)))
    return ev, U


def lda_whiten(m2, k):
    """lda.cpp:125-143: (W, unwhiten, singular_values), W and unwhiten V x k."""
    m2 = f64(m2)
    V = m2.shape[0]
    W, Uw, sv = np.zeros((V, k)), np.zeros((V, k)), np.zeros(k)
    _chk(lib().orc_lda_whiten(V, dp(m2), k, dp(W), dp(Uw), dp(sv)))
    return W, Uw, sv


def gen_planted_slice(n, rank, sigma, seed, i0=0, i1=None, dtype=np.float64):
    """BASELINE configs 0-2 planted tensor rows [i0, i1) (the device generator's noise model),
    restated here so CPU arms never load the product library. Returns (T_slice, lambda, V)."""
    i1 = n if i1 is None else i1
    T = np.empty((i1 - i0, n, n), dtype=dtype)
    lam = np.empty(rank)
    V = np.empty((rank, n))
    _chk(lib().orc_gen_planted_slice(n, rank, float(sigma), int(seed), int(i0), int(i1),
                                     int(np.dtype(dtype) == np.float32), T.ctypes.data_as(vp), dp(lam), dp(V)))
    return T, lam, np.ascontiguousarray(V.T)


def greedy_match(rec, truth):
    """metrics.cpp:8-45; rec (n, r), truth (n, g). Returns rows (rec, truth, cos, sqdist)."""
    R = np.asfortranarray(f64(rec))
    G = np.asfortranarray(f64(truth))
    n, r = R.shape
    g = G.shape[1]
    Rc = np.ascontiguousarray(R.T)
    Gc = np.ascontiguousarray(G.T)
    out = np.empty((r, 4))
    _chk(lib().orc_greedy_match(dp(Rc), r, dp(Gc), g, n, dp(out)))
    return out


def lda_recover_params(V, k, lam, A, unwhiten, alpha0):
    """lda.cpp:228-248 restated (sort-based simplex projection). A k x k, column i = component."""
    Phi, alpha = np.empty((V, k)), np.empty(k)
    _chk(lib().orc_lda_recover_params(V, k, dp(f64(lam)), dp(f64(A)), dp(f64(unwhiten)), float(alpha0), dp(Phi),
                                      dp(alpha)))
    return Phi, alpha


def lda_heldout_likelihood(Phi, Vh, doc_ptr, word, count):
    """lda.cpp:273-320 restated (documents in order)."""
    V, k = Phi.shape
    dpn = np.ascontiguousarray(doc_ptr, dtype=np.int64)
    wd = np.ascontiguousarray(word, dtype=np.int32)
    ct = np.ascontiguousarray(count, dtype=np.int32)
    ll, fl = C.c_double(), C.c_longlong()
    _chk(lib().orc_lda_heldout_likelihood(V, k, dp(f64(Phi)), int(Vh), dpn.size - 1, dpn.ctypes.data_as(ll_p),
                                          wd.ctypes.data_as(i_p), ct.ctypes.data_as(i_p), C.byref(ll), C.byref(fl)))
    return ll.value, fl.value
