"""ctypes wrapper of the reference's own sources compiled verbatim (oracle/_ref, built by
`make -C oracle ref` from /root/reference/proj/src; see oracle/ref_capi.cpp).

TEST INFRASTRUCTURE: used only by tests/test_ref_pins.py to pin the oracle restatement to
the reference itself."""
from __future__ import annotations

import ctypes as C
import pathlib

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
REF_LIB = ROOT / "oracle" / "_ref" / "libsketchcp_ref.so"

_lib = None
d_p = C.POINTER(C.c_double)
u32_p = C.POINTER(C.c_uint32)
u8_p = C.POINTER(C.c_uint8)
vp = C.c_void_p


def available() -> bool:
    return REF_LIB.exists()


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(str(REF_LIB))
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_derive_seed": (C.c_uint64, [C.c_uint64] * 4),
            "ref_unit_sphere": (C.c_int, [C.c_uint64, C.c_int, d_p]),
            "ref_fft": (C.c_int, [d_p, C.c_size_t, C.c_int]),
            "ref_sym_create": (C.c_int, [C.c_int, C.c_uint32, C.c_int, C.c_uint64, C.POINTER(vp)]),
            "ref_sym_destroy": (None, [vp]),
            "ref_sym_tables": (C.c_int, [vp, C.c_int, u32_p, u32_p, u32_p, u8_p]),
            "ref_sym_accumulate_dense": (C.c_int, [vp, d_p, C.c_int]),
            "ref_sym_add_scaled_rank1": (C.c_int, [vp, d_p, C.c_double]),
            "ref_sym_get_data": (C.c_int, [vp, d_p]),
            "ref_sym_set_data": (C.c_int, [vp, d_p]),
            "ref_sym_recover_entry": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, d_p]),
            "ref_sym_ivv": (C.c_int, [vp, d_p, d_p]),
            "ref_sym_vvv": (C.c_int, [vp, d_p, d_p]),
            "ref_sym_rtpm": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_double, d_p, d_p]),
            "ref_asym_create": (C.c_int, [C.c_int, C.c_uint32, C.c_int, C.c_uint64, C.POINTER(vp)]),
            "ref_asym_destroy": (None, [vp]),
            "ref_asym_accumulate_dense": (C.c_int, [vp, d_p]),
            "ref_asym_get_data": (C.c_int, [vp, d_p]),
            "ref_asym_vvv": (C.c_int, [vp, d_p, d_p]),
            "ref_asym_mode_contraction": (C.c_int, [vp, C.c_int, d_p, d_p, d_p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _chk(rc):
    if rc != 0:
        raise ValueError(lib().ref_last_error().decode())


def _dp(a):
    return a.ctypes.data_as(d_p)


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def unit_sphere(seed, n):
    out = np.empty(n)
    _chk(lib().ref_unit_sphere(seed, n, _dp(out)))
    return out


def fft(x, direction):
    y = np.ascontiguousarray(x, dtype=np.complex128).copy()
    _chk(lib().ref_fft(y.ctypes.data_as(d_p), y.size, direction))
    return y


class SymSet:
    def __init__(self, n, b, B, seed):
        self.n, self.b, self.B = n, b, B
        h = vp()
        _chk(lib().ref_sym_create(n, b, B, seed, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_sym_destroy(self.h)

    def tables(self, m):
        n = self.n
        b1, b2, b3 = (np.empty(n, np.uint32) for _ in range(3))
        e = np.empty(n, np.uint8)
        _chk(lib().ref_sym_tables(self.h, m, b1.ctypes.data_as(u32_p), b2.ctypes.data_as(u32_p),
                                  b3.ctypes.data_as(u32_p), e.ctypes.data_as(u8_p)))
        return b1, b2, b3, e

    def accumulate_dense(self, T, assume_symmetric=False):
        _chk(lib().ref_sym_accumulate_dense(self.h, _dp(_f(T)), int(assume_symmetric)))

    def add_scaled_rank1(self, u, alpha):
        _chk(lib().ref_sym_add_scaled_rank1(self.h, _dp(_f(u)), float(alpha)))

    def data(self):
        out = np.empty((self.B, self.b), np.complex128)
        _chk(lib().ref_sym_get_data(self.h, out.ctypes.data_as(d_p)))
        return out

    def set_data(self, d):
        d = np.ascontiguousarray(d, dtype=np.complex128)
        _chk(lib().ref_sym_set_data(self.h, d.ctypes.data_as(d_p)))

    def recover_entry(self, i, j, k):
        out = C.c_double()
        _chk(lib().ref_sym_recover_entry(self.h, i, j, k, C.byref(out)))
        return out.value

    def ivv(self, u):
        out = np.empty(self.n)
        _chk(lib().ref_sym_ivv(self.h, _dp(_f(u)), _dp(out)))
        return out

    def vvv(self, u):
        out = C.c_double()
        _chk(lib().ref_sym_vvv(self.h, _dp(_f(u)), C.byref(out)))
        return out.value

    def rtpm(self, k, L, T, seed=0, tol=1e-12):
        lam = np.empty(k)
        V = np.empty((k, self.n))
        _chk(lib().ref_sym_rtpm(self.h, k, L, T, seed, tol, _dp(lam), _dp(V)))
        return lam, V.T.copy()


class AsymSet:
    def __init__(self, n, b, B, seed):
        self.n, self.b, self.B = n, b, B
        h = vp()
        _chk(lib().ref_asym_create(n, b, B, seed, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_asym_destroy(self.h)

    def accumulate_dense(self, T):
        _chk(lib().ref_asym_accumulate_dense(self.h, _dp(_f(T))))

    def data(self):
        out = np.empty((self.B, self.b), np.complex128)
        _chk(lib().ref_asym_get_data(self.h, out.ctypes.data_as(d_p)))
        return out

    def vvv(self, u):
        out = C.c_double()
        _chk(lib().ref_asym_vvv(self.h, _dp(_f(u)), C.byref(out)))
        return out.value

    def mode_contraction(self, free_mode, x, y):
        out = np.empty(self.n)
        _chk(lib().ref_asym_mode_contraction(self.h, free_mode, _dp(_f(x)), _dp(_f(y)), _dp(out)))
        return out
