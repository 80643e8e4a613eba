"""B200-native FFT tensor-sketch hot path of arXiv 1506.04448.

Python mirror of the reference C++ API (proj/include/sketchcp/) over the C-ABI
in include/sketchcp_b200.h. Class and method names, argument meaning and error
behaviour follow the reference; numpy arrays stand in for Eigen vectors. All
compute runs in the sm_100a library ``_lib/libsketchcp_b200.so``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import (
    CudaError,
    DegenerateIterationError,
    FormatError,
    NumericalError,
    SKC_DEVICE,
    SKC_F32,
    SKC_F64,
    SKC_HOST,
    check,
    lib,
)

__all__ = [
    "Context",
    "default_context",
    "SymTensorSketchSet",
    "AsymTensorSketchSet",
    "SymContractionWorkspace",
    "AsymContractionWorkspace",
    "PowerConfig",
    "CpDecomposition",
    "robust_tpm_fast",
    "derive_seed",
    "unit_sphere",
    "power_inits",
    "gen_planted_tensor",
    "fft",
    "peek_sketch_mode",
    "kernel_launch_count",
    "transform_count",
    "NumericalError",
    "DegenerateIterationError",
    "FormatError",
    "CudaError",
]

SEED_TAG_POWER_INIT = 0x31  # rng.hpp:20


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a, shape=None) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None and x.shape != shape:
        raise ValueError(f"expected shape {shape}, got {x.shape}")
    return x


def derive_seed(master: int, tag: int, i0: int = 0, i1: int = 0) -> int:
    """rng.hpp:35-46"""
    return int(lib.skc_derive_seed(master, tag, i0, i1))


def unit_sphere(seed: int, n: int) -> np.ndarray:
    """Rng(seed).unit_sphere(n) (rng.hpp:100-106)."""
    out = np.empty(n)
    check(lib.skc_unit_sphere(seed, n, _dp(out)))
    return out


def power_inits(seed: int, n: int, k: int, L: int, c0: int = 0, tau0: int = 0) -> np.ndarray:
    """RTPM initial vectors (decompose.cpp:99-100): array (k, L, n)."""
    out = np.empty((k, L, n))
    check(lib.skc_power_inits(seed, n, c0, k, tau0, L, _dp(out)))
    return out


def kernel_launch_count() -> int:
    return int(lib.skc_kernel_launch_count())


def transform_count() -> int:
    """Analogue of fft::transform_count() (fft.hpp:25), in length-b transforms."""
    return int(lib.skc_transform_count())


class fft:  # noqa: N801 — mirrors namespace sketchcp::fft (fft.hpp:15-26)
    """In-place complex transforms of power-of-two length on the device."""

    @staticmethod
    def _run(x, direction):
        a = np.ascontiguousarray(np.asarray(x, dtype=np.complex128)).copy()
        check(lib.skc_fft(a.ctypes.data_as(C.POINTER(C.c_double)), a.size, direction))
        return a

    @staticmethod
    def forward(x):
        return fft._run(x, -1)

    @staticmethod
    def inverse(x):
        return fft._run(x, 1)

    @staticmethod
    def inverse_unscaled(x):
        return fft._run(x, 2)

    @staticmethod
    def circular_convolve(x, y):
        """fft.cpp:62-71"""
        x = np.asarray(x, dtype=np.complex128)
        y = np.asarray(y, dtype=np.complex128)
        if x.size != y.size:
            raise ValueError("circular_convolve: length mismatch")
        return fft.inverse(fft.forward(x) * fft.forward(y))


def peek_sketch_mode(path) -> str:
    """'sym' or 'asym' (sketch.cpp:445-449)."""
    m = C.c_int()
    check(lib.skc_peek_sketch_mode(str(path).encode(), C.byref(m)))
    return "sym" if m.value == 1 else "asym"


def device_count() -> int:
    c = C.c_int(0)
    check(lib.skc_device_count(C.byref(c)))
    return c.value


class Context:
    """One CUDA device + stream (the C-ABI skc_context)."""

    def __init__(self, device: int = 0, *, _handle=None):
        if _handle is not None:
            self._h = _handle
            self.device = device
            return
        h = C.c_void_p()
        check(lib.skc_context_create(device, C.byref(h)))
        self._h = h
        self.device = device

    def comm_init(self, nranks: int, rank: int, uid: bytes) -> None:
        """Join an NCCL communicator of nranks processes (one GPU each) with the id from
        nccl_unique_id() on rank 0 (skc_context_comm_init)."""
        check(lib.skc_context_comm_init(self._h, int(nranks), int(rank), bytes(uid)))

    def comm_info(self):
        """(nranks, rank) of this context's communicator ((1, 0) without one)."""
        a, b = C.c_int(), C.c_int()
        check(lib.skc_context_comm_info(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    @property
    def handle(self):
        return self._h

    def synchronize(self) -> None:
        check(lib.skc_context_synchronize(self._h))

    def build_retries(self) -> int:
        """fp32 dense builds repeated with two limbs after a one-limb overflow."""
        v = C.c_longlong()
        check(lib.skc_context_build_retries(self.handle, C.byref(v)))
        return v.value

    def build_banded(self) -> int:
        """Dense builds redone in magnitude bands (high-dynamic-range tensors)."""
        v = C.c_longlong()
        check(lib.skc_context_build_banded(self.handle, C.byref(v)))
        return v.value

    def stream(self) -> int:
        s = C.c_void_p()
        check(lib.skc_context_stream(self._h, C.byref(s)))
        return int(s.value or 0)

    def profile(self, on: bool = True) -> None:
        """Enable/disable per-kernel CUDA-event timing on this context's stream."""
        check(lib.skc_profile_enable(self._h, int(bool(on))))

    def profile_reset(self) -> None:
        check(lib.skc_profile_reset(self._h))

    def profile_get(self, kernel: str):
        """(total_ms, launches) for one kernel family since the last reset."""
        ms, cnt = C.c_double(), C.c_uint64()
        check(lib.skc_profile_get(self._h, kernel.encode(), C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.skc_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_DEFAULT: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _DEFAULT:
        _DEFAULT[device] = Context(device)
    return _DEFAULT[device]


def _order_after_torch(ctx: "Context", *tensors) -> None:
    """Orders the context stream after torch's current stream on the tensors' device, so a
    device input still being produced by an in-flight torch kernel (e.g. `.contiguous()`,
    `.to(float64)`, setitem) is complete before the library reads it
    (skc_context_wait_stream; no host synchronisation)."""
    import torch

    dev = next((t.device for t in tensors if t is not None), None)
    if dev is None:
        return
    check(lib.skc_context_wait_stream(ctx.handle, C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))


def _tensor_arg(T, n: int, ctx: "Context"):
    """Returns (pointer, dtype code, location, keepalive) for a dense n^3 tensor
    given as a numpy array (host) or a CUDA torch tensor (device)."""
    if hasattr(T, "is_cuda") and T.is_cuda:
        import torch

        if T.dtype not in (torch.float64, torch.float32):
            raise ValueError("accumulate_dense: tensor dtype must be float64 or float32")
        if T.numel() != n * n * n:
            raise ValueError("accumulate_dense: dimension mismatch")
        T = T.contiguous()
        _order_after_torch(ctx, T)
        return C.c_void_p(T.data_ptr()), (SKC_F64 if T.dtype == torch.float64 else SKC_F32), SKC_DEVICE, T
    a = np.asarray(T)
    if a.dtype not in (np.float64, np.float32):
        a = a.astype(np.float64)
    a = np.ascontiguousarray(a)
    if a.size != n * n * n:
        raise ValueError("accumulate_dense: dimension mismatch")
    return C.c_void_p(a.ctypes.data), (SKC_F64 if a.dtype == np.float64 else SKC_F32), SKC_HOST, a


@dataclass
class SymReplicate:
    """SymTensorSketchSet::Replicate (sketch.hpp:89-95), host copies."""

    bucket1: np.ndarray
    bucket2: np.ndarray
    bucket3: np.ndarray
    sexp: np.ndarray
    h_coefficients: np.ndarray
    sigma_coefficients: np.ndarray
    data: np.ndarray


class SymTensorSketchSet:
    """Colliding-hash sketch set for symmetric tensors (sketch.hpp:87-136)."""

    def __init__(self, n: int, b: int, B: int, master_seed: int, ctx: Context | None = None, *, _handle=None):
        self.ctx = ctx or default_context()
        if _handle is not None:
            self._h = _handle
            return
        h = C.c_void_p()
        check(lib.skc_sym_create(self.ctx.handle, int(n), int(b), int(B), int(master_seed), C.byref(h)))
        self._h = h

    @classmethod
    def from_coefficients(cls, n, b, B, master_seed, hcoef, scoef, data=None, ctx=None):
        """SymTensorSketchSet::load semantics (sketch.cpp:391-410)."""
        ctx = ctx or default_context()
        hc = np.ascontiguousarray(hcoef, dtype=np.uint64).reshape(-1)
        sc = np.ascontiguousarray(scoef, dtype=np.uint64).reshape(-1)
        if hc.size != B * 6 or sc.size != B * 6:
            raise ValueError("from_coefficients: need B*6 coefficients per hash")
        d = None if data is None else np.ascontiguousarray(np.asarray(data, dtype=np.complex128).reshape(B, b))
        h = C.c_void_p()
        check(
            lib.skc_sym_create_from_coefficients(
                ctx.handle,
                int(n),
                int(b),
                int(B),
                int(master_seed),
                hc.ctypes.data_as(C.POINTER(C.c_uint64)),
                sc.ctypes.data_as(C.POINTER(C.c_uint64)),
                None if d is None else d.ctypes.data_as(C.POINTER(C.c_double)),
                C.byref(h),
            )
        )
        return cls(n, b, B, master_seed, ctx, _handle=h)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib.skc_sym_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def _info(self):
        n, b, B, s, v = C.c_int(), C.c_uint32(), C.c_int(), C.c_uint64(), C.c_uint64()
        check(lib.skc_sym_info(self._h, C.byref(n), C.byref(b), C.byref(B), C.byref(s), C.byref(v)))
        return n.value, b.value, B.value, s.value, v.value

    def _dims(self):
        """(n, b, B): fixed for the life of a handle, so cached (one ctypes round trip saved per call)."""
        d = self.__dict__.get("_dims_cache")
        if d is None or d[0] != self._h:
            i = self._info()
            d = (self._h, i[:3])
            self.__dict__["_dims_cache"] = d
        return d[1]

    def n(self) -> int:
        return self._dims()[0]

    def b(self) -> int:
        return self._dims()[1]

    def replicates(self) -> int:
        return self._info()[2]

    def master_seed(self) -> int:
        return self._info()[3]

    def version(self) -> int:
        return self._info()[4]

    def coefficients(self):
        B = self.replicates()
        hc = np.empty(B * 6, dtype=np.uint64)
        sc = np.empty(B * 6, dtype=np.uint64)
        check(lib.skc_sym_coefficients(self._h, hc.ctypes.data_as(C.POINTER(C.c_uint64)),
                                       sc.ctypes.data_as(C.POINTER(C.c_uint64))))
        return hc.reshape(B, 6), sc.reshape(B, 6)

    def tables(self, m: int):
        n = self.n()
        b1, b2, b3 = (np.empty(n, dtype=np.uint32) for _ in range(3))
        se = np.empty(n, dtype=np.uint8)
        u32 = C.POINTER(C.c_uint32)
        check(
            lib.skc_sym_tables(
                self._h, int(m), b1.ctypes.data_as(u32), b2.ctypes.data_as(u32), b3.ctypes.data_as(u32),
                se.ctypes.data_as(C.POINTER(C.c_uint8)),
            )
        )
        return b1, b2, b3, se

    def replicate(self, m: int) -> SymReplicate:
        b1, b2, b3, se = self.tables(m)
        hc, sc = self.coefficients()
        return SymReplicate(b1, b2, b3, se, hc[m], sc[m], self.data(m))

    def data(self, m: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
        """replicate(m).data (or all B replicates as a (B, b) array). `out`: optional
        preallocated complex128 array of that shape (e.g. pinned host memory)."""
        b, B = self.b(), self.replicates()
        shape = (b,) if m is not None else (B, b)
        if out is None:
            out = np.empty(shape, dtype=np.complex128)
        elif out.shape != shape or out.dtype != np.complex128 or not out.flags.c_contiguous:
            raise ValueError(f"data: out must be a C-contiguous complex128 array of shape {shape}")
        check(lib.skc_sym_read_data(self._h, -1 if m is None else int(m), out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def set_data(self, m: int | None, values) -> None:
        """mutable_replicate(m).data = values (bumps version, sketch.hpp:105-108)."""
        b, B = self.b(), self.replicates()
        shape = (b,) if m is not None else (B, b)
        v = np.ascontiguousarray(np.asarray(values, dtype=np.complex128).reshape(shape))
        check(lib.skc_sym_write_data(self._h, -1 if m is None else int(m), v.ctypes.data_as(C.POINTER(C.c_double))))

    def accumulate_dense(self, T, assume_symmetric: bool = False, i0: int = 0, i1: int | None = None) -> None:
        """sketch.cpp:315-345; T numpy (host) or CUDA torch tensor (device), f64 or f32."""
        n = self.n()
        ptr, dt, loc, _keep = _tensor_arg(T, n, self.ctx)
        check(lib.skc_sym_accumulate_dense(self._h, ptr, dt, loc, int(bool(assume_symmetric)), int(i0),
                                           int(n if i1 is None else i1)))

    def add_scaled_rank1(self, u, alpha: float) -> None:
        """sketch.cpp:347-361"""
        n = self.n()
        u = np.asarray(u, dtype=np.float64)
        if u.shape != (n,):
            raise ValueError("add_scaled_rank1: dimension mismatch")
        u = np.ascontiguousarray(u)
        check(lib.skc_sym_add_scaled_rank1(self._h, _dp(u), float(alpha)))

    def accumulate_moment(self, X, w=None) -> None:
        """data += sum_i w_i sketch(x_i^(x)3); X (N, n) numpy or CUDA torch, w (N,) or None."""
        n = self.n()
        if hasattr(X, "is_cuda") and X.is_cuda:
            import torch

            X = X.to(torch.float64).contiguous()
            if X.ndim != 2 or X.shape[1] != n:
                raise ValueError("accumulate_moment: dimension mismatch")
            wp = None
            if w is not None:
                w = w.to(device=X.device, dtype=torch.float64).contiguous()
                wp = C.cast(C.c_void_p(w.data_ptr()), C.POINTER(C.c_double))
            _order_after_torch(self.ctx, X, w)
            check(lib.skc_sym_accumulate_moment(self._h, C.cast(C.c_void_p(X.data_ptr()), C.POINTER(C.c_double)),
                                                wp, X.shape[0], SKC_DEVICE))
            return
        X = _f64(X)
        if X.ndim != 2 or X.shape[1] != n:
            raise ValueError("accumulate_moment: dimension mismatch")
        wa = None if w is None else _f64(w, (X.shape[0],))
        check(lib.skc_sym_accumulate_moment(self._h, _dp(X), None if wa is None else _dp(wa), X.shape[0], SKC_HOST))

    def sketch_whitened_m3_shard(self, V: int, doc_ptr, word, count, W, alpha0: float, global_used: int, global_m1,
                                 add_q_cubed: bool):
        """Document-shard form (multi-GPU): sums over these documents, normalised by the
        whole corpus' global_used and M1; add_q_cubed on exactly one shard."""
        keep, (D, dpp, wdp, ctp) = _corpus_args(doc_ptr, word, count)
        Wm = _f64(W)
        m1 = _f64(global_m1, (int(V),))
        used, skipped = C.c_longlong(), C.c_longlong()
        check(lib.skc_sym_sketch_whitened_m3_shard(self._h, int(V), D, dpp, wdp, ctp, _dp(Wm), float(alpha0),
                                                   int(global_used), _dp(m1), 1 if add_q_cubed else 0,
                                                   C.byref(used), C.byref(skipped)))
        return used.value, skipped.value

    def sketch_whitened_m3_corpus(self, corpus: "LdaCorpus", W, alpha0: float):
        """sketch_whitened_m3 on a device-resident LdaCorpus (no re-upload)."""
        Wm = _f64(W)
        if Wm.shape != (corpus.V, self.n()):
            raise ValueError("sketch_whitened_m3: vocabulary mismatch")
        used, skipped = C.c_longlong(), C.c_longlong()
        check(lib.skc_sym_sketch_whitened_m3_corpus(self._h, corpus.handle, _dp(Wm), float(alpha0), C.byref(used),
                                                    C.byref(skipped)))
        return used.value, skipped.value

    def sketch_whitened_m3(self, V: int, doc_ptr, word, count, W, alpha0: float):
        """lda.cpp:145-226 on this set (n == whitening rank k). Corpus in CSR form; returns
        StreamStats as (used, skipped)."""
        dp = np.ascontiguousarray(doc_ptr, dtype=np.int64)
        wd = np.ascontiguousarray(word, dtype=np.int32)
        ct = np.ascontiguousarray(count, dtype=np.int32)
        Wm = _f64(W)
        if Wm.shape != (V, self.n()):
            raise ValueError("sketch_whitened_m3: vocabulary mismatch")
        used, skipped = C.c_longlong(), C.c_longlong()
        check(lib.skc_sym_sketch_whitened_m3(self._h, int(V), dp.size - 1, dp.ctypes.data_as(C.POINTER(C.c_longlong)),
                                             wd.ctypes.data_as(C.POINTER(C.c_int)), ct.ctypes.data_as(C.POINTER(C.c_int)),
                                             _dp(Wm), float(alpha0), C.byref(used), C.byref(skipped)))
        return used.value, skipped.value

    def aux_sketches(self, m: int, u):
        """sym_aux_sketches(replicate(m), b, u) (sketch.cpp:412-425) -> (s1, s2, s3)."""
        u = _f64(u, (self.n(),))
        b = self.b()
        out = [np.empty(b, dtype=np.complex128) for _ in range(3)]
        check(lib.skc_sym_aux_sketches(self._h, int(m), _dp(u), *[o.ctypes.data_as(C.POINTER(C.c_double)) for o in out]))
        return tuple(out)

    def rank1_truncated(self, m: int, u) -> np.ndarray:
        """sketch_rank1_sym(set, m, u) (sketch.cpp:427-443)."""
        u = _f64(u, (self.n(),))
        out = np.empty(self.b(), dtype=np.complex128)
        check(lib.skc_sym_rank1_truncated(self._h, int(m), _dp(u), out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def recover_entry(self, i: int, j: int, k: int) -> float:
        """sketch.cpp:363-377"""
        out = C.c_double()
        check(lib.skc_sym_recover_entry(self._h, int(i), int(j), int(k), C.byref(out)))
        return out.value

    def data_device(self):
        """(device pointer, bytes) of the B x b complex data, for collectives."""
        p, nb = C.c_void_p(), C.c_size_t()
        check(lib.skc_sym_data_device(self._h, C.byref(p), C.byref(nb)))
        return int(p.value), int(nb.value)

    def bump_version(self) -> None:
        check(lib.skc_sym_bump_version(self._h))

    def save(self, path) -> None:
        """sketch.cpp:379-389"""
        check(lib.skc_sym_save(self._h, str(path).encode()))

    @classmethod
    def load(cls, path, ctx: Context | None = None) -> "SymTensorSketchSet":
        """sketch.cpp:391-410"""
        ctx = ctx or default_context()
        h = C.c_void_p()
        check(lib.skc_sym_load(ctx.handle, str(path).encode(), C.byref(h)))
        obj = cls.__new__(cls)
        obj.ctx = ctx
        obj._h = h
        return obj


class SymContractionWorkspace:
    """contraction.hpp:14-41. Calls accept one n-vector or an (L, n) batch."""

    def __init__(self, set_: SymTensorSketchSet):
        self._set = set_

    def set(self) -> SymTensorSketchSet:
        return self._set

    def _batch(self, u):
        n = self._set.n()
        U = np.asarray(u, dtype=np.float64)
        single = U.ndim == 1
        U = np.ascontiguousarray(U.reshape(1, -1) if single else U)
        if U.shape[1] != n:
            raise ValueError("Ivv: dimension mismatch")
        return U, single

    def Ivv(self, u) -> np.ndarray:
        U, single = self._batch(u)
        out = np.empty_like(U)
        check(lib.skc_sym_ivv(self._set.handle, _dp(U), U.shape[0], _dp(out)))
        return out[0] if single else out

    def vvv(self, u):
        U, single = self._batch(u)
        out = np.empty(U.shape[0])
        check(lib.skc_sym_vvv(self._set.handle, _dp(U), U.shape[0], _dp(out)))
        return float(out[0]) if single else out

    def cached_transform(self, m: int) -> np.ndarray:
        b = self._set.b()
        out = np.empty(b, dtype=np.complex128)
        check(lib.skc_sym_cached_transform(self._set.handle, int(m), out.ctypes.data_as(C.POINTER(C.c_double))))
        return out


@dataclass
class PowerConfig:
    """decompose.hpp:9-17"""

    k: int = 1
    L: int = 30
    T_iters: int = 30
    b: int = 4096
    B: int = 20
    seed: int = 0
    tol: float = 1e-12


@dataclass
class CpDecomposition:
    """tensor.hpp:58-67 (symmetric_of: A = B = C copies, tensor.cpp:58-65)."""

    lambda_: np.ndarray
    A: np.ndarray
    B: np.ndarray
    C: np.ndarray
    best_tau: np.ndarray | None = None

    def rank(self) -> int:
        return int(self.lambda_.size)

    def dim(self) -> int:
        return int(self.A.shape[0])

    @staticmethod
    def symmetric_of(lam, V, best_tau=None) -> "CpDecomposition":
        return CpDecomposition(np.asarray(lam), V, V.copy(), V.copy(), best_tau)


def robust_tpm_fast(set_: SymTensorSketchSet, cfg: PowerConfig, inits=None) -> CpDecomposition:
    """decompose.cpp:83-115. inits: optional (k, L, n) initial vectors; default the
    reference's Rng(derive_seed(seed, 0x31, c, tau)).unit_sphere(n). The set is left deflated."""
    n = set_.n()
    lam = np.empty(max(cfg.k, 0))
    V = np.empty((max(cfg.k, 0), n))
    bt = (C.c_int * max(cfg.k, 1))()
    ip = None
    if inits is not None:
        inits = _f64(inits, (cfg.k, cfg.L, n))
        ip = _dp(inits)
    check(lib.skc_sym_rtpm(set_.handle, int(cfg.k), int(cfg.L), int(cfg.T_iters), int(cfg.seed), float(cfg.tol), ip,
                           _dp(lam), _dp(V), bt))
    A = np.ascontiguousarray(V.T)
    return CpDecomposition.symmetric_of(lam, A, np.array(bt[: cfg.k]))


class AsymTensorSketchSet:
    """Three-hash tensor sketch set (sketch.hpp:27-82)."""

    def __init__(self, n: int, b: int, B: int, master_seed: int, ctx: Context | None = None, *, _handle=None):
        self.ctx = ctx or default_context()
        if _handle is not None:
            self._h = _handle
            return
        h = C.c_void_p()
        check(lib.skc_asym_create(self.ctx.handle, int(n), int(b), int(B), int(master_seed), C.byref(h)))
        self._h = h

    @classmethod
    def from_coefficients(cls, n, b, B, master_seed, hcoef, xcoef, data=None, ctx=None):
        ctx = ctx or default_context()
        hc = np.ascontiguousarray(hcoef, dtype=np.uint64).reshape(-1)
        xc = np.ascontiguousarray(xcoef, dtype=np.uint64).reshape(-1)
        d = None if data is None else np.ascontiguousarray(np.asarray(data, dtype=np.complex128).reshape(B, b))
        h = C.c_void_p()
        check(
            lib.skc_asym_create_from_coefficients(
                ctx.handle, int(n), int(b), int(B), int(master_seed),
                hc.ctypes.data_as(C.POINTER(C.c_uint64)), xc.ctypes.data_as(C.POINTER(C.c_uint64)),
                None if d is None else d.ctypes.data_as(C.POINTER(C.c_double)), C.byref(h),
            )
        )
        return cls(n, b, B, master_seed, ctx, _handle=h)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib.skc_asym_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def _info(self):
        n, b, B, s, v = C.c_int(), C.c_uint32(), C.c_int(), C.c_uint64(), C.c_uint64()
        check(lib.skc_asym_info(self._h, C.byref(n), C.byref(b), C.byref(B), C.byref(s), C.byref(v)))
        return n.value, b.value, B.value, s.value, v.value

    def _dims(self):
        """(n, b, B): fixed for the life of a handle, so cached (one ctypes round trip saved per call)."""
        d = self.__dict__.get("_dims_cache")
        if d is None or d[0] != self._h:
            i = self._info()
            d = (self._h, i[:3])
            self.__dict__["_dims_cache"] = d
        return d[1]

    def n(self):
        return self._dims()[0]

    def b(self):
        return self._dims()[1]

    def replicates(self):
        return self._info()[2]

    def master_seed(self):
        return self._info()[3]

    def version(self):
        return self._info()[4]

    def coefficients(self):
        B = self.replicates()
        hc = np.empty(B * 6, dtype=np.uint64)
        xc = np.empty(B * 18, dtype=np.uint64)
        check(lib.skc_asym_coefficients(self._h, hc.ctypes.data_as(C.POINTER(C.c_uint64)),
                                        xc.ctypes.data_as(C.POINTER(C.c_uint64))))
        return hc.reshape(B, 3, 2), xc.reshape(B, 3, 6)

    def tables(self, m: int):
        n = self.n()
        bk = np.empty(3 * n, dtype=np.uint32)
        sg = np.empty(3 * n)
        check(lib.skc_asym_tables(self._h, int(m), bk.ctypes.data_as(C.POINTER(C.c_uint32)), _dp(sg)))
        return bk.reshape(3, n), sg.reshape(3, n)

    def data(self, m: int | None = None) -> np.ndarray:
        b, B = self.b(), self.replicates()
        out = np.empty((b,) if m is not None else (B, b), dtype=np.complex128)
        check(lib.skc_asym_read_data(self._h, -1 if m is None else int(m), out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def set_data(self, m, values):
        b, B = self.b(), self.replicates()
        shape = (b,) if m is not None else (B, b)
        v = np.ascontiguousarray(np.asarray(values, dtype=np.complex128).reshape(shape))
        check(lib.skc_asym_write_data(self._h, -1 if m is None else int(m), v.ctypes.data_as(C.POINTER(C.c_double))))

    def accumulate_dense(self, T, i0: int = 0, i1: int | None = None) -> None:
        """sketch.cpp:173-193"""
        n = self.n()
        ptr, dt, loc, _keep = _tensor_arg(T, n, self.ctx)
        check(lib.skc_asym_accumulate_dense(self._h, ptr, dt, loc, int(i0), int(n if i1 is None else i1)))

    def rank1_sketch(self, m: int, u, v, w) -> np.ndarray:
        """sketch.cpp:195-212"""
        n = self.n()
        u, v, w = (_f64(x, (n,)) for x in (u, v, w))
        out = np.empty(self.b(), dtype=np.complex128)
        check(lib.skc_asym_rank1_sketch(self._h, int(m), _dp(u), _dp(v), _dp(w), out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def add_rank1(self, alpha: float, u, v, w) -> None:
        """sketch.cpp:214-222"""
        n = self.n()
        u, v, w = (_f64(x, (n,)) for x in (u, v, w))
        check(lib.skc_asym_add_rank1(self._h, float(alpha), _dp(u), _dp(v), _dp(w)))

    def accumulate_factored(self, a, U, V, W) -> None:
        """sketch.cpp:224-248: components (a_i, u_i, v_i, w_i) as arrays (N,), (N, n) x 3."""
        n = self.n()
        a = _f64(a).reshape(-1)
        N = a.size
        U, V, W = (_f64(x, (N, n)) for x in (U, V, W))
        check(lib.skc_asym_accumulate_factored(self._h, N, _dp(a), _dp(U), _dp(V), _dp(W)))

    def recover_entry(self, i, j, k) -> float:
        out = C.c_double()
        check(lib.skc_asym_recover_entry(self._h, int(i), int(j), int(k), C.byref(out)))
        return out.value

    def data_device(self):
        p, nb = C.c_void_p(), C.c_size_t()
        check(lib.skc_asym_data_device(self._h, C.byref(p), C.byref(nb)))
        return int(p.value), int(nb.value)

    def bump_version(self) -> None:
        check(lib.skc_asym_bump_version(self._h))

    def save(self, path) -> None:
        """sketch.cpp:264-274"""
        check(lib.skc_asym_save(self._h, str(path).encode()))

    @classmethod
    def load(cls, path, ctx: Context | None = None) -> "AsymTensorSketchSet":
        """sketch.cpp:276-296"""
        ctx = ctx or default_context()
        h = C.c_void_p()
        check(lib.skc_asym_load(ctx.handle, str(path).encode(), C.byref(h)))
        obj = cls.__new__(cls)
        obj.ctx = ctx
        obj._h = h
        return obj


class AsymContractionWorkspace:
    """contraction.hpp:43-77"""

    def __init__(self, set_: AsymTensorSketchSet):
        self._set = set_

    def set(self):
        return self._set

    def _prep(self, x):
        n = self._set.n()
        X = np.asarray(x, dtype=np.float64)
        single = X.ndim == 1
        X = np.ascontiguousarray(X.reshape(1, -1) if single else X)
        if X.shape[1] != n:
            raise ValueError("mode_contraction: dimension mismatch")
        return X, single

    def mode_contraction(self, free_mode: int, x, y) -> np.ndarray:
        X, single = self._prep(x)
        Y, _ = self._prep(y)
        if X.shape != Y.shape:
            raise ValueError("mode_contraction: dimension mismatch")
        out = np.empty_like(X)
        check(lib.skc_asym_mode_contraction(self._set.handle, int(free_mode), _dp(X), _dp(Y), X.shape[0], _dp(out)))
        return out[0] if single else out

    def Ivv(self, u):
        return self.mode_contraction(0, u, u)

    def Ibc(self, bvec, cvec):
        return self.mode_contraction(0, bvec, cvec)

    def vvv(self, u):
        U, single = self._prep(u)
        out = np.empty(U.shape[0])
        check(lib.skc_asym_vvv(self._set.handle, _dp(U), U.shape[0], _dp(out)))
        return float(out[0]) if single else out

    def cached_transform(self, m: int) -> np.ndarray:
        out = np.empty(self._set.b(), dtype=np.complex128)
        check(lib.skc_asym_cached_transform(self._set.handle, int(m), out.ctypes.data_as(C.POINTER(C.c_double))))
        return out


class AlsConfig:
    """decompose.hpp:19-26"""

    def __init__(self, k=1, max_iters=1000, tol=1e-6, b=4096, B=40, seed=0):
        self.k, self.max_iters, self.tol, self.b, self.B, self.seed = k, max_iters, tol, b, B, seed


def als_fast(set_: "AsymTensorSketchSet", cfg: AlsConfig) -> CpDecomposition:
    """decompose.cpp:199-205: CP-ALS on the asymmetric sketch set (batched sketched mode
    contractions on the GPU). Returns CpDecomposition with A, B, C (n x k); the number of
    sweeps run is in .iters."""
    n = set_.n()
    k = int(cfg.k)
    lam = np.empty(k)
    A, B, Cm = (np.empty((k, n)) for _ in range(3))
    it = C.c_int()
    check(lib.skc_asym_als(set_.handle, k, int(cfg.max_iters), float(cfg.tol), C.c_uint64(cfg.seed), _dp(lam), _dp(A),
                           _dp(B), _dp(Cm), C.byref(it)))
    d = CpDecomposition(lam, A.T.copy(), B.T.copy(), Cm.T.copy())
    d.iters = it.value
    return d


# ---- LDA moments and whitening (lda.hpp:49-57, lda.cpp:88-143) ---------------------------
def _corpus_args(doc_ptr, word, count):
    dp = np.ascontiguousarray(doc_ptr, dtype=np.int64)
    wd = np.ascontiguousarray(word, dtype=np.int32)
    ct = np.ascontiguousarray(count, dtype=np.int32)
    return (dp, wd, ct), (dp.size - 1, dp.ctypes.data_as(C.POINTER(C.c_longlong)), wd.ctypes.data_as(C.POINTER(C.c_int)),
                          ct.ctypes.data_as(C.POINTER(C.c_int)))


class WhiteningMap:
    """lda.hpp:42-46: W (V x k, W' M2 W = I), unwhiten (V x k), singular_values (k)."""

    def __init__(self, W, unwhiten, singular_values):
        self.W, self.unwhiten, self.singular_values = W, unwhiten, singular_values


def compute_m1(V: int, doc_ptr, word, count, ctx: Context | None = None) -> np.ndarray:
    """lda.cpp:88-100 on the GPU (corpus in CSR form)."""
    ctx = ctx or default_context()
    keep, (D, dpp, wdp, ctp) = _corpus_args(doc_ptr, word, count)
    out = np.empty(V)
    check(lib.skc_lda_compute_m1(ctx.handle, int(V), D, dpp, wdp, ctp, _dp(out)))
    return out


def m2_apply(V: int, doc_ptr, word, count, alpha0: float, X, ctx: Context | None = None) -> np.ndarray:
    """M2 @ X for the implicit compute_m2(corpus, alpha0) (lda.cpp:102-123); X is V x p."""
    ctx = ctx or default_context()
    X = _f64(X)
    if X.ndim == 1:
        X = X.reshape(-1, 1)
    if X.shape[0] != V:
        raise ValueError("m2_apply: X must have V rows")
    keep, (D, dpp, wdp, ctp) = _corpus_args(doc_ptr, word, count)
    Y = np.empty_like(X)
    check(lib.skc_lda_m2_apply(ctx.handle, int(V), D, dpp, wdp, ctp, float(alpha0), X.shape[1], _dp(X), _dp(Y)))
    return Y


def whiten_corpus(V: int, doc_ptr, word, count, alpha0: float, k: int, oversample: int = -1, iters: int = -1,
                  seed: int = 0x5EED, ctx: Context | None = None) -> WhiteningMap:
    """whiten(compute_m2(corpus, alpha0), k) (lda.cpp:102-143) without forming M2:
    randomized subspace iteration + Rayleigh-Ritz on the GPU."""
    ctx = ctx or default_context()
    keep, (D, dpp, wdp, ctp) = _corpus_args(doc_ptr, word, count)
    W, U, sv = np.empty((V, k)), np.empty((V, k)), np.empty(k)
    check(lib.skc_lda_whiten_corpus(ctx.handle, int(V), D, dpp, wdp, ctp, float(alpha0), int(k), int(oversample),
                                    int(iters), C.c_uint64(seed), _dp(W), _dp(U), _dp(sv)))
    return WhiteningMap(W, U, sv)


def whiten(m2hat, k: int, oversample: int = -1, iters: int = -1, seed: int = 0x5EED,
           ctx: Context | None = None) -> WhiteningMap:
    """whiten(m2hat, k) (lda.cpp:125-143) for a dense symmetric matrix (lower triangle read)."""
    ctx = ctx or default_context()
    M = _f64(m2hat)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError("whiten: matrix must be square")
    V = M.shape[0]
    W, U, sv = np.empty((V, k)), np.empty((V, k)), np.empty(k)
    check(lib.skc_lda_whiten_dense(ctx.handle, V, _dp(M), int(k), int(oversample), int(iters), C.c_uint64(seed),
                                   _dp(W), _dp(U), _dp(sv)))
    return WhiteningMap(W, U, sv)


class LdaCorpus:
    """Device-resident corpus (B200 extension): CSR uploaded, validated and transposed
    once; whiten() and SymTensorSketchSet.sketch_whitened_m3(corpus=...) reuse it."""

    def __init__(self, V: int, doc_ptr, word, count, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        keep, (D, dpp, wdp, ctp) = _corpus_args(doc_ptr, word, count)
        h = C.c_void_p()
        check(lib.skc_lda_corpus_create(self.ctx.handle, int(V), D, dpp, wdp, ctp, C.byref(h)))
        self._h = h
        self.V = int(V)

    def __del__(self):
        if getattr(self, "_h", None):
            lib.skc_lda_corpus_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def info(self):
        V, D, nnz, u3 = C.c_int(), C.c_longlong(), C.c_longlong(), C.c_longlong()
        check(lib.skc_lda_corpus_info(self._h, C.byref(V), C.byref(D), C.byref(nnz), C.byref(u3)))
        return {"V": V.value, "D": D.value, "nnz": nnz.value, "docs_ge3": u3.value}

    def whiten(self, alpha0: float, k: int, oversample: int = -1, iters: int = -1, seed: int = 0x5EED):
        W, U, sv = np.empty((self.V, k)), np.empty((self.V, k)), np.empty(k)
        check(lib.skc_lda_whiten_corpus_handle(self._h, float(alpha0), int(k), int(oversample), int(iters),
                                               C.c_uint64(seed), _dp(W), _dp(U), _dp(sv)))
        return WhiteningMap(W, U, sv)


class LdaModel:
    """lda.hpp:33-39: Phi (V x k, column-stochastic) and alpha (k)."""

    def __init__(self, Phi, alpha):
        self.Phi, self.alpha = Phi, alpha

    def alpha0(self) -> float:
        return float(self.alpha.sum())


def recover_params(dec: "CpDecomposition", wm: WhiteningMap, alpha0: float, ctx: Context | None = None) -> LdaModel:
    """lda.cpp:228-248 on the device (topic vectors and their simplex projections)."""
    ctx = ctx or default_context()
    A = _f64(dec.A)
    k = A.shape[1]
    if A.shape[0] != wm.W.shape[1]:
        raise ValueError("recover_params: decomposition/whitening rank mismatch")
    lam = _f64(dec.lambda_)
    V = wm.unwhiten.shape[0]
    Phi, alpha = np.empty((V, k)), np.empty(k)
    check(lib.skc_lda_recover_params(ctx.handle, V, k, _dp(lam), _dp(A), _dp(_f64(wm.unwhiten)), float(alpha0),
                                     _dp(Phi), _dp(alpha)))
    return LdaModel(Phi, alpha)


def heldout_likelihood(model: LdaModel, V_held: int, doc_ptr, word, count, ctx: Context | None = None):
    """lda.cpp:273-320 on the device -> (mean per-word log-likelihood, floored word count)."""
    ctx = ctx or default_context()
    Phi = _f64(model.Phi)
    keep, (D, dpp, wdp, ctp) = _corpus_args(doc_ptr, word, count)
    ll, fl = C.c_double(), C.c_longlong()
    check(lib.skc_lda_heldout_likelihood(ctx.handle, Phi.shape[0], Phi.shape[1], _dp(Phi), int(V_held), D, dpp, wdp, ctp,
                                         C.byref(ll), C.byref(fl)))
    return ll.value, fl.value


def gen_planted_tensor(n: int, rank: int, sigma: float, seed: int, dtype=np.float64):
    """Host generator of the BASELINE planted tensors (configs 0-2). Returns (T, lambda, V)."""
    T = np.empty((n, n, n), dtype=dtype)
    lam = np.empty(rank)
    V = np.empty((rank, n))
    check(lib.skc_gen_planted_tensor(n, rank, float(sigma), int(seed), SKC_F64 if T.dtype == np.float64 else SKC_F32,
                                     C.c_void_p(T.ctypes.data), _dp(lam), _dp(V)))
    return T, lam, np.ascontiguousarray(V.T)


def gen_planted_tensor_device(ctx: Context, n: int, rank: int, sigma: float, seed: int, out_ptr: int, dtype=np.float64):
    """Device generator into a caller-owned buffer (e.g. a torch CUDA tensor's data_ptr)."""
    lam = np.empty(rank)
    V = np.empty((rank, n))
    check(lib.skc_gen_planted_tensor_device(ctx.handle, n, rank, float(sigma), int(seed),
                                            SKC_F64 if np.dtype(dtype) == np.float64 else SKC_F32,
                                            C.c_void_p(out_ptr), _dp(lam), _dp(V)))
    return lam, np.ascontiguousarray(V.T)


# ---------------------------------------------------------------- multi-GPU (NCCL)
def nccl_unique_id() -> bytes:
    """A fresh NCCL communicator id (128 bytes) for Context.comm_init on every rank."""
    buf = C.create_string_buffer(128)
    check(lib.skc_nccl_unique_id(buf))
    return buf.raw


def group_slices(n: int, world: int, sym: bool = True) -> list[tuple[int, int]]:
    """Equal-work i-slices of a dense build across `world` ranks (skc_group_slices)."""
    b = (C.c_int * (world + 1))()
    check(lib.skc_group_slices(int(n), int(bool(sym)), int(world), b))
    return [(b[r], b[r + 1]) for r in range(world)]


def group_restart_chunk(L: int, world: int, rank: int) -> tuple[int, int]:
    """Restarts [t0, t1) of a rank in a multi-GPU RTPM (skc_group_restart_chunk)."""
    a, b = C.c_int(), C.c_int()
    check(lib.skc_group_restart_chunk(int(L), int(world), int(rank), C.byref(a), C.byref(b)))
    return a.value, b.value


def group_contexts(devices) -> list[Context]:
    """One context per GPU in `devices`, joined by one NCCL communicator (ncclCommInitAll,
    skc_group_create), in rank order."""
    devices = [int(d) for d in devices]
    arr = (C.c_int * len(devices))(*devices)
    hs = (C.c_void_p * len(devices))()
    check(lib.skc_group_create(arr, len(devices), hs))
    return [Context(d, _handle=C.c_void_p(hs[i])) for i, d in enumerate(devices)]


class SymReplicas:
    """Replicas of one SymTensorSketchSet on the GPUs of an NCCL communicator: this
    process's local contexts (all of them after group_contexts(); one per process after
    Context.comm_init). Every operation is collective over all ranks and leaves every
    replica holding the same sketch (include/sketchcp_b200.h, multi-GPU section)."""

    def __init__(self, n: int, b: int, B: int, master_seed: int, contexts):
        self.contexts = list(contexts)
        self.sets = [SymTensorSketchSet(n, b, B, master_seed, c) for c in self.contexts]

    def _handles(self):
        return (C.c_void_p * len(self.sets))(*[s.handle.value for s in self.sets])

    def __len__(self):
        return len(self.sets)

    def accumulate_dense(self, T, assume_symmetric: bool = True) -> None:
        """sketch.cpp:315-345 over equal-work i-slices, exact accumulators all-reduced. T:
        one numpy array for all replicas, or one CUDA tensor per replica (on its device)."""
        Ts = T if isinstance(T, (list, tuple)) else [T] * len(self.sets)
        args = [_tensor_arg(t, s.n(), s.ctx) for t, s in zip(Ts, self.sets)]
        ptrs = (C.c_void_p * len(args))(*[a[0].value if isinstance(a[0], C.c_void_p) else a[0] for a in args])
        dt, loc = args[0][1], args[0][2]
        check(lib.skc_sym_accumulate_dense_group(self._handles(), len(self.sets), ptrs, dt, loc,
                                                 int(bool(assume_symmetric))))

    def accumulate_moment(self, X, w=None) -> None:
        """data += sum_i w_i sketch(x_i^(x)3) over sample blocks; X (N, n) host numpy."""
        n = self.sets[0].n()
        X = _f64(X)
        if X.ndim != 2 or X.shape[1] != n:
            raise ValueError("accumulate_moment: dimension mismatch")
        wa = None if w is None else _f64(w, (X.shape[0],))
        xs = (C.c_void_p * len(self.sets))(*([X.ctypes.data] * len(self.sets)))
        ws = None if wa is None else (C.c_void_p * len(self.sets))(*([wa.ctypes.data] * len(self.sets)))
        check(lib.skc_sym_accumulate_moment_group(self._handles(), len(self.sets), xs, ws, X.shape[0], SKC_HOST))

    def rtpm(self, cfg: "PowerConfig", inits=None) -> "CpDecomposition":
        """decompose.cpp:83-115 with the L restarts split across ranks; the replicas are left
        deflated."""
        n = self.sets[0].n()
        lam = np.empty(cfg.k)
        V = np.empty((cfg.k, n))
        bt = (C.c_int * cfg.k)()
        ip = None
        if inits is not None:
            inits = _f64(inits, (cfg.k, cfg.L, n))
            ip = _dp(inits)
        check(lib.skc_sym_rtpm_group(self._handles(), len(self.sets), int(cfg.k), int(cfg.L), int(cfg.T_iters),
                                     int(cfg.seed), float(cfg.tol), ip, _dp(lam), _dp(V), bt))
        return CpDecomposition.symmetric_of(lam, np.ascontiguousarray(V.T), np.array(bt[: cfg.k]))

    def sketch_whitened_m3(self, V: int, doc_ptr, word, count, W, alpha0: float):
        """lda.cpp:145-226 over document blocks; returns (used, skipped) of the whole corpus."""
        _keep, (D, dpp, wdp, ctp) = _corpus_args(doc_ptr, word, count)
        Wm = _f64(W)
        used, skipped = C.c_longlong(), C.c_longlong()
        check(lib.skc_sym_sketch_whitened_m3_group(self._handles(), len(self.sets), int(V), D, dpp, wdp, ctp, _dp(Wm),
                                                   float(alpha0), C.byref(used), C.byref(skipped)))
        return used.value, skipped.value

    def data(self, r: int = 0) -> np.ndarray:
        return self.sets[r].data()
