"""ctypes binding of the C-ABI in include/sketchcp_b200.h.

Loads the in-tree sm_100a library ``_lib/libsketchcp_b200.so``. There is no CPU
fallback: if the library is missing, importing the package raises; if no B200
is visible, every compute call raises :class:`CudaError`.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

_HERE = pathlib.Path(__file__).resolve().parent
# SKC_LIB_DIR: alternate build directory (instrumented experiment builds); default _lib/
LIB_PATH = pathlib.Path(os.environ["SKC_LIB_DIR"]) / "libsketchcp_b200.so" if os.environ.get("SKC_LIB_DIR") \
    else _HERE / "_lib" / "libsketchcp_b200.so"

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(this package has no CPU fallback)"
    )

def _preload_nccl() -> None:
    """The library links libnccl.so.2 (multi-GPU paths). When torch's bundled NCCL is
    installed, load that copy first, so the process holds one NCCL (the soname resolves to
    the loaded copy) whichever of torch and this library is imported first."""
    import sys

    for base in sys.path:
        cand = pathlib.Path(base or ".") / "nvidia" / "nccl" / "lib" / "libnccl.so.2"
        if cand.exists():
            try:
                C.CDLL(str(cand), mode=C.RTLD_GLOBAL)
            except OSError:
                pass
            return


_preload_nccl()
lib = C.CDLL(str(LIB_PATH))

c_int, c_u32, c_u64, c_ll, c_double, c_size = C.c_int, C.c_uint32, C.c_uint64, C.c_longlong, C.c_double, C.c_size_t
p_void, p_double, p_u32, p_u64, p_u8, p_int, p_ll = (
    C.c_void_p,
    C.POINTER(C.c_double),
    C.POINTER(C.c_uint32),
    C.POINTER(C.c_uint64),
    C.POINTER(C.c_uint8),
    C.POINTER(C.c_int),
    C.POINTER(C.c_longlong),
)
pp_void = C.POINTER(C.c_void_p)

# name -> (restype, argtypes)
SIGNATURES = {
    "skc_last_error": (C.c_char_p, []),
    "skc_version": (c_int, []),
    "skc_kernel_launch_count": (c_u64, []),
    "skc_transform_count": (c_u64, []),
    "skc_context_create": (c_int, [c_int, pp_void]),
    "skc_context_destroy": (c_int, [p_void]),
    "skc_context_synchronize": (c_int, [p_void]),
    "skc_context_stream": (c_int, [p_void, pp_void]),
    "skc_context_wait_stream": (c_int, [p_void, p_void]),
    "skc_context_build_retries": (c_int, [p_void, p_ll]),
    "skc_context_build_banded": (c_int, [p_void, p_ll]),
    "skc_device_count": (c_int, [p_int]),
    "skc_profile_enable": (c_int, [p_void, c_int]),
    "skc_profile_reset": (c_int, [p_void]),
    "skc_profile_get": (c_int, [p_void, C.c_char_p, p_double, p_u64]),
    "skc_derive_seed": (c_u64, [c_u64, c_u64, c_u64, c_u64]),
    "skc_unit_sphere": (c_int, [c_u64, c_int, p_double]),
    "skc_power_inits": (c_int, [c_u64, c_int, c_int, c_int, c_int, c_int, p_double]),
    "skc_poly_coefficients": (c_int, [c_int, c_u64, p_u64]),
    "skc_poly_eval": (c_u32, [p_u64, c_int, c_u32, c_u64]),
    "skc_sym_create": (c_int, [p_void, c_int, c_u32, c_int, c_u64, pp_void]),
    "skc_sym_create_from_coefficients": (
        c_int,
        [p_void, c_int, c_u32, c_int, c_u64, p_u64, p_u64, p_double, pp_void],
    ),
    "skc_sym_destroy": (c_int, [p_void]),
    "skc_sym_info": (c_int, [p_void, p_int, p_u32, p_int, p_u64, p_u64]),
    "skc_sym_tables": (c_int, [p_void, c_int, p_u32, p_u32, p_u32, p_u8]),
    "skc_sym_coefficients": (c_int, [p_void, p_u64, p_u64]),
    "skc_sym_accumulate_dense": (c_int, [p_void, p_void, c_int, c_int, c_int, c_int, c_int]),
    "skc_sym_add_scaled_rank1": (c_int, [p_void, p_double, c_double]),
    "skc_sym_accumulate_moment": (c_int, [p_void, p_double, p_double, c_ll, c_int]),
    "skc_sym_sketch_whitened_m3": (c_int, [p_void, c_int, c_ll, p_ll, p_int, p_int, p_double, c_double, p_ll, p_ll]),
    "skc_asym_als": (c_int, [p_void, c_int, c_int, c_double, c_u64, p_double, p_double, p_double, p_double, p_int]),
    "skc_sym_sketch_whitened_m3_shard": (c_int, [p_void, c_int, c_ll, p_ll, p_int, p_int, p_double, c_double, c_ll,
                                                 p_double, c_int, p_ll, p_ll]),
    "skc_lda_corpus_create": (c_int, [p_void, c_int, c_ll, p_ll, p_int, p_int, C.POINTER(p_void)]),
    "skc_lda_corpus_destroy": (c_int, [p_void]),
    "skc_lda_corpus_info": (c_int, [p_void, p_int, p_ll, p_ll, p_ll]),
    "skc_lda_whiten_corpus_handle": (c_int, [p_void, c_double, c_int, c_int, c_int, c_u64, p_double, p_double,
                                             p_double]),
    "skc_sym_sketch_whitened_m3_corpus": (c_int, [p_void, p_void, p_double, c_double, p_ll, p_ll]),
    "skc_lda_compute_m1": (c_int, [p_void, c_int, c_ll, p_ll, p_int, p_int, p_double]),
    "skc_lda_m2_apply": (c_int, [p_void, c_int, c_ll, p_ll, p_int, p_int, c_double, c_int, p_double, p_double]),
    "skc_lda_whiten_corpus": (c_int, [p_void, c_int, c_ll, p_ll, p_int, p_int, c_double, c_int, c_int, c_int, c_u64,
                                      p_double, p_double, p_double]),
    "skc_lda_recover_params": (c_int, [p_void, c_int, c_int, p_double, p_double, p_double, c_double, p_double, p_double]),
    "skc_lda_heldout_likelihood": (c_int, [p_void, c_int, c_int, p_double, c_int, c_ll, p_ll, p_int, p_int, p_double, p_ll]),
    "skc_lda_whiten_dense": (c_int, [p_void, c_int, p_double, c_int, c_int, c_int, c_u64, p_double, p_double,
                                     p_double]),
    "skc_sym_aux_sketches": (c_int, [p_void, c_int, p_double, p_double, p_double, p_double]),
    "skc_sym_rank1_truncated": (c_int, [p_void, c_int, p_double, p_double]),
    "skc_sym_read_data": (c_int, [p_void, c_int, p_double]),
    "skc_sym_write_data": (c_int, [p_void, c_int, p_double]),
    "skc_sym_data_device": (c_int, [p_void, pp_void, C.POINTER(c_size)]),
    "skc_sym_bump_version": (c_int, [p_void]),
    "skc_sym_recover_entry": (c_int, [p_void, c_int, c_int, c_int, p_double]),
    "skc_sym_ivv": (c_int, [p_void, p_double, c_int, p_double]),
    "skc_sym_vvv": (c_int, [p_void, p_double, c_int, p_double]),
    "skc_sym_cached_transform": (c_int, [p_void, c_int, p_double]),
    "skc_sym_rtpm": (c_int, [p_void, c_int, c_int, c_int, c_u64, c_double, p_double, p_double, p_double, p_int]),
    "skc_sym_rtpm_restarts": (c_int, [p_void, p_double, c_int, c_int, c_double, p_double, p_double]),
    "skc_nccl_unique_id": (c_int, [C.c_char_p]),
    "skc_context_comm_init": (c_int, [p_void, c_int, c_int, C.c_char_p]),
    "skc_group_create": (c_int, [p_int, c_int, pp_void]),
    "skc_context_comm_info": (c_int, [p_void, p_int, p_int]),
    "skc_group_slices": (c_int, [c_int, c_int, c_int, p_int]),
    "skc_group_restart_chunk": (c_int, [c_int, c_int, c_int, p_int, p_int]),
    "skc_sym_accumulate_dense_group": (c_int, [pp_void, c_int, pp_void, c_int, c_int, c_int]),
    "skc_sym_accumulate_moment_group": (c_int, [pp_void, c_int, pp_void, pp_void, c_ll, c_int]),
    "skc_sym_rtpm_group": (c_int, [pp_void, c_int, c_int, c_int, c_int, c_u64, c_double, p_double, p_double,
                                   p_double, p_int]),
    "skc_sym_sketch_whitened_m3_group": (c_int, [pp_void, c_int, c_int, c_ll, p_ll, p_int, p_int, p_double, c_double,
                                                 p_ll, p_ll]),
    "skc_asym_create": (c_int, [p_void, c_int, c_u32, c_int, c_u64, pp_void]),
    "skc_asym_create_from_coefficients": (
        c_int,
        [p_void, c_int, c_u32, c_int, c_u64, p_u64, p_u64, p_double, pp_void],
    ),
    "skc_asym_destroy": (c_int, [p_void]),
    "skc_asym_info": (c_int, [p_void, p_int, p_u32, p_int, p_u64, p_u64]),
    "skc_asym_tables": (c_int, [p_void, c_int, p_u32, p_double]),
    "skc_asym_coefficients": (c_int, [p_void, p_u64, p_u64]),
    "skc_asym_accumulate_dense": (c_int, [p_void, p_void, c_int, c_int, c_int, c_int]),
    "skc_asym_add_rank1": (c_int, [p_void, c_double, p_double, p_double, p_double]),
    "skc_asym_accumulate_factored": (c_int, [p_void, c_ll, p_double, p_double, p_double, p_double]),
    "skc_asym_rank1_sketch": (c_int, [p_void, c_int, p_double, p_double, p_double, p_double]),
    "skc_asym_read_data": (c_int, [p_void, c_int, p_double]),
    "skc_asym_write_data": (c_int, [p_void, c_int, p_double]),
    "skc_asym_data_device": (c_int, [p_void, pp_void, C.POINTER(c_size)]),
    "skc_asym_bump_version": (c_int, [p_void]),
    "skc_asym_recover_entry": (c_int, [p_void, c_int, c_int, c_int, p_double]),
    "skc_asym_mode_contraction": (c_int, [p_void, c_int, p_double, p_double, c_int, p_double]),
    "skc_asym_vvv": (c_int, [p_void, p_double, c_int, p_double]),
    "skc_asym_cached_transform": (c_int, [p_void, c_int, p_double]),
    "skc_fft": (c_int, [p_double, c_size, c_int]),
    "skc_peek_sketch_mode": (c_int, [C.c_char_p, p_int]),
    "skc_sym_save": (c_int, [p_void, C.c_char_p]),
    "skc_sym_load": (c_int, [p_void, C.c_char_p, pp_void]),
    "skc_asym_save": (c_int, [p_void, C.c_char_p]),
    "skc_asym_load": (c_int, [p_void, C.c_char_p, pp_void]),
    "skc_gen_planted_tensor": (c_int, [c_int, c_int, c_double, c_u64, c_int, p_void, p_double, p_double]),
    "skc_gen_planted_tensor_device": (
        c_int,
        [p_void, c_int, c_int, c_double, c_u64, c_int, p_void, p_double, p_double],
    ),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

SKC_OK, SKC_INVALID_ARGUMENT, SKC_NUMERICAL_ERROR, SKC_DEGENERATE, SKC_FORMAT_ERROR, SKC_CUDA_ERROR, SKC_OOM = range(7)
SKC_HOST, SKC_DEVICE = 0, 1
SKC_F64, SKC_F32 = 0, 1


class NumericalError(RuntimeError):
    """sketchcp::NumericalError (common.hpp:20-23)."""


class DegenerateIterationError(NumericalError):
    """sketchcp::DegenerateIterationError (common.hpp:25-28)."""


class FormatError(RuntimeError):
    """sketchcp::FormatError (common.hpp:15-18)."""


class CudaError(RuntimeError):
    """No usable sm_100 device, or a CUDA failure (there is no CPU fallback)."""


def check(status: int) -> None:
    if status == SKC_OK:
        return
    msg = lib.skc_last_error().decode(errors="replace")
    if status == SKC_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if status == SKC_DEGENERATE:
        raise DegenerateIterationError(msg)
    if status == SKC_NUMERICAL_ERROR:
        raise NumericalError(msg)
    if status == SKC_FORMAT_ERROR:
        raise FormatError(msg)
    if status == SKC_OOM:
        raise MemoryError(msg)
    raise CudaError(msg)


def loaded_path() -> str:
    return os.fspath(LIB_PATH)
