"""ctypes binding of the C ABI (include/paro_b200.h) -> paro_b200/_lib/libparo_b200.so.

There is no CPU fallback: if the native library or a GPU is missing, the
product path raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libparo_b200.so"

_P = C.c_void_p
_D = C.c_double
_DP = C.POINTER(C.c_double)
_SZ = C.c_size_t
_SZP = C.POINTER(C.c_size_t)
_LL = C.c_longlong
_I = C.c_int


class Error(RuntimeError):
    """paro::Error (proj/include/paro/errors.hpp:10-13)."""

    code = 1

    def __init__(self, msg: str = "", residual: float = 0.0):
        super().__init__(msg)
        self.residual = residual


class InvalidArgumentError(Error):
    code = 2


class NotSpdError(Error):
    code = 3


class IterationLimitError(Error):
    """Carries the final relative residual (errors.hpp:30-33)."""

    code = 4


class DegenerateSpanError(Error):
    code = 5


class PencilError(Error):
    code = 6


class EmptyBasisError(Error):
    code = 7


class CapacityError(Error):
    code = 8


class LineageError(Error):
    code = 9


class CudaError(Error):
    code = 20


class ScfDivergenceError(Error):
    """paro::ScfDivergenceError (errors.hpp): raised by the run-level stop test, not the library."""

    code = 30


class ParseError(Error):
    """paro::ParseError (errors.hpp): run configuration / molecule file syntax."""

    code = 31


ERRORS = {c.code: c for c in (Error, InvalidArgumentError, NotSpdError, IterationLimitError, DegenerateSpanError,
                              PencilError, EmptyBasisError, CapacityError, LineageError, CudaError,
                              ScfDivergenceError, ParseError)}

# name -> (restype, argtypes)
SIGNATURES = {
    "paro_ctx_create": (_I, [_I, _P, C.POINTER(_P)]),
    "paro_ctx_destroy": (_I, [_P]),
    "paro_ctx_set_stream": (_I, [_P, _P]),
    "paro_ctx_last_error": (C.c_char_p, [_P]),
    "paro_ctx_last_residual": (_D, [_P]),
    "paro_ctx_launches": (C.c_ulonglong, [_P]),
    "paro_ctx_synchronize": (_I, [_P]),
    "paro_ctx_set_ritz_mode": (_I, [_P, _I]),
    "paro_ctx_set_hartree_mode": (_I, [_P, _I]),
    "paro_ctx_set_ritz_copyout": (_I, [_P, _P, _P, _LL, _I, _I]),
    "paro_ctx_stats": (_I, [_P, _DP, _I]),
    "paro_malloc": (_I, [_P, _SZ, C.POINTER(_P)]),
    "paro_free": (_I, [_P, _P]),
    "paro_memcpy_h2d": (_I, [_P, _P, _P, _SZ]),
    "paro_memcpy_d2h": (_I, [_P, _P, _P, _SZ]),
    "paro_upload_columns": (_I, [_P, _I, C.POINTER(_P), _SZ, _P, _LL]),
    "paro_download_columns": (_I, [_P, _I, _P, _LL, _SZ, C.POINTER(_P)]),
    "paro_grid_init": (_I, [_P, _I, _D, _D]),
    "paro_grid_dofs": (_LL, [_P]),
    "paro_op_create_const": (_I, [_P, _DP, C.POINTER(_P)]),
    "paro_op_create_var": (_I, [_P, C.POINTER(_P)]),
    "paro_op_from_csr": (_I, [_P, _SZ, _SZP, C.POINTER(C.c_uint32), _DP, C.POINTER(_P)]),
    "paro_op_to_csr": (_I, [_P, _P, _SZP, _SZP, C.POINTER(C.c_uint32), _DP]),
    "paro_op_coefficients": (_I, [_P, C.POINTER(_DP)]),
    "paro_op_weights": (_I, [_P, _DP, C.POINTER(_I)]),
    "paro_op_destroy": (_I, [_P]),
    "paro_op_apply": (_I, [_P, _P, _P, _D, _I, _P, _LL, _P, _LL]),
    "paro_cg_solve": (_I, [_P, _P, _I, _P, _P, _LL, _D, _SZ, _I, _P, _SZP, _DP]),
    "paro_source_solve_step": (_I, [_P, _P, _P, _I, _P, _LL, _DP, _D, _SZ, _D, _P, _SZP, _DP]),
    "paro_source_solve_columns": (_I, [_P, _P, _P, _I, _P, _LL, _DP, _D, _SZ, _D, _P, _SZP, _DP, C.POINTER(_I),
                                       C.POINTER(_I)]),
    "paro_shifted_source_step": (_I, [_P, _P, _P, _I, _P, _LL, _DP, _D, _SZ, _P, _DP, _SZP, _DP]),
    "paro_hartree_solve": (_I, [_P, _P, _P, _P, _D, _P, _SZP]),
    "paro_rayleigh_ritz": (_I, [_P, _P, _P, _I, _P, _LL, _SZ, _D, _DP, _P, _LL, C.POINTER(_I), _DP]),
    "paro_dense_sym_geneig": (_I, [_P, _I, _DP, _DP, _DP, _DP]),
    "paro_baseline_geneig": (_I, [_P, _P, _P, _I, _SZ, C.c_ulonglong, _DP, _P, _LL, C.POINTER(_I)]),
    "paro_b_orthonormalize": (_I, [_P, _P, _I, _P, _D, _P, C.POINTER(_I), C.POINTER(_I)]),
    "paro_fix_sign": (_I, [_P, _I, _P, _LL]),
    "paro_mesh_dump": (_I, [_I, _D, _D, C.c_char_p]),
    "paro_op_apply_planes": (_I, [_P, _P, _I, _P, _LL, _P, _I, _I]),
    "paro_gram_sym": (_I, [_P, _I, _P, _LL, _P, _LL, _LL, _LL, _P]),
    "paro_gram_rect": (_I, [_P, _I, _P, _LL, _I, _P, _LL, _LL, _LL, _P]),
    "paro_rotate": (_I, [_P, _I, _P, _LL, _P, _I, _I, _P, _LL, _LL, _LL, _I]),
    "paro_ritz_ortho": (_I, [_P, _I, _P, _D, _P, C.POINTER(_I), _DP]),
    "paro_ritz_second_pass": (_I, [_P, _I, _P, _P, _P]),
    "paro_ritz_congruence": (_I, [_P, _I, _P, _P, _P]),
    "paro_ritz_pencil": (_I, [_P, _I, _P, _P, _P, _P, _DP, _P]),
    "paro_gram_defect": (_I, [_P, _I, _P, _DP]),
    "paro_sign_init": (_I, [_P, _I, _P, _P]),
    "paro_colmax": (_I, [_P, _I, _P, _LL, _LL, _LL, _P]),
    "paro_first_above": (_I, [_P, _I, _P, _LL, _LL, _LL, _P, _P]),
    "paro_sign_flags": (_I, [_P, _I, _P, _LL, _LL, _LL, _P, _P, _P]),
    "paro_negate_columns": (_I, [_P, _I, _P, _LL, _LL, _LL, _P]),
    "paro_assemble_mass": (_I, [_P, C.POINTER(_P)]),
    "paro_assemble_stiffness": (_I, [_P, _D, C.POINTER(_P)]),
    "paro_assemble_vext": (_I, [_P, _I, _DP, _DP, _D, C.POINTER(_P)]),
    "paro_assemble_harmonic": (_I, [_P, _D, C.POINTER(_P)]),
    "paro_op_add_scaled": (_I, [_P, _P, _P, _D]),
    "paro_csr_create": (_I, [_P, _SZ, _SZP, C.POINTER(C.c_uint32), _DP, C.POINTER(_P)]),
    "paro_csr_destroy": (_I, [_P]),
    "paro_csr_add_scaled": (_I, [_P, _P, _P, _D]),
    "paro_csr_apply": (_I, [_P, _P, _I, _P, _LL, _P]),
    "paro_csr_cg_solve": (_I, [_P, _P, _I, _P, _P, _LL, _D, _SZ, _I, _P, _SZP, _DP]),
    "paro_csr_source_solve_step": (_I, [_P, _P, _P, _I, _P, _LL, _DP, _D, _SZ, _D, _P, _SZP, _DP]),
    "paro_ks_form": (_I, [_P, _P, _P, _P, _P, _I, _P, C.POINTER(_LL)]),
    "paro_ks_form_planes": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _P, C.POINTER(_LL)]),
    "paro_density": (_I, [_P, _I, _P, _LL, _DP, _P, _DP]),
    "paro_mix_density": (_I, [_P, _P, _P, _D, _P]),
    "paro_density_rows": (_I, [_P, _I, _P, _LL, _DP, _LL, _LL, _P]),
    "paro_density_normalize": (_I, [_P, _D, _P, _DP]),
    "paro_integrate": (_I, [_P, _P, _DP]),
    "paro_norm_l2": (_I, [_P, _P, _DP]),
    "paro_integrate_product": (_I, [_P, _P, _P, _DP]),
    "paro_rho_residual": (_I, [_P, _P, _P, _P, _DP]),
    "paro_total_energy": (_I, [_P, _I, _DP, _I, _DP, _P, _P, _I, _I, _DP, _DP, _DP]),
    "paro_energy_xc_layers": (_I, [_P, _P, _I, _I, _I, _DP]),
    "paro_total_energy_with_xc": (_I, [_P, _I, _DP, _I, _DP, _P, _P, _I, _DP, _DP, C.c_double, _DP]),
    "paro_estimate_eta": (_I, [_P, _I, _P, _LL, _DP, _D, _I, _D, _I, _DP, _DP, _D, _P, _P, _I, _P, _DP]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise ImportError(f"paro_b200 native library missing ({_LIB_PATH}); run `python -m paro_b200.build`")
        L = C.CDLL(str(_LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name, None)
            if f is None:
                continue
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def library_path() -> Path:
    return _LIB_PATH


def check(ctx_handle, status: int) -> None:
    if status != 0:
        L = lib()
        msg = (L.paro_ctx_last_error(ctx_handle) or b"").decode()
        res = L.paro_ctx_last_residual(ctx_handle)
        raise ERRORS.get(status, Error)(msg, res)
