"""The C-ABI library loads without a GPU and exports every symbol that
include/paro_b200.h declares (no compute calls here)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "paro_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(paro_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("paro_source_solve_step", "paro_rayleigh_ritz", "paro_cg_solve", "paro_hartree_solve",
                 "paro_ks_form", "paro_density", "paro_total_energy", "paro_op_from_csr", "paro_op_apply",
                 "paro_dense_sym_geneig", "paro_b_orthonormalize", "paro_mix_density"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paro_b200 import _native

    path = _native.library_path()
    if not path.exists():
        pytest.skip("native library not built")
    lib = ctypes.CDLL(str(path))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    bound = _native.lib()
    for name in _native.SIGNATURES:
        assert hasattr(bound, name)


def test_no_gpu_error_path():
    """Without a device the context call fails loudly (no CPU fallback)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paro_b200 import _native

    lib = _native.lib()
    h = ctypes.c_void_p()
    st = lib.paro_ctx_create(0, None, ctypes.byref(h))
    assert st != 0
    assert lib.paro_ctx_last_error(None)
