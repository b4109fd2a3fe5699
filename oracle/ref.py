"""ctypes binding of oracle/_ref/libparo_ref.so — TEST INFRASTRUCTURE ONLY.

The library is the *unmodified* reference implementation (/root/reference/proj,
C++20) compiled by oracle/Makefile together with oracle/harness/ref_capi.cpp.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module, as the checker / CPU baseline. The product (paro_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "libparo_ref.so"

_P = C.c_void_p
_D = C.c_double
_DP = C.POINTER(C.c_double)
_SZ = C.c_size_t
_SZP = C.POINTER(C.c_size_t)


class RefError(RuntimeError):
    """Reference exception re-raised across the C boundary."""

    code = 1

    def __init__(self, msg: str, residual: float = 0.0):
        super().__init__(msg)
        self.residual = residual


class RefInvalidArgument(RefError):
    code = 2


class RefNotSpd(RefError):
    code = 3


class RefIterationLimit(RefError):
    code = 4


class RefDegenerateSpan(RefError):
    code = 5


class RefPencilError(RefError):
    code = 6


class RefEmptyBasis(RefError):
    code = 7


_ERRS = {c.code: c for c in (RefError, RefInvalidArgument, RefNotSpd, RefIterationLimit,
                              RefDegenerateSpan, RefPencilError, RefEmptyBasis)}

_lib = None


def available() -> bool:
    return LIB_PATH.exists()


def build() -> None:
    """Compile oracle/_ref from /root/reference (only where the reference exists)."""
    if not Path("/root/reference/proj/src").exists():
        return
    import subprocess

    subprocess.run(["make", "-s", "-j8", "-C", str(HERE), "all"], check=True)
    gpu_lib = HERE.parent / "paro_b200" / "_lib" / "libparo_b200.so"
    if gpu_lib.exists():  # the C++ drop-in check links the product library
        subprocess.run(["make", "-s", "-C", str(HERE), "dropin"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle` where /root/reference exists")
        L = C.CDLL(str(LIB_PATH))
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_last_residual": (_D, []),
            "ref_space_create": (_P, [C.c_int, _D, _D, C.c_int]),
            "ref_space_free": (None, [_P]),
            "ref_space_dofs": (_SZ, [_P]),
            "ref_space_elements": (_SZ, [_P]),
            "ref_space_dump": (C.c_int, [_P, C.c_char_p]),
            "ref_run_config": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.c_char_p, C.c_int]),
            "ref_op_mass": (_P, [_P]),
            "ref_op_stiffness": (_P, [_P, _D]),
            "ref_op_wmass_coulomb": (_P, [_P, C.c_int, _DP, _DP, _D]),
            "ref_op_wmass_harmonic": (_P, [_P, _D]),
            "ref_op_wmass_nodal": (_P, [_P, _DP]),
            "ref_op_copy": (_P, [_P]),
            "ref_op_add_scaled": (C.c_int, [_P, _P, _D]),
            "ref_op_free": (None, [_P]),
            "ref_op_nnz": (_SZ, [_P]),
            "ref_op_dim": (_SZ, [_P]),
            "ref_op_csr": (None, [_P, _SZP, C.POINTER(C.c_uint32), _DP]),
            "ref_op_from_csr": (_P, [_SZ, _SZP, C.POINTER(C.c_uint32), _DP, C.c_int]),
            "ref_matvec": (None, [_P, _DP, _DP]),
            "ref_cg": (C.c_int, [_P, _DP, _DP, _D, _SZ, C.c_int, C.c_int, _DP, _SZP, _DP, C.POINTER(C.c_int)]),
            "ref_source_solve": (C.c_int, [_P, _P, _SZ, _DP, _DP, _D, _SZ, C.c_int, _D, _DP]),
            "ref_shifted_source": (C.c_int, [_P, _P, _P, _SZ, _DP, _DP, _D, _SZ, C.c_int, _DP, _DP]),
            "ref_source_pinned": (C.c_int, [_P, _P, _SZ, _DP, _DP, _D, _SZ, C.c_int]),
            "ref_rayleigh_ritz": (C.c_int, [_P, _SZ, _DP, _P, _P, _SZ, _D, _DP, _DP, _SZP, _DP, _DP]),
            "ref_b_orthonormalize": (C.c_int, [_SZ, _SZ, _DP, _P, _D, _DP, _SZP, _SZP, _SZP]),
            "ref_gram_defect": (C.c_int, [_SZ, _SZ, _DP, _P, _DP]),
            "ref_dense_sym_geneig": (C.c_int, [_SZ, _DP, _DP, _DP, _DP]),
            "ref_baseline_geneig": (C.c_int, [_P, _P, _SZ, _SZ, C.c_uint64, _DP, _DP]),
            "ref_jacobi_eig": (C.c_int, [_SZ, _DP, _D, C.c_int, _DP, _DP]),
            "ref_fix_sign": (None, [_SZ, _DP]),
            "ref_density": (C.c_int, [_P, _SZ, _DP, _DP, _DP, _DP]),
            "ref_mix": (C.c_int, [_P, _DP, _DP, _D, _DP]),
            "ref_hartree": (C.c_int, [_P, _P, _P, _DP, _D, _DP]),
            "ref_lda": (C.c_int, [_D, C.c_int, _DP, _DP]),
            "ref_total_energy": (C.c_int, [_P, _SZ, _DP, _SZ, _DP, _DP, C.c_int, C.c_int, _DP, _DP, _DP]),
            "ref_norm_l2": (_D, [_P, _DP]),
            "ref_integrate": (_D, [_P, _DP]),
            "ref_nuclear_repulsion": (_D, [C.c_int, _DP, _DP]),
            "ref_quad_rule": (_SZ, [C.c_int, C.c_int, C.c_int, _DP, _DP]),
            "ref_ks_create": (_P, [_P, C.c_int, _DP, _DP, C.c_int, _D, C.c_int]),
            "ref_ks_free": (None, [_P]),
            "ref_ks_op": (_P, [_P, C.c_int]),
            "ref_ks_form": (_P, [_P, _DP, _DP, C.POINTER(C.c_long)]),
            "ref_ks_state_create": (_P, [_P, _SZ, _DP, _D, _D, _D, _SZ, _D, _D, C.c_int]),
            "ref_ks_state_free": (None, [_P]),
            "ref_ks_state_k": (_SZ, [_P]),
            "ref_ks_state_step": (C.c_int, [_P, C.c_int, _DP, _DP]),
            "ref_ks_state_get": (None, [_P, C.c_int, _DP]),
            "ref_ks_eta_total": (C.c_int, [_P, C.c_size_t, _DP, _DP, _DP, _DP, _DP, _DP]),
            "ref_lin_eta_total": (C.c_int, [_P, C.c_size_t, _DP, _DP, _D, C.c_int, _D, C.c_int, _DP, _DP, _D, _DP,
                                            _DP]),
            "ref_ks_state_clamped": (C.c_long, [_P]),
            "ref_lin_state_create": (_P, [_P, _P, _P, _SZ, _SZ, _DP, _D, _D, _D, _SZ, _D, C.c_int]),
            "ref_lin_state_free": (None, [_P]),
            "ref_lin_state_step": (C.c_int, [_P, C.c_int, _DP, _DP]),
            "ref_lin_state_get": (None, [_P, C.c_int, _DP]),
            "ref_lin_state_k": (_SZ, [_P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name, None)
            if f is None:  # an older build of the harness: that entry point fails when called
                continue
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_DP)


def _check(st: int):
    if st != 0:
        L = lib()
        msg = L.ref_last_error().decode()
        cls = _ERRS.get(st, RefError)
        raise cls(msg, L.ref_last_residual())


def _checkp(p):
    if not p:
        raise RefError(lib().ref_last_error().decode())
    return p


class Space:
    def __init__(self, subdivisions: int, lo: float, hi: float, dim: int = 3):
        self.h = _checkp(lib().ref_space_create(subdivisions, lo, hi, dim))
        self.s, self.lo, self.hi, self.dim = subdivisions, lo, hi, dim
        self.n = lib().ref_space_dofs(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_space_free(self.h)
            self.h = None


class Op:
    def __init__(self, handle, keep=None):
        self.h = _checkp(handle)
        self._keep = keep
        self.n = lib().ref_op_dim(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_op_free(self.h)
            self.h = None

    @staticmethod
    def mass(sp: Space) -> "Op":
        return Op(lib().ref_op_mass(sp.h), sp)

    @staticmethod
    def stiffness(sp: Space, scale: float) -> "Op":
        return Op(lib().ref_op_stiffness(sp.h, scale), sp)

    @staticmethod
    def wmass_coulomb(sp: Space, Z, R, eps: float) -> "Op":
        Z = np.ascontiguousarray(Z, np.float64)
        R = np.ascontiguousarray(R, np.float64).reshape(-1)
        return Op(lib().ref_op_wmass_coulomb(sp.h, len(Z), _dp(Z), _dp(R), eps), sp)

    @staticmethod
    def wmass_harmonic(sp: Space, c: float) -> "Op":
        return Op(lib().ref_op_wmass_harmonic(sp.h, c), sp)

    @staticmethod
    def wmass_nodal(sp: Space, w) -> "Op":
        w = np.ascontiguousarray(w, np.float64)
        return Op(lib().ref_op_wmass_nodal(sp.h, _dp(w)), sp)

    @staticmethod
    def from_csr(rows, cols, vals, symmetric=True) -> "Op":
        rows = np.ascontiguousarray(rows, np.uintp)
        cols = np.ascontiguousarray(cols, np.uint32)
        vals = np.ascontiguousarray(vals, np.float64)
        return Op(lib().ref_op_from_csr(len(rows) - 1, rows.ctypes.data_as(_SZP),
                                        cols.ctypes.data_as(C.POINTER(C.c_uint32)), _dp(vals), int(symmetric)))

    def copy(self) -> "Op":
        return Op(lib().ref_op_copy(self.h), self._keep)

    def add_scaled(self, other: "Op", s: float = 1.0) -> "Op":
        _check(lib().ref_op_add_scaled(self.h, other.h, s))
        return self

    def csr(self):
        L = lib()
        nnz = L.ref_op_nnz(self.h)
        rows = np.zeros(self.n + 1, np.uintp)
        cols = np.zeros(nnz, np.uint32)
        vals = np.zeros(nnz, np.float64)
        L.ref_op_csr(self.h, rows.ctypes.data_as(_SZP), cols.ctypes.data_as(C.POINTER(C.c_uint32)), _dp(vals))
        return rows.astype(np.int64), cols, vals

    def matvec(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(self.n)
        lib().ref_matvec(self.h, _dp(x), _dp(y))
        return y


def cg(op: Op, b, x0=None, tol=1e-10, max_iter=10000, precond=True, throw=True):
    b = np.ascontiguousarray(b, np.float64)
    x = np.empty(op.n)
    it = C.c_size_t(0)
    res = C.c_double(0)
    conv = C.c_int(0)
    x0p = _dp(np.ascontiguousarray(x0, np.float64)) if x0 is not None else None
    _check(lib().ref_cg(op.h, _dp(b), x0p, tol, max_iter, int(precond), int(throw), _dp(x),
                        C.byref(it), C.byref(res), C.byref(conv)))
    return x, it.value, res.value, bool(conv.value)


def source_solve(a: Op, b: Op, U, lambdas, tol, max_iter=100000, workers=1, sigma=0.0):
    U = np.ascontiguousarray(U, np.float64)
    lam = np.ascontiguousarray(lambdas, np.float64)
    out = np.empty_like(U)
    _check(lib().ref_source_solve(a.h, b.h, U.shape[0], _dp(U), _dp(lam), tol, max_iter, workers, sigma, _dp(out)))
    return out


def shifted_source(a: Op, b: Op, sp: Space, U, lambdas, tol, max_iter=100000, workers=1):
    U = np.ascontiguousarray(U, np.float64)
    lam = np.ascontiguousarray(lambdas, np.float64)
    out = np.empty_like(U)
    sig = C.c_double(0)
    _check(lib().ref_shifted_source(a.h, b.h, sp.h, U.shape[0], _dp(U), _dp(lam), tol, max_iter, workers,
                                    _dp(out), C.byref(sig)))
    return out, sig.value


def source_pinned(a: Op, b: Op, U, lambdas, sigma, iters, workers=1):
    U = np.ascontiguousarray(U, np.float64)
    lam = np.ascontiguousarray(lambdas, np.float64)
    _check(lib().ref_source_pinned(a.h, b.h, U.shape[0], _dp(U), _dp(lam), sigma, iters, workers))


def rayleigh_ritz(sp: Space, cands, a: Op, b: Op, min_keep, drop_tol=1e-8):
    cands = np.ascontiguousarray(cands, np.float64)
    k = cands.shape[0]
    lam = np.zeros(k)
    orbs = np.zeros_like(cands)
    kout = C.c_size_t(0)
    defect = C.c_double(0)
    t4 = np.zeros(4)
    _check(lib().ref_rayleigh_ritz(sp.h, k, _dp(cands), a.h, b.h, min_keep, drop_tol, _dp(lam), _dp(orbs),
                                   C.byref(kout), C.byref(defect), _dp(t4)))
    kk = kout.value
    return lam[:kk].copy(), orbs[:kk].copy(), defect.value, t4


def b_orthonormalize(U, b: Op, drop_tol):
    U = np.ascontiguousarray(U, np.float64)
    k, n = U.shape
    out = np.zeros_like(U)
    kout = C.c_size_t(0)
    dropped = np.zeros(max(k, 1), np.uintp)
    nd = C.c_size_t(0)
    _check(lib().ref_b_orthonormalize(k, n, _dp(U), b.h, drop_tol, _dp(out), C.byref(kout),
                                      dropped.ctypes.data_as(_SZP), C.byref(nd)))
    return out[: kout.value].copy(), [int(i) for i in dropped[: nd.value]]


def gram_defect(U, b: Op) -> float:
    U = np.ascontiguousarray(U, np.float64)
    d = C.c_double(0)
    _check(lib().ref_gram_defect(U.shape[0], U.shape[1], _dp(U), b.h, C.byref(d)))
    return d.value


def baseline_geneig(a: "Op", b: "Op", count: int, max_iter: int = 400, seed: int = 7):
    """baseline_geneig (linalg.cpp:615-623): dense (Eigen shim) up to 5,000 dofs,
    else baseline_subspace; -> (values[count], vectors[count, n])."""
    n = a.n
    vals = np.zeros(count)
    vecs = np.zeros((count, n))
    _check(lib().ref_baseline_geneig(a.h, b.h, count, max_iter, seed, _dp(vals), _dp(vecs)))
    return vals, vecs


def dense_sym_geneig(A, B):
    A = np.ascontiguousarray(A, np.float64)
    B = np.ascontiguousarray(B, np.float64)
    m = A.shape[0]
    vals = np.zeros(m)
    vecs = np.zeros((m, m))
    _check(lib().ref_dense_sym_geneig(m, _dp(A), _dp(B), _dp(vals), _dp(vecs)))
    return vals, vecs


def jacobi_eig(A, tol=1e-12, sweeps=60):
    A = np.ascontiguousarray(A, np.float64)
    m = A.shape[0]
    vals = np.zeros(m)
    vecs = np.zeros((m, m))
    _check(lib().ref_jacobi_eig(m, _dp(A), tol, sweeps, _dp(vals), _dp(vecs)))
    return vals, vecs


def fix_sign(v):
    v = np.array(v, np.float64)
    lib().ref_fix_sign(len(v), _dp(v))
    return v


def density(sp: Space, U, occ):
    U = np.ascontiguousarray(U, np.float64)
    occ = np.ascontiguousarray(occ, np.float64)
    rho = np.zeros(sp.n)
    raw = C.c_double(0)
    _check(lib().ref_density(sp.h, U.shape[0], _dp(U), _dp(occ), _dp(rho), C.byref(raw)))
    return rho, raw.value


def mix(sp: Space, rin, rout, alpha):
    out = np.zeros(sp.n)
    _check(lib().ref_mix(sp.h, _dp(np.ascontiguousarray(rin, np.float64)),
                         _dp(np.ascontiguousarray(rout, np.float64)), alpha, _dp(out)))
    return out


def hartree(sp: Space, poisson: Op, mass: Op, rho, tol=1e-11):
    out = np.zeros(sp.n)
    _check(lib().ref_hartree(sp.h, poisson.h, mass.h, _dp(np.ascontiguousarray(rho, np.float64)), tol, _dp(out)))
    return out


def lda(rho: float, exchange_only=False):
    v = C.c_double(0)
    e = C.c_double(0)
    cl = lib().ref_lda(rho, int(exchange_only), C.byref(v), C.byref(e))
    return v.value, e.value, bool(cl)


def total_energy(sp: Space, lambdas, nocc, rho, vh, Z, R, exchange_only=False):
    lam = np.ascontiguousarray(lambdas, np.float64)
    Z = np.ascontiguousarray(Z, np.float64)
    R = np.ascontiguousarray(R, np.float64).reshape(-1)
    e = C.c_double(0)
    _check(lib().ref_total_energy(sp.h, len(lam), _dp(lam), nocc, _dp(np.ascontiguousarray(rho, np.float64)),
                                  _dp(np.ascontiguousarray(vh, np.float64)), int(exchange_only), len(Z),
                                  _dp(Z), _dp(R), C.byref(e)))
    return e.value


def norm_l2(sp: Space, f) -> float:
    return lib().ref_norm_l2(sp.h, _dp(np.ascontiguousarray(f, np.float64)))


def integrate(sp: Space, f) -> float:
    return lib().ref_integrate(sp.h, _dp(np.ascontiguousarray(f, np.float64)))


def nuclear_repulsion(Z, R) -> float:
    Z = np.ascontiguousarray(Z, np.float64)
    R = np.ascontiguousarray(R, np.float64).reshape(-1)
    return lib().ref_nuclear_repulsion(len(Z), _dp(Z), _dp(R))


def quad_rule(dim: int, degree: int, levels: int = -1):
    L = lib()
    m = L.ref_quad_rule(dim, degree, levels, None, None)
    pts = np.zeros((m, 4))
    w = np.zeros(m)
    L.ref_quad_rule(dim, degree, levels, _dp(pts), _dp(w))
    return pts, w


class KsSystem:
    """Reference Kohn-Sham model + static operators (assemble_ks_operators)."""

    def __init__(self, sp: Space, Z, R, n_electrons: int, eps: float = 0.0, exchange_only=False):
        self.sp = sp
        self.Z = np.ascontiguousarray(Z, np.float64)
        self.R = np.ascontiguousarray(R, np.float64).reshape(-1, 3)
        self.nocc = n_electrons // 2
        self.exchange_only = exchange_only
        Rf = np.ascontiguousarray(self.R.reshape(-1))
        self.h = _checkp(lib().ref_ks_create(sp.h, len(self.Z), _dp(self.Z), _dp(Rf), n_electrons, eps,
                                             int(exchange_only)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_ks_free(self.h)
            self.h = None

    def op(self, which: str) -> Op:
        idx = {"mass": 0, "kinetic": 1, "vext": 2, "poisson": 3}[which]
        return Op(lib().ref_ks_op(self.h, idx), self)

    def eta_total(self, U, lambdas, rho, vh, with_eta=False):
        """Step 2 of the KS driver (paro.cpp:521-538) on the first N orbitals."""
        U = np.ascontiguousarray(U, np.float64)
        lam = np.ascontiguousarray(lambdas, np.float64)
        eta = _eta_out(self.sp, with_eta)
        tot = C.c_double(0.0)
        _check(lib().ref_ks_eta_total(self.h, U.shape[0], _dp(U), _dp(lam), _dp(np.ascontiguousarray(rho, np.float64)),
                                      _dp(np.ascontiguousarray(vh, np.float64)),
                                      _dp(eta) if eta is not None else None, C.byref(tot)))
        return (tot.value, eta) if with_eta else tot.value

    def form(self, rho, vh):
        cl = C.c_long(0)
        op = Op(lib().ref_ks_form(self.h, _dp(np.ascontiguousarray(rho, np.float64)),
                                  _dp(np.ascontiguousarray(vh, np.float64)), C.byref(cl)), self)
        return op, cl.value


def _eta_out(sp, with_eta):
    return np.empty(6 * sp.s ** 3) if with_eta else None


def lin_eta_total(sp: Space, U, lambdas, diffusion: float, reaction: str, c: float = 0.0, Z=(), R=(), eps=0.0,
                  with_eta=False):
    """Step-2 estimator of the linear driver (paro.cpp:306-315): combine_max over the
    orbitals of estimate_eigen_residual (adapt.cpp:104-115) and its total."""
    U = np.ascontiguousarray(U, np.float64)
    lam = np.ascontiguousarray(lambdas, np.float64)
    Z = np.ascontiguousarray(Z, np.float64)
    Rf = np.ascontiguousarray(np.asarray(R, np.float64).reshape(-1))
    eta = _eta_out(sp, with_eta)
    tot = C.c_double(0.0)
    kind = {"harmonic": 1, "well": 2}[reaction]
    _check(lib().ref_lin_eta_total(sp.h, U.shape[0], _dp(U), _dp(lam), diffusion, kind, c, len(Z),
                                   _dp(Z) if len(Z) else None, _dp(Rf) if len(Z) else None, eps,
                                   _dp(eta) if eta is not None else None, C.byref(tot)))
    return (tot.value, eta) if with_eta else tot.value


class KsLoop:
    """Fixed-mesh KS outer iterations through the reference (paro.cpp:514-638)."""

    def __init__(self, ks: KsSystem, guess, cg_tol_start=1e-8, cg_tol=1e-12, cg_tol_factor=0.25,
                 cg_max_iter=100000, mixing_alpha=0.3, drop_tol=1e-8, workers=1):
        self.ks = ks
        guess = np.ascontiguousarray(guess, np.float64)
        self.h = _checkp(lib().ref_ks_state_create(ks.h, guess.shape[0], _dp(guess), cg_tol_start, cg_tol,
                                                   cg_tol_factor, cg_max_iter, mixing_alpha, drop_tol, workers))
        self.k = lib().ref_ks_state_k(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_ks_state_free(self.h)
            self.h = None

    def step(self, n: int):
        lam = np.zeros(self.k)
        out = np.zeros(6)
        _check(lib().ref_ks_state_step(self.h, n, _dp(lam), _dp(out)))
        return {"lambdas": lam, "e_tot": out[0], "rho_residual": out[1], "sigma": out[2],
                "gram_defect": out[3], "t_source": out[4], "t_project": out[5]}

    def get(self, which: str):
        n = self.ks.sp.n
        idx = {"orbitals": 0, "rho_in": 1, "rho_out": 2, "lambdas": 3}[which]
        out = np.zeros((self.k, n)) if idx == 0 else np.zeros(self.k if idx == 3 else n)
        lib().ref_ks_state_get(self.h, idx, _dp(out))
        return out


class LinLoop:
    """Fixed-mesh linear ParO iterations through the reference (paro.cpp:302-370)."""

    def __init__(self, sp: Space, a: Op, b: Op, guess, n_orbitals, cg_tol_start=1e-8, cg_tol=1e-12,
                 cg_tol_factor=0.25, cg_max_iter=100000, drop_tol=1e-8, workers=1):
        guess = np.ascontiguousarray(guess, np.float64)
        self.sp, self.a, self.b = sp, a, b
        self.h = _checkp(lib().ref_lin_state_create(sp.h, a.h, b.h, guess.shape[0], n_orbitals, _dp(guess),
                                                    cg_tol_start, cg_tol, cg_tol_factor, cg_max_iter, drop_tol,
                                                    workers))
        self.k = lib().ref_lin_state_k(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_lin_state_free(self.h)
            self.h = None

    def step(self, n: int):
        lam = np.zeros(self.k)
        out = np.zeros(4)
        _check(lib().ref_lin_state_step(self.h, n, _dp(lam), _dp(out)))
        return {"lambdas": lam, "sigma": out[0], "gram_defect": out[1], "t_source": out[2], "t_project": out[3]}

    def get(self, which: str):
        idx = {"orbitals": 0, "lambdas": 3}[which]
        out = np.zeros((self.k, self.sp.n)) if idx == 0 else np.zeros(self.k)
        lib().ref_lin_state_get(self.h, idx, _dp(out))
        return out


def space_dump(sp: "Space", path) -> None:
    """Mesh::dump (mesh.cpp:198-217) of the space's mesh into `path`."""
    if lib().ref_space_dump(sp.h, str(path).encode()) != 0:
        raise RefError(lib().ref_last_error().decode())


def run_config(config_path, out_dir, workers: int = 0):
    """The reference runner (run_experiment, runner.cpp:67-121) on a config file:
    returns (exit code as tools/main.cpp maps it, summary line, error text).
    Runs in a subprocess without numpy (oracle/run_config.py)."""
    import subprocess
    import sys

    r = subprocess.run([sys.executable, str(HERE / "run_config.py"), str(config_path), str(out_dir), str(int(workers))],
                       capture_output=True, text=True, timeout=3600)
    if r.returncode != 0:
        raise RefError(f"reference runner crashed (rc {r.returncode}): {r.stderr[-500:]}")
    rc, summary, err = r.stdout.rstrip("\n").split("\t")
    return int(rc), summary, err


def workers_default() -> int:
    return os.cpu_count() or 1
