"""Host mirror of the reference's solver/operator interface over the C ABI.

Names, argument meaning and error behaviour follow proj/include/paro
(linalg.hpp, paro.hpp, model.hpp); vectors are torch float64 CUDA tensors of
shape [n] or [k, n] (k orbitals, interior-dof order). The heavy lifting (CG
loop, Gram/pencil, assembly) runs natively; this module only marshals.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N

_DP = C.POINTER(C.c_double)


def _ptr(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


def _as_cols(x: torch.Tensor, n: int) -> torch.Tensor:
    if x.dim() == 1:
        x = x.unsqueeze(0)
    if x.dtype != torch.float64 or not x.is_cuda:
        raise N.InvalidArgumentError("paro_b200: vectors must be float64 CUDA tensors")
    if x.shape[1] != n or x.stride(1) != 1:
        raise N.InvalidArgumentError("paro_b200: vector length does not match the grid")
    return x


class Context:
    """One paro_ctx bound to a CUDA device and (by default) torch's current stream."""

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("paro_b200 requires a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", device)
        self.stream = stream or torch.cuda.current_stream(self.device)
        h = C.c_void_p()
        st = N.lib().paro_ctx_create(device, C.c_void_p(self.stream.cuda_stream), C.byref(h))
        if st != 0:
            raise N.ERRORS.get(st, N.Error)(N.lib().paro_ctx_last_error(None).decode())
        self.h = h
        self.s = None
        self.n = 0

    def close(self):
        if getattr(self, "h", None):
            N.lib().paro_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, st: int):
        N.check(self.h, st)

    def set_stream(self, stream: torch.cuda.Stream):
        self.stream = stream
        self.check(N.lib().paro_ctx_set_stream(self.h, C.c_void_p(stream.cuda_stream)))

    def grid(self, subdivisions: int, lo: float, hi: float) -> "Context":
        """create_box_mesh([lo,hi]^3, subdivisions) + FeSpace::create (mesh.cpp:411-478)."""
        self.check(N.lib().paro_grid_init(self.h, subdivisions, lo, hi))
        self.s, self.lo, self.hi = subdivisions, lo, hi
        self.S = subdivisions - 1
        self.n = N.lib().paro_grid_dofs(self.h)
        self.hgrid = (hi - lo) / subdivisions
        return self

    def launches(self) -> int:
        return int(N.lib().paro_ctx_launches(self.h))

    def stats(self, reset: bool = False) -> dict:
        """Live PCG accounting (seconds, algorithmic bytes, column-iterations)."""
        out = (C.c_double * 8)()
        N.lib().paro_ctx_stats(self.h, out, int(reset))
        return {"step3_s": out[0], "step3_bytes": out[1], "step3_col_iters": out[2],
                "hartree_s": out[3], "hartree_bytes": out[4], "hartree_col_iters": out[5]}

    def synchronize(self):
        self.check(N.lib().paro_ctx_synchronize(self.h))

    def set_ritz_copyout(self, stream: torch.cuda.Stream, host: torch.Tensor, c0: int, c1: int):
        """One-shot: the next rayleigh_ritz copies its orbital columns [c0, c1)
        to the pinned host tensor `host` [K, n] on `stream` as soon as they are
        final (overlapping the Gram certificate); synchronise `stream` to use them."""
        self.check(N.lib().paro_ctx_set_ritz_copyout(self.h, C.c_void_p(stream.cuda_stream), _ptr(host),
                                                      host.stride(0), c0, c1))

    def set_hartree_mode(self, mode: str) -> "Context":
        """'cg': Jacobi-PCG to tol (reference algorithm); 'dst': exact DST-I solve when applicable."""
        self.check(N.lib().paro_ctx_set_hartree_mode(self.h, {"cg": 0, "dst": 1}[mode]))
        return self

    def set_ritz_mode(self, mode: str) -> "Context":
        """'cholqr': Cholesky-QR (one K x K pass for well-conditioned candidates, else twice) with
        Gram-Schmidt fallback; 'cholqr2': always twice; 'cgs2': always Gram-Schmidt."""
        self.check(N.lib().paro_ctx_set_ritz_mode(self.h, {"cholqr": 0, "cgs2": 1, "cholqr2": 2}[mode]))
        return self

    def empty(self, *shape) -> torch.Tensor:
        return torch.empty(*shape, dtype=torch.float64, device=self.device)

    def zeros(self, *shape) -> torch.Tensor:
        return torch.zeros(*shape, dtype=torch.float64, device=self.device)


class Operator:
    """SparseOperator (linalg.hpp:14-50) as a 15-point P1/Kuhn stencil."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self.h = handle
        w = (C.c_double * 8)()
        var = C.c_int(0)
        ctx.check(N.lib().paro_op_weights(self.h, w, C.byref(var)))
        self.variable = bool(var.value)
        self.weights = np.array(list(w))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                N.lib().paro_op_destroy(self.h)
                self.h = None
        except Exception:
            pass

    @classmethod
    def constant(cls, ctx: Context, w) -> "Operator":
        arr = (C.c_double * 8)(*[float(v) for v in w])
        h = C.c_void_p()
        ctx.check(N.lib().paro_op_create_const(ctx.h, arr, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def variable_empty(cls, ctx: Context) -> "Operator":
        h = C.c_void_p()
        ctx.check(N.lib().paro_op_create_var(ctx.h, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_csr(cls, ctx: Context, rows, cols, vals) -> "Operator":
        """SparseOperator(n, row_offsets, cols, vals) -> stencil (pattern-checked)."""
        rows = np.ascontiguousarray(rows, np.uintp)
        cols = np.ascontiguousarray(cols, np.uint32)
        vals = np.ascontiguousarray(vals, np.float64)
        h = C.c_void_p()
        ctx.check(N.lib().paro_op_from_csr(ctx.h, len(rows) - 1, rows.ctypes.data_as(C.POINTER(C.c_size_t)),
                                           cols.ctypes.data_as(C.POINTER(C.c_uint32)), vals.ctypes.data_as(_DP),
                                           C.byref(h)))
        return cls(ctx, h)

    def coefficients(self) -> torch.Tensor:
        """Device view [8, n] of a variable operator's SoA coefficients."""
        p = _DP()
        self.ctx.check(N.lib().paro_op_coefficients(self.h, C.byref(p)))
        n = self.ctx.n
        addr = C.cast(p, C.c_void_p).value
        return _wrap_device(addr, (8, n), self.ctx.device, owner=self)

    def to_csr(self):
        nnz = C.c_size_t(0)
        self.ctx.check(N.lib().paro_op_to_csr(self.ctx.h, self.h, C.byref(nnz), None, None, None))
        rows = np.zeros(self.ctx.n + 1, np.uintp)
        cols = np.zeros(nnz.value, np.uint32)
        vals = np.zeros(nnz.value, np.float64)
        self.ctx.check(N.lib().paro_op_to_csr(self.ctx.h, self.h, C.byref(nnz),
                                              rows.ctypes.data_as(C.POINTER(C.c_size_t)),
                                              cols.ctypes.data_as(C.POINTER(C.c_uint32)), vals.ctypes.data_as(_DP)))
        return rows.astype(np.int64), cols, vals

    def apply(self, x: torch.Tensor, shift: "Operator | None" = None, sigma: float = 0.0,
              out: torch.Tensor | None = None) -> torch.Tensor:
        """y = (A + sigma*shift) x  (SparseOperator::apply / matvec, linalg.cpp:88-100)."""
        squeeze = x.dim() == 1
        xc = _as_cols(x, self.ctx.n)
        y = out if out is not None else torch.empty_like(xc)
        y = _as_cols(y, self.ctx.n)
        if xc.stride(0) != y.stride(0):
            raise N.InvalidArgumentError("apply: x and y strides differ")
        ld = xc.stride(0) if xc.shape[0] > 1 else self.ctx.n
        self.ctx.check(N.lib().paro_op_apply(self.ctx.h, self.h, shift.h if shift else None, sigma, xc.shape[0],
                                             _ptr(xc), ld, _ptr(y), ld))
        return y[0] if squeeze else y


def _wrap_device(addr: int, shape, device, owner=None) -> torch.Tensor:
    """Zero-copy torch view of device memory owned by the native library."""
    numel = int(np.prod(shape))

    class _Holder:
        __cuda_array_interface__ = {"shape": (numel,), "typestr": "<f8", "data": (addr, False), "version": 3,
                                    "strides": None}

    h = _Holder()
    t = torch.as_tensor(h, device=device).view(*shape)
    t._paro_owner = owner  # keep the operator alive while the view exists
    return t


@dataclass
class CgResult:
    """CgResult (linalg.hpp:107-112), per column."""

    x: torch.Tensor
    iterations: list = field(default_factory=list)
    residual: list = field(default_factory=list)
    converged: list = field(default_factory=list)


def cg_solve(a: Operator, b: torch.Tensor, x0: torch.Tensor | None = None, tol: float = 1e-10,
             max_iter: int = 10000, throw_on_max_iter: bool = True) -> CgResult:
    """cg_solve (linalg.cpp:143-223), Jacobi preconditioner, k right-hand sides at once."""
    ctx = a.ctx
    squeeze = b.dim() == 1
    bc = _as_cols(b, ctx.n).contiguous()
    k = bc.shape[0]
    x = torch.empty_like(bc)
    x0c = _as_cols(x0, ctx.n).contiguous() if x0 is not None else None
    it = (C.c_size_t * k)()
    res = (C.c_double * k)()
    st = N.lib().paro_cg_solve(ctx.h, a.h, k, _ptr(bc), _ptr(x0c) if x0c is not None else None, ctx.n, tol,
                               max_iter, int(throw_on_max_iter), _ptr(x), it, res)
    ctx.check(st)
    iters = list(it)
    resid = list(res)
    conv = [r <= tol for r in resid]
    return CgResult(x[0] if squeeze else x, iters, resid, conv)


def source_solve_step(a: Operator, b: Operator, u_prev: torch.Tensor, lambdas, tol: float = 1e-10,
                      max_iter: int = 100000, sigma: float = 0.0, out: torch.Tensor | None = None,
                      report: dict | None = None) -> torch.Tensor:
    """Step 3, source_solve_step (paro.cpp:81-119), all K orbitals in one batch."""
    ctx = a.ctx
    u = _as_cols(u_prev, ctx.n)
    k = u.shape[0]
    if len(lambdas) != k:
        raise N.InvalidArgumentError("source_solve_step: orbital/lambda count mismatch")
    if u.stride(0) != ctx.n:
        u = u.contiguous()
    y = out if out is not None else torch.empty_like(u)
    lam = (C.c_double * k)(*[float(v) for v in lambdas])
    it = (C.c_size_t * k)()
    res = (C.c_double * k)()
    st = N.lib().paro_source_solve_step(ctx.h, a.h, b.h, k, _ptr(u), ctx.n, lam, tol, max_iter, sigma, _ptr(y),
                                        it, res)
    if report is not None:
        report.update(iterations=list(it), residual=list(res))
    ctx.check(st)
    return y


def source_solve_columns(a: Operator, b: Operator, u_prev: torch.Tensor, lambdas, tol: float, max_iter: int,
                         sigma: float, out: torch.Tensor):
    """Batched Step 3 with per-column outcomes (no exception collapsing).

    Returns (first_status, final_status, iterations, residual) lists; the
    caller applies source_solve_step's exception order (paro.cpp:110-117)."""
    ctx = a.ctx
    u = _as_cols(u_prev, ctx.n)
    k = u.shape[0]
    lam = (C.c_double * k)(*[float(v) for v in lambdas])
    it = (C.c_size_t * k)()
    res = (C.c_double * k)()
    fs = (C.c_int * k)()
    ls = (C.c_int * k)()
    st = N.lib().paro_source_solve_columns(ctx.h, a.h, b.h, k, _ptr(u), u.stride(0) if k > 1 else ctx.n, lam, tol,
                                           max_iter, sigma, _ptr(out), it, res, fs, ls)
    if st not in (0, N.NotSpdError.code, N.IterationLimitError.code):
        ctx.check(st)
    return list(fs), list(ls), list(it), list(res)


def shifted_source_step(a: Operator, b: Operator, u_prev: torch.Tensor, lambdas, tol: float = 1e-10,
                        max_iter: int = 100000, out: torch.Tensor | None = None, report: dict | None = None):
    """shifted_source_step (paro.cpp:194-210) -> (u_half, sigma)."""
    ctx = a.ctx
    u = _as_cols(u_prev, ctx.n)
    if u.stride(0) != ctx.n:
        u = u.contiguous()
    k = u.shape[0]
    y = out if out is not None else torch.empty_like(u)
    lam = (C.c_double * k)(*[float(v) for v in lambdas])
    it = (C.c_size_t * k)()
    res = (C.c_double * k)()
    sig = C.c_double(0.0)
    st = N.lib().paro_shifted_source_step(ctx.h, a.h, b.h, k, _ptr(u), ctx.n, lam, tol, max_iter, _ptr(y),
                                          C.byref(sig), it, res)
    if report is not None:
        report.update(iterations=list(it), residual=list(res), sigma=sig.value)
    ctx.check(st)
    return y, sig.value


def hartree_solve_with(poisson: Operator, mass: Operator, rho: torch.Tensor, tol: float = 1e-11,
                       out: torch.Tensor | None = None, report: dict | None = None) -> torch.Tensor:
    """hartree_solve_with (model.cpp:242-255)."""
    ctx = poisson.ctx
    r = _as_cols(rho, ctx.n).contiguous()
    vh = out if out is not None else ctx.empty(ctx.n)
    it = C.c_size_t(0)
    st = N.lib().paro_hartree_solve(ctx.h, poisson.h, mass.h, _ptr(r), tol, _ptr(vh), C.byref(it))
    if report is not None:
        report.update(iterations=it.value)
    ctx.check(st)
    return vh


@dataclass
class OrbitalSet:
    """OrbitalSet (paro.hpp:16-23): B-orthonormal orbitals [k, n] + ascending lambdas."""

    orbitals: torch.Tensor
    lambdas: list
    gram_defect: float = 0.0

    def count(self) -> int:
        return len(self.lambdas)


def rayleigh_ritz(candidates: torch.Tensor, a_form: Operator, b: Operator, min_keep: int, drop_tol: float = 1e-8,
                  out: torch.Tensor | None = None) -> OrbitalSet:
    """Step 4, rayleigh_ritz (paro.cpp:121-177)."""
    ctx = a_form.ctx
    U = _as_cols(candidates, ctx.n).contiguous()
    k = U.shape[0]
    V = out if out is not None else torch.empty_like(U)
    lam = (C.c_double * k)()
    kout = C.c_int(0)
    defect = C.c_double(0.0)
    st = N.lib().paro_rayleigh_ritz(ctx.h, a_form.h, b.h, k, _ptr(U), ctx.n, min_keep, drop_tol, lam, _ptr(V), ctx.n,
                                    C.byref(kout), C.byref(defect))
    ctx.check(st)
    kk = kout.value
    return OrbitalSet(V[:kk], list(lam)[:kk], defect.value)


def baseline_geneig(a: Operator, b: Operator, count: int, max_iter: int = 400, seed: int = 7):
    """baseline_geneig (linalg.cpp:615-623): the lowest `count` eigenpairs of
    (A, B) -> (lambdas, vectors [count, n], outer iterations). Device block
    subspace iteration (baseline_subspace, linalg.cpp:531-611) with no dof cap;
    raises IterationLimitError if it does not converge in max_iter."""
    ctx = a.ctx
    V = ctx.empty(count, ctx.n)
    lam = (C.c_double * count)()
    its = C.c_int(0)
    ctx.check(N.lib().paro_baseline_geneig(ctx.h, a.h, b.h, int(count), int(max_iter), int(seed), lam, _ptr(V), ctx.n,
                                           C.byref(its)))
    return list(lam), V, its.value


def initial_guess(a0: Operator, b: Operator, count: int, max_iter: int = 400, seed: int = 7) -> OrbitalSet:
    """initial_guess (paro.cpp:63-79): baseline eigenpairs of the core operator
    as the starting orbital set, with its B-Gram defect."""
    if count <= 0:
        raise N.InvalidArgumentError("initial_guess: count must be positive")
    if count > a0.ctx.n:
        raise N.InvalidArgumentError("initial_guess: more orbitals requested than coarse dofs")
    lam, V, _ = baseline_geneig(a0, b, count, max_iter, seed)
    G = torch.empty((count, a0.ctx.n), dtype=torch.float64, device=V.device)
    b.apply(V, out=G)
    gram = V @ G.T
    defect = float((gram - torch.eye(count, dtype=gram.dtype, device=gram.device)).abs().tril().max())
    return OrbitalSet(V, lam, defect)


def b_orthonormalize(vectors: torch.Tensor, b: Operator, drop_tol: float) -> torch.Tensor:
    """b_orthonormalize (linalg.cpp:409-439) -> accepted B-orthonormal vectors [k, n]."""
    ctx = b.ctx
    U = _as_cols(vectors, ctx.n).contiguous()
    Q = torch.empty_like(U)
    k = C.c_int(0)
    acc = (C.c_int * max(1, U.shape[0]))()
    ctx.check(N.lib().paro_b_orthonormalize(ctx.h, b.h, U.shape[0], _ptr(U), float(drop_tol), _ptr(Q), C.byref(k),
                                            acc))
    return Q[: k.value]


def dense_sym_geneig(ctx: Context, A, B):
    """dense_sym_geneig (linalg.cpp:341-393) on the device; host row-major in/out."""
    A = np.ascontiguousarray(A, np.float64)
    B = np.ascontiguousarray(B, np.float64)
    m = A.shape[0]
    vals = np.zeros(m)
    vecs = np.zeros((m, m))
    ctx.check(N.lib().paro_dense_sym_geneig(ctx.h, m, A.ctypes.data_as(_DP), B.ctypes.data_as(_DP),
                                            vals.ctypes.data_as(_DP), vecs.ctypes.data_as(_DP)))
    return vals, vecs


def fix_sign(ctx: Context, v: torch.Tensor) -> torch.Tensor:
    """fix_sign (linalg.cpp:229-241) in place on [k, n] device columns."""
    vc = _as_cols(v, ctx.n)
    ctx.check(N.lib().paro_fix_sign(ctx.h, vc.shape[0], _ptr(vc), vc.stride(0)))
    return v


# ---------------------------------------------------------------- assembly --

def _new_op(ctx: Context, fn, *args) -> Operator:
    h = C.c_void_p()
    ctx.check(fn(ctx.h, *args, C.byref(h)))
    return Operator(ctx, h)


def assemble_mass(ctx: Context) -> Operator:
    """assemble_mass (fem.cpp:253-268), on the device."""
    return _new_op(ctx, N.lib().paro_assemble_mass)


def assemble_stiffness(ctx: Context, scale: float) -> Operator:
    """assemble_stiffness(constant_diffusion(scale), 0) (fem.cpp:221-251)."""
    return _new_op(ctx, N.lib().paro_assemble_stiffness, float(scale))


def assemble_vext(ctx: Context, charges, positions, eps: float = 0.0) -> Operator:
    """Weighted mass of external_potential(molecule, eps) with the singular policy."""
    Z = np.ascontiguousarray(charges, np.float64)
    R = np.ascontiguousarray(positions, np.float64).reshape(-1)
    return _new_op(ctx, N.lib().paro_assemble_vext, len(Z), Z.ctypes.data_as(_DP), R.ctypes.data_as(_DP), float(eps))


def assemble_harmonic(ctx: Context, c: float) -> Operator:
    """Weighted mass of c*|x|^2 (4-point rule)."""
    return _new_op(ctx, N.lib().paro_assemble_harmonic, float(c))


def add_scaled(a: Operator, b: Operator, s: float = 1.0) -> Operator:
    """a += s*b (SparseOperator::add_scaled, linalg.cpp:120-125)."""
    a.ctx.check(N.lib().paro_op_add_scaled(a.ctx.h, a.h, b.h, float(s)))
    w = (C.c_double * 8)()
    var = C.c_int(0)
    a.ctx.check(N.lib().paro_op_weights(a.h, w, C.byref(var)))
    a.variable, a.weights = bool(var.value), np.array(list(w))
    return a


def ks_form_matrix(kinetic: Operator, vext: Operator, rho: torch.Tensor, vh: torch.Tensor,
                   exchange_only: bool = False, out: Operator | None = None):
    """ks_form_matrix (paro.cpp:446-454) -> (operator, clamped density points)."""
    ctx = kinetic.ctx
    op = out if out is not None else Operator.variable_empty(ctx)
    cl = C.c_longlong(0)
    ctx.check(N.lib().paro_ks_form(ctx.h, kinetic.h, vext.h, _ptr(rho), _ptr(vh), int(exchange_only), op.h,
                                   C.byref(cl)))
    return op, cl.value


def ks_form_planes(kinetic: Operator, vext: Operator, rho: torch.Tensor, vh: torch.Tensor, z0: int, z1: int,
                   out: Operator, exchange_only: bool = False) -> int:
    """ks_form_matrix for the dofs of lattice planes [z0, z1) only (a rank's row slab); returns the
    clamp count of the slab's cells (the ranks' counts add up to the full form's)."""
    ctx = kinetic.ctx
    cl = C.c_longlong(0)
    ctx.check(N.lib().paro_ks_form_planes(ctx.h, kinetic.h, vext.h, _ptr(rho), _ptr(vh), int(exchange_only),
                                          int(z0), int(z1), out.h, C.byref(cl)))
    return cl.value


# ------------------------------------------------------------------ fields --

def density_from_orbitals(ctx: Context, orbitals: torch.Tensor, occupations, out: torch.Tensor | None = None):
    """density_from_orbitals (model.cpp:192-223) -> (rho, raw_integral)."""
    U = _as_cols(orbitals, ctx.n)
    nocc = len(occupations)
    if nocc == 0 or U.shape[0] < nocc:
        raise N.InvalidArgumentError("density: orbital/occupation count mismatch")
    rho = out if out is not None else ctx.empty(ctx.n)
    occ = (C.c_double * nocc)(*[float(f) for f in occupations])
    raw = C.c_double(0.0)
    ld = U.stride(0) if U.shape[0] > 1 else ctx.n
    ctx.check(N.lib().paro_density(ctx.h, nocc, _ptr(U), ld, occ, _ptr(rho), C.byref(raw)))
    return rho, raw.value


def mix_density(ctx: Context, rho_in: torch.Tensor, rho_out: torch.Tensor, alpha: float,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """mix_density (model.cpp:225-236)."""
    o = out if out is not None else ctx.empty(ctx.n)
    ctx.check(N.lib().paro_mix_density(ctx.h, _ptr(rho_in), _ptr(rho_out), float(alpha), _ptr(o)))
    return o


def _scalar(ctx: Context, fn, *args) -> float:
    out = C.c_double(0.0)
    ctx.check(fn(ctx.h, *args, C.byref(out)))
    return out.value


def integrate(ctx: Context, f: torch.Tensor) -> float:
    return _scalar(ctx, N.lib().paro_integrate, _ptr(f))


def norm_l2(ctx: Context, f: torch.Tensor) -> float:
    return _scalar(ctx, N.lib().paro_norm_l2, _ptr(f))


def integrate_product(ctx: Context, u: torch.Tensor, v: torch.Tensor) -> float:
    return _scalar(ctx, N.lib().paro_integrate_product, _ptr(u), _ptr(v))


def rho_residual(ctx: Context, rho_out: torch.Tensor, rho_in: torch.Tensor, scratch: torch.Tensor) -> float:
    return _scalar(ctx, N.lib().paro_rho_residual, _ptr(rho_out), _ptr(rho_in), _ptr(scratch))


def total_energy(ctx: Context, lambdas, occupations, rho: torch.Tensor, vh: torch.Tensor, charges, positions,
                 exchange_only: bool = False) -> float:
    """total_energy (model.cpp:329-360)."""
    lam = (C.c_double * len(lambdas))(*[float(v) for v in lambdas])
    occ = (C.c_double * len(occupations))(*[float(v) for v in occupations])
    Z = np.ascontiguousarray(charges, np.float64)
    R = np.ascontiguousarray(positions, np.float64).reshape(-1)
    return _scalar(ctx, N.lib().paro_total_energy, len(lambdas), lam, len(occupations), occ, _ptr(rho), _ptr(vh),
                   int(exchange_only), len(Z), Z.ctypes.data_as(_DP), R.ctypes.data_as(_DP))


def energy_xc_layers(ctx: Context, rho: torch.Tensor, k0: int, k1: int, exchange_only: bool = False) -> float:
    """The XC term of total_energy, int rho (e_xc - v_xc), over the cell layers [k0, k1)."""
    return _scalar(ctx, N.lib().paro_energy_xc_layers, _ptr(rho), int(exchange_only), int(k0), int(k1))


def total_energy_with_xc(ctx: Context, lambdas, occupations, rho: torch.Tensor, vh: torch.Tensor, charges, positions,
                         xc_term: float) -> float:
    """total_energy (model.cpp:329-360) with the XC term summed elsewhere (energy_xc_layers over the ranks)."""
    lam = (C.c_double * len(lambdas))(*[float(v) for v in lambdas])
    occ = (C.c_double * len(occupations))(*[float(v) for v in occupations])
    Z = np.ascontiguousarray(charges, np.float64)
    R = np.ascontiguousarray(positions, np.float64).reshape(-1)
    return _scalar(ctx, N.lib().paro_total_energy_with_xc, len(lambdas), lam, len(occupations), occ, _ptr(rho),
                   _ptr(vh), len(Z), Z.ctypes.data_as(_DP), R.ctypes.data_as(_DP), float(xc_term))


def estimate_eta(ctx: Context, orbitals: torch.Tensor, lambdas, *, diffusion: float = 0.5, reaction: str = "ks",
                 c: float = 0.0, charges=(), positions=(), eps: float = 0.0, rho: torch.Tensor | None = None,
                 vh: torch.Tensor | None = None, exchange_only: bool = False, with_eta: bool = False):
    """Step 2 on a fixed mesh: combine_max over the orbitals (rows of
    `orbitals`) of estimate_eigen_residual (adapt.cpp:104-129) and its total,
    as the drivers run it every iteration (paro.cpp:521-538 Kohn-Sham with
    reaction "ks"; paro.cpp:306-315 linear with "harmonic" (c |x|^2) or "well"
    (external_potential)). Returns eta_total, or (eta_total, eta[6 s^3]) in
    the reference element order."""
    U = _as_cols(orbitals, ctx.n)
    k = U.shape[0]
    lam = (C.c_double * k)(*[float(v) for v in lambdas[:k]])
    kind = {"ks": 0, "harmonic": 1, "well": 2}[reaction]
    Z = np.ascontiguousarray(charges, np.float64)
    R = np.ascontiguousarray(positions, np.float64).reshape(-1)
    eta = torch.empty(6 * ctx.s ** 3, dtype=torch.float64, device=ctx.device) if with_eta else None
    tot = C.c_double(0.0)
    ctx.check(N.lib().paro_estimate_eta(ctx.h, k, _ptr(U), U.stride(0) if k > 1 else ctx.n, lam, diffusion, kind, c,
                                        len(Z), Z.ctypes.data_as(_DP) if len(Z) else None,
                                        R.ctypes.data_as(_DP) if len(Z) else None, eps,
                                        _ptr(rho) if rho is not None else None, _ptr(vh) if vh is not None else None,
                                        int(exchange_only), _ptr(eta) if eta is not None else None, C.byref(tot)))
    return (tot.value, eta) if with_eta else tot.value

class CsrOperator:
    """SparseOperator (linalg.hpp:14-50) for general sparse matrices (adapted
    meshes): CSR on the device, independent of the uniform
    grid. Same call surface as the stencil Operator for apply / add_scaled /
    cg_solve / source_solve_step."""

    def __init__(self, ctx: Context, rows, cols, vals):
        rows = np.ascontiguousarray(rows, np.uintp)
        cols = np.ascontiguousarray(cols, np.uint32)
        vals = np.ascontiguousarray(vals, np.float64)
        self.ctx = ctx
        self.n = len(rows) - 1
        self.h = None
        h = C.c_void_p()
        ctx.check(N.lib().paro_csr_create(ctx.h, self.n, rows.ctypes.data_as(C.POINTER(C.c_size_t)),
                                          cols.ctypes.data_as(C.POINTER(C.c_uint32)), vals.ctypes.data_as(_DP),
                                          C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None):
                N.lib().paro_csr_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def add_scaled(self, other: "CsrOperator", s: float = 1.0) -> "CsrOperator":
        """this += s * other on identical structures (linalg.cpp:120-125)."""
        self.ctx.check(N.lib().paro_csr_add_scaled(self.ctx.h, self.h, other.h, s))
        return self

    def apply(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """y = A x for k columns (matvec, linalg.cpp:88-94)."""
        squeeze = x.dim() == 1
        xc = _as_cols(x, self.n).contiguous()
        y = out if out is not None else torch.empty_like(xc)
        self.ctx.check(N.lib().paro_csr_apply(self.ctx.h, self.h, xc.shape[0], _ptr(xc), self.n, _ptr(y)))
        return y[0] if squeeze else y


def csr_cg_solve(a: CsrOperator, b: torch.Tensor, x0: torch.Tensor | None = None, tol: float = 1e-10,
                 max_iter: int = 10000, throw_on_max_iter: bool = True) -> CgResult:
    """cg_solve (linalg.cpp:143-223) on a general CSR operator, k right-hand sides."""
    ctx = a.ctx
    squeeze = b.dim() == 1
    bc = _as_cols(b, a.n).contiguous()
    k = bc.shape[0]
    x = torch.empty_like(bc)
    x0c = _as_cols(x0, a.n).contiguous() if x0 is not None else None
    it = (C.c_size_t * k)()
    res = (C.c_double * k)()
    st = N.lib().paro_csr_cg_solve(ctx.h, a.h, k, _ptr(bc), _ptr(x0c) if x0c is not None else None, a.n, tol,
                                   max_iter, int(throw_on_max_iter), _ptr(x), it, res)
    ctx.check(st)
    iters, resid = list(it), list(res)
    return CgResult(x[0] if squeeze else x, iters, resid, [r <= tol for r in resid])


def csr_source_solve_step(a: CsrOperator, b: CsrOperator, u_prev: torch.Tensor, lambdas, tol: float = 1e-10,
                          max_iter: int = 100000, sigma: float = 0.0, report: dict | None = None) -> torch.Tensor:
    """source_solve_step (paro.cpp:81-119) on general CSR operators."""
    ctx = a.ctx
    u = _as_cols(u_prev, a.n).contiguous()
    k = u.shape[0]
    if len(lambdas) != k:
        raise N.InvalidArgumentError("source_solve_step: orbital/lambda count mismatch")
    y = torch.empty_like(u)
    lam = (C.c_double * k)(*[float(v) for v in lambdas])
    it = (C.c_size_t * k)()
    res = (C.c_double * k)()
    st = N.lib().paro_csr_source_solve_step(ctx.h, a.h, b.h, k, _ptr(u), a.n, lam, tol, max_iter, sigma, _ptr(y),
                                            it, res)
    if report is not None:
        report.update(iterations=list(it), residual=list(res))
    ctx.check(st)
    return y


# ----------------------------------------------------------------------------
# Step 4 building blocks on row ranges (row-slab sharded rayleigh_ritz,
# paro_b200/step4.py). Vectors are [k, n] device tensors with column stride
# n; small matrices are flat device tensors in column-major order.

def _ld(X: torch.Tensor, n: int) -> int:
    return X.stride(0) if X.dim() == 2 and X.shape[0] > 1 else n


def apply_planes(op: Operator, X: torch.Tensor, k: int, Y: torch.Tensor, z0: int, z1: int):
    """Y = A X on the rows of planes [z0, z1); X valid on planes z0-1 .. z1."""
    ctx = op.ctx
    ctx.check(N.lib().paro_op_apply_planes(ctx.h, op.h, int(k), _ptr(X), _ld(X, ctx.n), _ptr(Y), int(z0), int(z1)))


def gram_sym(ctx: Context, X: torch.Tensor, Y: torch.Tensor, k: int, r0: int, r1: int, out=None) -> torch.Tensor:
    """X[:k]^T Y[:k] over rows [r0, r1) of a symmetric product (k x k, column-major)."""
    G = out if out is not None else torch.empty(k * k, dtype=torch.float64, device=ctx.device)
    ctx.check(N.lib().paro_gram_sym(ctx.h, int(k), _ptr(X), _ld(X, ctx.n), _ptr(Y), _ld(Y, ctx.n), int(r0), int(r1),
                                    _ptr(G)))
    return G


def gram_rect(ctx: Context, X: torch.Tensor, k1: int, Y: torch.Tensor, k2: int, r0: int, r1: int,
              out=None) -> torch.Tensor:
    """X[:k1]^T Y[:k2] over rows [r0, r1) (k1 x k2, column-major; k1 <= 80, k2 <= 16)."""
    G = out if out is not None else torch.empty(k1 * k2, dtype=torch.float64, device=ctx.device)
    ctx.check(N.lib().paro_gram_rect(ctx.h, int(k1), _ptr(X), _ld(X, ctx.n), int(k2), _ptr(Y), _ld(Y, ctx.n),
                                     int(r0), int(r1), _ptr(G)))
    return G


def rotate(ctx: Context, X: torch.Tensor, k1: int, Cm: torch.Tensor, ldc: int, k2: int, Z: torch.Tensor, r0: int,
           r1: int, mode: int = 0):
    """Z[:k2] = X[:k1] C over rows [r0, r1) (mode 1: Z -= X C, 4: Z += X C, 2: C triangular)."""
    ctx.check(N.lib().paro_rotate(ctx.h, int(k1), _ptr(X), _ld(X, ctx.n), _ptr(Cm), int(ldc), int(k2), _ptr(Z),
                                  _ld(Z, ctx.n), int(r0), int(r1), int(mode)))


def ritz_ortho(ctx: Context, G: torch.Tensor, K: int, drop_tol: float, C1: torch.Tensor):
    """Ordered Cholesky with the MGS drop rule of the raw Gram -> (k, min pivot ratio); C1 = K x k basis change."""
    k = C.c_int(0)
    rmin = C.c_double(0.0)
    ctx.check(N.lib().paro_ritz_ortho(ctx.h, int(K), _ptr(G), float(drop_tol), _ptr(C1), C.byref(k), C.byref(rmin)))
    return k.value, rmin.value


def ritz_second_pass(ctx: Context, G2: torch.Tensor, k: int, C2: torch.Tensor, Bt: torch.Tensor) -> bool:
    st = N.lib().paro_ritz_second_pass(ctx.h, int(k), _ptr(G2), _ptr(C2), _ptr(Bt))
    if st == 6:  # PencilError: the pass is not positive definite -> the caller falls back to CGS2
        return False
    ctx.check(st)
    return True


def ritz_congruence(ctx: Context, G: torch.Tensor, C1: torch.Tensor, k: int, Bt: torch.Tensor):
    """Bt = sym(C1^T sym(G) C1): the B-Gram of U C1 in k x k arithmetic (one-pass Step 4)."""
    ctx.check(N.lib().paro_ritz_congruence(ctx.h, int(k), _ptr(G), _ptr(C1), _ptr(Bt)))


def ritz_pencil(ctx: Context, GA: torch.Tensor, C2, Bt, GB, k: int, Y: torch.Tensor) -> list:
    """The k x k pencil (in the Q basis from GA, C2, Bt, or directly from GA, GB) -> eigenvalues; Y = lift."""
    vals = (C.c_double * k)()
    ctx.check(N.lib().paro_ritz_pencil(ctx.h, int(k), _ptr(GA), _ptr(C2) if C2 is not None else None,
                                       _ptr(Bt) if Bt is not None else None, _ptr(GB) if GB is not None else None,
                                       vals, _ptr(Y)))
    return list(vals)


def gram_defect_of(ctx: Context, G: torch.Tensor, k: int) -> float:
    out = C.c_double(0.0)
    ctx.check(N.lib().paro_gram_defect(ctx.h, int(k), _ptr(G), C.byref(out)))
    return out.value


def sign_buffers(ctx: Context, k: int):
    amax = torch.empty(k, dtype=torch.float64, device=ctx.device)
    first = torch.empty(k, dtype=torch.int64, device=ctx.device)
    flip = torch.empty(k, dtype=torch.float64, device=ctx.device)
    ctx.check(N.lib().paro_sign_init(ctx.h, int(k), _ptr(amax), _ptr(first)))
    return amax, first, flip


def colmax(ctx: Context, V, k, r0, r1, amax):
    ctx.check(N.lib().paro_colmax(ctx.h, int(k), _ptr(V), _ld(V, ctx.n), int(r0), int(r1), _ptr(amax)))


def first_above(ctx: Context, V, k, r0, r1, amax, first):
    ctx.check(N.lib().paro_first_above(ctx.h, int(k), _ptr(V), _ld(V, ctx.n), int(r0), int(r1), _ptr(amax),
                                       _ptr(first)))


def sign_flags(ctx: Context, V, k, r0, r1, amax, first, flip):
    ctx.check(N.lib().paro_sign_flags(ctx.h, int(k), _ptr(V), _ld(V, ctx.n), int(r0), int(r1), _ptr(amax),
                                      _ptr(first), _ptr(flip)))


def negate_columns(ctx: Context, V, k, r0, r1, flip):
    ctx.check(N.lib().paro_negate_columns(ctx.h, int(k), _ptr(V), _ld(V, ctx.n), int(r0), int(r1), _ptr(flip)))


def density_rows(ctx: Context, U: torch.Tensor, occupations, r0: int, r1: int, rho: torch.Tensor) -> float:
    """Nodal sum of density_from_orbitals on rows [r0, r1) of rho; returns sum occ."""
    nocc = len(occupations)
    if nocc == 0 or U.shape[0] < nocc:
        raise N.InvalidArgumentError("density: orbital/occupation count mismatch")
    occ = (C.c_double * nocc)(*[float(f) for f in occupations])
    ctx.check(N.lib().paro_density_rows(ctx.h, nocc, _ptr(U), _ld(U, ctx.n), occ, int(r0), int(r1), _ptr(rho)))
    return float(sum(occupations))


def density_normalize(ctx: Context, total_occ: float, rho: torch.Tensor) -> float:
    raw = C.c_double(0.0)
    ctx.check(N.lib().paro_density_normalize(ctx.h, float(total_occ), _ptr(rho), C.byref(raw)))
    return raw.value
