"""CPU backend for paro_b200.driver built on the oracle — TEST INFRASTRUCTURE.

Lets the rank-sharded orchestration (driver.ParoRun + Dist) run under gloo on
CPU: operators come from the compiled reference (oracle/_ref), the algebra from
the numpy restatement (oracle/port.py). Never used by the product path.
"""
import numpy as np
import torch

from oracle import port as P
from oracle import ref as R

OK, NOT_SPD, ITER_LIMIT = 0, 3, 4


class _Form:
    def __init__(self, A):
        self.A = A


class PortBackend:
    device = torch.device("cpu")

    def __init__(self, w):
        self.w = w
        self.sp = R.Space(w.subdivisions, w.lo, w.hi)
        self.n = self.sp.n
        if w.kind == "ks":
            self.ks = R.KsSystem(self.sp, w.charges, w.positions, w.n_electrons, w.eps)
            self.M = P.csr(*self.ks.op("mass").csr())
            self.K = P.csr(*self.ks.op("poisson").csr())
            self.kin = P.csr(*self.ks.op("kinetic").csr())
            self.vext = P.csr(*self.ks.op("vext").csr())
        else:
            a = R.Op.stiffness(self.sp, 0.5)
            a.add_scaled(R.Op.wmass_harmonic(self.sp, 0.5) if w.potential == "harmonic"
                         else R.Op.wmass_coulomb(self.sp, w.charges, w.positions, w.eps))
            self.form = _Form(P.csr(*a.csr()))
            self.M = P.csr(*R.Op.mass(self.sp).csr())
        self.calls = 0

    def empty(self, *shape):
        return torch.zeros(*shape, dtype=torch.float64)

    def from_host(self, a):
        return torch.as_tensor(np.ascontiguousarray(a))

    def sync(self):
        pass

    def launches(self):
        return self.calls

    def core_hamiltonian(self):
        return _Form(self.kin + self.vext)

    def ks_form(self, rho, vh, slot):
        op, cl = self.ks.form(rho.numpy(), vh.numpy())
        return _Form(P.csr(*op.csr())), cl

    def hartree(self, rho, out=None):
        v = torch.as_tensor(P.hartree(self.K, self.M, rho.numpy()))
        if out is not None:
            out.copy_(v)
            return out
        return v

    def source_solve(self, a, u, lambdas, sigma, tol, max_iter, out):
        """Per-column Step 3 with the per-orbital retry (paro.cpp:95-113)."""
        S = a.A + sigma * self.M if sigma != 0.0 else a.A
        first, final, iters = [], [], []
        for c in range(u.shape[0]):
            x0 = u[c].numpy()
            rhs = (self.M @ x0) * (lambdas[c] + sigma)
            f = g = OK
            it = 0
            try:
                x, it, _, _ = P.cg_solve(S, rhs, x0, tol, max_iter)
            except P.IterationLimitError:
                f = ITER_LIMIT
                try:
                    x, it, _, _ = P.cg_solve(S, rhs, x0, tol * 100.0, max_iter * 4)
                except P.IterationLimitError:
                    g, x = ITER_LIMIT, x0
                except P.NotSpdError:
                    g, x = NOT_SPD, x0
            except P.NotSpdError:
                f = g = NOT_SPD
                x = x0
            if f != ITER_LIMIT:
                g = f
            out[c].copy_(torch.as_tensor(x))
            first.append(f)
            final.append(g)
            iters.append(it)
        self.calls += 1
        return first, final, iters, [0.0] * len(first)

    def ritz(self, cands, a, min_keep, drop_tol, out):
        vals, V, d = P.rayleigh_ritz(cands.numpy(), a.A, self.M, min_keep, drop_tol)
        out[: len(V)].copy_(torch.as_tensor(V))
        return out[: len(V)], list(vals), d

    def density(self, U, occ, out=None):
        rho, _ = P.density(U.numpy(), occ, self.w.subdivisions, self.w.lo, self.w.hi)
        t = torch.as_tensor(rho)
        if out is not None:
            out.copy_(t)
            return out
        return t

    def energy(self, lambdas, occ, rho, vh):
        return P.total_energy(lambdas, occ, rho.numpy(), vh.numpy(), self.w.charges, self.w.positions,
                              self.w.subdivisions, self.w.lo, self.w.hi)

    def mix(self, rin, rout, alpha, out):
        out.copy_(torch.as_tensor(P.mix(rin.numpy(), rout.numpy(), alpha)))
        return out

    def rho_residual(self, rout, rin):
        return P.norm_l2((rout - rin).numpy(), self.w.subdivisions, self.w.lo, self.w.hi)
