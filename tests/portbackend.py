"""CPU backend for paro_b200.driver built on the oracle — TEST INFRASTRUCTURE.

Lets the rank-sharded orchestration (driver.ParoRun + Dist + step4.Step4)
run under gloo on CPU: operators come from the compiled reference
(oracle/_ref), the algebra from the numpy restatement (oracle/port.py), and
the Step-4 building blocks are numpy restatements of the device kernels
(ritz.cu / step4.cu / dense.cu: row-range Grams, rotations, the K x K
Cholesky-QR stages, the fix_sign pieces). Never used by the product path.
"""
import math

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

    # ---- Step 4 building blocks (step4.py), numpy restatements of the kernels
    @property
    def S(self):
        return self.w.subdivisions - 1

    def mass_op(self):
        return _Form(self.M)

    def apply_planes(self, op, X, k, Y, z0, z1):
        p = self.S * self.S
        r0, r1 = z0 * p, z1 * p
        A = op.A[r0:r1]
        Y[:k, r0:r1] = torch.as_tensor(np.asarray(A @ X[:k].numpy().T).T)

    @staticmethod
    def _flat(M):
        return torch.as_tensor(np.asarray(M, float).reshape(-1, order="F").copy())

    @staticmethod
    def _mat(t, rows, cols, ld=None):
        ld = rows if ld is None else ld
        return t.numpy()[: ld * cols].reshape(cols, ld).T[:rows, :cols]

    def gram_sym(self, X, Y, k, r0, r1):
        G = X[:k, r0:r1].numpy() @ Y[:k, r0:r1].numpy().T
        G = np.triu(G) + np.triu(G, 1).T  # the upper triangle, mirrored (ritz.cu)
        return self._flat(G)

    def gram_rect(self, X, k1, Y, k2, r0, r1):
        return self._flat(X[:k1, r0:r1].numpy() @ Y[:k2, r0:r1].numpy().T)

    def rotate(self, X, k1, Cm, ldc, k2, Z, r0, r1, mode):
        C = self._mat(Cm, k1, k2, ldc)
        R = C.T @ X[:k1, r0:r1].numpy()
        if mode & 1:
            Z[:k2, r0:r1] -= torch.as_tensor(R)
        elif mode & 4:
            Z[:k2, r0:r1] += torch.as_tensor(R)
        else:
            Z[:k2, r0:r1] = torch.as_tensor(R)

    def kk(self, m):
        return torch.zeros(max(m, 1), dtype=torch.float64)

    def ritz_ortho(self, G, K, drop_tol, C1):
        """ortho_from_gram_kernel (dense.cu): ordered Cholesky with the MGS drop rule."""
        a = self._mat(G, K, K)
        a = 0.5 * (a + a.T)
        L = np.zeros((K, K))
        acc, rmin = [], 1e300
        for j in range(K):
            g = a[j, j]
            orig = math.sqrt(max(0.0, g))
            if not orig > 0.0:
                rmin = 0.0
                continue
            k = len(acc)
            lrow = np.zeros(k)
            d2 = g
            for c in range(k):
                sv = a[j, acc[c]] - lrow[:c] @ L[c, :c]
                lrow[c] = sv / L[c, c]
                d2 -= lrow[c] * lrow[c]
            nb = math.sqrt(max(0.0, d2))
            rmin = min(rmin, nb / orig)
            if nb <= drop_tol * orig:
                continue
            L[k, :k] = lrow
            L[k, k] = nb
            acc.append(j)
        k = len(acc)
        Linv = np.linalg.inv(L[:k, :k]) if k else np.zeros((0, 0))
        C = np.zeros((K, k))
        for i in range(k):
            C[acc[i], :] = Linv[:, i]  # C[acc[i], j] = Linv[j][i]
        C1.zero_()
        C1[: K * k] = self._flat(C)
        return k, rmin

    def ritz_second_pass(self, G2, k, C2, Bt):
        a = self._mat(G2, k, k)
        a = 0.5 * (a + a.T)
        try:
            L = P.cholesky(a)
        except P.PencilError:
            return False
        Li = np.linalg.inv(L)
        b = Li @ a @ Li.T
        b = 0.5 * (b + b.T)
        C2[: k * k] = self._flat(Li.T)
        Bt[: k * k] = self._flat(b)
        return True

    def ritz_congruence(self, G, C1, k, Bt):
        g = self._mat(G, k, k)
        g = 0.5 * (g + g.T)
        c = self._mat(C1, k, k)
        b = c.T @ g @ c
        Bt[: k * k] = self._flat(0.5 * (b + b.T))

    def ritz_pencil(self, GA, C2, Bt, GB, k, Y):
        ga = self._mat(GA, k, k)
        ga = 0.5 * (ga + ga.T)
        if GB is None:
            c2 = self._mat(C2, k, k)
            At = c2.T @ ga @ c2
            At = 0.5 * (At + At.T)
            B = self._mat(Bt, k, k)
        else:
            At = ga
            B = self._mat(GB, k, k)
            B = 0.5 * (B + B.T)
        vals, X = P.dense_sym_geneig(At, B)
        Yk = (self._mat(C2, k, k) @ X) if GB is None else X
        Y[: k * k] = self._flat(Yk)
        return list(vals)

    def gram_defect(self, G, k):
        g = self._mat(G, k, k)
        return float(np.max(np.abs(np.tril(g - np.eye(k))))) if k else 0.0

    def sign_buffers(self, k):
        return (torch.zeros(k, dtype=torch.float64), torch.full((k,), 2 ** 63 - 1, dtype=torch.int64),
                torch.zeros(k, dtype=torch.float64))

    def colmax(self, V, k, r0, r1, amax):
        if r1 > r0:
            amax[:k] = torch.maximum(amax[:k], V[:k, r0:r1].abs().amax(dim=1))

    def first_above(self, V, k, r0, r1, amax, first):
        for c in range(k):
            if amax[c] > 0.0 and r1 > r0:
                idx = torch.nonzero(V[c, r0:r1].abs() > 1e-12 * amax[c])
                if len(idx):
                    first[c] = min(int(first[c]), r0 + int(idx[0, 0]))

    def sign_flags(self, V, k, r0, r1, amax, first, flip):
        for c in range(k):
            f = int(first[c])
            flip[c] = 1.0 if (amax[c] > 0.0 and r0 <= f < r1 and V[c, f] < 0.0) else 0.0

    def negate_columns(self, V, k, r0, r1, flip):
        for c in range(k):
            if flip[c] != 0.0:
                V[c, r0:r1] = -V[c, r0:r1]

    def copy_rows(self, src, dst, r0, r1):
        dst[:, r0:r1] = src[:, r0:r1]

    def div_rows(self, src, d, dst, r0, r1):
        dst[:, r0:r1] = src[:, r0:r1] / d

    def to_host(self, t):
        return t.tolist()

    def density_rows(self, U, occ, r0, r1, rho):
        r = np.zeros(r1 - r0)
        for f, u in zip(occ, U.numpy()):
            r += f * u[r0:r1] * u[r0:r1]
        rho[r0:r1] = torch.as_tensor(r)
        return float(sum(occ))

    def density_normalize(self, total, rho):
        w = self.w
        raw = P.integrate(rho.numpy(), w.subdivisions, w.lo, w.hi)
        if total > 0.0 and raw > 0.0:
            rho.mul_(total / raw)
        return raw

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
