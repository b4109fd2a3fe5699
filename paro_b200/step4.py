"""Step 4 of the ParO outer iteration, rayleigh_ritz (proj/src/paro.cpp:121-177),
orchestrated over row slabs so that it shards across ranks.

Each rank owns the rows of a contiguous block of lattice planes (RowSlab) for
ALL K candidate columns, plus one halo plane on each side (the reach of the
15-point stencil). Everything the reference does per dof is local to the slab:
the B / A applies (rows of the owned planes, reading the halo planes), the
basis changes and the lift (row-local rotations, applied to the halo planes
too so they stay consistent without an exchange), the sign flips. What is
global is small and goes through the `dist` reductions: the K x K Gram
partials (summed in rank order, so every rank then runs the identical K x K
stage), the fix_sign pieces (max / min / max of K numbers) and the CGS2
projections. At world size 1 the slab is the whole lattice and the sequence of
kernels is the one of the C ABI's monolithic paro_rayleigh_ritz (ritz.cu), so
both give bit-identical orbitals.

Numerics: Cholesky-QR twice with the MGS drop rule of
b_orthonormalize (linalg.cpp:409-439) on the Gram, the pencil solved in the
orthonormal basis, lift, fix_sign, certificate max |V^T B V - I| <= 1e-8
(paro.cpp:171-174); candidates whose pivot ratio falls below 1e-5, or a failed
second pass / certificate, go through a blocked two-pass Gram-Schmidt
(`cgs2`) with the reference's drop rule instead.

The backend supplies the primitives (GpuBackend: the native sm_100a library;
tests' PortBackend: numpy) and `dist` the reductions (driver.Dist), so this
orchestration is the same code on one GPU, on N GPUs over NCCL and in the
gloo world-size-2/4 CPU tests.
"""
from __future__ import annotations

from dataclasses import dataclass

CERT_TOL = 1e-8          # paro.cpp:171
CGS_RATIO = 1e-5         # pivot/original ratio below which Cholesky-QR hands over to CGS2
CGS_BLOCK = 8            # candidates per CGS2 block
ONE_PASS_RATIO = 0.5     # pivot ratio from which the basis change stays in K x K arithmetic (ritz.cu kOnePassRatio)


class Step4Error(RuntimeError):
    pass


@dataclass
class RowSlab:
    """Planes [z0, z1) of the S^3 interior lattice owned by one rank, rows
    [r0, r1) = [z0 S^2, z1 S^2); the extended range [e0, e1) adds the halo
    planes z0 - 1 and z1 (clipped to the lattice)."""

    S: int
    z0: int
    z1: int

    @property
    def plane(self) -> int:
        return self.S * self.S

    @property
    def r0(self) -> int:
        return self.z0 * self.plane

    @property
    def r1(self) -> int:
        return self.z1 * self.plane

    @property
    def e0(self) -> int:
        return max(0, self.z0 - 1) * self.plane

    @property
    def e1(self) -> int:
        return min(self.S, self.z1 + 1) * self.plane

    @staticmethod
    def split(S: int, world: int, rank: int) -> "RowSlab":
        base, rem = divmod(S, world)
        counts = [base + (1 if r < rem else 0) for r in range(world)]
        z0 = sum(counts[:rank])
        return RowSlab(S, z0, z0 + counts[rank])

    @staticmethod
    def all(S: int, world: int) -> list:
        return [RowSlab.split(S, world, r) for r in range(world)]


@dataclass
class RitzInfo:
    k: int = 0
    min_ratio: float = 0.0
    cgs2: bool = False
    one_pass: bool = False


class Step4:
    """rayleigh_ritz over this rank's row slab. `be` provides the primitives
    (see GpuBackend in driver.py), `dist` the cross-rank reductions."""

    def __init__(self, be, dist, slab: RowSlab):
        self.be = be
        self.d = dist
        self.slab = slab
        self._ws = {}
        self.force_cgs2 = False
        self.two_pass_only = False
        self.info = RitzInfo()

    # work buffers [k, n] reused across calls
    def _buf(self, name, k):
        t = self._ws.get(name)
        if t is None or t.shape[0] < k:
            t = self.be.empty(max(k, 1), self.be.n)
            self._ws[name] = t
        return t

    def _gram(self, X, Y, k):
        s = self.slab
        G = self.be.gram_sym(X, Y, k, s.r0, s.r1)
        self.d.allsum_(G)
        return G

    def _apply(self, op, X, k, Y):
        self.be.apply_planes(op, X, k, Y, self.slab.z0, self.slab.z1)

    def fix_sign(self, V, k):
        """fix_sign (linalg.cpp:229-241) of k columns across the slabs."""
        be, d, s = self.be, self.d, self.slab
        amax, first, flip = be.sign_buffers(k)
        be.colmax(V, k, s.r0, s.r1, amax)
        d.allmax_(amax)
        be.first_above(V, k, s.r0, s.r1, amax, first)
        d.allmin_(first)
        be.sign_flags(V, k, s.r0, s.r1, amax, first, flip)
        d.allmax_(flip)
        be.negate_columns(V, k, s.e0, s.e1, flip)

    def _check_count(self, k, min_keep):
        from . import _native as N

        if k == 0:
            raise N.EmptyBasisError("b_orthonormalize: all vectors dropped")
        if k < min_keep:
            raise N.DegenerateSpanError(f"rayleigh_ritz: candidate span collapsed to {k} < {min_keep}")

    def ritz(self, U, A, B, min_keep: int, drop_tol: float, V, on_final=None):
        """Candidates U [K, n] (valid on the extended slab rows) -> V[:k] (the
        Ritz orbitals, valid on the extended rows), eigenvalues (host list) and
        the B-orthonormality defect. on_final(V, k) runs once the orbitals are
        final (before the certificate), e.g. to start their host copy-out; it
        may return a callable that orders later writes of V after that use
        (called if a CGS2 retry produces the orbitals again)."""
        from . import _native as N

        be, s = self.be, self.slab
        K = U.shape[0]
        if K <= 0:
            raise N.EmptyBasisError("b_orthonormalize: all vectors dropped")
        W = self._buf("W", K)
        Q1 = self._buf("Q1", K)
        self._pending = None  # a started host copy-out of V that must finish before V is rewritten
        info = RitzInfo()
        lam, d = None, 0.0
        use_cgs = self.force_cgs2
        if not use_cgs:
            # Cholesky-QR pass 1: Gram of the candidates, ordered Cholesky with drops
            self._apply(B, U, K, W)
            G = self._gram(U, W, K)
            C1 = be.kk(K * K)
            k, rmin = be.ritz_ortho(G, K, drop_tol, C1)
            info.min_ratio = rmin
            # Cholesky pivots lose ~eps/ratio^2 relative accuracy: near-dependent
            # candidates (and every drop decision) go through CGS2 instead
            use_cgs = rmin < CGS_RATIO
        one_pass = False
        if not use_cgs and k == K and rmin >= ONE_PASS_RATIO and not self.two_pass_only \
                and U.data_ptr() != V.data_ptr():
            # well-conditioned candidates (the steady state: Step-3 solutions are nearly
            # B-orthonormal): the basis change stays in K x K arithmetic. Both Grams are those of
            # the actual candidates, At = C1^T (U^T A U) C1, Bt = C1^T (U^T B U) C1, and the lift is
            # V = U (C1 X): one rotation, one apply and one Gram less than forming Q1. The
            # certificate still measures the actual V; a failure falls back to the two-pass path.
            self._check_count(k, min_keep)
            Bt = be.kk(k * k)
            be.ritz_congruence(G, C1, k, Bt)
            self._apply(A, U, k, W)
            GA = self._gram(U, W, k)
            Y = be.kk(k * k)
            try:
                lam = be.ritz_pencil(GA, C1, Bt, None, k, Y)
            except N.PencilError:
                lam = None
            if lam is not None:
                d = self._finish(U, Y, k, V, W, B, on_final)
                one_pass = d <= CERT_TOL
        info.one_pass = one_pass
        if not use_cgs and not one_pass:
            self._check_count(k, min_keep)
            be.rotate(U, K, C1, K, k, Q1, s.e0, s.e1, 2)
            self._apply(B, Q1, k, W)
            G2 = self._gram(Q1, W, k)
            C2, Bt = be.kk(k * k), be.kk(k * k)
            if not be.ritz_second_pass(G2, k, C2, Bt):
                use_cgs = True
            else:
                self._apply(A, Q1, k, W)
                GA = self._gram(Q1, W, k)
                Y = be.kk(k * k)
                lam = be.ritz_pencil(GA, C2, Bt, None, k, Y)
                d = self._finish(Q1, Y, k, V, W, B, on_final)
                use_cgs = d > CERT_TOL  # retry with explicit Gram-Schmidt before failing the certificate
        if use_cgs:
            info.cgs2 = True
            BQ = W
            k, _ = self.cgs2(U, K, B, drop_tol, Q1, BQ)
            self._check_count(k, min_keep)
            AQ = self._buf("AQ", k)
            self._apply(A, Q1, k, AQ)
            GA = self._gram(Q1, AQ, k)
            G2 = self._gram(Q1, BQ, k)
            Y = be.kk(k * k)
            lam = be.ritz_pencil(GA, None, None, G2, k, Y)
            d = self._finish(Q1, Y, k, V, W, B, on_final)
        info.k = k
        self.info = info
        if d > CERT_TOL:
            raise N.Error(f"rayleigh_ritz: orthonormality certificate violated (defect {d})")
        return V[:k], list(lam)[:k], d

    def _finish(self, Qb, Y, k, V, W, B, on_final):
        """lift, sign convention, certificate (paro.cpp:157-174)"""
        be, s = self.be, self.slab
        if self._pending is not None:  # the CGS2 retry rewrites V: the earlier copy-out must have read it
            self._pending()
            self._pending = None
        be.rotate(Qb, k, Y, k, k, V, s.e0, s.e1, 0)
        self.fix_sign(V, k)
        if on_final is not None:
            self._pending = on_final(V, k)
        self._apply(B, V, k, W)
        G3 = self._gram(V, W, k)
        return be.gram_defect(G3, k)

    def cgs2(self, U, K, B, drop_tol, Q, BQ):
        """b_orthonormalize (linalg.cpp:409-439) as blocked two-pass Gram-Schmidt
        in the B inner product: each block of CGS_BLOCK candidates is projected
        twice against the basis accepted before it (block Grams + rotations),
        then its candidates are finished one by one (twice against the
        block's own accepted vectors, B-norm of the projected vector against
        the original one for the drop rule, normalisation). Returns
        (k, accepted candidate indices); Q[:k], BQ[:k] = B Q valid on the slab
        (Q on the extended rows)."""
        be, d, s = self.be, self.d, self.slab
        H = self._buf("H", CGS_BLOCK)
        BH = self._buf("BH", CGS_BLOCK)
        k, acc = 0, []
        for j0 in range(0, K, CGS_BLOCK):
            nb_ = min(CGS_BLOCK, K - j0)
            be.copy_rows(U[j0:j0 + nb_], H[:nb_], s.e0, s.e1)
            self._apply(B, H, nb_, BH)
            Gh = be.gram_rect(H, nb_, BH, nb_, s.r0, s.r1)
            d.allsum_(Gh)
            diag = be.to_host(Gh)
            orig = [max(0.0, diag[i + i * nb_]) ** 0.5 for i in range(nb_)]
            for _ in range(2):
                self._project(Q, BQ, 0, k, H, nb_)
            kb = k
            for jj in range(nb_):
                if not orig[jj] > 0.0:
                    continue
                h, bh = H[jj:jj + 1], BH[jj:jj + 1]
                for _ in range(2):
                    self._project(Q, BQ, kb, k, h, 1)
                self._apply(B, h, 1, bh)
                g = be.gram_rect(h, 1, bh, 1, s.r0, s.r1)
                d.allsum_(g)
                nb = max(0.0, be.to_host(g)[0]) ** 0.5
                if nb <= drop_tol * orig[jj]:
                    continue
                be.div_rows(h, nb, Q[k:k + 1], s.e0, s.e1)
                self._apply(B, Q[k:k + 1], 1, BQ[k:k + 1])
                acc.append(j0 + jj)
                k += 1
        return k, acc

    def _project(self, Q, BQ, q0, q1, H, m):
        """H -= Q[q0:q1] (BQ[q0:q1]^T H) over the slab (80-column slices)."""
        be, d, s = self.be, self.d, self.slab
        for a in range(q0, q1, 80):
            b = min(q1, a + 80)
            C = be.gram_rect(BQ[a:b], b - a, H, m, s.r0, s.r1)
            d.allsum_(C)
            be.rotate(Q[a:b], b - a, C, b - a, m, H, s.e0, s.e1, 1)
