"""CPU restatement of the reference's ParO hot path — TEST INFRASTRUCTURE ONLY.

numpy / pure-Python restatement of the reference algorithms, each function
citing the reference file:line it follows (paths under /root/reference/proj).
Pinned by tests/test_oracle.py against (a) the known-answer vectors of the
reference's own tests and (b) the unmodified reference compiled into
oracle/_ref (oracle/ref.py). Only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs may use it; the product path never does.

Operators are scipy CSR matrices in the reference's dof order; the uniform-box
Kuhn geometry helpers build element lists for integrate / norm_l2 / energy.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp


class NotSpdError(RuntimeError):
    pass


class IterationLimitError(RuntimeError):
    def __init__(self, msg, residual):
        super().__init__(msg)
        self.residual = residual


class DegenerateSpanError(RuntimeError):
    pass


class PencilError(RuntimeError):
    pass


class EmptyBasisError(RuntimeError):
    pass


def csr(rows, cols, vals, n=None) -> sp.csr_matrix:
    n = len(rows) - 1 if n is None else n
    return sp.csr_matrix((np.asarray(vals, float), np.asarray(cols), np.asarray(rows)), shape=(n, n))


# --------------------------------------------------------------- linalg ----

def cg_solve(A: sp.csr_matrix, b, x0=None, tol=1e-10, max_iter=10000, precond=True, throw_on_max_iter=True):
    """cg_solve, linalg.cpp:143-223 (Jacobi preconditioner)."""
    b = np.asarray(b, float)
    if not np.all(np.isfinite(b)):
        raise ValueError("cg: right-hand side not finite")
    x = np.zeros_like(b) if x0 is None else np.array(x0, float)
    bnorm = math.sqrt(float(b @ b))
    if bnorm == 0.0:
        return np.zeros_like(b), 0, 0.0, True
    d = A.diagonal()
    if np.any(d <= 0.0):
        raise NotSpdError("cg: operator has a non-positive diagonal entry")
    inv = 1.0 / d if precond else np.ones_like(d)
    r = b - A @ x
    z = inv * r
    p = z.copy()
    rz = float(r @ z)
    rnorm = math.sqrt(float(r @ r))
    for it in range(max_iter):
        if rnorm / bnorm <= tol:
            return x, it, rnorm / bnorm, True
        q = A @ p
        pq = float(p @ q)
        if pq <= 0.0:
            raise NotSpdError("cg: operator not positive definite (p'Ap <= 0)")
        alpha = rz / pq
        x += alpha * p
        r -= alpha * q
        z = inv * r
        rz_next = float(r @ z)
        beta = rz_next / rz
        rz = rz_next
        p = z + beta * p
        rnorm = math.sqrt(float(r @ r))
    res = rnorm / bnorm
    conv = res <= tol
    if not conv and throw_on_max_iter:
        raise IterationLimitError("cg: iteration limit reached", res)
    return x, max_iter, res, conv


def source_solve_step(A, B, U, lambdas, tol=1e-10, max_iter=100000, sigma=0.0):
    """source_solve_step, paro.cpp:81-119 (serial worker order)."""
    S = A + sigma * B if sigma != 0.0 else A
    half = [None] * len(U)
    failures = [None] * len(U)
    for i, u in enumerate(U):
        rhs = (B @ u) * (lambdas[i] + sigma)
        try:
            half[i] = cg_solve(S, rhs, u, tol, max_iter)[0]
        except IterationLimitError:
            half[i] = cg_solve(S, rhs, u, tol * 100.0, max_iter * 4)[0]  # escapes if it fails
        except Exception as e:  # noqa: BLE001
            failures[i] = e
    for f in failures:
        if f is not None:
            raise f
    return np.array(half)


def shifted_source_step(A, B, U, lambdas, tol, max_iter=100000):
    """shifted_source_step, paro.cpp:194-210."""
    sigma = max(0.0, 0.5 - lambdas[0])
    for attempt in range(5):
        try:
            return source_solve_step(A, B, U, lambdas, tol, max_iter, sigma), sigma
        except NotSpdError:
            if attempt >= 4:
                raise
            sigma = 2.0 * sigma + 1.0


def fix_sign(v):
    """fix_sign, linalg.cpp:229-241."""
    v = np.array(v, float)
    amax = float(np.max(np.abs(v))) if v.size else 0.0
    if amax == 0.0:
        return v
    idx = np.nonzero(np.abs(v) > 1e-12 * amax)[0]
    if idx.size and v[idx[0]] < 0.0:
        v = -v
    return v


def cholesky(b):
    """cholesky, linalg.cpp:307-323."""
    n = b.shape[0]
    L = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1):
            s = b[i, j]
            for k in range(j):
                s -= L[i, k] * L[j, k]
            if i == j:
                if s <= 0.0:
                    raise PencilError("pencil: B is not positive definite")
                L[i, i] = math.sqrt(s)
            else:
                L[i, j] = s / L[j, j]
    return L


def jacobi_eig(a0, tol=1e-12, max_sweeps=60):
    """jacobi_eig, linalg.cpp:243-302 (cyclic sweeps, ascending order)."""
    a = np.array(a0, float)
    n = a.shape[0]
    v = np.eye(n)
    fro = math.sqrt(float(np.sum(a * a))) or 1.0
    for _ in range(max_sweeps):
        off = 2.0 * float(np.sum(np.triu(a, 1) ** 2))
        if math.sqrt(off) <= tol * fro:
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = a[p, q]
                if abs(apq) <= 1e-300:
                    continue
                tau = (a[q, q] - a[p, p]) / (2.0 * apq)
                t = (1.0 if tau >= 0.0 else -1.0) / (abs(tau) + math.sqrt(1.0 + tau * tau))
                c = 1.0 / math.sqrt(1.0 + t * t)
                s = t * c
                akp, akq = a[:, p].copy(), a[:, q].copy()
                a[:, p], a[:, q] = c * akp - s * akq, s * akp + c * akq
                apk, aqk = a[p, :].copy(), a[q, :].copy()
                a[p, :], a[q, :] = c * apk - s * aqk, s * apk + c * aqk
                vkp, vkq = v[:, p].copy(), v[:, q].copy()
                v[:, p], v[:, q] = c * vkp - s * vkq, s * vkp + c * vkq
    order = np.argsort(np.diag(a), kind="stable")
    return np.diag(a)[order].copy(), v[:, order].copy()


def dense_sym_geneig(A, B):
    """dense_sym_geneig, linalg.cpp:341-393."""
    A, B = np.asarray(A, float), np.asarray(B, float)
    for M in (A, B):
        scale = max(1.0, float(np.max(np.abs(M))) if M.size else 0.0)
        if np.any(np.abs(M - M.T) > 1e-12 * scale):
            raise PencilError("pencil: not symmetric")
    L = cholesky(B)
    W = np.linalg.solve(L, A)          # L^{-1} A
    C = np.linalg.solve(L, W.T).T      # W L^{-T}
    C = 0.5 * (C + C.T)
    vals, Y = jacobi_eig(C, 1e-12, 60)
    X = np.linalg.solve(L.T, Y)
    for j in range(X.shape[1]):
        X[:, j] = fix_sign(X[:, j])
    return vals, X


def b_orthonormalize(U, B, drop_tol):
    """b_orthonormalize, linalg.cpp:409-439 (MGS, two passes, relative drop)."""
    out, bq, dropped = [], [], []
    for idx, u in enumerate(U):
        h = np.array(u, float)
        orig = math.sqrt(max(0.0, float(h @ (B @ h))))
        if not orig > 0.0:
            dropped.append(idx)
            continue
        for _ in range(2):
            for q, bqk in zip(out, bq):
                h -= float(h @ bqk) * q
        nb = math.sqrt(max(0.0, float(h @ (B @ h))))
        if nb <= drop_tol * orig:
            dropped.append(idx)
            continue
        h /= nb
        out.append(h)
        bq.append(B @ h)
    if not out and len(U):
        raise EmptyBasisError("b_orthonormalize: all vectors dropped")
    return np.array(out), dropped


def gram_defect(V, B):
    """gram_defect, paro.cpp:50-61."""
    G = V @ (B @ V.T)
    return float(np.max(np.abs(np.tril(G - np.eye(len(V))))))


def rayleigh_ritz(cands, A, B, min_keep, drop_tol=1e-8):
    """rayleigh_ritz, paro.cpp:121-177."""
    Q, _ = b_orthonormalize(cands, B, drop_tol)
    k = len(Q)
    if k < min_keep:
        raise DegenerateSpanError(f"rayleigh_ritz: candidate span collapsed to {k} < {min_keep}")
    AQ = (A @ Q.T).T
    BQ = (B @ Q.T).T
    GA = Q @ AQ.T
    GB = Q @ BQ.T
    vals, X = dense_sym_geneig(0.5 * (GA + GA.T), 0.5 * (GB + GB.T))
    V = X.T @ Q
    V = np.array([fix_sign(v) for v in V])
    d = gram_defect(V, B)
    if d > 1e-8:
        raise RuntimeError(f"rayleigh_ritz: orthonormality certificate violated (defect {d})")
    return vals, V, d


# ------------------------------------------------- uniform Kuhn geometry ----

PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


def kuhn_elements(s: int):
    """Tet vertex lattice indices (mesh.cpp:455-474): [6 s^3, 4, 3] in element order."""
    c = np.arange(s)
    K, J, I = np.meshgrid(c, c, c, indexing="ij")
    base = np.stack([I.ravel(), J.ravel(), K.ravel()], axis=1)
    tets = []
    for p in PERMS:
        v = [base.copy()]
        cur = base.copy()
        for step in range(3):
            cur = cur.copy()
            cur[:, p[step]] += 1
            v.append(cur)
        tets.append(np.stack(v, axis=1))
    return np.stack(tets, axis=1).reshape(-1, 4, 3)


def vertex_values(f, s):
    """vertex_values (fem.cpp:359-366): zero-padded (s+1)^3 field, x fastest."""
    S = s - 1
    g = np.zeros((s + 1, s + 1, s + 1))
    g[1:s, 1:s, 1:s] = np.asarray(f, float).reshape(S, S, S)
    return g


def _elem_values(f, s, tets):
    g = vertex_values(f, s)
    return g[tets[:, :, 2], tets[:, :, 1], tets[:, :, 0]]


def element_volume(lo, hi, s):
    h = (hi - lo) / s
    return h ** 3 / 6.0


def integrate(f, s, lo, hi):
    """integrate, fem.cpp:419-430 (exact for P1)."""
    t = kuhn_elements(s)
    return float(np.sum(element_volume(lo, hi, s) * _elem_values(f, s, t).sum(1) / 4))


def norm_l2(f, s, lo, hi):
    """norm_l2, fem.cpp:432-448."""
    v = _elem_values(f, s, kuhn_elements(s))
    tot = np.sum(element_volume(lo, hi, s) * ((v * v).sum(1) + v.sum(1) ** 2) / 20.0)
    return math.sqrt(max(0.0, float(tot)))


def integrate_product(u, w, s, lo, hi):
    """integrate_product, model.cpp:306-327."""
    t = kuhn_elements(s)
    a, b = _elem_values(u, s, t), _elem_values(w, s, t)
    return float(np.sum(element_volume(lo, hi, s) * ((a * b).sum(1) + a.sum(1) * b.sum(1)) / 20.0))


# ------------------------------------------------------------------ model ----

def lda_vxc(rho, exchange_only=False):
    """lda_vxc, model.cpp:268-300 (Dirac exchange + PZ81), vectorised."""
    rho = np.asarray(rho, float)
    clamped = rho < 0.0
    r = np.where(clamped, 0.0, rho)
    v = np.zeros_like(r)
    e = np.zeros_like(r)
    nz = r > 0.0
    cx = np.cbrt(3.0 / math.pi)
    r13 = np.cbrt(r[nz])
    v[nz] = -cx * r13
    e[nz] = -0.75 * cx * r13
    if not exchange_only:
        with np.errstate(divide="ignore", over="ignore", invalid="ignore"):
            rs = np.cbrt(3.0 / (4.0 * math.pi * r[nz]))
            a, b, c, dd = 0.0311, -0.048, 0.0020, -0.0116
            g, b1, b2 = -0.1423, 1.0529, 0.3334
            ln = np.log(np.where(rs < 1.0, rs, 1.0))
            sq = np.sqrt(rs)
            den = 1.0 + b1 * sq + b2 * rs
            ec = np.where(rs < 1.0, a * ln + b + c * rs * ln + dd * rs, g / den)
            vc = np.where(rs < 1.0, a * ln + (b - a / 3.0) + (2.0 / 3.0) * c * rs * ln + ((2.0 * dd - c) / 3.0) * rs,
                          (g / den) * (1.0 + (7.0 / 6.0) * b1 * sq + (4.0 / 3.0) * b2 * rs) / den)
        e[nz] += ec
        v[nz] += vc
    return v, e, clamped


def density(U, occ, s, lo, hi):
    """density_from_orbitals, model.cpp:192-223 -> (rho, raw_integral)."""
    rho = np.zeros(U.shape[1])
    for f, u in zip(occ, U):
        rho += f * u * u
    raw = integrate(rho, s, lo, hi)
    tot = float(sum(occ))
    if tot > 0.0 and raw > 0.0:
        rho = rho * (tot / raw)
    return rho, raw


def mix(rin, rout, alpha):
    """mix_density, model.cpp:225-236."""
    return (1.0 - alpha) * np.asarray(rin) + alpha * np.asarray(rout)


def hartree(K, M, rho, tol=1e-11):
    """hartree_solve_with, model.cpp:242-255."""
    return cg_solve(K, (M @ rho) * (4.0 * math.pi), None, tol, 200000)[0]


def nuclear_repulsion(Z, R):
    """nuclear_repulsion, model.cpp:177-186."""
    e = 0.0
    for k in range(len(Z)):
        for m in range(k + 1, len(Z)):
            e += Z[k] * Z[m] / float(np.linalg.norm(np.asarray(R[k]) - np.asarray(R[m])))
    return e


QUAD4_A = (5.0 + 3.0 * math.sqrt(5.0)) / 20.0
QUAD4_B = (5.0 - math.sqrt(5.0)) / 20.0


def total_energy(lambdas, occ, rho, vh, Z, R, s, lo, hi, exchange_only=False):
    """total_energy, model.cpp:329-360 (4-point rule for E_xc)."""
    e_band = float(sum(f * lam for f, lam in zip(occ, lambdas)))
    e_h = 0.5 * integrate_product(vh, rho, s, lo, hi)
    t = kuhn_elements(s)
    v = _elem_values(rho, s, t)
    vol = element_volume(lo, hi, s)
    e_xc = 0.0
    for q in range(4):
        w = np.full(4, QUAD4_B)
        w[q] = QUAD4_A
        rq = np.maximum(0.0, v @ w)
        vx, ex, _ = lda_vxc(rq, exchange_only)
        e_xc += float(np.sum(0.25 * vol * (ex - vx) * rq))
    return e_band - e_h + e_xc + nuclear_repulsion(Z, R)


# -------------------------------------------------------------- Step 2 ----

def _tet_geometry(s, lo, hi):
    """Vertex coordinates (mesh.cpp:432-434), diameters (mesh.cpp:109-118),
    volumes and barycentric gradients (fem.cpp:65-88) of every Kuhn tet."""
    t = kuhn_elements(s)
    P = lo + (hi - lo) * t.astype(float) / s
    diam = np.zeros(len(t))
    for i in range(4):
        for j in range(i + 1, 4):
            diam = np.maximum(diam, np.linalg.norm(P[:, i] - P[:, j], axis=1))
    a, b, c = P[:, 1] - P[:, 0], P[:, 2] - P[:, 0], P[:, 3] - P[:, 0]
    det = np.einsum("ij,ij->i", a, np.cross(b, c))
    g = np.zeros((len(t), 4, 3))
    g[:, 1] = np.cross(b, c) / det[:, None]
    g[:, 2] = np.cross(c, a) / det[:, None]
    g[:, 3] = np.cross(a, b) / det[:, None]
    g[:, 0] = -(g[:, 1] + g[:, 2] + g[:, 3])
    return t, P, diam, np.abs(det) / 6.0, g


def _interior_faces(t, s):
    """Interior faces (two tets sharing three vertices): elem pair, normal,
    diameter and measure (adapt.cpp:27-56)."""
    vid = (t[:, :, 2] * (s + 1) + t[:, :, 1]) * (s + 1) + t[:, :, 0]
    owner = {}
    pairs = []
    for e in range(len(t)):
        for k in range(4):
            key = tuple(sorted(int(vid[e, m]) for m in range(4) if m != k))
            if key in owner:
                pairs.append((owner.pop(key), e, key))
            else:
                owner[key] = e
    return pairs


def estimate_eta(U, lambdas, s, lo, hi, reaction, diffusion=0.5):
    """combine_max over the columns of estimate_eigen_residual and its total
    (adapt.cpp:58-129): eta2_e = h_e^2 sum_q w_q |e| (lambda u - c u)^2(x_q)
    + sum_faces 1/2 diam |f| ((F_e - F_e').n)^2 with F = diffusion grad u.
    `reaction(x [E,4,3], bary [4,4]) -> [E,4]` evaluates c at the quadrature
    points. Returns (total, eta [6 s^3])."""
    t, P, diam, vol, g = _tet_geometry(s, lo, hi)
    bary = np.full((4, 4), QUAD4_B)
    np.fill_diagonal(bary, QUAD4_A)
    X = np.einsum("qi,eid->eqd", bary, P)
    react = reaction(X, bary, t)
    faces = _interior_faces(t, s)
    coords = lambda key: np.array([[k % (s + 1), (k // (s + 1)) % (s + 1), k // (s + 1) ** 2] for k in key],
                                  float) * (hi - lo) / s + lo
    fgeo = []
    for e0, e1, key in faces:
        A, B, Cc = coords(key)
        n = np.cross(B - A, Cc - A)
        area = 0.5 * np.linalg.norm(n)
        fd = max(np.linalg.norm(A - B), np.linalg.norm(B - Cc), np.linalg.norm(A - Cc))
        fgeo.append((e0, e1, n / np.linalg.norm(n), 0.5 * fd * area))
    e0 = np.array([f[0] for f in fgeo])
    e1 = np.array([f[1] for f in fgeo])
    nrm = np.array([f[2] for f in fgeo])
    fac = np.array([f[3] for f in fgeo])
    best = np.zeros(len(t))
    for col, lam in zip(np.atleast_2d(U), lambdas):
        v = _elem_values(col, s, t)
        uh = v @ bary.T
        r = lam * uh - react * uh
        eta2 = diam * diam * np.sum(0.25 * vol[:, None] * r * r, axis=1)
        flux = diffusion * np.einsum("ei,eid->ed", v, g)
        jump = np.einsum("fd,fd->f", flux[e0] - flux[e1], nrm)
        contrib = fac * jump * jump
        np.add.at(eta2, e0, contrib)
        np.add.at(eta2, e1, contrib)
        best = np.maximum(best, np.sqrt(np.maximum(0.0, eta2)))
    return math.sqrt(float(np.sum(best * best))), best


def ks_reaction(Z, R, rho, vh, s, eps=0.0, exchange_only=False):
    """V_ext(x) + V_H(x) + v_xc(rho(x)) at the quadrature points (paro.cpp:525-531)."""
    Z = np.asarray(Z, float)
    R = np.asarray(R, float).reshape(-1, 3)

    def f(X, bary, t):
        d2 = ((X[:, :, None, :] - R[None, None]) ** 2).sum(-1)
        vext = -(Z / np.sqrt(d2 + eps * eps)).sum(-1)
        rq = _elem_values(rho, s, t) @ bary.T
        vq = _elem_values(vh, s, t) @ bary.T
        return vext + vq + lda_vxc(rq, exchange_only)[0]
    return f

