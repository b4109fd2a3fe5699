"""GPU checks of the Step-4 building blocks on row ranges (step4.cu, ritz.cu)
and of the row-slab orchestration (paro_b200/step4.py):

* the DMMA rotation / rectangular Gram against a float64 torch reference;
* every piece computed on a split of the rows equals the whole-range result
  (bitwise for the row-local kernels, to rounding for the Gram partial sums),
  which is what the sharded Step 4 relies on;
* the orchestrated Step 4 at world size 1 is bit-identical to the C ABI's
  monolithic paro_rayleigh_ritz (same kernels, same order), and its CGS2 path
  agrees with the monolithic CGS2 to rounding.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ctx(s=24, lo=-6.0, hi=6.0):
    from paro_b200 import core

    return core.Context(0).grid(s, lo, hi)


def _rand(shape, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.rand(shape, generator=g, dtype=torch.float64).mul_(2).sub_(1).cuda()


@pytest.mark.parametrize("k1,k2", [(76, 76), (5, 3), (80, 17), (33, 1), (100, 90), (81, 7)])
def test_rotate_matches_torch(k1, k2):
    from paro_b200 import core

    ctx = _ctx()
    n = ctx.n
    X = _rand((k1, n), 1)
    Cm = _rand((k2, k1), 2)  # column-major k1 x k2 == row-major [k2][k1]
    Z = torch.empty((k2, n), dtype=torch.float64, device="cuda")
    core.rotate(ctx, X, k1, Cm.reshape(-1), k1, k2, Z, 0, n, 0)
    ref = Cm @ X  # Z_j = sum_i C[i][j] X_i
    torch.testing.assert_close(Z, ref, rtol=1e-12, atol=1e-12)
    Z2 = Z.clone()
    core.rotate(ctx, X, k1, Cm.reshape(-1), k1, k2, Z2, 0, n, 1)  # Z -= X C
    assert Z2.abs().max().item() <= 1e-12
    core.rotate(ctx, X, k1, Cm.reshape(-1), k1, k2, Z2, 0, n, 4)  # Z += X C
    torch.testing.assert_close(Z2, ref, rtol=1e-12, atol=1e-12)


def test_rotate_triangular_and_row_split_bitwise():
    from paro_b200 import core

    ctx = _ctx()
    n, K = ctx.n, 40
    X = _rand((K, n), 3)
    Cm = torch.triu(_rand((K, K), 4)).T.contiguous()  # column-major upper triangular
    full = torch.empty((K, n), dtype=torch.float64, device="cuda")
    core.rotate(ctx, X, K, Cm.reshape(-1), K, K, full, 0, n, 0)
    tri = torch.empty_like(full)
    core.rotate(ctx, X, K, Cm.reshape(-1), K, K, tri, 0, n, 2)
    torch.testing.assert_close(tri, full, rtol=1e-13, atol=1e-13)
    part = torch.zeros_like(full)
    cut = 23 * 23 * 7 + 5  # not a multiple of the 32-row chunk
    core.rotate(ctx, X, K, Cm.reshape(-1), K, K, part, 0, cut, 0)
    core.rotate(ctx, X, K, Cm.reshape(-1), K, K, part, cut, n, 0)
    assert torch.equal(part, full)


@pytest.mark.parametrize("k1,k2", [(76, 8), (7, 1), (80, 16)])
def test_gram_rect_matches_torch(k1, k2):
    from paro_b200 import core

    ctx = _ctx()
    n = ctx.n
    X, Y = _rand((k1, n), 5), _rand((k2, n), 6)
    G = core.gram_rect(ctx, X, k1, Y, k2, 0, n)
    ref = (X @ Y.T).T.reshape(-1)  # column-major k1 x k2
    torch.testing.assert_close(G, ref, rtol=1e-12, atol=1e-10)
    r = 1000
    G2 = core.gram_rect(ctx, X, k1, Y, k2, 0, r) + core.gram_rect(ctx, X, k1, Y, k2, r, n)
    torch.testing.assert_close(G2, ref, rtol=1e-12, atol=1e-10)


def test_gram_sym_and_apply_on_slabs():
    from paro_b200 import core
    from paro_b200.step4 import RowSlab

    ctx = _ctx()
    S, n, K = ctx.S, ctx.n, 12
    M = core.assemble_mass(ctx)
    U = _rand((K, n), 7)
    W = M.apply(U)
    Gf = core.gram_sym(ctx, U, W, K, 0, n)
    for world in (2, 3):
        Wp = torch.full_like(W, float("nan"))
        Gp = torch.zeros_like(Gf)
        for sl in RowSlab.all(S, world):
            core.apply_planes(M, U, K, Wp, sl.z0, sl.z1)
            assert torch.equal(Wp[:, sl.r0:sl.r1], W[:, sl.r0:sl.r1])
            Gp += core.gram_sym(ctx, U, Wp, K, sl.r0, sl.r1)
        assert torch.equal(Wp, W)
        torch.testing.assert_close(Gp, Gf, rtol=1e-12, atol=1e-12)


def test_fix_sign_pieces_split_equals_whole():
    from paro_b200 import core
    from paro_b200.step4 import RowSlab

    ctx = _ctx()
    S, n, k = ctx.S, ctx.n, 9
    V = _rand((k, n), 8)
    V[2, : 3 * S * S] = 0.0  # pivot in a later slab
    V[4] = 0.0               # zero column: no flip
    whole = V.clone()
    amax, first, flip = core.sign_buffers(ctx, k)
    core.colmax(ctx, whole, k, 0, n, amax)
    core.first_above(ctx, whole, k, 0, n, amax, first)
    core.sign_flags(ctx, whole, k, 0, n, amax, first, flip)
    core.negate_columns(ctx, whole, k, 0, n, flip)
    ref = V.cpu().numpy().copy()
    for c in range(k):  # fix_sign, linalg.cpp:229-241
        v = ref[c]
        m = np.abs(v).max()
        if m > 0:
            i = np.nonzero(np.abs(v) > 1e-12 * m)[0][0]
            if v[i] < 0:
                ref[c] = -v
    assert np.array_equal(whole.cpu().numpy(), ref)
    slabs = RowSlab.all(S, 3)
    bufs = [core.sign_buffers(ctx, k) for _ in slabs]
    for sl, (a, _, _) in zip(slabs, bufs):
        core.colmax(ctx, V, k, sl.r0, sl.r1, a)
    amax = torch.stack([b[0] for b in bufs]).amax(0)
    for sl, (_, f, _) in zip(slabs, bufs):
        core.first_above(ctx, V, k, sl.r0, sl.r1, amax, f)
    first = torch.stack([b[1] for b in bufs]).amin(0)
    for sl, (_, _, fl) in zip(slabs, bufs):
        core.sign_flags(ctx, V, k, sl.r0, sl.r1, amax, first, fl)
    flip = torch.stack([b[2] for b in bufs]).amax(0)
    split = V.clone()
    for sl in slabs:
        core.negate_columns(ctx, split, k, sl.r0, sl.r1, flip)
    assert torch.equal(split, whole)


@pytest.mark.parametrize("force_cgs2", [False, True])
def test_orchestrated_ritz_equals_monolithic(force_cgs2):
    """Step4.ritz at world size 1 vs paro_rayleigh_ritz on the same KS pencil."""
    from paro_b200 import configs, core
    from paro_b200.driver import Dist, GpuBackend
    from paro_b200.step4 import RowSlab, Step4

    w = configs.get("water@s24")
    be = GpuBackend(w)
    g = be.from_host(configs.guess_vectors(w))
    a0 = be.core_hamiltonian()
    K = g.shape[0]
    s4 = Step4(be, Dist(), RowSlab.split(be.S, 1, 0))
    s4.force_cgs2 = force_cgs2
    V1 = be.empty(K, be.n)
    orb1, lam1, d1 = s4.ritz(g, a0, be.mass, K, w.drop_tol, V1)
    be.ctx.set_ritz_mode("cgs2" if force_cgs2 else "cholqr")
    r = core.rayleigh_ritz(g, a0, be.mass, K, w.drop_tol)
    be.ctx.set_ritz_mode("cholqr")
    assert s4.info.cgs2 == force_cgs2
    assert len(lam1) == len(r.lambdas)
    if not force_cgs2:
        assert lam1 == r.lambdas and d1 == r.gram_defect
        assert torch.equal(orb1, r.orbitals)
    else:  # blocked vs one-by-one Gram-Schmidt: same span, rounding-level differences
        np.testing.assert_allclose(lam1, r.lambdas, rtol=1e-11)
        torch.testing.assert_close(orb1, r.orbitals, rtol=0, atol=1e-8 * r.orbitals.abs().max().item())
        assert d1 <= 1e-8


def test_one_pass_ritz_matches_two_pass():
    """Well-conditioned candidates (Step-3 solutions of a running KS iteration,
    pivot ratios ~1) take the one-pass basis change (K x K congruence, lift
    from the candidates themselves): same Ritz values to 1e-12 relative and the
    same orbitals to rounding as the two-pass Cholesky-QR, bit-identical
    between the orchestrated and the monolithic Step 4, certificate <= 1e-8."""
    from paro_b200 import configs, core
    from paro_b200.driver import GpuBackend, ParoRun

    w = configs.get("water@s24")
    be = GpuBackend(w)
    run = ParoRun(w, be, timers=False)
    for i in range(2):
        run.step(i)
    assert run.s4.info.one_pass and not run.s4.info.cgs2
    K = run.k
    half = run.half[:K].clone()
    a_half = be.forms["half"]
    s4 = run.s4
    V1, V2 = be.empty(K, be.n), be.empty(K, be.n)
    o1, l1, d1 = s4.ritz(half, a_half, be.mass, K, w.drop_tol, V1)
    assert s4.info.one_pass and s4.info.min_ratio >= 0.5
    s4.two_pass_only = True
    o2, l2, d2 = s4.ritz(half, a_half, be.mass, K, w.drop_tol, V2)
    s4.two_pass_only = False
    assert not s4.info.one_pass
    assert d1 <= 1e-8 and d2 <= 1e-8
    np.testing.assert_allclose(l1, l2, rtol=1e-12, atol=1e-13)
    torch.testing.assert_close(o1, o2, rtol=0, atol=1e-9 * o2.abs().max().item())
    # the monolithic C-ABI Step 4 takes the same path with the same kernels
    r = core.rayleigh_ritz(half, a_half, be.mass, K, w.drop_tol)
    assert l1 == r.lambdas and d1 == r.gram_defect and torch.equal(o1, r.orbitals)
    be.ctx.set_ritz_mode("cholqr2")
    r2 = core.rayleigh_ritz(half, a_half, be.mass, K, w.drop_tol)
    be.ctx.set_ritz_mode("cholqr")
    assert l2 == r2.lambdas and torch.equal(o2, r2.orbitals)


@pytest.mark.parametrize("K,dependent", [(9, ()), (76, ()), (140, ()), (12, (5,)), (40, (0, 17, 39))])
def test_ritz_ortho_parallel_and_drop_paths(K, dependent):
    """ortho_from_gram_kernel: the column-parallel Cholesky (no drops) and the
    ordered row loop (taken from the first dropped candidate on) against the
    numpy restatement of the same ordered Cholesky (tests/portbackend.py):
    same accepted set, pivot ratio and basis change."""
    from portbackend import PortBackend

    from paro_b200 import core

    ctx = core.Context(0).grid(8, -1.0, 1.0)
    rng = np.random.default_rng(K)
    n = 400
    U = rng.standard_normal((n, K))
    for j in dependent:  # candidate j in the span of the others (dropped), or zero (j == 0)
        U[:, j] = 0.0 if j == 0 else U[:, :j] @ rng.standard_normal(j)
    G = U.T @ U
    Gd = torch.as_tensor(G.T.reshape(-1).copy(), device="cuda")  # column-major
    C1 = torch.zeros(K * K, dtype=torch.float64, device="cuda")
    k, rmin = core.ritz_ortho(ctx, Gd, K, 1e-6, C1)
    pb = PortBackend.__new__(PortBackend)
    C1p = torch.zeros(K * K, dtype=torch.float64)
    kp, rminp = PortBackend.ritz_ortho(pb, torch.as_tensor(G.T.reshape(-1).copy()), K, 1e-6, C1p)
    assert k == kp == K - len(dependent)
    if dependent:
        assert rmin <= 1e-6 and rminp <= 1e-6     # a dropped candidate: ratio at rounding level (~1e-8)
    else:
        assert abs(rmin - rminp) <= 1e-12 * rminp
    Cg = C1.cpu().numpy()[: K * k].reshape(k, K).T
    Cp = C1p.numpy()[: K * k].reshape(k, K).T
    np.testing.assert_allclose(Cg, Cp, rtol=0, atol=1e-9 * np.abs(Cp).max())
    Q = U @ Cg
    np.testing.assert_allclose(Q.T @ Q, np.eye(k), atol=1e-8)
