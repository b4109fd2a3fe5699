"""GPU parity: operator apply, cg_solve, Step 3 and the Hartree solve against
the compiled reference (oracle/_ref) on identical inputs."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ops(ref, s=12, lo=-6.0, hi=6.0):
    sp = ref.Space(s, lo, hi)
    Z = np.array([1.0, 1.0])
    R = np.array([[0.7, 0.0, 0.0], [-0.7, 0.0, 0.0]])
    ks = ref.KsSystem(sp, Z, R, 2)
    return sp, ks


def _dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda")


def test_apply_bit_exact_vs_csr_matvec(ref, gpu_ctx_factory):
    from paro_b200 import core

    sp, ks = _ops(ref)
    ctx = gpu_ctx_factory(sp.s, sp.lo, sp.hi)
    rng = np.random.default_rng(1)
    X = rng.standard_normal((3, sp.n))
    mass, kin, vext, poi = (ks.op(w) for w in ("mass", "kinetic", "vext", "poisson"))
    a0 = kin.copy().add_scaled(vext)  # core Hamiltonian (paro.cpp:500-501)
    for op in (mass, kin, vext, poi, a0):
        g = core.Operator.from_csr(ctx, *op.csr())
        Y = g.apply(_dev(X)).cpu().numpy()
        for c in range(3):
            np.testing.assert_array_equal(Y[c], op.matvec(X[c]))
    # shifted operator A + sigma B == add_scaled(b, sigma) (paro.cpp:89-90)
    sigma = 0.8123
    gm = core.Operator.from_csr(ctx, *mass.csr())
    ga = core.Operator.from_csr(ctx, *a0.csr())
    Y = ga.apply(_dev(X), shift=gm, sigma=sigma).cpu().numpy()
    sh = a0.copy().add_scaled(mass, sigma)
    for c in range(3):
        np.testing.assert_array_equal(Y[c], sh.matvec(X[c]))
    assert gm.variable is False and ga.variable is True


def test_to_csr_roundtrip(ref, gpu_ctx_factory):
    from paro_b200 import core

    sp, ks = _ops(ref, s=8)
    ctx = gpu_ctx_factory(sp.s, sp.lo, sp.hi)
    for w in ("mass", "vext"):
        op = ks.op(w)
        rows, cols, vals = op.csr()
        g = core.Operator.from_csr(ctx, rows, cols, vals)
        r2, c2, v2 = g.to_csr()
        np.testing.assert_array_equal(rows, r2)
        np.testing.assert_array_equal(cols, c2)
        np.testing.assert_array_equal(vals, v2)


def test_cg_solve_matches_reference(ref, gpu_ctx_factory):
    from paro_b200 import core

    sp, ks = _ops(ref)
    ctx = gpu_ctx_factory(sp.s, sp.lo, sp.hi)
    poi = ks.op("poisson")
    g = core.Operator.from_csr(ctx, *poi.csr())
    rng = np.random.default_rng(2)
    B = rng.standard_normal((2, sp.n))
    X0 = rng.standard_normal((2, sp.n))
    res = core.cg_solve(g, _dev(B), _dev(X0), tol=1e-10, max_iter=5000)
    for c in range(2):
        x, it, r, conv = ref.cg(poi, B[c], X0[c], tol=1e-10, max_iter=5000)
        assert abs(res.iterations[c] - it) <= 1
        np.testing.assert_allclose(res.x[c].cpu().numpy(), x, rtol=0, atol=1e-8 * np.abs(x).max())


def test_cg_limits_and_not_spd(ref, gpu_ctx_factory):
    from paro_b200 import IterationLimitError, NotSpdError, core

    sp, ks = _ops(ref, s=8)
    ctx = gpu_ctx_factory(sp.s, sp.lo, sp.hi)
    g = core.Operator.from_csr(ctx, *ks.op("poisson").csr())
    b = _dev(np.ones(sp.n))
    with pytest.raises(IterationLimitError) as e:
        core.cg_solve(g, b, tol=1e-14, max_iter=2)
    assert e.value.residual > 0
    with pytest.raises(ref.RefIterationLimit):
        ref.cg(ks.op("poisson"), np.ones(sp.n), tol=1e-14, max_iter=2)
    neg = core.Operator.constant(ctx, -g.weights)
    with pytest.raises(NotSpdError):
        core.cg_solve(neg, b, tol=1e-10)
    # zero right-hand side: x = 0 in 0 iterations (linalg.cpp:158-162)
    r = core.cg_solve(g, _dev(np.zeros(sp.n)), _dev(np.ones(sp.n)))
    assert r.iterations[0] == 0 and float(r.x.abs().max()) == 0.0


def test_source_solve_step_matches_reference(ref, gpu_ctx_factory):
    from paro_b200 import core

    sp, ks = _ops(ref)
    ctx = gpu_ctx_factory(sp.s, sp.lo, sp.hi)
    mass = ks.op("mass")
    a0 = ks.op("kinetic").copy().add_scaled(ks.op("vext"))
    rng = np.random.default_rng(3)
    G = rng.uniform(-1, 1, (4, sp.n))
    lam, U, _, _ = ref.rayleigh_ritz(sp, G, a0, mass, 4)
    ga = core.Operator.from_csr(ctx, *a0.csr())
    gm = core.Operator.from_csr(ctx, *mass.csr())
    for tol in (1e-8, 1e-12):
        rep = {}
        half, sigma = core.shifted_source_step(ga, gm, _dev(U), lam, tol=tol, report=rep)
        half_ref, sigma_ref = ref.shifted_source(a0, mass, sp, U, lam, tol)
        assert sigma == sigma_ref
        h = half.cpu().numpy()
        for c in range(4):
            scale = np.abs(half_ref[c]).max()
            np.testing.assert_allclose(h[c], half_ref[c], rtol=0, atol=50 * tol * scale)


def test_hartree_matches_reference(ref, gpu_ctx_factory):
    from paro_b200 import core

    sp, ks = _ops(ref)
    ctx = gpu_ctx_factory(sp.s, sp.lo, sp.hi)
    rng = np.random.default_rng(4)
    U = rng.uniform(-1, 1, (1, sp.n))
    rho, _ = ref.density(sp, U, [2.0])
    vh_ref = ref.hartree(sp, ks.op("poisson"), ks.op("mass"), rho, 1e-11)
    gp = core.Operator.from_csr(ctx, *ks.op("poisson").csr())
    gm = core.Operator.from_csr(ctx, *ks.op("mass").csr())
    assert not gp.variable and not gm.variable
    for mode, tol in (("cg", 1e-9), ("dst", 1e-10)):
        ctx.set_hartree_mode(mode)
        rep = {}
        vh = core.hartree_solve_with(gp, gm, _dev(rho), 1e-11, report=rep).cpu().numpy()
        np.testing.assert_allclose(vh, vh_ref, rtol=0, atol=tol * np.abs(vh_ref).max())
        assert (rep["iterations"] == 0) == (mode == "dst")
    # the exact DST solution satisfies the discrete system to round-off
    b = ks.op("mass").matvec(rho) * 4 * np.pi
    r = ks.op("poisson").matvec(vh) - b
    assert np.linalg.norm(r) <= 1e-12 * np.linalg.norm(b)


@pytest.mark.parametrize("s", [17, 20, 33])
def test_source_step_even_and_odd_rows(ref, gpu_ctx_factory, s):
    """Step 3 through the TMA PCG passes: even and odd interior row length
    S = s - 1 (row-padded solver layout with P = S or S + 1), tiles that
    overhang the lattice in x and y, several z-chunks, K = 6 (a 4-column group
    plus a partial one) and K = 2, against the reference at the solver
    tolerance."""
    from paro_b200 import core

    sp = ref.Space(s, -6.0, 6.0)
    Z = np.array([1.0, 1.0])
    R = np.array([[0.7, 0.0, 0.0], [-0.7, 0.0, 0.0]])
    ks = ref.KsSystem(sp, Z, R, 2)
    ctx = gpu_ctx_factory(sp.s, sp.lo, sp.hi)
    mass = ks.op("mass")
    a0 = ks.op("kinetic").copy().add_scaled(ks.op("vext"))
    rng = np.random.default_rng(s)
    G = rng.uniform(-1, 1, (6, sp.n))
    lam, U, _, _ = ref.rayleigh_ritz(sp, G, a0, mass, 6)
    ga = core.Operator.from_csr(ctx, *a0.csr())
    gm = core.Operator.from_csr(ctx, *mass.csr())
    tol = 1e-10
    for k in (6, 2):
        half, sigma = core.shifted_source_step(ga, gm, _dev(U[:k]), lam[:k], tol=tol)
        half_ref, sigma_ref = ref.shifted_source(a0, mass, sp, U[:k], lam[:k], tol)
        assert sigma == sigma_ref
        h = half.cpu().numpy()
        for c in range(k):
            np.testing.assert_allclose(h[c], half_ref[c], rtol=0, atol=50 * tol * np.abs(half_ref[c]).max())


@pytest.mark.parametrize("k", [1, 3, 5, 9])
def test_variable_cg_column_groups(ref, gpu_ctx_factory, k):
    """Batched Jacobi-PCG on a variable operator (TMA passes with staged
    coefficients, symmetric p'Ap) for column counts that leave partial
    column groups and columns that stop at different iterations, against the
    reference cg_solve column by column (linalg.cpp:143-223)."""
    from paro_b200 import core

    sp, ks = _ops(ref, s=21)
    ctx = gpu_ctx_factory(sp.s, sp.lo, sp.hi)
    a0 = ks.op("kinetic").copy().add_scaled(ks.op("vext")).add_scaled(ks.op("mass"), 3.0)
    ga = core.Operator.from_csr(ctx, *a0.csr())
    assert ga.variable
    rng = np.random.default_rng(100 + k)
    # right-hand sides of different smoothness converge in different counts
    B = rng.standard_normal((k, sp.n)) * np.linspace(0.2, 1.0, k)[:, None]
    B[::2] = np.cumsum(B[::2], axis=1) / np.sqrt(sp.n)
    X0 = rng.standard_normal((k, sp.n)) * 1e-3
    if k > 2:  # column 1 starts next to its solution and stops early
        xs = rng.standard_normal(sp.n)
        B[1] = a0.matvec(xs)
        X0[1] = xs + 1e-9 * rng.standard_normal(sp.n)
    res = core.cg_solve(ga, _dev(B), _dev(X0), tol=1e-11, max_iter=5000)
    iters = []
    for c in range(k):
        x, it, r, conv = ref.cg(a0, B[c], X0[c], tol=1e-11, max_iter=5000)
        iters.append(it)
        assert abs(res.iterations[c] - it) <= 1, (c, res.iterations[c], it)
        np.testing.assert_allclose(res.x[c].cpu().numpy(), x, rtol=0, atol=1e-8 * np.abs(x).max())
    if k > 2:
        assert len(set(iters)) > 1  # the batch really ran with mixed active masks


@pytest.mark.parametrize("s,K", [(12, 1), (12, 4), (40, 5), (40, 9), (70, 2), (34, 3)])
def test_apply_flat_view_bit_exact(ref, gpu_ctx_factory, s, K):
    """The dense-layout TMA apply (tma.cu k3f_kernel: x through the flat
    2S-wide view, parity boxes, lattice masks) against the reference CSR
    matvec: odd S with partial tiles, column counts that leave partial column
    groups and odd lattice-row totals, variable and constant operators, plus
    an 8-byte-misaligned column view (which stays on stream_kernel)."""
    from paro_b200 import core

    sp, ks = _ops(ref, s=s, lo=-7.0, hi=7.0)
    ctx = gpu_ctx_factory(sp.s, sp.lo, sp.hi)
    rng = np.random.default_rng(s * 100 + K)
    X = rng.standard_normal((K + 1, sp.n))
    Xd = _dev(X)
    mass, kin, vext = (ks.op(w) for w in ("mass", "kinetic", "vext"))
    a0 = kin.copy().add_scaled(vext)
    for op in (mass, a0):
        g = core.Operator.from_csr(ctx, *op.csr())
        for view, rows in ((Xd[:K], range(K)), (Xd[1:], range(1, K + 1))):
            Y = g.apply(view).cpu().numpy()
            for i, c in enumerate(rows):
                np.testing.assert_array_equal(Y[i], op.matvec(X[c]))
