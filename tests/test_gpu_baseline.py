"""GPU baseline_geneig / initial_guess (linalg.cpp:615-623,
paro.cpp:63-79) against the compiled reference on the same pencil: both
converge to the same lowest eigenpairs (fix_sign convention), so eigenvalues
and sign-fixed eigenvectors are compared, not the random starts. Beyond the
reference's 50,000-dof cap the defining properties are checked instead."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _pencil_ref(ref, w):
    sp = ref.Space(w.subdivisions, w.lo, w.hi)
    a = ref.Op.stiffness(sp, 0.5)
    a.add_scaled(ref.Op.wmass_coulomb(sp, w.charges, w.positions, w.eps))
    return sp, a, ref.Op.mass(sp)


def _pencil_gpu(w):
    from paro_b200 import core

    ctx = core.Context(0).grid(w.subdivisions, w.lo, w.hi)
    a = core.assemble_stiffness(ctx, 0.5)
    core.add_scaled(a, core.assemble_vext(ctx, w.charges, w.positions, w.eps))
    return ctx, a, core.assemble_mass(ctx)


def test_baseline_geneig_matches_reference(ref):
    from paro_b200 import configs, core

    w = configs.get("source64").scaled(20)  # n = 6859: the reference's subspace route
    sp, ra, rb = _pencil_ref(ref, w)
    vals_r, vecs_r = ref.baseline_geneig(ra, rb, 6)
    ctx, a, b = _pencil_gpu(w)
    vals, V, its = core.baseline_geneig(a, b, 6)
    assert its >= 1
    np.testing.assert_allclose(vals, vals_r, rtol=1e-9, atol=1e-12)
    Vh = V.cpu().numpy()
    for j in range(6):
        scale = np.abs(vecs_r[j]).max()
        assert np.abs(Vh[j] - vecs_r[j]).max() <= 1e-6 * scale, j


def test_initial_guess_is_b_orthonormal_and_errors(ref):
    from paro_b200 import _native as N
    from paro_b200 import configs, core

    w = configs.get("source64").scaled(20)
    ctx, a, b = _pencil_gpu(w)
    og = core.initial_guess(a, b, 4)
    assert og.gram_defect <= 1e-10
    assert og.lambdas == sorted(og.lambdas)
    with pytest.raises(N.InvalidArgumentError):
        core.initial_guess(a, b, 0)
    with pytest.raises(N.InvalidArgumentError):
        core.baseline_geneig(a, b, ctx.n + 1)


def test_baseline_geneig_beyond_the_reference_cap():
    """65^3 nodes (n = 250,047, five times the reference's hard cap): residuals
    within the reference's own convergence bar, B-orthonormal, ascending."""
    from paro_b200 import configs, core

    w = configs.get("source64").scaled(64)
    ctx, a, b = _pencil_gpu(w)
    vals, V, _ = core.baseline_geneig(a, b, 8)
    AV = a.apply(V)
    BV = b.apply(V)
    lam = torch.tensor(vals, dtype=torch.float64, device=V.device)[:, None]
    res = torch.linalg.vector_norm(AV - lam * BV, dim=1).cpu().numpy()
    amax = float(a.coefficients().abs().max()) if a.variable else float(np.abs(a.weights).max())
    bmax = float(np.abs(b.weights).max()) if not b.variable else float(b.coefficients().abs().max())
    for j, l in enumerate(vals):
        assert res[j] <= 1e-9 * max(1.0, amax + abs(l) * bmax), (j, res[j])
    G = (V @ BV.T).cpu().numpy()
    assert np.abs(G - np.eye(8)).max() <= 1e-10
    assert list(vals) == sorted(vals)


def test_paro_from_baseline_start_matches_reference(ref):
    """The reference drivers' own start (initial_guess = baseline eigenpairs of
    the core Hamiltonian, paro.cpp:499-505) on both sides, then two Kohn-Sham
    outer iterations: water on a 21^3-node mesh (the reference's subspace route)."""
    from paro_b200 import configs
    from paro_b200.driver import GpuBackend, ParoRun

    w = configs.get("water").scaled(20)
    sp = ref.Space(w.subdivisions, w.lo, w.hi)
    ks = ref.KsSystem(sp, w.charges, w.positions, w.n_electrons, w.eps)
    a0 = ks.op("kinetic").copy().add_scaled(ks.op("vext"))
    _, guess = ref.baseline_geneig(a0, ks.op("mass"), w.K)
    loop = ref.KsLoop(ks, guess, w.cg_tol_start, w.cg_tol, w.cg_tol_factor, w.cg_max_iter, w.mixing_alpha,
                      w.drop_tol)
    run = ParoRun(w, GpuBackend(w), guess="baseline")
    np.testing.assert_allclose(run.lambdas, loop.get("lambdas")[: w.K], rtol=1e-9)
    for it in range(2):
        tr = run.step(it)
        rr = loop.step(it)
        np.testing.assert_allclose(tr.lambdas, rr["lambdas"][: w.n_orbitals], rtol=1e-8, atol=1e-10)
        assert abs(tr.e_tot - rr["e_tot"]) <= 1e-8
