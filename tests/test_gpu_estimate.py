"""GPU parity of the Step-2 residual estimator against the
compiled reference (estimate_eigen_residual + combine_max + total,
proj/src/adapt.cpp:58-129) on identical inputs: the Kohn-Sham reaction
V_ext + V_H + v_xc (paro.cpp:521-538) and the linear drivers' reactions
(paro.cpp:306-315). The device evaluates the element geometry from the
uniform spacing and the reference from vertex coordinates, so the bar is
rounding-level agreement (1e-10 relative), not bit equality."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

RTOL = 1e-10


def _check(tot_g, eta_g, tot_r, eta_r):
    assert abs(tot_g - tot_r) <= RTOL * abs(tot_r), (tot_g, tot_r)
    e = eta_g.cpu().numpy()
    np.testing.assert_allclose(e, eta_r, rtol=RTOL, atol=RTOL * np.abs(eta_r).max())


@pytest.mark.parametrize("name,s", [("h2", 16), ("water", 24)])
def test_ks_estimator_matches_reference(ref, name, s):
    from paro_b200 import configs, core
    from paro_b200.driver import GpuBackend, ParoRun

    w = configs.get(f"{name}@s{s}")
    be = GpuBackend(w)
    run = ParoRun(w, be)
    run.step(0)
    N = w.n_orbitals
    vh = be.hartree(run.rho_in, out=be.empty(be.n))
    tot, eta = core.estimate_eta(be.ctx, run.orb[:N], run.lambdas[:N], reaction="ks", charges=w.charges,
                                 positions=w.positions, eps=w.eps, rho=run.rho_in, vh=vh, with_eta=True)
    sp = ref.Space(w.subdivisions, w.lo, w.hi)
    ks = ref.KsSystem(sp, w.charges, w.positions, w.n_electrons, w.eps)
    tot_r, eta_r = ks.eta_total(run.orb[:N].cpu().numpy(), run.lambdas[:N], run.rho_in.cpu().numpy(),
                                vh.cpu().numpy(), with_eta=True)
    _check(tot, eta, tot_r, eta_r)
    assert tot > 0 and np.isfinite(tot)


def test_linear_estimators_match_reference(ref):
    from paro_b200 import configs, core

    rng = np.random.default_rng(7)
    for w, reaction in ((configs.oscillator().scaled(16), "harmonic"), (configs.get("source64@s12"), "well")):
        ctx = core.Context(0).grid(w.subdivisions, w.lo, w.hi)
        U = rng.uniform(-1, 1, (3, ctx.n))
        lam = [0.7, 1.9, 2.4]
        kw = dict(c=0.5) if reaction == "harmonic" else dict(charges=w.charges, positions=w.positions, eps=w.eps)
        tot, eta = core.estimate_eta(ctx, torch.as_tensor(U, device="cuda"), lam, reaction=reaction,
                                     with_eta=True, **kw)
        sp = ref.Space(w.subdivisions, w.lo, w.hi)
        rkw = dict(c=0.5) if reaction == "harmonic" else dict(Z=w.charges, R=w.positions, eps=w.eps)
        tot_r, eta_r = ref.lin_eta_total(sp, U, lam, 0.5, reaction, with_eta=True, **rkw)
        _check(tot, eta, tot_r, eta_r)


def test_estimator_argument_errors():
    from paro_b200 import InvalidArgumentError, core

    ctx = core.Context(0).grid(8, -4.0, 4.0)
    U = torch.zeros((1, ctx.n), dtype=torch.float64, device="cuda")
    with pytest.raises(InvalidArgumentError):
        core.estimate_eta(ctx, U, [1.0], reaction="ks")  # no rho / V_H / nuclei
    with pytest.raises(InvalidArgumentError):
        core.estimate_eta(ctx, U, [1.0], reaction="well")  # no nuclei
    assert core.estimate_eta(ctx, U, [1.0], reaction="harmonic", c=0.5) == 0.0


def test_driver_step2_eta_total(ref):
    """ParoRun(estimate=True) reports the reference's eta_total of the state
    each outer iteration starts from (Step 2 precedes Step 3)."""
    from paro_b200 import configs
    from paro_b200.driver import GpuBackend, ParoRun

    w = configs.get("h2@s16")
    be = GpuBackend(w)
    run = ParoRun(w, be, estimate=True)
    sp = ref.Space(w.subdivisions, w.lo, w.hi)
    ks = ref.KsSystem(sp, w.charges, w.positions, w.n_electrons, w.eps)
    for it in range(2):
        N = w.n_orbitals
        U, lam, rho = run.orb[:N].cpu().numpy(), list(run.lambdas[:N]), run.rho_in.cpu().numpy()
        vh = be.hartree(run.rho_in, out=be.empty(be.n)).cpu().numpy()
        tr = run.step(it)
        assert abs(tr.eta_total - ks.eta_total(U, lam, rho, vh)) <= RTOL * tr.eta_total
