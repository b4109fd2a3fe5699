"""GPU runs of the BASELINE generators (scaled meshes) against the committed
golden fixtures produced by the compiled reference (tests/golden/make_golden.py).
North-star tolerances: eigenvalues 1e-8 relative (for |lambda| < 1e-2 a 1e-10 Ha
absolute floor, a hundredth of the energy bar, replaces it), energy 1e-8 Ha.
These fixtures carry only the density's checksums (integral, L2 norm, the
residual ||rho_out - rho_in||); the density difference itself is bounded in
test_gpu_driver.py (live reference, small meshes) and test_gpu_golden_big.py
(stored reference vectors and sketches at the config sizes)."""
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def check_lambdas(got, ref):
    got, ref = np.asarray(got), np.asarray(ref)
    small = np.abs(ref) < 1e-2
    np.testing.assert_allclose(got[~small], ref[~small], rtol=1e-8, atol=0)
    np.testing.assert_allclose(got[small], ref[small], rtol=0, atol=1e-10)


@pytest.mark.parametrize("name", ["h2_s16", "water_s24", "cluster32_s24", "oscillator_s16", "source64_s24"])
def test_gpu_matches_golden_trace(name):
    from paro_b200 import configs, core
    from paro_b200.driver import GpuBackend, ParoRun

    fx = json.loads((GOLDEN / f"{name}.json").read_text())
    w = configs.get(fx["workload"])
    run = ParoRun(w, GpuBackend(w))
    np.testing.assert_allclose(run.lambdas[: len(fx["lambdas0"])], fx["lambdas0"], rtol=1e-10)
    for row in fx["trace"]:
        tr = run.step(row["iter"] - 1)
        check_lambdas(tr.lambdas, row["lambdas"])
        assert tr.sigma == pytest.approx(row["sigma"], rel=1e-12, abs=1e-14)
        if "e_tot" in row:
            assert abs(tr.e_tot - row["e_tot"]) <= 1e-8
            ctx = run.be.ctx
            assert core.integrate(ctx, run.rho_out) == pytest.approx(row["rho_integral"], rel=1e-12)
            assert abs(core.norm_l2(ctx, run.rho_out) - row["rho_l2"]) <= 1e-7
            assert abs(tr.rho_residual - row["rho_residual"]) <= 1e-7


# the Kohn-Sham configs at full size have stored reference densities (big_*.json)
FULL = sorted(p.stem for p in GOLDEN.glob("full_*.json"))


@pytest.mark.parametrize("name", FULL)
def test_gpu_matches_golden_trace_full_size(name):
    """BASELINE configs[1] at its full size and iteration count (oscillator
    65^3 x 40) and configs[3]'s generator on a 65^3 mesh (source64, noise
    start: the Gram-Schmidt path of Step 4); tests/golden/make_golden.py full."""
    test_gpu_matches_golden_trace(name)
