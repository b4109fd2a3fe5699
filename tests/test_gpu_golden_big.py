"""Config-size parity (BASELINE configs[2] water at 129^3 for all 30 outer
iterations; configs[4]'s 32-atom cluster generator at 65^3 for all 15) against
golden traces of the compiled reference (tests/golden/make_golden_big.py).

North-star bar, checked on the density vector itself:
* eigenvalues: 1e-8 relative; for |lambda| < 1e-2 an absolute floor of 1e-10 Ha
  (a hundredth of the energy bar) replaces it;
* total energy: 1e-8 Ha; the Step-3 shift sigma (derived from lambda_1 and
  the NotSpd escalations) to 1e-9 relative;
* density: ||rho_gpu - rho_ref||_L2 <= 1e-7 (FE norm) at the iterations whose
  reference rho is stored in full; at every iteration a 32-row sketch of the
  difference bounds it as well: ||d||_L2 <= h^1.5 ||d||_2 (the P1 mass matrix
  is at most h^3 times the identity), with ||d||_2 estimated from the sketch.

Non-converging SCF trajectories. The water runs (65^3 and the full 129^3) do
not converge under alpha = 0.3 linear mixing: the energy sloshes by tens of Ha
between iterations, and such a trajectory amplifies any rounding-level
difference by ~1.5x per outer iteration. tests/golden/sensitivity.py measures
that on the reference itself: its own trajectory from the guess perturbed by
1e-12 (relative) moves by s(k) at iteration k (s_E reaches 1e-8 Ha by iteration
29 at 65^3: the reference fails the energy bar against itself). The device
path differs from the reference by ~1e-12 in lambda after the first iteration
(~100 s(1): CG stop decisions at the loose early tolerances, reduction order),
so where a sensitivity_<tag>.json exists each bar is max(bar, 1e3 s(k)), the
reference's own amplification with a 10x margin; elsewhere the bars are
strict. cluster32 (converging) and H2 are checked at the strict bars.
"""
import json
import math
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(GOLDEN))

CASES = sorted(p.stem[4:] for p in GOLDEN.glob("big_*.json"))


AMPLIFY = 1e3  # device-vs-reference difference level over the reference's 1e-12 sensitivity, x10


def check_lambdas(got, ref, s_rel=0.0, s_abs=0.0):
    got, ref = np.asarray(got), np.asarray(ref)
    small = np.abs(ref) < 1e-2
    np.testing.assert_allclose(got[~small], ref[~small], rtol=max(1e-8, AMPLIFY * s_rel), atol=0)
    np.testing.assert_allclose(got[small], ref[small], rtol=0, atol=max(1e-10, AMPLIFY * s_abs))


@pytest.mark.parametrize("tag", CASES)
def test_config_size_trace_and_density(tag):
    from make_golden_big import sketch_matrix, unshuffle

    from paro_b200 import configs, core
    from paro_b200.driver import GpuBackend, ParoRun

    fx = json.loads((GOLDEN / f"big_{tag}.json").read_text())
    vecs = np.load(GOLDEN / f"big_{tag}_rho.npz")
    sens_path = GOLDEN / f"sensitivity_{tag}.json"
    sens = {r["iter"]: r for r in json.loads(sens_path.read_text())["trace"]} if sens_path.exists() else {}
    w = configs.get(fx["workload"])
    run = ParoRun(w, GpuBackend(w))
    ctx = run.be.ctx
    check_lambdas(run.lambdas[: len(fx["lambdas0"])], fx["lambdas0"])
    S = torch.as_tensor(sketch_matrix(w.n), device="cuda")
    hh = w.h ** 1.5
    worst = 0.0
    for row in fx["trace"]:
        tr = run.step(row["iter"] - 1)
        sk = sens.get(row["iter"], {})
        check_lambdas(tr.lambdas, row["lambdas"], sk.get("max_rel_lambda", 0.0), sk.get("max_abs_lambda", 0.0))
        e_bar = max(1e-8, AMPLIFY * sk.get("abs_e_tot", 0.0))
        rho_bar = max(1e-7, AMPLIFY * sk.get("rho_l2_est", 0.0))
        assert abs(tr.e_tot - row["e_tot"]) <= e_bar, (row["iter"], tr.e_tot, row["e_tot"])
        # sigma = max(0, 0.5 - lambda_1 of the previous iteration) escalated by
        # the NotSpd policy: the same escalation count, the value within the
        # eigenvalue bar of the iteration it comes from
        s_prev = sens.get(row["iter"] - 1, {}).get("max_rel_lambda", 0.0)
        assert tr.sigma == pytest.approx(row["sigma"], rel=max(1e-9, AMPLIFY * max(s_prev, sk.get("max_rel_lambda", 0.0))),
                                         abs=1e-12)
        d_sketch = (S @ run.rho_out).cpu().numpy() - np.asarray(row["rho_sketch"])
        est = math.sqrt(3.0 * float(np.mean(d_sketch ** 2)))  # ~ ||d||_2
        assert hh * est <= 0.5 * rho_bar, (row["iter"], hh * est)
        key = f"it{row['iter']:02d}"
        if key in vecs.files:
            ref = torch.as_tensor(unshuffle(vecs[key]), device="cuda")
            err = core.norm_l2(ctx, run.rho_out - ref)
            worst = max(worst, err)
            assert err <= rho_bar, (row["iter"], err)
    assert worst > 0.0 or not vecs.files
