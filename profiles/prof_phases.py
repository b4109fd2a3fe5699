"""Per-phase device times of one fixed-mesh outer iteration (synchronised timers).

  python profiles/prof_phases.py [--workload cluster32] [--warmup 2]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paro_b200 import configs, core  # noqa: E402
from paro_b200.driver import GpuBackend, ParoRun  # noqa: E402


def timed(fn, reps=3):
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cluster32")
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    w = configs.get(a.workload)
    t0 = time.perf_counter()
    be = GpuBackend(w)
    run = ParoRun(w, be)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    for i in range(a.warmup):
        run.step(i)
    N = w.n_orbitals
    res = {"workload": w.name, "setup_s": setup}
    res["step_s"], tr = timed(lambda: run.step(a.warmup), reps=1)
    res["t_source"] = tr.t_source
    res["hartree_s"], _ = timed(lambda: be.hartree(run.rho_in, out=run.vh))
    res["ks_form_s"], _ = timed(lambda: be.ks_form(run.rho_in, run.vh, "in"))
    res["density_s"], _ = timed(lambda: be.density(run.orb[:N], run.occ, out=run.rho_half))
    res["energy_s"], _ = timed(lambda: be.energy(run.lambdas, run.occ, run.rho_out, run.vh))
    a_half = be.forms["half"]
    half = run.half[: run.k].clone()
    res["ritz_s"], _ = timed(lambda: be.ritz(half, a_half, N, w.drop_tol, run.orb), reps=2)
    res["apply_K_s"], _ = timed(lambda: a_half.apply(half, out=run.orb[: run.k]))
    res["mass_apply_K_s"], _ = timed(lambda: be.mass.apply(half, out=run.orb[: run.k]))
    res["step2_estimator_s"], res["eta_total"] = timed(
        lambda: be.estimate(run.orb[:N], run.lambdas[:N], run.rho_in, run.vh), reps=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
