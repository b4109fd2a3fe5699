"""Which columns meet NotSpd at the first sigma of a steady-state outer iteration, and when?
The failing attempt of shifted_source_step (paro.cpp:194-210) replayed through
cg_solve (no batch abort): per-column status and iteration of the p'Ap <= 0 event.

  python profiles/probe_columns.py [--workload cluster32] [--warmup 10]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paro_b200 import configs, core  # noqa: E402
from paro_b200.driver import GpuBackend, ParoRun  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cluster32")
    ap.add_argument("--warmup", type=int, default=10)
    a = ap.parse_args()
    w = configs.get(a.workload)
    be = GpuBackend(w)
    run = ParoRun(w, be, timers=False)
    for i in range(a.warmup):
        run.step(i)
    K = run.k
    # the next step's Step-3 inputs: form at rho_in, sigma_0 = max(0, 0.5 - lambda_1)
    vh = be.hartree(run.rho_in, out=run.vh)
    a_in, _ = be.ks_form(run.rho_in, vh, "in")
    sigma0 = max(0.0, 0.5 - run.lambdas[0])
    tol = w.cg_tol_for_iteration(a.warmup)
    shifted = core.add_scaled(core.add_scaled(core.assemble_stiffness(be.ctx, 0.0), a_in, 1.0), be.mass, sigma0)
    u = run.orb[:K]
    b = be.mass.apply(u)
    b.mul_(torch.tensor([l + sigma0 for l in run.lambdas[:K]], device=b.device, dtype=b.dtype)[:, None])
    # the C ABI directly: per-column iteration counts and residuals whatever the call's status
    from paro_b200 import _native as N
    import ctypes as C

    x = torch.empty_like(b)
    x0 = u.clone()
    it = (C.c_size_t * K)()
    res = (C.c_double * K)()
    n = be.n
    stat = N.lib().paro_cg_solve(be.ctx.h, shifted.h, K, core._ptr(b), core._ptr(x0), n, tol, 400, 0, core._ptr(x), it, res)
    its, rs = list(it), list(res)
    print("status", stat, "probe list:", run._notspd_probe, "sigma0", sigma0, "tol", tol)
    failed = [(c, its[c]) for c in range(K) if rs[c] > tol]
    print("columns that stopped above the tolerance (NotSpd) and the iteration of the event:", sorted(failed, key=lambda t: t[1]))
    print("converged columns:", [(c, its[c]) for c in range(K) if rs[c] <= tol])


if __name__ == "__main__":
    main()
