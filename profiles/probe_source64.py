"""Where configs[3] (source64, noise start) meets NotSpd: the lowest
generalized eigenvalue of its operator pencil at a mesh size, the Ritz start
and the sigma sequence of one Step-3 pass. python profiles/probe_source64.py 128"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paro_b200 import configs, core  # noqa: E402
from paro_b200.driver import GpuBackend, ParoRun  # noqa: E402

s = int(sys.argv[1]) if len(sys.argv) > 1 else 128
w = configs.get(f"source64@s{s}")
be = GpuBackend(w)
lam, V, its = core.baseline_geneig(be.form, be.mass, 2)
print(f"s={s} lowest eigenvalues of (A, M): {lam} ({its} subspace iterations)", flush=True)
run = ParoRun(w, be)
print(f"Ritz start lambda_1..3 = {run.lambdas[:3]}", flush=True)
try:
    tr = run.step(0)
    print(f"pass ok: sigma={tr.sigma}, attempts={run.last_attempts}, lambda_1={tr.lambdas[0]}")
except Exception as e:
    print(f"pass failed after {run.last_attempts} attempts: {type(e).__name__}: {e}")
