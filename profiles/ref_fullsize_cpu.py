"""The reference's Step-3 hot path measured directly at the full mesh (257^3
nodes, 16.6 M dofs) on the host cores: cg_solve at a pinned iteration count
(tol 1e-30, no throw; harness ref_source_pinned, precedent proj/src/suites.cpp:
439-457) on the shifted operator A + sigma M with the reference's own
orbital-level parallel_for. The operator is stiffness + a weighted mass (the
sparsity, and so the SpMV cost, of the Kohn-Sham form). Checks the
reduced-mesh extrapolation of bench.py's cpu_baseline.

  python profiles/ref_fullsize_cpu.py [--s 256] [--cols 16] [--iters 10] [--workers 16]
"""
import argparse
import json
import os
import resource
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402


def rss_gb():
    return round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6, 2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", type=int, default=256)
    ap.add_argument("--cols", type=int, default=16)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    from oracle import ref

    out = {"subdivisions": a.s, "workers": a.workers, "host_cpus": os.cpu_count()}
    t = time.time()
    sp = ref.Space(a.s, -18.0, 18.0)
    out["space_build_s"] = round(time.time() - t, 1)
    out["n_dofs"] = sp.n
    out["rss_after_space_gb"] = rss_gb()
    print(out, flush=True)
    t = time.time()
    m = ref.Op.mass(sp)
    op = ref.Op.stiffness(sp, 0.5)
    op.add_scaled(ref.Op.wmass_harmonic(sp, 0.5))
    out["operators_s"] = round(time.time() - t, 1)
    out["rss_after_operators_gb"] = rss_gb()
    print(out, flush=True)
    rng = np.random.default_rng(0)
    U = rng.standard_normal((a.cols, sp.n))
    lam = np.full(a.cols, -1.0)
    runs = []
    for cols, workers in ((1, 1), (a.cols, a.workers), (a.cols, a.workers)):
        t = time.time()
        ref.source_pinned(op, m, U[:cols], lam[:cols], 5.0, a.iters, workers=workers)
        w = time.time() - t
        runs.append({"columns": cols, "workers": workers, "iterations": a.iters, "wall_s": round(w, 2),
                     "col_iters_per_s": round(cols * a.iters / w, 2)})
        print(runs[-1], flush=True)
    out["pinned"] = runs
    best = max(r["col_iters_per_s"] for r in runs if r["workers"] == a.workers)
    # one cluster32 outer iteration: 3,246 column-iterations of Step 3 (bench breakdown), 76 columns on
    # `workers` threads (5 rounds of 16 for 76 columns: the last round is 12/16 full)
    rounds = -(-76 // a.workers)
    out["step3_s_per_outer_iteration"] = round(3246.4 / best * (rounds * a.workers / 76.0), 1)
    out["rss_peak_gb"] = rss_gb()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
