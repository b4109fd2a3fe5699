"""Generate the golden fixtures in tests/golden/ from the unmodified reference
(oracle/_ref, built from /root/reference by oracle/Makefile).

  python tests/golden/make_golden.py

Fixtures: fixed-mesh ParO traces on identical seeded inputs (paro_b200.configs
generators), per outer iteration: the first N eigenvalues, the total energy,
sigma, and size-independent density checksums (integral, L2 norm) of rho_out,
plus the P1/Kuhn mass and stiffness stencils of a grid.
"""
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from paro_b200 import configs  # noqa: E402

OUT = Path(__file__).resolve().parent
WORKERS = os.cpu_count() or 1  # per-column results do not depend on the worker count (parallel.hpp:10-12)


def ks_trace(name, iters):
    w = configs.get(name)
    sp = ref.Space(w.subdivisions, w.lo, w.hi)
    ks = ref.KsSystem(sp, w.charges, w.positions, w.n_electrons, w.eps)
    g = configs.guess_vectors(w)
    loop = ref.KsLoop(ks, g, w.cg_tol_start, w.cg_tol, w.cg_tol_factor, w.cg_max_iter, w.mixing_alpha, w.drop_tol,
                      WORKERS)
    rows = []
    lam0 = loop.get("lambdas").tolist()
    for it in range(iters):
        r = loop.step(it)
        rho = loop.get("rho_out")
        rows.append({"iter": it + 1, "lambdas": r["lambdas"][: w.n_orbitals].tolist(), "e_tot": r["e_tot"],
                     "sigma": r["sigma"], "rho_residual": r["rho_residual"],
                     "rho_integral": ref.integrate(sp, rho), "rho_l2": ref.norm_l2(sp, rho)})
    return {"workload": name, "kind": "ks", "iterations": iters, "lambdas0": lam0, "trace": rows}


def linear_trace(name, iters):
    w = configs.get(name)
    sp = ref.Space(w.subdivisions, w.lo, w.hi)
    a = ref.Op.stiffness(sp, 0.5)
    a.add_scaled(ref.Op.wmass_harmonic(sp, 0.5) if w.potential == "harmonic"
                 else ref.Op.wmass_coulomb(sp, w.charges, w.positions, w.eps))
    b = ref.Op.mass(sp)
    g = configs.guess_vectors(w)
    loop = ref.LinLoop(sp, a, b, g, w.n_orbitals, w.cg_tol_start, w.cg_tol, w.cg_tol_factor, w.cg_max_iter,
                       w.drop_tol, WORKERS)
    lam0 = loop.get("lambdas").tolist()
    rows = []
    for it in range(iters):
        r = loop.step(it)
        rows.append({"iter": it + 1, "lambdas": r["lambdas"][: w.n_orbitals].tolist(), "sigma": r["sigma"]})
    return {"workload": name, "kind": "linear", "iterations": iters, "lambdas0": lam0, "trace": rows}


def stencils():
    out = {}
    for s, lo, hi in ((32, -10.0, 10.0), (12, -6.0, 6.0)):
        sp = ref.Space(s, lo, hi)
        S = s - 1
        c = (S * S + S + 1) * (S // 2)  # an interior row
        res = {}
        for nm, op in (("mass", ref.Op.mass(sp)), ("kinetic", ref.Op.stiffness(sp, 0.5)),
                       ("poisson", ref.Op.stiffness(sp, 1.0))):
            rows, cols, vals = op.csr()
            res[nm] = {str(int(cols[k]) - c): float(vals[k]) for k in range(rows[c], rows[c + 1])}
        out[f"s{s}_{lo}_{hi}"] = res
    return out


# BASELINE configs at full size where the reference finishes here (configs[0]
# H2 at 33^3 for all 20 iterations, configs[1] the oscillator at 65^3 for all
# 40), and configs[2..4] on 65^3 meshes of the same generators (SURVEY 8d:
# "run configs 4 and 5 scaled down (same generators at s = 64) fully on both
# sides").  python tests/golden/make_golden.py full
# The Kohn-Sham configs at these sizes (h2, water@s64, cluster32@s64, and
# water at its full 129^3) have traces with stored reference densities:
# tests/golden/make_golden_big.py.
FULL = {
    "oscillator": ("linear", 40),
    "source64@s64": ("linear", 1),
}


def main_full(names=None):
    for name, (kind, iters) in FULL.items():
        if names and name not in names:
            continue
        fx = ks_trace(name, iters) if kind == "ks" else linear_trace(name, iters)
        (OUT / f"full_{name.replace('@', '_')}.json").write_text(json.dumps(fx, indent=1))
        print("wrote", name, flush=True)


def main():
    fixtures = {
        "h2@s16": ks_trace("h2@s16", 6),
        "water@s24": ks_trace("water@s24", 4),
        "cluster32@s24": ks_trace("cluster32@s24", 3),
        "oscillator@s16": linear_trace("oscillator@s16", 8),
        "source64@s24": linear_trace("source64@s24", 1),
        "stencils": stencils(),
    }
    for k, v in fixtures.items():
        (OUT / f"{k.replace('@', '_')}.json").write_text(json.dumps(v, indent=1))
        print("wrote", k)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "full":
        main_full(sys.argv[2:])
    else:
        main()
