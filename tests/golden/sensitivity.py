"""How far the reference's own Kohn-Sham trajectory moves under a tiny
perturbation of its input (TEST INFRASTRUCTURE): the compiled reference
(oracle/_ref) runs the same workload from the generator's guess with every
entry multiplied by (1 + 1e-12), and each iteration's eigenvalues / energy /
density are compared with the unperturbed golden trace. 1e-12 is the level at
which two correct implementations differ after one outer iteration (the
CG stop test at the loose early tolerances moves by one iteration, e.g.);
a non-converging (sloshing) SCF amplifies such differences by a roughly fixed
factor per outer iteration, which bounds the parity horizon of ANY
implementation whose rounding differs from the reference's.

  python tests/golden/sensitivity.py water@s64 [workers]   -> tests/golden/sensitivity_<tag>.json
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

from oracle import ref  # noqa: E402
from paro_b200 import configs  # noqa: E402


def main(name, workers):
    tag = name.replace("@", "_")
    gold = json.loads((Path(__file__).resolve().parent / f"big_{tag}.json").read_text())
    w = configs.get(name)
    sp = ref.Space(w.subdivisions, w.lo, w.hi)
    ks = ref.KsSystem(sp, w.charges, w.positions, w.n_electrons, w.eps)
    g = configs.guess_vectors(w) * (1.0 + 1e-12)
    from make_golden_big import sketch_matrix

    S = sketch_matrix(w.n)
    loop = ref.KsLoop(ks, g, w.cg_tol_start, w.cg_tol, w.cg_tol_factor, w.cg_max_iter, w.mixing_alpha, w.drop_tol,
                      workers)
    rows = []
    for it, row in enumerate(gold["trace"]):
        r = loop.step(it)
        lam = np.asarray(r["lambdas"][: w.n_orbitals])
        ref_lam = np.asarray(row["lambdas"])
        rows.append({"iter": it + 1, "max_rel_lambda": float(np.max(np.abs(lam - ref_lam) / np.abs(ref_lam))),
                     "max_abs_lambda": float(np.max(np.abs(lam - ref_lam))),
                     "abs_e_tot": float(abs(r["e_tot"] - row["e_tot"])),
                     "rho_l2_est": float(w.h ** 1.5 * np.sqrt(3.0 * np.mean((S @ loop.get("rho_out")
                                                                               - np.asarray(row["rho_sketch"])) ** 2)))})
        print(rows[-1], flush=True)
    out = {"workload": name, "perturbation": "guess * (1 + 1e-12)", "trace": rows}
    (Path(__file__).resolve().parent / f"sensitivity_{tag}.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 8)
