"""Config-size golden traces with the density vectors, from the unmodified
reference (oracle/_ref).  TEST INFRASTRUCTURE ONLY.

  python tests/golden/make_golden_big.py water [workers]        # configs[2]: 129^3, N=5, all 30 iterations
  python tests/golden/make_golden_big.py cluster32@s64 [workers] # configs[4] generator at 65^3, all 15 iterations

Writes tests/golden/big_<name>.json (per-iteration eigenvalues, energy, sigma,
rho checksums) and tests/golden/big_<name>_rho.npz: rho_out of the selected
iterations, byte-shuffled + zlib (numpy savez_compressed of the uint8 planes
of the float64 array), so tests can form ||rho_gpu - rho_ref||_L2 directly.
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from paro_b200 import configs  # noqa: E402

OUT = Path(__file__).resolve().parent
SCRATCH = ROOT / "scratch"

# iterations whose rho_out is stored as a full vector (all iterations keep
# their checksums); config-size vectors are 16 MB (129^3) / 2 MB (65^3) each
RHO_ITERS = {"water": None, "cluster32@s64": None}  # None: decided by --keep below


def shuffle(v: np.ndarray) -> np.ndarray:
    """float64 -> [8, n] uint8 byte planes (compresses ~2x better than raw)."""
    return np.ascontiguousarray(v.astype("<f8").view(np.uint8).reshape(-1, 8).T)


def unshuffle(b: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(b.T).reshape(-1).view("<f8")


def run(name: str, workers: int):
    w = configs.get(name)
    iters = w.iterations
    sp = ref.Space(w.subdivisions, w.lo, w.hi)
    ks = ref.KsSystem(sp, w.charges, w.positions, w.n_electrons, w.eps)
    g = configs.guess_vectors(w)
    t0 = time.time()
    loop = ref.KsLoop(ks, g, w.cg_tol_start, w.cg_tol, w.cg_tol_factor, w.cg_max_iter, w.mixing_alpha, w.drop_tol,
                      workers)
    rows = []
    lam0 = loop.get("lambdas").tolist()
    print(f"{name}: setup {time.time() - t0:.1f} s", flush=True)
    tag = name.replace("@", "_")
    for it in range(iters):
        t1 = time.time()
        r = loop.step(it)
        rho = loop.get("rho_out")
        rows.append({"iter": it + 1, "lambdas": r["lambdas"][: w.n_orbitals].tolist(), "e_tot": r["e_tot"],
                     "sigma": r["sigma"], "rho_residual": r["rho_residual"], "gram_defect": r["gram_defect"],
                     "rho_integral": ref.integrate(sp, rho), "rho_l2": ref.norm_l2(sp, rho),
                     "t_step_s": time.time() - t1})
        np.save(SCRATCH / f"{tag}_rho_{it + 1:02d}.npy", rho)
        print(f"{name}: iter {it + 1} {time.time() - t1:.1f} s E={r['e_tot']:.12f}", flush=True)
        fx = {"workload": name, "kind": "ks", "iterations": it + 1, "lambdas0": lam0, "workers": workers,
              "trace": rows}
        (SCRATCH / f"big_{tag}.json").write_text(json.dumps(fx, indent=1))
    return fx


SKETCH_ROWS = 32
SKETCH_SEED = 20261020


def sketch_matrix(n: int) -> np.ndarray:
    """[SKETCH_ROWS, n] uniform[-1, 1) rows (configs.SplitMix64, seeded): for a
    difference d, mean((S d)^2) * 3 estimates ||d||_2^2 (E s^2 = 1/3)."""
    rng = configs.SplitMix64(SKETCH_SEED)
    return rng.sym_array(SKETCH_ROWS * n).reshape(SKETCH_ROWS, n)


def pack(name: str, keep):
    """Commit step: the trace json (plus a 32-row sketch of every iteration's
    rho_out) and the full rho vectors of iterations `keep`."""
    tag = name.replace("@", "_")
    fx = json.loads((SCRATCH / f"big_{tag}.json").read_text())
    n = configs.get(name).n
    S = sketch_matrix(n)
    for row in fx["trace"]:
        rho = np.load(SCRATCH / f"{tag}_rho_{row['iter']:02d}.npy")
        row["rho_sketch"] = (S @ rho).tolist()
    fx["rho_vectors"] = list(keep)
    fx["sketch"] = {"rows": SKETCH_ROWS, "seed": SKETCH_SEED, "dist": "uniform[-1,1) SplitMix64"}
    (OUT / f"big_{tag}.json").write_text(json.dumps(fx, indent=1))
    arrs = {f"it{k:02d}": shuffle(np.load(SCRATCH / f"{tag}_rho_{k:02d}.npy")) for k in keep}
    np.savez_compressed(OUT / f"big_{tag}_rho.npz", **arrs)


if __name__ == "__main__":
    SCRATCH.mkdir(exist_ok=True)
    if sys.argv[1] == "pack":
        pack(sys.argv[2], [int(k) for k in sys.argv[3].split(",")])
    else:
        run(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 8)
