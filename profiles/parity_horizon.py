"""Per-iteration distance of the device trajectory from a config-size golden
trace (tests/golden/big_<tag>.json): max relative eigenvalue error, energy
error, density sketch estimate, for the default exact (DST) Hartree solve and
for the reference's own Jacobi-PCG Hartree algorithm (ctx hartree mode "cg").

  python profiles/parity_horizon.py water_s64 [--mode dst|cg]
"""
import argparse
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from make_golden_big import sketch_matrix  # noqa: E402
from paro_b200 import configs  # noqa: E402
from paro_b200.driver import GpuBackend, ParoRun  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--mode", default="dst")
    a = ap.parse_args()
    fx = json.loads((ROOT / "tests" / "golden" / f"big_{a.tag}.json").read_text())
    w = configs.get(fx["workload"])
    be = GpuBackend(w)
    be.ctx.set_hartree_mode(a.mode)
    run = ParoRun(w, be)
    S = torch.as_tensor(sketch_matrix(w.n), device="cuda")
    out = []
    for row in fx["trace"]:
        tr = run.step(row["iter"] - 1)
        lam, ref = np.asarray(tr.lambdas), np.asarray(row["lambdas"])
        d = (S @ run.rho_out).cpu().numpy() - np.asarray(row["rho_sketch"])
        out.append({"iter": row["iter"], "max_rel_lambda": float(np.max(np.abs(lam - ref) / np.abs(ref))),
                    "max_abs_lambda": float(np.max(np.abs(lam - ref))), "abs_e_tot": abs(tr.e_tot - row["e_tot"]),
                    "rho_l2_est": w.h ** 1.5 * math.sqrt(3.0 * float(np.mean(d ** 2)))})
        print(json.dumps(out[-1]), flush=True)
    Path(ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / f"horizon_{a.tag}_{a.mode}.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
