"""Step-3 Jacobi-PCG kernels at the bench's per-GPU shape, for ncu and timing.

Runs a pinned number of batched PCG iterations (tol 1e-30, no throw) of a
variable-coefficient P1/Kuhn operator (0.5*stiffness + harmonic mass) on
K random columns, plus a single-column constant-stencil (Hartree-like) solve,
and prints per-iteration times and algorithmic GB/s (SURVEY.md §8d:
n*(88 k + 64) bytes per PCG iteration).

  python profiles/prof_pcg.py [--s 256] [--k 76] [--iters 6]
  PARO_NO_GRAPH=1 ncu --set full -k 'regex:march_kernel<[12], true, 8>' -c 2 ... python profiles/prof_pcg.py
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paro_b200 import core  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", type=int, default=256)
    ap.add_argument("--k", type=int, default=76)
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--shifted", action="store_true", help="also time source_solve_columns with sigma = 16")
    ap.add_argument("--const", action="store_true", help="constant-coefficient operator (no coefficient loads)")
    a = ap.parse_args()
    ctx = core.Context(0).grid(a.s, -18.0, 18.0)
    op = core.assemble_stiffness(ctx, 0.5)
    if not a.const:
        core.add_scaled(op, core.assemble_harmonic(ctx, 0.01))
    poisson = core.assemble_stiffness(ctx, 1.0)
    n = ctx.n
    g = torch.Generator(device="cuda").manual_seed(0)
    b = torch.randn((a.k, n), dtype=torch.float64, device="cuda", generator=g)
    x0 = torch.randn((a.k, n), dtype=torch.float64, device="cuda", generator=g)
    out = {}
    if a.shifted:
        # Step 3 proper: source_solve_step with a spectral shift and the mass rhs
        mass = core.assemble_mass(ctx)
        lam = [-15.0] * a.k
        half = torch.empty_like(x0)
        for rep in range(a.reps):
            ctx.stats(reset=True)
            f, g2, it, _ = core.source_solve_columns(op, mass, x0, lam, 1e-30, a.iters, 16.0, half)
            st = ctx.stats()
            out[f"source_step_rep{rep}"] = {"ms_per_iter": 1e3 * st["step3_s"] / max(it),
                                            "achieved_gbs": st["step3_bytes"] / st["step3_s"] / 1e9,
                                            "col_iters": st["step3_col_iters"]}
    for name, A, B, X0 in (("step3", op, b, x0), ("hartree", poisson, b[:1], None)):
        best = None
        for _ in range(a.reps):
            ctx.stats(reset=True)
            r = core.cg_solve(A, B, X0, tol=1e-30, max_iter=a.iters, throw_on_max_iter=False)
            st = ctx.stats()
            key = "step3" if name == "step3" and not a.const else "hartree"  # stats bucket: variable / constant operator
            sec, byt = st[f"{key}_s"], st[f"{key}_bytes"]
            cur = {"ms_per_iter": 1e3 * sec / a.iters, "achieved_gbs": byt / sec / 1e9, "iters": r.iterations[0]}
            best = cur if best is None or cur["ms_per_iter"] < best["ms_per_iter"] else best
        out[name] = best
    print(json.dumps({"s": a.s, "n": n, "k": a.k, **out}))


if __name__ == "__main__":
    main()
