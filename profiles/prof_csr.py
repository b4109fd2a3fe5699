"""General-CSR path (csr.cu) at scale: the Kohn-Sham core operator of a
uniform mesh exported as CSR (15 nnz per row, the worst case for a stencil
pattern held as a general matrix), K columns: batched SpMV and PCG iteration
times, with the bytes the CSR formulation must move.

  python profiles/prof_csr.py [--s 128] [--k 8] [--iters 20]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paro_b200 import core  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", type=int, default=128)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    ctx = core.Context(0).grid(a.s, -12.0, 12.0)
    op = core.assemble_stiffness(ctx, 0.5)
    core.add_scaled(op, core.assemble_harmonic(ctx, 0.01))
    rows, cols, vals = op.to_csr()
    A = core.CsrOperator(ctx, rows, cols, vals)
    n, nnz = len(rows) - 1, len(vals)
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn((a.k, n), dtype=torch.float64, device="cuda", generator=g)
    Y = A.apply(X)
    # bit-exact against the stencil apply of the same operator
    assert torch.equal(Y, op.apply(X))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    best = 1e30
    for _ in range(5):
        torch.cuda.synchronize()
        ev[0].record()
        A.apply(X, out=Y)
        ev[1].record()
        torch.cuda.synchronize()
        best = min(best, ev[0].elapsed_time(ev[1]))
    # the apply includes the two boundary transposes (2 x 2 x 8 n k bytes)
    spmv_bytes = nnz * 12 + (n + 1) * 8 + 2 * 8 * n * a.k
    t0 = time.perf_counter()
    r = core.csr_cg_solve(A, X, None, tol=1e-30, max_iter=a.iters, throw_on_max_iter=False)
    torch.cuda.synchronize()
    cg_s = time.perf_counter() - t0
    # per PCG iteration: SpMV (matrix + p read + q write) + update (x, r, p, q read; x, r write) + direction (r, p read; p write)
    it_bytes = nnz * 12 + (n + 1) * 8 + 8 * n * a.k * (2 + 6 + 3) + 8 * n * 3
    print(json.dumps({"s": a.s, "n": n, "nnz": nnz, "k": a.k, "apply_ms": best,
                      "apply_gbs_incl_transposes": (spmv_bytes + 4 * 8 * n * a.k) / best / 1e6,
                      "cg_iters": r.iterations[0], "cg_ms_per_iter_wall": 1e3 * cg_s / max(1, r.iterations[0]),
                      "cg_gbs_wall": it_bytes * r.iterations[0] / cg_s / 1e9}))


if __name__ == "__main__":
    main()
