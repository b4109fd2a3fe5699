"""Batched operator apply y = A x at the bench shape (257^3 nodes, K columns):
variable (KS-like) and constant (mass) operators, CUDA events, algorithmic
n(16k + 64) / n(16k) bytes.

  python profiles/prof_apply.py [--s 256] [--k 76] [--reps 5]
  PARO_NO_FLAT_APPLY=1 ...   (the previous stream_kernel path)
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paro_b200 import configs, core  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", type=int, default=256)
    ap.add_argument("--k", type=int, default=76)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    w = configs.get("cluster32").scaled(a.s)
    ctx = core.Context(0).grid(w.subdivisions, w.lo, w.hi)
    n = ctx.n
    mass = core.assemble_mass(ctx)
    kin = core.assemble_stiffness(ctx, 0.5)
    var = core.add_scaled(kin, core.assemble_harmonic(ctx, 0.5))
    x = torch.randn((a.k, n), dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    out = {"s": a.s, "n": n, "k": a.k}
    for name, op, cb in (("variable", var, 64), ("constant", mass, 0)):
        op.apply(x, out=y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            op.apply(x, out=y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        b = n * (16 * a.k + cb)
        out[name] = {"ms": ms, "gbs": b / ms / 1e6, "variable_op": op.variable}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
