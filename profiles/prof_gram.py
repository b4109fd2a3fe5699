"""Step-4 Gram (upper-triangle DMMA) and rotation at the bench shape: CUDA-event times.

  python profiles/prof_gram.py [--s 256] [--k 76] [--reps 10]
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
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    ctx = core.Context(0).grid(a.s, -18.0, 18.0)
    n, k = ctx.n, a.k
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn((k, n), dtype=torch.float64, device="cuda", generator=g)
    Y = torch.randn((k, n), dtype=torch.float64, device="cuda", generator=g)
    Z = torch.empty_like(X)
    Cm = torch.randn(k * k, dtype=torch.float64, device="cuda", generator=g)
    out = {}
    for name, fn in (("gram_sym", lambda: core.gram_sym(ctx, X, Y, k, 0, n)),
                     ("rotate", lambda: core.rotate(ctx, X, k, Cm, k, k, Z, 0, n, 0))):
        fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out[name + "_ms"] = e0.elapsed_time(e1) / a.reps
    out["gram_tflops"] = k * (k + 1) * n / (out["gram_sym_ms"] * 1e-3) / 1e12
    out["rotate_tflops"] = 2.0 * n * k * k / (out["rotate_ms"] * 1e-3) / 1e12
    print(json.dumps(out))


if __name__ == "__main__":
    main()
