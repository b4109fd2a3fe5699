"""Time the K x K pencil solve (dense_sym_geneig on the device, the Jacobi
rotations of Step 4) on a near-diagonal 76 x 76 pencil like the ones a
converging outer iteration produces. python profiles/prof_pencil.py [--k 76]"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paro_b200 import core  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=76)
    a = ap.parse_args()
    rng = np.random.default_rng(1)
    k = a.k
    A = np.diag(np.sort(rng.uniform(-20, 2, k))) + 1e-3 * rng.standard_normal((k, k))
    A = 0.5 * (A + A.T)
    B = np.eye(k) + 1e-6 * rng.standard_normal((k, k))
    B = 0.5 * (B + B.T)
    ctx = core.Context(0).grid(8, -1.0, 1.0)
    core.dense_sym_geneig(ctx, A, B)
    t = time.perf_counter()
    for _ in range(5):
        vals, X = core.dense_sym_geneig(ctx, A, B)
    print(f"k={k} {1e3 * (time.perf_counter() - t) / 5:.2f} ms per pencil, lambda_1 {vals[0]:.12f}")


if __name__ == "__main__":
    main()
