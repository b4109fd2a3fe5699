"""Time the Step-4 rotation Z = X C (rotate_kernel) at the bench shape:
n = 255^3 rows, 76 x 76, dense and triangular. python profiles/prof_rotate.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paro_b200 import core  # noqa: E402


def main():
    ctx = core.Context(0).grid(256, -18.0, 18.0)
    n, k = ctx.n, 76
    X = torch.randn((k, n), dtype=torch.float64, device="cuda")
    Z = torch.empty_like(X)
    C = torch.triu(torch.randn((k, k), dtype=torch.float64, device="cuda")).T.contiguous().reshape(-1)
    for mode, name in ((0, "dense"), (2, "triangular")):
        core.rotate(ctx, X, k, C, k, k, Z, 0, n, mode)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(5):
            core.rotate(ctx, X, k, C, k, k, Z, 0, n, mode)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        fl = 2.0 * n * k * k * (1.0 if mode == 0 else 109.0 / 190.0)
        print(f"{name}: {ms:.2f} ms, {fl / ms / 1e9:.1f} TF/s, {16.0 * n * k / ms / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
