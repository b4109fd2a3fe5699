"""FP64 peak probe: cuBLAS DGEMM throughput on this B200 (the
FP64 tensor-core path, DMMA), square n^3 and the Step-4 tall-skinny shape,
best of R runs with CUDA events. Writes profiles/r02/fp64_peak.json.

  python profiles/fp64_peak.py
"""
import json
import sys
from pathlib import Path

import torch


def best(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return min(out)


def main():
    res = {"gpu": torch.cuda.get_device_name(0)}
    for n in (4096, 8192):
        x = torch.randn(n, n, dtype=torch.float64, device="cuda")
        y = torch.randn(n, n, dtype=torch.float64, device="cuda")
        ms = best(lambda: torch.mm(x, y))
        res[f"dgemm_{n}^3_tflops"] = 2 * n ** 3 / ms / 1e9
    # Step-4 shapes: Gram (76 x n)(n x 76) and rotation (n x 76)(76 x 76), n = 255^3
    n, k = 255 ** 3, 76
    u = torch.randn(k, n, dtype=torch.float64, device="cuda")
    c = torch.randn(k, k, dtype=torch.float64, device="cuda")
    ms = best(lambda: u @ u.T, 5)
    res["gram_76xn_ms"] = ms
    res["gram_76xn_tflops"] = 2 * n * k * k / ms / 1e9
    ms = best(lambda: c @ u, 5)
    res["rotate_nx76_ms"] = ms
    res["rotate_nx76_tflops"] = 2 * n * k * k / ms / 1e9
    res["rotate_nx76_gbs"] = 2 * 8 * n * k / ms / 1e6
    res["fp64_peak_tflops"] = max(res["dgemm_4096^3_tflops"], res["dgemm_8192^3_tflops"])
    out = Path(__file__).resolve().parent / "r02" / "fp64_peak.json"
    out.write_text(json.dumps(res, indent=1))
    print(json.dumps(res))


if __name__ == "__main__":
    sys.exit(main())
