"""Step-3 anatomy of one steady-state outer iteration: every batched_pcg call
(probe and batch) with its phases (PARO_PCG_TRACE=1, synchronising) and the
step's phase marks.

  python profiles/prof_step3.py [--workload cluster32] [--warmup 10]
"""
import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cluster32")
    ap.add_argument("--warmup", type=int, default=10)
    a = ap.parse_args()
    import torch

    from paro_b200 import configs
    from paro_b200.driver import GpuBackend, ParoRun

    w = configs.get(a.workload)
    run = ParoRun(w, GpuBackend(w), timers=False)
    for i in range(a.warmup):
        run.step(i)
    torch.cuda.synchronize()
    # untraced step with marks
    run.timeline = []
    s = torch.cuda.Event(enable_timing=True)
    s.record()
    t0 = time.perf_counter()
    tr = run.step(a.warmup)
    torch.cuda.synchronize()
    print(f"step {a.warmup}: wall {1e3 * (time.perf_counter() - t0):.1f} ms, probe {run._notspd_probe}, "
          f"attempts {run.last_attempts}, sigma {tr.sigma}")
    print({lbl: round(s.elapsed_time(ev), 2) for lbl, ev in run.timeline})
    run.timeline = None
    # wall time of every source_solve call (synchronised) against the step-3 span
    be = run.be
    orig = be.source_solve
    spans = []

    def timed_solve(*a_, **k_):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = orig(*a_, **k_)
        torch.cuda.synchronize()
        spans.append(round(1e3 * (time.perf_counter() - t), 2))
        return out

    be.source_solve = timed_solve
    run.timeline = []
    s = torch.cuda.Event(enable_timing=True)
    s.record()
    run.step(a.warmup + 1)
    torch.cuda.synchronize()
    print("source_solve calls (ms):", spans, {lbl: round(s.elapsed_time(ev), 2) for lbl, ev in run.timeline})
    run.timeline = None
    be.source_solve = orig
    os.environ["PARO_PCG_TRACE"] = "1"
    t0 = time.perf_counter()
    run.step(a.warmup + 2)
    torch.cuda.synchronize()
    print(f"traced step wall {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)


if __name__ == "__main__":
    main()
