"""Timeline of back-to-back host-memory steps (ParoRun.step_host): blocking
calls against stream-ordered (pipelined) calls, marks on the compute and copy
streams relative to one start event.

  python profiles/prof_e2e_pipeline.py [--workload cluster32] [--steps 3]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paro_b200 import configs  # noqa: E402
from paro_b200.driver import GpuBackend, ParoRun  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cluster32")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=6)
    a = ap.parse_args()
    w = configs.get(a.workload)
    run = ParoRun(w, GpuBackend(w), timers=False)
    for i in range(a.warmup):
        run.step(i)
    K, n = run.k, run.be.n
    h_orb = torch.empty((K, n), dtype=torch.float64, pin_memory=True)
    h_rho = torch.empty((n,), dtype=torch.float64, pin_memory=True) if w.kind == "ks" else None
    h_orb.copy_(run.orb[:K])
    if h_rho is not None:
        h_rho.copy_(run.rho_in)
    torch.cuda.synchronize()
    it = a.warmup
    for pipelined in (True, False):
        run.host_join()
        torch.cuda.synchronize()
        run.step_host(it, h_orb, h_rho, pipelined=pipelined)  # prime the pipeline
        it += 1
        run.timeline = []
        start = torch.cuda.Event(enable_timing=True)
        start.record()
        for i in range(a.steps):
            run._mark(f"call{i}")
            run.step_host(it, h_orb, h_rho, pipelined=pipelined)
            it += 1
        run.host_join()
        end = torch.cuda.Event(enable_timing=True)
        end.record()
        torch.cuda.synchronize()
        print("pipelined" if pipelined else "blocking", f"{start.elapsed_time(end) / a.steps:.1f} ms per step")
        print([(lbl, round(start.elapsed_time(ev), 1)) for lbl, ev in run.timeline])
        run.timeline = None


if __name__ == "__main__":
    main()
