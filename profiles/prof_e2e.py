"""End-to-end step with host-resident state: device step vs step_host vs the
bare copies (CUDA events on the current stream).

  python profiles/prof_e2e.py [--workload cluster32] [--chunks 2]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paro_b200 import configs  # noqa: E402
from paro_b200.driver import GpuBackend, ParoRun  # noqa: E402


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cluster32")
    ap.add_argument("--chunks", type=int, default=2)
    a = ap.parse_args()
    w = configs.get(a.workload)
    run = ParoRun(w, GpuBackend(w), timers=False)
    for i in range(2):
        run.step(i)
    K, n = run.k, run.be.n
    h_orb = torch.empty((K, n), dtype=torch.float64, pin_memory=True)
    h_rho = torch.empty((n,), dtype=torch.float64, pin_memory=True)
    h_orb.copy_(run.orb[:K])
    h_rho.copy_(run.rho_in)
    res = {}
    res["h2d_s"], _ = timed(lambda: run.orb[:K].copy_(h_orb, non_blocking=True))
    res["d2h_s"], _ = timed(lambda: h_orb.copy_(run.orb[:K], non_blocking=True))
    res["step_s"], _ = timed(lambda: run.step(2))
    h_orb.copy_(run.orb[:K])
    h_rho.copy_(run.rho_in)
    res["step_host_s"], _ = timed(lambda: run.step_host(3, h_orb, h_rho, chunks=a.chunks))
    res["step_host2_s"], _ = timed(lambda: run.step_host(4, h_orb, h_rho, chunks=a.chunks))
    res["serial_estimate_s"] = res["h2d_s"] + res["step_s"] + res["d2h_s"]
    # both directions at once (full-duplex PCIe)
    scratch = torch.empty_like(run.half[:K])
    cs = torch.cuda.Stream()

    def both():
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            h_orb.copy_(scratch, non_blocking=True)
        run.orb[:K].copy_(h_orb_b, non_blocking=True)
        torch.cuda.current_stream().wait_stream(cs)

    h_orb_b = torch.empty_like(h_orb, pin_memory=True)
    h_orb_b.copy_(h_orb)
    res["h2d_plus_d2h_concurrent_s"], _ = timed(both)
    h_orb.copy_(run.orb[:K])
    h_rho.copy_(run.rho_in)
    # timeline of one step_host: marks on the main and the copy stream
    run.timeline = []
    start = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record()
    run.step_host(5, h_orb, h_rho, chunks=a.chunks)
    end = torch.cuda.Event(enable_timing=True)
    end.record()
    torch.cuda.synchronize()
    res["timeline_ms"] = {lbl: round(start.elapsed_time(ev), 2) for lbl, ev in run.timeline}
    res["timeline_ms"]["returned"] = round(start.elapsed_time(end), 2)
    run.timeline = None
    print(json.dumps(res))


if __name__ == "__main__":
    main()
