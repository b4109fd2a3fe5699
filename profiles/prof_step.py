"""One outer iteration inside an NVTX range "prof" (for an ncu launch list):

  PARO_NO_GRAPH=1 ncu --nvtx --nvtx-include "prof/" --metrics gpu__time_duration.sum \\
      --clock-control none --csv --log-file launches.csv python profiles/prof_step.py
  python profiles/prof_step.py --summarize launches.csv
"""
import argparse
import collections
import csv
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def summarize(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    iN, iV = h.index("Kernel Name"), h.index("Metric Value")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[1:]:
        name = r[iN].split("(")[0].replace("paro_b200::<unnamed>::", "").replace("void ", "")
        tot[name] += float(r[iV]) * 1e-6
        cnt[name] += 1
    total = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'ms':>9s} {'share':>6s}")
    for k, v in tot.most_common(25):
        print(f"{k[:60]:60s} {cnt[k]:8d} {v:9.2f} {100 * v / total:5.1f}%")
    print(f"{'total':60s} {sum(cnt.values()):8d} {total:9.2f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cluster32")
    ap.add_argument("--summarize")
    ap.add_argument("--phase", default="step", choices=["step", "ritz"])
    a = ap.parse_args()
    if a.summarize:
        return summarize(a.summarize)
    import torch

    from paro_b200 import configs
    from paro_b200.driver import GpuBackend, ParoRun

    w = configs.get(a.workload)
    run = ParoRun(w, GpuBackend(w), timers=False)
    run.step(0)
    torch.cuda.synchronize()
    half = run.half[: run.k].clone()
    a_half = run.be.forms["half"]
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("prof")
    if a.phase == "ritz":
        run.s4.ritz(half, a_half, run.be.mass, w.n_orbitals, w.drop_tol, run.orb)
    else:
        run.step(1)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()


if __name__ == "__main__":
    main()
