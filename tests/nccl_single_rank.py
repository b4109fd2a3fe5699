"""Single-rank NCCL run of the multi-rank code path (TEST HELPER, GPU):
driver.Dist(collectives=True) sends every exchange of the orbital-sharded
Step 3 / row-slab Step 4 iteration through NCCL (all_to_all_single,
all_gather_into_tensor, all_reduce MIN / MAX on device tensors) although the
world has one rank; the trace must equal the shortcut run bit for bit.

  python tests/nccl_single_rank.py <workload> <iterations>   (prints OK)
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import torch.distributed as td

    from paro_b200 import configs
    from paro_b200.driver import Dist, GpuBackend, ParoRun

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29611")
    torch.cuda.set_device(0)
    td.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    name, iters = sys.argv[1], int(sys.argv[2])
    w = configs.get(name)
    out = []
    for coll in (False, True):
        d = Dist(collectives=coll)
        assert d.solo == (not coll)
        run = ParoRun(w, GpuBackend(w), d)
        tr = [run.step(i) for i in range(iters)]
        out.append(([t.lambdas for t in tr], [t.e_tot for t in tr], [t.sigma for t in tr],
                    [t.cg_iterations for t in tr], run.orb[: run.k].cpu()))
    a, b = out
    assert a[:4] == b[:4], (a[:4], b[:4])
    assert torch.equal(a[4], b[4])
    td.destroy_process_group()
    print("OK")


if __name__ == "__main__":
    main()
