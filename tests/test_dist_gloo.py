"""The N > 1 orchestration on CPU: world_size 2 over gloo, orbitals sharded
across ranks, half-step orbitals all-gathered, Step 4 and the potential
rebuild replicated. The compute comes from the oracle-backed PortBackend, so
this checks the sharding / collective / exception logic of driver.py: the
2-rank trace must be identical to the 1-rank trace."""
import os
import socket

import pytest
import torch.multiprocessing as mp

CASES = [("oscillator@s8", 3), ("water@s12", 2), ("h2@s8", 2), ("source64@s8", 3)]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _trace(name, iters, dist=None):
    from paro_b200 import configs
    from paro_b200.driver import Dist, ParoRun
    from portbackend import PortBackend

    w = configs.get(name)
    run = ParoRun(w, PortBackend(w), dist or Dist(), timers=False)
    out = []
    for i in range(iters):
        t = run.step(i)
        out.append((list(t.lambdas), t.e_tot, t.sigma, list(t.cg_iterations)))
    return out, run.orb[: run.k].numpy().copy()


def _worker(rank, world, port, name, iters, q):
    import torch.distributed as td

    from paro_b200.driver import Dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr, orb = _trace(name, iters, Dist())
        q.put((rank, tr, orb))
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("name,iters", CASES)
def test_two_ranks_match_one_rank(ref, name, iters):
    single, orb1 = _trace(name, iters)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, iters, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, tr, orb in results:
        assert tr == single, f"rank {rank} trace differs from the single-rank run"
        assert (orb == orb1).all()


def test_shard_and_outcome_logic():
    from paro_b200.driver import ITER_LIMIT, NOT_SPD, OK, Dist, step3_outcome

    d = Dist()
    d.world, d.rank = 3, 1
    assert d.shard(76) == (26, 51, [26, 25, 25])
    d.rank = 2
    assert d.shard(2)[:2] == (2, 2)
    # a failure inside the retry escapes first; otherwise the first failed first attempt
    assert step3_outcome([OK, NOT_SPD, ITER_LIMIT], [OK, NOT_SPD, ITER_LIMIT]) == (ITER_LIMIT, 2)
    assert step3_outcome([OK, NOT_SPD, ITER_LIMIT], [OK, NOT_SPD, OK]) == (NOT_SPD, 1)
    assert step3_outcome([ITER_LIMIT, OK], [OK, OK]) == (OK, -1)


def test_notspd_probe_keeps_the_trace():
    """source64 escalates sigma every outer iteration (the first Step-3
    attempt meets NotSpd); from the second iteration on the probe decides that
    attempt from the previously failing orbital alone, and a probe that
    passes hands its solution to the batch. The trace (lambdas,
    sigma, CG iterations, orbitals) must equal the full-batch run's."""
    from paro_b200 import configs
    from paro_b200.driver import Dist, ParoRun
    from portbackend import PortBackend

    w = configs.get("source64@s8")

    def run(probe):
        r = ParoRun(w, PortBackend(w), Dist(), timers=False)
        if not probe:
            r._probe = lambda *a, **k: (False, {})
        out = [r.step(i) for i in range(3)]
        return r, [(list(t.lambdas), t.sigma, list(t.cg_iterations)) for t in out]

    rp, tp = run(True)
    rf, tf = run(False)
    assert rp.probe_hits >= 1 and rf.probe_hits == 0
    assert tp == tf
    assert (rp.orb[: rp.k].numpy() == rf.orb[: rf.k].numpy()).all()
