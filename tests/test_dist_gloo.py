"""The N > 1 orchestration on CPU: world sizes 2 and 4 over gloo, orbitals
sharded across ranks for Step 3, then transposed (all-to-all) into row slabs
for the sharded Step 4 (step4.py: Gram partials summed in rank order, fix_sign
pieces reduced, densities all-gathered) and back. The compute comes from the
oracle-backed PortBackend, so this checks the sharding / collective /
exception logic of driver.py and step4.py: every rank's trace must match the
1-rank trace to well inside the north-star bar (eigenvalues 1e-8 relative,
energy 1e-8 Ha); the only difference is the summation order of the Gram
partials."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

CASES = [("oscillator@s8", 3), ("water@s12", 2), ("h2@s8", 2), ("source64@s8", 3), ("cgs2:water@s12", 2)]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _trace(name, iters, dist=None):
    from paro_b200 import configs
    from paro_b200.driver import Dist, ParoRun
    from portbackend import PortBackend

    force = name.startswith("cgs2:")  # Step 4 through the blocked Gram-Schmidt path
    w = configs.get(name.split(":")[-1])
    d = dist or Dist()
    run = ParoRun(w, PortBackend(w), d, timers=False)
    run.s4.force_cgs2 = force
    out = []
    for i in range(iters):
        t = run.step(i)
        out.append((list(t.lambdas), t.e_tot, t.sigma, list(t.cg_iterations)))
        assert run.s4.info.cgs2 or not force
    c0, c1, _ = d.shard(run.k)  # this rank's columns hold every row
    return out, (c0, c1, run.orb[c0:c1].numpy().copy())


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


def _run_world(world, name, iters):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, iters, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return results


def _close(tr, single):
    assert len(tr) == len(single)
    for (lam, e, sig, its), (lam1, e1, sig1, its1) in zip(tr, single):
        np.testing.assert_allclose(lam, lam1, rtol=1e-10, atol=1e-12)
        if e1 is not None:
            assert abs(e - e1) <= 1e-10
        assert sig == pytest.approx(sig1, rel=1e-10, abs=1e-12)
        assert its == its1


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name,iters", CASES)
def test_ranks_match_one_rank(ref, name, iters, world):
    single, (_, _, orb1) = _trace(name, iters)
    results = _run_world(world, name, iters)
    ranks = sorted(results, key=lambda r: r[0])
    for rank, tr, _ in ranks:
        _close(tr, single)
        assert tr == ranks[0][1], f"rank {rank} disagrees with rank 0"  # identical K x K stage on every rank
    orb = np.concatenate([o for _, _, (_, _, o) in ranks])
    np.testing.assert_allclose(orb, orb1, rtol=0, atol=1e-9 * np.abs(orb1).max())


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
