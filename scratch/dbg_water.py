import numpy as np, torch, sys
sys.path.insert(0, '.')
from paro_b200 import configs, core
from paro_b200.driver import GpuBackend, ParoRun
from oracle import ref
w = configs.water().scaled(24)
be = GpuBackend(w)
g = configs.guess_vectors(w)
run = ParoRun(w, be, guess=g)
sp = ref.Space(w.subdivisions, w.lo, w.hi)
ks = ref.KsSystem(sp, w.charges, w.positions, w.n_electrons, w.eps)
loop = ref.KsLoop(ks, g)
for it in range(4):
    fin = lambda t: torch.isfinite(t).all().item()
    print('it', it, 'rho_in', fin(run.rho_in), 'orb', fin(run.orb[:run.k]), 'k', run.k, flush=True)
    try:
        tr = run.step(it)
        print('  gpu', tr.lambdas, tr.e_tot, tr.sigma, tr.cg_iterations, flush=True)
    except Exception as e:
        print('  gpu FAIL', e)
        vh = be.hartree(run.rho_in, out=run.vh)
        print('  vh', fin(vh), 'half', fin(run.half[:run.k]))
        r = run.rho_in.cpu().numpy(); print('  rho min/max', r.min(), r.max(), np.abs(r[r!=0]).min())
        break
    rr = loop.step(it)
    print('  ref', rr['lambdas'][:5], rr['e_tot'], rr['sigma'], flush=True)
