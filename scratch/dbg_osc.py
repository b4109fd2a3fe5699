import numpy as np, torch, sys
sys.path.insert(0, '.')
from paro_b200 import configs, core
from paro_b200.driver import GpuBackend, ParoRun
from oracle import ref
w = configs.oscillator().scaled(16)
sp = ref.Space(w.subdivisions, w.lo, w.hi)
a = ref.Op.stiffness(sp, 0.5).add_scaled(ref.Op.wmass_harmonic(sp, 0.5)); b = ref.Op.mass(sp)
g = configs.guess_vectors(w)
lam0, U0, _, _ = ref.rayleigh_ritz(sp, g, a, b, w.K)
half_ref, sig = ref.shifted_source(a, b, sp, U0, lam0, 1e-8)
print('lam0', lam0[:3], 'sigma', sig)
be = GpuBackend(w)
run = ParoRun(w, be, guess=g)
print('gpu lam0', run.lambdas[:3])
sigma, iters = run.step3(be.form, 0)
h = run.half.cpu().numpy()
print('iters', iters, 'sigma', sigma)
print('half rel diff', [float(np.abs(h[c]-half_ref[c]).max()/np.abs(half_ref[c]).max()) for c in range(w.K)])
# conditioning of the half-step candidates
G = half_ref @ np.stack([b.matvec(x) for x in half_ref]).T
ev = np.linalg.eigvalsh(0.5*(G+G.T)); print('kappa(G)', ev.max()/ev.min())
try:
    lam_r, orb_r, d_r, _ = ref.rayleigh_ritz(sp, half_ref, a, b, w.n_orbitals); print('ref ritz ok', lam_r[:4], d_r)
except Exception as e: print('ref ritz FAIL', e)
from paro_b200 import _native as N
for mode in (0, 1):
    be.ctx.check(N.lib().paro_ctx_set_ritz_mode(be.ctx.h, mode))
    try:
        o = core.rayleigh_ritz(torch.as_tensor(half_ref, device='cuda'), be.form, be.mass, w.n_orbitals)
        print('gpu ritz mode', mode, o.lambdas[:4], o.gram_defect)
    except Exception as e: print('gpu ritz mode', mode, 'FAIL', e)
Qr, dropped = ref.b_orthonormalize(half_ref, b, 1e-8)
Q = core.b_orthonormalize(torch.as_tensor(half_ref, device='cuda'), be.mass, 1e-8).cpu().numpy()
print('k', Q.shape[0], Qr.shape[0], dropped)
print([float(np.abs(Q[j]-Qr[j]).max()/np.abs(Qr[j]).max()) for j in range(Q.shape[0])])
BQ = np.stack([b.matvec(q) for q in Q]); print('gram err', np.abs(Q @ BQ.T - np.eye(len(Q))).max())
ga2 = core.Operator.from_csr(be.ctx, *a.csr())
print('form vs from_csr var', be.form.variable, ga2.variable)
r1, c1, v1 = be.form.to_csr(); r2, c2, v2 = a.csr(); print('form csr equal', np.array_equal(v1, v2))
be.ctx.check(N.lib().paro_ctx_set_ritz_mode(be.ctx.h, 1))
for op, name in ((ga2, 'from_csr'), (be.form, 'form')):
    try:
        o = core.rayleigh_ritz(torch.as_tensor(half_ref, device='cuda'), op, be.mass, w.n_orbitals)
        print(name, o.lambdas[:4], o.gram_defect)
    except Exception as e: print(name, 'FAIL', e)
gm2 = core.Operator.from_csr(be.ctx, *b.csr())
print('mass const', be.mass.variable, gm2.variable, np.array_equal(be.mass.weights, gm2.weights))
try:
    o = core.rayleigh_ritz(torch.as_tensor(half_ref, device='cuda'), ga2, gm2, w.n_orbitals); print('both from_csr', o.lambdas[:4], o.gram_defect)
except Exception as e: print('both FAIL', e)
ctx2 = core.Context(0).grid(w.subdivisions, w.lo, w.hi)
ga3 = core.Operator.from_csr(ctx2, *a.csr()); gm3 = core.Operator.from_csr(ctx2, *b.csr())
ctx2.check(N.lib().paro_ctx_set_ritz_mode(ctx2.h, 1))
try:
    o = core.rayleigh_ritz(torch.as_tensor(half_ref, device='cuda'), ga3, gm3, w.n_orbitals); print('fresh ctx', o.lambdas[:4], o.gram_defect)
except Exception as e: print('fresh FAIL', e)
