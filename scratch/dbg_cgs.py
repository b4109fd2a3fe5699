import numpy as np, torch, sys
sys.path.insert(0, '.')
from paro_b200 import core
from oracle import ref
sp = ref.Space(8, -4.0, 4.0)
b = ref.Op.mass(sp)
ctx = core.Context(0).grid(8, -4.0, 4.0)
gb = core.Operator.from_csr(ctx, *b.csr())
rng = np.random.default_rng(3)
U = rng.uniform(-1, 1, (4, sp.n))
Qr, dropped = ref.b_orthonormalize(U, b, 1e-8)
Q = core.b_orthonormalize(torch.as_tensor(U, device='cuda'), gb, 1e-8).cpu().numpy()
print('k', Q.shape[0], Qr.shape[0], dropped)
for j in range(Q.shape[0]):
    print(j, np.abs(Q[j]-Qr[j]).max(), np.abs(Qr[j]).max())
BQ = np.stack([b.matvec(q) for q in Q]); print('gram', np.round(Q @ BQ.T, 10))
from paro_b200 import _native as N
a = ref.Op.stiffness(sp, 0.5).add_scaled(ref.Op.wmass_harmonic(sp, 0.5))
ga = core.Operator.from_csr(ctx, *a.csr())
lr, orr, dr, _ = ref.rayleigh_ritz(sp, U, a, b, 4)
print('ref', lr, dr)
for mode in (0, 1):
    ctx.check(N.lib().paro_ctx_set_ritz_mode(ctx.h, mode))
    try:
        o = core.rayleigh_ritz(torch.as_tensor(U, device='cuda'), ga, gb, 4)
        print('mode', mode, o.lambdas, o.gram_defect)
    except Exception as e:
        print('mode', mode, 'FAIL', e)
AQ = np.stack([a.matvec(q) for q in Q]); GA = Q @ AQ.T; GB = Q @ BQ.T
print('numpy pencil eig', np.linalg.eigvals(np.linalg.solve(GB, GA)).real.round(8))
