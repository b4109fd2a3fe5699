import numpy as np, torch, sys
sys.path.insert(0, '.')
from paro_b200 import core
from oracle import ref
sp = ref.Space(16, -8.0, 8.0)
a = ref.Op.stiffness(sp, 0.5).add_scaled(ref.Op.wmass_harmonic(sp, 0.5)); b = ref.Op.mass(sp)
rng = np.random.default_rng(0)
for trial in range(2):
    ctx = core.Context(0).grid(16, -8.0, 8.0)
    ga = core.Operator.from_csr(ctx, *a.csr()); gb = core.Operator.from_csr(ctx, *b.csr())
    for K in (10, 1, 2, 3, 4, 5, 8, 9, 12, 16, 17):
        X = rng.standard_normal((K, sp.n))
        for op, r in ((ga, a), (gb, b)):
            Y = op.apply(torch.as_tensor(X, device='cuda')).cpu().numpy()
            bad = [c for c in range(K) if not np.array_equal(Y[c], r.matvec(X[c]))]
            if bad: print('trial', trial, 'K', K, 'var' if op.variable else 'const', 'bad cols', bad, flush=True)
print('done')
