import numpy as np, torch, sys
sys.path.insert(0, '.')
from paro_b200 import configs, core, _native as N
from oracle import ref
w = configs.oscillator().scaled(16)
sp = ref.Space(w.subdivisions, w.lo, w.hi)
a = ref.Op.stiffness(sp, 0.5).add_scaled(ref.Op.wmass_harmonic(sp, 0.5)); b = ref.Op.mass(sp)
g = configs.guess_vectors(w)
lam0, U0, _, _ = ref.rayleigh_ritz(sp, g, a, b, w.K)
half_ref, sig = ref.shifted_source(a, b, sp, U0, lam0, 1e-8)
H = torch.as_tensor(half_ref, device='cuda')
def trial(seq):
    ctx = core.Context(0).grid(w.subdivisions, w.lo, w.hi)
    ga = core.Operator.from_csr(ctx, *a.csr()); gm = core.Operator.from_csr(ctx, *b.csr())
    out = []
    for mode, K in seq:
        ctx.check(N.lib().paro_ctx_set_ritz_mode(ctx.h, mode))
        try:
            o = core.rayleigh_ritz(H[:K], ga, gm, min(K, w.n_orbitals)); out.append((mode, K, 'ok', round(o.gram_defect, 18)))
        except Exception as e: out.append((mode, K, 'FAIL', str(e)[-20:]))
    print(seq, out, flush=True)
trial([(1, 10), (1, 10)])
trial([(0, 10), (1, 10)])
trial([(1, 4), (1, 10)])
trial([(1, 10), (1, 4)])
trial([(0, 4), (1, 10)])
