"""GPU parity: Step 4 (rayleigh_ritz) and the dense pencil solve vs the reference."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda")


def _system(ref, s=12, lo=-6.0, hi=6.0):
    sp = ref.Space(s, lo, hi)
    ks = ref.KsSystem(sp, np.array([1.0, 1.0]), np.array([[0.7, 0, 0], [-0.7, 0, 0]]), 2)
    a0 = ks.op("kinetic").copy().add_scaled(ks.op("vext"))
    return sp, ks, a0, ks.op("mass")


def test_dense_sym_geneig_bit_exact(ref, gpu_ctx_factory):
    from paro_b200 import core

    ctx = gpu_ctx_factory(4, 0.0, 1.0)
    rng = np.random.default_rng(5)
    for m in (1, 2, 7, 12, 40, 76, 131):  # 131 > the block's thread count: strided rows
        X = rng.standard_normal((m, m))
        A = X + X.T
        Y = rng.standard_normal((m, m))
        B = Y @ Y.T + m * np.eye(m)
        v_ref, V_ref = ref.dense_sym_geneig(A, B)
        v, V = core.dense_sym_geneig(ctx, A, B)
        np.testing.assert_array_equal(v, v_ref)
        np.testing.assert_array_equal(V, V_ref)
    # known answers (test_linalg.cpp:143-283)
    v, _ = core.dense_sym_geneig(ctx, np.diag([2.0, 3.0]), np.eye(2))
    assert list(v) == [2.0, 3.0]
    v, _ = core.dense_sym_geneig(ctx, np.array([[2.0, 1.0], [1.0, 2.0]]), np.eye(2))
    np.testing.assert_allclose(v, [1.0, 3.0], atol=1e-14)
    from paro_b200 import PencilError

    with pytest.raises(PencilError):
        core.dense_sym_geneig(ctx, np.eye(2), np.diag([1.0, -1.0]))
    with pytest.raises(PencilError):  # check_symmetric (linalg.cpp:325-337)
        core.dense_sym_geneig(ctx, np.array([[1.0, 2.0], [2.0 + 1e-6, 1.0]]), np.eye(2))
    B40 = np.eye(40)
    B40[37, 37] = -1.0  # the pivot fails late: every earlier column is already final
    with pytest.raises(PencilError):
        core.dense_sym_geneig(ctx, np.eye(40), B40)


def test_rayleigh_ritz_matches_reference(ref, gpu_ctx_factory):
    from paro_b200 import core

    sp, ks, a0, mass = _system(ref)
    ctx = gpu_ctx_factory(sp.s, sp.lo, sp.hi)
    ga = core.Operator.from_csr(ctx, *a0.csr())
    gm = core.Operator.from_csr(ctx, *mass.csr())
    rng = np.random.default_rng(6)
    cands = rng.uniform(-1, 1, (6, sp.n))
    lam_ref, orb_ref, defect_ref, _ = ref.rayleigh_ritz(sp, cands, a0, mass, 6)
    out = core.rayleigh_ritz(_dev(cands), ga, gm, 6)
    lam = np.array(out.lambdas)
    np.testing.assert_allclose(lam, lam_ref, rtol=1e-11, atol=0)
    assert out.gram_defect <= 1e-8
    orb = out.orbitals.cpu().numpy()
    for j in range(6):
        np.testing.assert_allclose(orb[j], orb_ref[j], rtol=0, atol=1e-8 * np.abs(orb_ref[j]).max())


def test_rayleigh_ritz_gram_schmidt_path(ref, gpu_ctx_factory):
    """The explicit two-pass Gram-Schmidt path (used for near-dependent
    candidates) gives the same Ritz pairs; near-parallel candidates included."""
    from paro_b200 import _native as N
    from paro_b200 import core

    sp, ks, a0, mass = _system(ref)
    ctx = gpu_ctx_factory(sp.s, sp.lo, sp.hi)
    ga = core.Operator.from_csr(ctx, *a0.csr())
    gm = core.Operator.from_csr(ctx, *mass.csr())
    rng = np.random.default_rng(11)
    base = rng.uniform(-1, 1, (5, sp.n))
    cands = np.concatenate([base, base[:2] + 1e-7 * rng.uniform(-1, 1, (2, sp.n))])  # ratio ~1e-7
    lam_ref, orb_ref, _, _ = ref.rayleigh_ritz(sp, cands, a0, mass, 5)
    for mode in (0, 1):
        ctx.check(N.lib().paro_ctx_set_ritz_mode(ctx.h, mode))
        out = core.rayleigh_ritz(_dev(cands), ga, gm, 5)
        assert len(out.lambdas) == len(lam_ref)
        np.testing.assert_allclose(out.lambdas[:5], lam_ref[:5], rtol=1e-9)
        assert out.gram_defect <= 1e-8
    ctx.check(N.lib().paro_ctx_set_ritz_mode(ctx.h, 0))


def test_rayleigh_ritz_known_answers(ref, gpu_ctx_factory):
    """test_paro.cpp:156-218: invariant subspace, K=1 Rayleigh quotient, degenerate span."""
    from paro_b200 import DegenerateSpanError, core

    sp, ks, a0, mass = _system(ref, s=8)
    ctx = gpu_ctx_factory(sp.s, sp.lo, sp.hi)
    ga = core.Operator.from_csr(ctx, *a0.csr())
    gm = core.Operator.from_csr(ctx, *mass.csr())
    rng = np.random.default_rng(7)
    v = rng.standard_normal(sp.n)
    single = core.rayleigh_ritz(_dev(v[None]), ga, gm, 1, 1e-10)
    rq = v @ a0.matvec(v) / (v @ mass.matvec(v))
    assert abs(single.lambdas[0] - rq) <= 1e-10 * abs(rq)
    # exact Ritz vectors reproduce their values
    lam, orb, _, _ = ref.rayleigh_ritz(sp, rng.uniform(-1, 1, (4, sp.n)), a0, mass, 4)
    back = core.rayleigh_ritz(_dev(orb), ga, gm, 4, 1e-10)
    np.testing.assert_allclose(back.lambdas, lam, rtol=1e-10)
    e = np.zeros(sp.n)
    e[0] = 1.0
    with pytest.raises(DegenerateSpanError):
        core.rayleigh_ritz(_dev(np.stack([e, e])), ga, gm, 2, 1e-8)
    with pytest.raises(ref.RefDegenerateSpan):
        ref.rayleigh_ritz(sp, np.stack([e, e]), a0, mass, 2, 1e-8)


def test_fix_sign_device(ref, gpu_ctx_factory):
    from paro_b200 import core

    ctx = gpu_ctx_factory(8, 0.0, 1.0)
    rng = np.random.default_rng(8)
    V = rng.standard_normal((3, ctx.n))
    V[1, :5] = 0.0
    V[1, 5] = -1e-3
    V[2, 0] = 1e-14  # below 1e-12 * max: skipped
    V[2, 1] = -2.0
    got = core.fix_sign(ctx, _dev(V)).cpu().numpy()
    for j in range(3):
        np.testing.assert_array_equal(got[j], ref.fix_sign(V[j]))
