"""GPU parity: device operator assembly and nodal fields vs the reference."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

H2_Z = np.array([1.0, 1.0])
H2_R = np.array([[0.7, 0.0, 0.0], [-0.7, 0.0, 0.0]])


def _dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda")


def _same_csr(g, r, rtol=0.0):
    gr, gc, gv = g.to_csr()
    rr, rc, rv = r.csr()
    np.testing.assert_array_equal(gr, rr)
    np.testing.assert_array_equal(gc, rc)
    if rtol == 0.0:
        np.testing.assert_array_equal(gv, rv)
    else:
        np.testing.assert_allclose(gv, rv, rtol=rtol, atol=rtol * np.abs(rv).max())


@pytest.mark.parametrize("s,lo,hi", [(8, -4.0, 4.0), (12, -6.0, 6.0), (10, -5.0, 5.0)])
def test_static_operators_bit_exact(ref, gpu_ctx_factory, s, lo, hi):
    from paro_b200 import core

    sp = ref.Space(s, lo, hi)
    ks = ref.KsSystem(sp, H2_Z, H2_R, 2)
    ctx = gpu_ctx_factory(s, lo, hi)
    _same_csr(core.assemble_mass(ctx), ks.op("mass"))
    _same_csr(core.assemble_stiffness(ctx, 0.5), ks.op("kinetic"))
    _same_csr(core.assemble_stiffness(ctx, 1.0), ks.op("poisson"))
    # bare Coulomb with the singular-quadrature policy (64/256-point rules)
    _same_csr(core.assemble_vext(ctx, H2_Z, H2_R, 0.0), ks.op("vext"))


def test_uniform_operators_become_constant(gpu_ctx_factory):
    from paro_b200 import core

    ctx = gpu_ctx_factory(32, -10.0, 10.0)  # h = 0.625, exact coordinates
    m = core.assemble_mass(ctx)
    k = core.assemble_stiffness(ctx, 1.0)
    assert not m.variable and not k.variable
    h = 0.625
    np.testing.assert_allclose(m.weights / h**3, [0.4, 0.05, 0.05, 1 / 30, 0.05, 1 / 30, 1 / 30, 0.05], rtol=1e-14)
    np.testing.assert_allclose(k.weights / h, [6, -1, -1, 0, -1, 0, 0, 0], atol=1e-14)


def test_other_potentials(ref, gpu_ctx_factory):
    from paro_b200 import core

    sp = ref.Space(10, -5.0, 5.0)
    ctx = gpu_ctx_factory(10, -5.0, 5.0)
    Z = np.array([3.0, 1.0, 2.0])
    R = np.array([[0.3, -1.1, 0.7], [1.9, 0.2, -0.4], [-2.2, 1.0, 1.5]])
    _same_csr(core.assemble_vext(ctx, Z, R, 0.0), ref.Op.wmass_coulomb(sp, Z, R, 0.0))
    eps = np.sqrt(0.1)
    _same_csr(core.assemble_vext(ctx, Z, R, eps), ref.Op.wmass_coulomb(sp, Z, R, eps))
    _same_csr(core.assemble_harmonic(ctx, 0.5), ref.Op.wmass_harmonic(sp, 0.5))
    # linear form: stiffness + weighted mass (paro.cpp:270-274)
    a = core.add_scaled(core.assemble_stiffness(ctx, 0.5), core.assemble_harmonic(ctx, 0.5))
    b = ref.Op.stiffness(sp, 0.5).add_scaled(ref.Op.wmass_harmonic(sp, 0.5))
    _same_csr(a, b)


def test_ks_form_and_fields(ref, gpu_ctx_factory):
    from paro_b200 import core

    sp = ref.Space(12, -6.0, 6.0)
    ks = ref.KsSystem(sp, H2_Z, H2_R, 2)
    ctx = gpu_ctx_factory(12, -6.0, 6.0)
    rng = np.random.default_rng(9)
    U = rng.uniform(-1, 1, (3, sp.n))
    occ = [2.0, 2.0]
    rho_ref, raw_ref = ref.density(sp, U[:2], occ)
    rho, raw = core.density_from_orbitals(ctx, _dev(U), occ)
    np.testing.assert_allclose(rho.cpu().numpy(), rho_ref, rtol=1e-13)
    assert abs(raw - raw_ref) <= 1e-12 * abs(raw_ref)
    assert abs(core.integrate(ctx, rho) - ref.integrate(sp, rho_ref)) <= 1e-12 * 4
    vh_ref = ref.hartree(sp, ks.op("poisson"), ks.op("mass"), rho_ref, 1e-11)
    vh = _dev(vh_ref)
    kin = core.assemble_stiffness(ctx, 0.5)
    vext = core.assemble_vext(ctx, H2_Z, H2_R, 0.0)
    form, clamped = core.ks_form_matrix(kin, vext, _dev(rho_ref), vh)
    form_ref, clamped_ref = ks.form(rho_ref, vh_ref)
    assert clamped == clamped_ref
    _same_csr(form, form_ref, rtol=1e-14)
    # energy, norms, mixing
    lam = [-0.6, -0.2, 0.1]
    e_ref = ref.total_energy(sp, lam, 2, rho_ref, vh_ref, H2_Z, H2_R)
    e = core.total_energy(ctx, lam, occ, _dev(rho_ref), vh, H2_Z, H2_R)
    assert abs(e - e_ref) <= 1e-12 * abs(e_ref)
    r2 = np.abs(rho_ref[::-1]).copy()
    mixed = core.mix_density(ctx, _dev(rho_ref), _dev(r2), 0.3).cpu().numpy()
    np.testing.assert_array_equal(mixed, ref.mix(sp, rho_ref, r2, 0.3))
    assert abs(core.norm_l2(ctx, _dev(r2)) - ref.norm_l2(sp, r2)) <= 1e-13 * ref.norm_l2(sp, r2)


@pytest.mark.parametrize("s,lo,hi,uniform", [(12, -6.0, 6.0, True), (16, -10.0, 10.0, True), (10, -7.0, 7.0, False)])
def test_nodal_sums_match_element_sums(ref, gpu_ctx_factory, s, lo, hi, uniform):
    """integrate / norm_l2 / integrate_product (fem.cpp:419-448, model.cpp:306-327):
    once the context knows the grid's mass as one constant stencil
    (exact-binary spacings) they run as nodal sums f' M g / (int phi) sum f;
    both forms against the reference's element loops, and against each other
    (a second context that never assembled the mass stays on the element loop)."""
    from paro_b200 import core

    sp = ref.Space(s, lo, hi)
    ctx_el = gpu_ctx_factory(s, lo, hi)          # element loops
    ctx = gpu_ctx_factory(s, lo, hi)
    m = core.assemble_mass(ctx)                  # records the stencil
    assert m.variable is (not uniform)
    rng = np.random.default_rng(s)
    f = rng.uniform(0.0, 2.0, sp.n)
    g = rng.standard_normal(sp.n)
    fd, gd = _dev(f), _dev(g)
    mass = ref.Op.mass(sp)
    for c in (ctx, ctx_el):
        i_ref = ref.integrate(sp, f)
        assert abs(core.integrate(c, fd) - i_ref) <= 1e-13 * abs(i_ref)
        n_ref = ref.norm_l2(sp, g)
        assert abs(core.norm_l2(c, gd) - n_ref) <= 1e-13 * n_ref
        p_ref = float(f @ mass.matvec(g))        # integrate_product == f' M g on Dirichlet functions
        scale = float(np.abs(f) @ mass.matvec(np.abs(g)))
        assert abs(core.integrate_product(c, fd, gd) - p_ref) <= 1e-13 * scale


@pytest.mark.parametrize("s,parts", [(12, 3), (17, 4), (9, 8)])
def test_ks_form_planes_union_is_the_full_form(ref, gpu_ctx_factory, s, parts):
    """paro_ks_form_planes: the KS form assembled slab by slab (the row-sharded
    run: each rank its planes, then an all-gather of the 8 coefficient slots)
    is the full form bit for bit, the slabs' clamp counts add up to the full
    count (a density with negative lobes, so the count is not zero), and a slab
    call leaves the other planes' coefficients untouched."""
    from paro_b200 import core
    from paro_b200.step4 import RowSlab

    sp = ref.Space(s, -6.0, 6.0)
    ctx = gpu_ctx_factory(s, -6.0, 6.0)
    rng = np.random.default_rng(s)
    rho = _dev(rng.uniform(-0.05, 1.0, sp.n))          # some quadrature points interpolate below zero
    vh = _dev(rng.standard_normal(sp.n))
    kin = core.assemble_stiffness(ctx, 0.5)
    vext = core.assemble_vext(ctx, H2_Z, H2_R, 0.0)
    full, cl_full = core.ks_form_matrix(kin, vext, rho, vh)
    assert cl_full > 0
    S = ctx.S
    out = core.Operator.variable_empty(ctx)
    coef = out.coefficients()
    coef.fill_(123.0)
    total = 0
    for r in range(parts):
        sl = RowSlab.split(S, parts, r)
        total += core.ks_form_planes(kin, vext, rho, vh, sl.z0, sl.z1, out)
        assert torch.equal(coef[:, sl.r0:sl.r1], full.coefficients()[:, sl.r0:sl.r1])
        if sl.r1 < ctx.n:
            assert bool((coef[:, sl.r1:] == 123.0).all())   # later slabs not written yet
    assert torch.equal(coef, full.coefficients())
    assert total == cl_full
    # an empty slab (more ranks than planes) is a no-op
    assert core.ks_form_planes(kin, vext, rho, vh, 3, 3, out) == 0
    assert torch.equal(coef, full.coefficients())


def test_energy_xc_layers_add_up(ref, gpu_ctx_factory):
    """The XC term of total_energy summed over cell-layer slabs (the sharded
    run) against the one-call form: equal to rounding, and with the full layer
    range bit for bit; total_energy_with_xc with that term is total_energy."""
    from paro_b200 import core
    from paro_b200.step4 import RowSlab

    s = 14
    sp = ref.Space(s, -6.0, 6.0)
    ctx = gpu_ctx_factory(s, -6.0, 6.0)
    rng = np.random.default_rng(3)
    rho = _dev(rng.uniform(0.0, 1.0, sp.n))
    vh = _dev(rng.standard_normal(sp.n))
    lam, occ = [-0.7, -0.3], [2.0, 2.0]
    full = core.energy_xc_layers(ctx, rho, 0, s)
    S = ctx.S
    for parts in (2, 5):
        tot = 0.0
        for r in range(parts):
            sl = RowSlab.split(S, parts, r)
            tot += core.energy_xc_layers(ctx, rho, sl.z0, sl.z1 + 1 if sl.z1 == S else sl.z1)
        assert abs(tot - full) <= 1e-13 * abs(full)
    assert core.energy_xc_layers(ctx, rho, 4, 4) == 0.0
    e = core.total_energy(ctx, lam, occ, rho, vh, H2_Z, H2_R)
    assert core.total_energy_with_xc(ctx, lam, occ, rho, vh, H2_Z, H2_R, full) == e
    e_ref = ref.total_energy(sp, lam, 2, rho.cpu().numpy(), vh.cpu().numpy(), H2_Z, H2_R)
    assert abs(e - e_ref) <= 1e-12 * abs(e_ref)
