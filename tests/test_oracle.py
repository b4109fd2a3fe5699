"""CPU tests of the oracle (no GPU): the compiled reference (oracle/_ref) and
the numpy restatement (oracle/port.py) are pinned against the reference's own
known-answer tests and against each other, and the committed golden fixtures
are reproduced."""
import json
import math
from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def port():
    from oracle import port as P

    return P


# ------------------------------------------- reference known answers -------

def test_lda_frozen_values(ref, port):
    """test_model.cpp:211-254."""
    v, e, cl = ref.lda(1.0, exchange_only=True)
    assert v == pytest.approx(-0.9847450218426965, rel=1e-12) and e == pytest.approx(0.75 * v, rel=1e-12)
    rho = 3.0 / (4.0 * math.pi)
    ec = ref.lda(rho)[1] - ref.lda(rho, True)[1]
    vc = ref.lda(rho)[0] - ref.lda(rho, True)[0]
    assert ec == pytest.approx(-0.05963206637891296, rel=1e-12)
    assert vc == pytest.approx(-0.06679442823281624, rel=1e-12)
    assert ref.lda(-0.5)[2] and ref.lda(-0.5)[0] == 0.0 and ref.lda(0.0)[:2] == (0.0, 0.0)
    pv, pe, pcl = port.lda_vxc(np.array([1.0, rho, -0.5, 0.0]))
    pvx, pex, _ = port.lda_vxc(np.array([1.0, rho]), exchange_only=True)
    assert pvx[0] == pytest.approx(-0.9847450218426965, rel=1e-12)
    assert pe[1] - pex[1] == pytest.approx(-0.05963206637891296, rel=1e-12)
    assert pv[1] - pvx[1] == pytest.approx(-0.06679442823281624, rel=1e-12)
    assert pcl[2] and pv[2] == 0.0 and pv[3] == 0.0


def test_cg_known_answers(ref, port):
    """test_linalg.cpp:67-141: identity, 2x2 SPD solution, NotSpd, IterationLimit."""
    A = ref.Op.from_csr([0, 2, 4], [0, 1, 0, 1], [4.0, 1.0, 1.0, 3.0])
    x, it, res, conv = ref.cg(A, [1.0, 2.0], tol=1e-14)
    np.testing.assert_allclose(x, [1 / 11, 7 / 11], rtol=1e-12)
    Ap = port.csr([0, 2, 4], [0, 1, 0, 1], [4.0, 1.0, 1.0, 3.0])
    xp = port.cg_solve(Ap, [1.0, 2.0], tol=1e-14)[0]
    np.testing.assert_allclose(xp, [1 / 11, 7 / 11], rtol=1e-12)
    eye = ref.Op.from_csr(np.arange(6), np.arange(5), np.ones(5))
    assert ref.cg(eye, [1, -2, 3, 0.5, 4])[1] <= 1
    neg = ref.Op.from_csr([0, 1, 2], [0, 1], [-5.0, 3.0])
    with pytest.raises(ref.RefNotSpd):
        ref.cg(neg, [1.0, 1.0])
    with pytest.raises(port.NotSpdError):
        port.cg_solve(port.csr([0, 1, 2], [0, 1], [-5.0, 3.0]), [1.0, 1.0])
    n = 50
    rows = [0]
    cols, vals = [], []
    for i in range(n):
        for j, v in ((i - 1, -1.0), (i, 2.0), (i + 1, -1.0)):
            if 0 <= j < n:
                cols.append(j)
                vals.append(v * 51 * 51)
        rows.append(len(cols))
    with pytest.raises(ref.RefIterationLimit) as e:
        ref.cg(ref.Op.from_csr(rows, cols, vals), np.ones(n), tol=1e-14, max_iter=2)
    assert e.value.residual > 0
    with pytest.raises(port.IterationLimitError):
        port.cg_solve(port.csr(rows, cols, vals), np.ones(n), tol=1e-14, max_iter=2)


def test_dense_pencil_known_answers(ref, port):
    """test_linalg.cpp:143-283."""
    for impl in (ref.dense_sym_geneig, port.dense_sym_geneig):
        v, _ = impl(np.diag([2.0, 3.0]), np.eye(2))
        np.testing.assert_allclose(v, [2.0, 3.0])
        v, _ = impl(np.array([[2.0, 1.0], [1.0, 2.0]]), np.eye(2))
        np.testing.assert_allclose(v, [1.0, 3.0], atol=1e-14)
        v, V = impl(np.diag([1.0, 4.0]), np.diag([1.0, 4.0]))
        np.testing.assert_allclose(v, [1.0, 1.0], atol=1e-14)
        np.testing.assert_allclose(V.T @ np.diag([1.0, 4.0]) @ V, np.eye(2), atol=1e-12)
    with pytest.raises(ref.RefPencilError):
        ref.dense_sym_geneig(np.eye(2), np.diag([1.0, -1.0]))
    with pytest.raises(port.PencilError):
        port.dense_sym_geneig(np.eye(2), np.diag([1.0, -1.0]))
    rng = np.random.default_rng(0)
    X = rng.standard_normal((12, 12))
    A = X + X.T
    Y = rng.standard_normal((12, 12))
    B = Y @ Y.T + 12 * np.eye(12)
    v1, V1 = ref.dense_sym_geneig(A, B)
    v2, V2 = port.dense_sym_geneig(A, B)
    np.testing.assert_allclose(v2, v1, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(np.abs(V2), np.abs(V1), atol=1e-9)
    assert np.max(np.abs(A @ V1 - B @ V1 * v1)) <= 50e-10 * np.abs(A).max()


def test_quadrature_rules(ref):
    """test_fem.cpp:89-96: weights sum to 1, exact to the declared degree."""
    for deg, lev, npts in ((2, -1, 4), (5, -1, 64), (5, 2, 256)):
        p, w = ref.quad_rule(3, deg, lev)
        assert len(w) == npts and w.sum() == pytest.approx(1.0, abs=1e-14)
        # int_T x^2 y over the reference tet (barycentric monomial) = 2!1!/(5+3)! * 3!
        val = np.sum(w * p[:, 1] ** 2 * p[:, 2]) / 6.0
        if deg >= 3:
            assert val == pytest.approx(2 * 1 * 6 / math.factorial(6) / 6.0, rel=1e-12)


def test_stencil_fixture_and_constants():
    """Mass and stiffness on the uniform Kuhn mesh are 15-point stencils:
    mass h^3{0.4, 0.05 axis, 1/30 face diagonal, 0.05 body diagonal};
    stiffness h{6, -1 axis, 0 diagonals}."""
    st = json.loads((GOLDEN / "stencils.json").read_text())
    g = st["s32_-10.0_10.0"]
    h = 0.625
    S = 31
    m = {int(k): v for k, v in g["mass"].items()}
    assert m[0] / h**3 == pytest.approx(0.4, rel=1e-14)
    assert m[1] / h**3 == pytest.approx(0.05, rel=1e-14)
    assert m[1 + S] / h**3 == pytest.approx(1 / 30, rel=1e-14)
    assert m[1 + S + S * S] / h**3 == pytest.approx(0.05, rel=1e-14)
    k = {int(k): v for k, v in g["poisson"].items()}
    assert k[0] / h == pytest.approx(6.0, rel=1e-14) and k[S * S] / h == pytest.approx(-1.0, rel=1e-14)
    assert k[1 + S] == 0.0 and k[1 + S + S * S] == 0.0
    assert len(m) == 15 and len(k) == 15


def test_port_matches_compiled_reference(ref, port):
    """The numpy restatement reproduces the compiled reference on one KS system."""
    sp = ref.Space(8, -4.0, 4.0)
    Z = np.array([1.0, 1.0])
    R = np.array([[0.7, 0, 0], [-0.7, 0, 0]])
    ks = ref.KsSystem(sp, Z, R, 2)
    ops = {k: port.csr(*ks.op(k).csr()) for k in ("mass", "kinetic", "vext", "poisson")}
    M = ops["mass"]
    A0 = ops["kinetic"] + ops["vext"]
    rng = np.random.default_rng(1)
    C = rng.uniform(-1, 1, (3, sp.n))
    a0 = ks.op("kinetic").copy().add_scaled(ks.op("vext"))
    lam_r, orb_r, _, _ = ref.rayleigh_ritz(sp, C, a0, ks.op("mass"), 3)
    lam_p, orb_p, _ = port.rayleigh_ritz(C, A0, M, 3)
    np.testing.assert_allclose(lam_p, lam_r, rtol=1e-11)
    np.testing.assert_allclose(orb_p, orb_r, atol=1e-9)
    half_r, sig_r = ref.shifted_source(a0, ks.op("mass"), sp, orb_r, lam_r, 1e-10)
    half_p, sig_p = port.shifted_source_step(A0, M, orb_r, lam_r, 1e-10)
    assert sig_p == sig_r
    np.testing.assert_allclose(half_p, half_r, atol=1e-8 * np.abs(half_r).max())
    rho_r, raw_r = ref.density(sp, orb_r[:1], [2.0])
    rho_p, raw_p = port.density(orb_r[:1], [2.0], 8, -4.0, 4.0)
    np.testing.assert_allclose(rho_p, rho_r, rtol=1e-12)
    vh_r = ref.hartree(sp, ks.op("poisson"), ks.op("mass"), rho_r)
    vh_p = port.hartree(ops["poisson"], M, rho_r)
    np.testing.assert_allclose(vh_p, vh_r, atol=1e-9 * np.abs(vh_r).max())
    e_r = ref.total_energy(sp, lam_r, 1, rho_r, vh_r, Z, R)
    e_p = port.total_energy(lam_r, [2.0], rho_r, vh_r, Z, R, 8, -4.0, 4.0)
    assert e_p == pytest.approx(e_r, rel=1e-12)
    assert port.norm_l2(rho_r, 8, -4.0, 4.0) == pytest.approx(ref.norm_l2(sp, rho_r), rel=1e-12)
    np.testing.assert_array_equal(port.fix_sign(-orb_r[0]), ref.fix_sign(-orb_r[0]))
    with pytest.raises(port.DegenerateSpanError):
        e = np.zeros(sp.n)
        e[0] = 1.0
        port.rayleigh_ritz(np.stack([e, e]), A0, M, 2)


@pytest.mark.parametrize("name", ["h2_s16", "oscillator_s16"])
def test_reference_reproduces_golden(ref, name):
    """Re-running the compiled reference reproduces the committed fixtures."""
    from paro_b200 import configs

    fx = json.loads((GOLDEN / f"{name}.json").read_text())
    w = configs.get(fx["workload"])
    sp = ref.Space(w.subdivisions, w.lo, w.hi)
    g = configs.guess_vectors(w)
    if fx["kind"] == "ks":
        ks = ref.KsSystem(sp, w.charges, w.positions, w.n_electrons, w.eps)
        loop = ref.KsLoop(ks, g, w.cg_tol_start, w.cg_tol, w.cg_tol_factor, w.cg_max_iter, w.mixing_alpha,
                          w.drop_tol)
    else:
        a = ref.Op.stiffness(sp, 0.5).add_scaled(ref.Op.wmass_harmonic(sp, 0.5))
        loop = ref.LinLoop(sp, a, ref.Op.mass(sp), g, w.n_orbitals, w.cg_tol_start, w.cg_tol, w.cg_tol_factor,
                           w.cg_max_iter, w.drop_tol)
    for row in fx["trace"]:
        r = loop.step(row["iter"] - 1)
        np.testing.assert_allclose(r["lambdas"][: w.n_orbitals], row["lambdas"], rtol=1e-12)
        if "e_tot" in row:
            assert r["e_tot"] == pytest.approx(row["e_tot"], rel=1e-12)


def test_port_estimator_matches_reference(ref):
    """Step-2 estimator (adapt.cpp:58-129): numpy restatement vs the compiled
    reference, Kohn-Sham and linear reactions, on a 6^3-cell mesh."""
    from oracle import port

    s, lo, hi = 6, -4.0, 4.0
    sp = ref.Space(s, lo, hi)
    rng = np.random.default_rng(11)
    U = rng.uniform(-1, 1, (2, sp.n))
    lam = [-0.4, 0.3]
    Z, R = np.array([1.0, 1.0]), np.array([[0.7, 0.1, 0.05], [-0.7, -0.1, 0.05]])
    ks = ref.KsSystem(sp, Z, R, 4)
    rho = rng.uniform(0, 0.5, sp.n)
    vh = rng.uniform(0, 1, sp.n)
    tot_r, eta_r = ks.eta_total(U, lam, rho, vh, with_eta=True)
    tot_p, eta_p = port.estimate_eta(U, lam, s, lo, hi, port.ks_reaction(Z, R, rho, vh, s))
    assert abs(tot_p - tot_r) <= 1e-10 * tot_r
    np.testing.assert_allclose(eta_p, eta_r, rtol=1e-10, atol=1e-12 * eta_r.max())
    harm = lambda X, b, t: 0.5 * (X * X).sum(-1)
    tot_r = ref.lin_eta_total(sp, U, lam, 0.5, "harmonic", c=0.5)
    tot_p, _ = port.estimate_eta(U, lam, s, lo, hi, harm)
    assert abs(tot_p - tot_r) <= 1e-10 * tot_r


def test_big_golden_fixtures_are_consistent():
    """The committed config-size rho vectors reproduce their trace's checksums
    (integral, L2 norm) and sketches, so the GPU parity test compares against
    what the reference produced (tests/golden/make_golden_big.py)."""
    import json
    import sys
    from pathlib import Path

    import numpy as np

    from oracle import port as P
    from paro_b200 import configs

    gold = Path(__file__).resolve().parent / "golden"
    sys.path.insert(0, str(gold))
    from make_golden_big import sketch_matrix, unshuffle

    for js in sorted(gold.glob("big_*.json")):
        fx = json.loads(js.read_text())
        w = configs.get(fx["workload"])
        vecs = np.load(js.with_name(js.stem + "_rho.npz"))
        S = sketch_matrix(w.n)
        rows = {r["iter"]: r for r in fx["trace"]}
        assert len(rows) == w.iterations
        for key in vecs.files:
            rho = unshuffle(vecs[key])
            r = rows[int(key[2:])]
            # numpy's pairwise sums vs the reference's sequential ones: 1e-12-level at 2M dofs
            assert P.integrate(rho, w.subdivisions, w.lo, w.hi) == pytest.approx(r["rho_integral"], rel=1e-10)
            assert P.norm_l2(rho, w.subdivisions, w.lo, w.hi) == pytest.approx(r["rho_l2"], rel=1e-10)
            np.testing.assert_allclose(S @ rho, r["rho_sketch"], rtol=1e-12, atol=1e-12)


def test_quad_tables_are_the_reference_rules(ref):
    """paro_b200/csrc/quad_tables.inc holds the reference's tetrahedral rules
    bit for bit (generated by oracle/gen_quad_tables.py)."""
    import re
    from pathlib import Path

    text = (Path(__file__).resolve().parents[1] / "paro_b200" / "csrc" / "quad_tables.inc").read_text()
    for name, degree, levels in (("kSimplex2", 2, -1), ("kSimplex5", 5, -1), ("kSubdivided5x2", 5, 2)):
        body = text.split(f"constexpr double {name}[")[1].split("};")[0]
        rows = [[float.fromhex(v) for v in r.split(",")] for r in re.findall(r"\{([^{}]+)\}", body)]
        pts, w = ref.quad_rule(3, degree, levels)
        assert len(rows) == len(w)
        for row, p, wt in zip(rows, pts, w):
            assert row[:4] == list(p) and row[4] == wt
