"""GPU parity of the general-CSR path: matrices that are not
the uniform Kuhn stencil (irregular sparsity, as after mesh adaptation) through
paro_csr_* against the compiled reference's SparseOperator / cg_solve /
source_solve_step on identical inputs."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda")


def _random_spd(n, seed, avg_deg=12, shift=0.05):
    """Symmetric irregular sparse matrix: weighted graph Laplacian of a random
    geometric-ish graph plus a positive diagonal; rows of varying length."""
    rng = np.random.default_rng(seed)
    pts = rng.uniform(0, 1, (n, 3))
    deg = rng.integers(2, 2 * avg_deg, n)
    rows_i, rows_j = [], []
    order = np.argsort(pts[:, 0])
    for a in range(n):
        # neighbours among points close in the sorted order (irregular, local)
        i = order[a]
        for b in range(1, int(deg[i]) // 2 + 1):
            if a + b < n:
                j = order[a + b]
                rows_i += [i, j]
                rows_j += [j, i]
    w = {}
    for i, j in zip(rows_i, rows_j):
        key = (min(i, j), max(i, j))
        if key not in w:
            w[key] = rng.uniform(0.1, 1.0)
    A = {}
    for (i, j), v in w.items():
        A[(i, j)] = A.get((i, j), 0.0) - v
        A[(j, i)] = A.get((j, i), 0.0) - v
        A[(i, i)] = A.get((i, i), 0.0) + v
        A[(j, j)] = A.get((j, j), 0.0) + v
    for i in range(n):
        A[(i, i)] = A.get((i, i), 0.0) + shift * (1.0 + rng.uniform())
    keys = sorted(A)
    rows = np.zeros(n + 1, np.int64)
    cols = np.array([k[1] for k in keys], np.uint32)
    vals = np.array([A[k] for k in keys], np.float64)
    for (i, _) in keys:
        rows[i + 1] += 1
    return np.cumsum(rows), cols, vals


def _ctx():
    from paro_b200 import core

    return core.Context(0)


def test_csr_apply_bit_exact(ref):
    from paro_b200 import core

    rows, cols, vals = _random_spd(3000, 1)
    ctx = _ctx()
    A = core.CsrOperator(ctx, rows, cols, vals)
    R = ref.Op.from_csr(rows, cols, vals)
    X = np.random.default_rng(2).standard_normal((5, 3000))
    Y = A.apply(_dev(X)).cpu().numpy()
    for c in range(5):
        np.testing.assert_array_equal(Y[c], R.matvec(X[c]))


@pytest.mark.parametrize("k", [1, 5, 40])
def test_csr_cg_matches_reference(ref, k):
    from paro_b200 import core

    rows, cols, vals = _random_spd(2500, 10 + k)
    ctx = _ctx()
    A = core.CsrOperator(ctx, rows, cols, vals)
    R = ref.Op.from_csr(rows, cols, vals)
    rng = np.random.default_rng(k)
    B = rng.standard_normal((k, 2500))
    X0 = rng.standard_normal((k, 2500)) * 0.01
    res = core.csr_cg_solve(A, _dev(B), _dev(X0), tol=1e-10, max_iter=20000)
    for c in range(k):
        x, it, r, conv = ref.cg(R, B[c], X0[c], tol=1e-10, max_iter=20000)
        assert abs(res.iterations[c] - it) <= 1, (c, res.iterations[c], it)
        np.testing.assert_allclose(res.x[c].cpu().numpy(), x, rtol=0, atol=1e-8 * np.abs(x).max())


def test_csr_cg_error_semantics(ref):
    from paro_b200 import IterationLimitError, InvalidArgumentError, NotSpdError, core

    rows, cols, vals = _random_spd(800, 5)
    ctx = _ctx()
    A = core.CsrOperator(ctx, rows, cols, vals)
    b = _dev(np.ones(800))
    with pytest.raises(IterationLimitError) as e:
        core.csr_cg_solve(A, b, tol=1e-14, max_iter=3)
    assert e.value.residual > 0
    r = core.csr_cg_solve(A, b, tol=1e-14, max_iter=3, throw_on_max_iter=False)
    assert r.iterations[0] == 3 and not r.converged[0]
    # zero right-hand side: x = 0, no iterations (linalg.cpp:158-162)
    r = core.csr_cg_solve(A, _dev(np.zeros(800)), _dev(np.ones(800)))
    assert r.iterations[0] == 0 and float(r.x.abs().max()) == 0.0
    # a non-positive diagonal entry -> NotSpd (linalg.cpp:165-167), like the reference
    v2 = vals.copy()
    d0 = np.flatnonzero((cols == 0) & (np.arange(len(cols)) < rows[1]))[0]
    v2[d0] = -1.0
    Aneg = core.CsrOperator(ctx, rows, cols, v2)
    with pytest.raises(NotSpdError):
        core.csr_cg_solve(Aneg, b)
    with pytest.raises(ref.RefNotSpd):
        ref.cg(ref.Op.from_csr(rows, cols, v2, symmetric=False), np.ones(800))
    # add_scaled needs identical structures (linalg.cpp:120-125)
    r2, c2, v3 = _random_spd(800, 6)
    with pytest.raises(InvalidArgumentError):
        A.add_scaled(core.CsrOperator(ctx, r2, c2, v3), 1.0)
    # malformed input is rejected at upload
    bad = cols.copy()
    bad[1], bad[0] = bad[0], bad[1]
    with pytest.raises(InvalidArgumentError):
        core.CsrOperator(ctx, rows, bad, vals)


def test_csr_add_scaled_and_source_step(ref):
    """source_solve_step on general CSR operators: (A + sigma B) u_half =
    (lambda + sigma) B u with x0 = u (paro.cpp:81-119), against the reference."""
    from paro_b200 import core

    n, k = 2000, 6
    rows, cols, vals = _random_spd(n, 21, shift=0.5)
    rng = np.random.default_rng(22)
    mvals = np.where(cols == np.repeat(np.arange(n), np.diff(rows)), 1.0, 0.0) + 0.01 * np.abs(vals)
    # B symmetric positive definite with A's structure (a mass-like matrix)
    ctx = _ctx()
    A = core.CsrOperator(ctx, rows, cols, vals)
    Bm = core.CsrOperator(ctx, rows, cols, mvals)
    Ra = ref.Op.from_csr(rows, cols, vals)
    Rb = ref.Op.from_csr(rows, cols, mvals)
    # add_scaled values equal the reference's
    A2 = core.CsrOperator(ctx, rows, cols, vals).add_scaled(Bm, 0.37)
    Ra2 = ref.Op.from_csr(rows, cols, vals).add_scaled(Rb, 0.37)
    X = rng.standard_normal((2, n))
    np.testing.assert_array_equal(A2.apply(_dev(X)).cpu().numpy()[0], Ra2.matvec(X[0]))
    U = rng.standard_normal((k, n))
    lam = list(np.linspace(0.1, 0.9, k))
    for sigma in (0.0, 0.8):
        half = core.csr_source_solve_step(A, Bm, _dev(U), lam, tol=1e-10, sigma=sigma).cpu().numpy()
        half_ref = ref.source_solve(Ra, Rb, U, lam, 1e-10, sigma=sigma)
        for c in range(k):
            np.testing.assert_allclose(half[c], half_ref[c], rtol=0, atol=1e-8 * np.abs(half_ref[c]).max())
