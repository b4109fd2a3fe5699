"""Synthetic BASELINE workload generators (shared by both sides of every parity test)."""
import numpy as np
import pytest

from paro_b200 import configs


def test_splitmix64_reference_values():
    # SplitMix64 (Steele, Lea, Flood 2014) with seed 0: published first outputs
    r = configs.SplitMix64(0)
    assert [r.next() for _ in range(3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    a, b = configs.SplitMix64(7), configs.SplitMix64(7)
    np.testing.assert_array_equal(a.sym_array(1000), [b.sym() for _ in range(1000)])
    v = configs.SplitMix64(1).sym_array(100000)
    assert v.min() >= -1.0 and v.max() < 1.0 and abs(v.mean()) < 0.01


def test_workloads_match_baseline_json():
    h2, osc, wat, src, cl = (configs.get(n) for n in ("h2", "oscillator", "water", "source64", "cluster32"))
    assert (h2.subdivisions + 1, h2.K, h2.iterations, h2.lo, h2.hi) == (33, 1, 20, -10.0, 10.0)
    assert (osc.subdivisions + 1, osc.K, osc.lo, osc.hi) == (65, 10, -8.0, 8.0)
    assert (wat.subdivisions + 1, wat.K, wat.iterations, wat.lo) == (129, 5, 30, -12.0)
    assert np.allclose(np.linalg.norm(wat.positions[1]), 1.809) and np.allclose(np.linalg.norm(wat.positions[2]), 1.809)
    cosang = wat.positions[1] @ wat.positions[2] / 1.809**2
    assert np.degrees(np.arccos(cosang)) == pytest.approx(104.5)
    assert (src.subdivisions + 1, src.K, src.lo, len(src.charges)) == (257, 64, -16.0, 16)
    assert set(src.charges) <= {1.0, 2.0, 3.0, 4.0, 5.0, 6.0} and np.abs(src.positions).max() <= 10.0
    assert (cl.subdivisions + 1, cl.K, cl.n_electrons, cl.iterations, cl.lo) == (257, 76, 152, 15, -18.0)
    assert list(cl.charges).count(6.0) == 24 and list(cl.charges).count(1.0) == 8
    d = np.linalg.norm(cl.positions[:, None] - cl.positions[None], axis=-1) + 1e9 * np.eye(32)
    assert d.min() >= 2.0 and np.abs(cl.positions).max() <= 9.0


def test_guess_vectors():
    w = configs.get("water@s24")
    g = configs.guess_vectors(w)
    assert g.shape == (5, w.n) and np.isfinite(g).all()
    assert np.all((g == 0) | (np.abs(g) >= configs.GUESS_FLUSH))
    n = configs.get("oscillator@s8")
    gn = configs.guess_vectors(n)
    assert gn.shape == (10, n.n)
    np.testing.assert_array_equal(gn.reshape(-1), configs.SplitMix64(n.seed).sym_array(10 * n.n))
