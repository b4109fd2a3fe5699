"""The run-configuration front end (paro_b200/runner.py) on CPU: the
reference's key = value format and validation (runconfig.cpp:133-240), the
molecule format (model.cpp:97-138), the device-path scope checks, and the
CLI exit codes (tools/main.cpp:46-67) for failures that need no GPU."""
import pytest

from paro_b200 import _native as N
from paro_b200 import runner as R


def test_builtin_defaults_and_overrides():
    c = R.parse_run_config("problem = molecule\nmolecule_file = h2.mol\nsubdivisions = 12  # comment\n"
                           "adaptive = off\naugment = 0\ntol_energy = 1e-8\n")
    assert (c.problem, c.box_lo, c.box_hi, c.subdivisions, c.augment, c.adaptive) == ("molecule", -8.0, 8.0, 12, 0,
                                                                                      False)
    assert c.tol_energy == 1e-8 and c.max_dofs == 30000
    h = R.parse_run_config("problem = hydrogen")
    assert (h.box_lo, h.box_hi, h.subdivisions, h.n_orbitals, h.augment, h.tol_energy) == (-10.0, 10.0, 4, 1, 2, 1e-7)


@pytest.mark.parametrize("text,msg", [
    ("problem = nope", "unknown problem"),
    ("subdivisions", "expected 'key = value'"),
    ("subdivisions = ", "empty key or value"),
    ("subdivisions = 4x", "expected an integer"),
    ("theta = 1.5", "theta must lie"),
    ("mixing_alpha = 0", "mixing_alpha must lie"),
    ("frobnicate = 1", "unknown key"),
    ("problem = molecule", "requires molecule_file"),
    ("adaptive = maybe", "expected on/off"),
    ("box_lo = 2\nbox_hi = 1", "box_hi must exceed"),
])
def test_config_errors(text, msg):
    with pytest.raises(N.ParseError, match=msg):
        R.parse_run_config(text)


def test_molecule_format():
    Z, Rr, ne = R.parse_molecule("# water-ish\n8 0 0 0\n1 1.4 1.1 0\n1 -1.4 1.1 0\n")
    assert list(Z) == [8.0, 1.0, 1.0] and ne == 10 and Rr.shape == (3, 3)
    assert R.parse_molecule("1 0.7 0 0\n1 -0.7 0 0\nelectrons 2\n")[2] == 2
    for bad in ("", "x 0 0 0", "1 0 0", "-1 0 0 0", "electrons x\n1 0 0 0"):
        with pytest.raises(N.ParseError):
            R.parse_molecule(bad)


def test_scope_checks():
    with pytest.raises(N.InvalidArgumentError, match="2-D"):
        R.workload_of(R.parse_run_config("problem = oscillator\nadaptive = off"))
    with pytest.raises(N.InvalidArgumentError, match="adaptive"):
        R.workload_of(R.parse_run_config("problem = hydrogen"))
    w = R.workload_of(R.parse_run_config("problem = hydrogen\nadaptive = off\nvext_smoothing = 0.5"))
    assert (w.kind, w.potential, w.eps, w.K, w.tol_energy) == ("linear", "softwell", 0.5, 3, 1e-7)
    w = R.workload_of(R.parse_run_config("problem = laplace-cube\nadaptive = off"))
    assert (w.potential, w.diffusion) == ("none", 1.0)


def test_cli_exit_codes(tmp_path, capsys):
    assert R.main([]) == 2
    bad = tmp_path / "bad.cfg"
    bad.write_text("problem = nope\n")
    assert R.main(["--config", str(bad)]) == 2
    assert R.main(["--config", str(tmp_path / "missing.cfg")]) == 2
    adaptive = tmp_path / "adaptive.cfg"
    adaptive.write_text("problem = hydrogen\n")
    assert R.main(["--config", str(adaptive)]) == 2
    err = capsys.readouterr().err
    assert "config error" in err and "adaptive" in err


def test_summary_and_mesh_dump(tmp_path):
    """summary.txt / mesh.txt formats (runner.cpp:107-121, mesh.cpp:198-217)."""
    from paro_b200 import artifacts

    assert artifacts.summary_line(True, 7, True, -1.2345678901234, None, 29791) == \
        "converged, 7 iterations, E_tot = -1.23456789012, 29791 DOFs"
    assert artifacts.summary_line(False, 3, False, None, 1.5, 343) == "failed, 3 iterations, lambda_1 = 1.5, 343 DOFs"
    p = tmp_path / "mesh.txt"
    artifacts.mesh_dump(p, 2, -1.0, 1.0)
    lines = p.read_text().splitlines()
    assert lines[0] == "3 27 48"
    assert lines[1] == "-1 -1 -1" and lines[2] == "0 -1 -1" and lines[27] == "1 1 1"
    assert lines[28] == "0 1 4 13 2 0"  # cell (0,0,0), perm (x, y, z): 0 -> +x 1 -> +y 4 -> +z 13
    assert len(lines) == 1 + 27 + 48
