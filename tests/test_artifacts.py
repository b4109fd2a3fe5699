"""Artifact formats of the reference runner (runner.cpp:15-19, 50-65, 97-101)."""
from paro_b200.artifacts import eigenvalues_txt, trace_csv
from paro_b200.driver import Trace


def _tr(i, lam, e):
    return Trace(i, lam, e, 0.1, 0.0, 0.0, [3], 0.25, 0.125, 0.5, eta_total=1.5e-3, t_meshgen=0.0625, dofs=29791)


def test_trace_csv_format():
    text = trace_csv([_tr(1, [-0.5, 0.25], -1.1), _tr(2, [-0.5000000001], None)], 2, kohn_sham=True)
    lines = text.splitlines()
    assert lines[0] == "iter,dofs,lambda_1,lambda_2,e_tot,eta_total,t_meshgen,t_source,t_project"
    assert lines[1] == "1,29791,-0.5,0.25,-1.1,0.0015,0.062500,0.250000,0.125000"
    assert lines[2] == "2,29791,-0.5000000001,nan,nan,0.0015,0.062500,0.250000,0.125000"
    lin = trace_csv([_tr(1, [1.5], None)], 1, kohn_sham=False).splitlines()
    assert lin[0] == "iter,dofs,lambda_1,eta_total,t_meshgen,t_source,t_project"


def test_eigenvalues_txt_format():
    assert eigenvalues_txt([1.5, 2.4999999999999996]) == "1 1.5\n2 2.5\n"
    assert eigenvalues_txt([-0.123456789012345678]) == "1 -0.123456789012346\n"
