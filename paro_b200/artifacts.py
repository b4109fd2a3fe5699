"""Run artifacts in the reference's formats, so a run of
this driver can be diffed against `paro --config` output:

  trace.csv        write_trace_csv   proj/src/runner.cpp:50-65
                   header iter,dofs,lambda_1..N[,e_tot],eta_total,t_meshgen,t_source,t_project;
                   values "%.12g", times "%.6f", missing values "nan"
  eigenvalues.txt  proj/src/runner.cpp:97-101   "<i> <lambda_i %.15g>" per line
  mesh.txt         Mesh::dump proj/src/mesh.cpp:198-217 of the uniform Kuhn box
                   mesh (C ABI paro_mesh_dump, streamed by the native library)
  summary.txt      proj/src/runner.cpp:107-121  "<converged|failed>, <n> iterations,
                   E_tot = %.12g | lambda_1 = %.12g, <dofs> DOFs"
"""
from __future__ import annotations

import math
from pathlib import Path


def _fmt(v, spec="%.12g") -> str:
    """fmt (runner.cpp:15-19): C printf formatting of a double."""
    if v is None:
        return "nan"
    v = float(v)
    if math.isnan(v):
        return "nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return spec % v


def trace_csv(traces, n_lambdas: int, kohn_sham: bool) -> str:
    head = "iter,dofs" + "".join(f",lambda_{i}" for i in range(1, n_lambdas + 1))
    if kohn_sham:
        head += ",e_tot"
    lines = [head + ",eta_total,t_meshgen,t_source,t_project"]
    for tr in traces:
        row = [str(tr.iter), str(tr.dofs)]
        row += [_fmt(tr.lambdas[i]) if i < len(tr.lambdas) else "nan" for i in range(n_lambdas)]
        if kohn_sham:
            row.append(_fmt(tr.e_tot))
        # eta_total is 0 when Step 2 did not run (the reference always runs it)
        row.append(_fmt(tr.eta_total if tr.eta_total is not None else 0.0))
        row += [_fmt(tr.t_meshgen, "%.6f"), _fmt(tr.t_source, "%.6f"), _fmt(tr.t_project, "%.6f")]
        lines.append(",".join(row))
    return "\n".join(lines) + "\n"


def eigenvalues_txt(lambdas) -> str:
    return "".join(f"{i + 1} {_fmt(v, '%.15g')}\n" for i, v in enumerate(lambdas))


def summary_line(converged: bool, iterations: int, kohn_sham: bool, e_tot, lambda_1, dofs: int) -> str:
    """run_experiment's summary (runner.cpp:107-116)."""
    s = f"{'converged' if converged else 'failed'}, {iterations} iterations, "
    s += f"E_tot = {_fmt(e_tot or 0.0)}" if kohn_sham else f"lambda_1 = {_fmt(lambda_1 or 0.0)}"
    return s + f", {dofs} DOFs"


def mesh_dump(path, subdivisions: int, lo: float, hi: float) -> None:
    """mesh.txt: Mesh::dump of create_box_mesh([lo, hi]^3, subdivisions)."""
    from . import _native as N

    st = N.lib().paro_mesh_dump(int(subdivisions), float(lo), float(hi), str(path).encode())
    if st != 0:
        raise N.ERRORS.get(st, N.Error)((N.lib().paro_ctx_last_error(None) or b"").decode())


def write_run(out_dir, traces, final_lambdas, n_lambdas: int, kohn_sham: bool, *, converged: bool | None = None,
              mesh=None) -> str | None:
    """The run_experiment artifacts (runner.cpp:79-121) under out_dir:
    trace.csv + eigenvalues.txt, and with mesh = (subdivisions, lo, hi)
    mesh.txt, with `converged` given summary.txt. Returns the summary line."""
    d = Path(out_dir)
    d.mkdir(parents=True, exist_ok=True)
    (d / "trace.csv").write_text(trace_csv(traces, n_lambdas, kohn_sham))
    (d / "eigenvalues.txt").write_text(eigenvalues_txt(final_lambdas))
    if mesh is not None:
        mesh_dump(d / "mesh.txt", *mesh)
    if converged is None:
        return None
    last = traces[-1] if traces else None
    line = summary_line(converged, len(traces), kohn_sham, last.e_tot if last else None,
                        final_lambdas[0] if len(final_lambdas) else None, last.dofs if last else 0)
    (d / "summary.txt").write_text(line + "\n")
    return line
