"""`paro --config` for the fixed-mesh device path: the reference's run
configuration format, run_experiment and exit codes, on the B200 driver.

  python -m paro_b200 --config run.cfg [-o out_dir] [-w workers]

Mirrors (proj/):
  parse_run_config   src/runconfig.cpp:133-240  key = value lines, '#' comments,
                     builtin problem defaults (:39-88), the same validation
  parse_molecule     src/model.cpp:97-138       "Z x y z" lines, optional "electrons N"
  run_experiment     src/runner.cpp:67-121      trace.csv, eigenvalues.txt, mesh.txt,
                     summary.txt; paro_kohn_sham / paro_linear with their
                     degenerate-span restarts (src/paro.cpp:377-392, 646-662)
                     and stop tests (driver.StopTests)
  main               tools/main.cpp:46-67       exit codes: 0 converged, 1 not
                     converged, 2 config / invalid argument, 3 solver (NotSpd,
                     IterationLimit), 4 capacity, 5 SCF divergence, 6 other

Scope: the device path is the fixed-mesh outer iteration on 3-D boxes, so a
configuration must set `adaptive = off`; the 2-D builtins (laplace-square,
oscillator) and adaptive refinement are host-side in the reference and are
rejected here with exit code 2. The initial guess is the reference drivers'
own (initial_guess = baseline eigenpairs, paro.cpp:63-79) on the device.
"""
from __future__ import annotations

import argparse
import sys
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _native as N
from .configs import Workload

PROBLEMS = ("laplace-square", "laplace-cube", "oscillator", "hydrogen", "molecule")
DIM2 = ("laplace-square", "oscillator")


@dataclass
class RunConfig:
    """RunConfig + ParoConfig (runconfig.hpp, paro.hpp:28-54) fields the device path reads."""

    problem: str = "laplace-square"
    box_lo: float = 0.0
    box_hi: float = 1.0
    subdivisions: int = 8
    out_dir: str = "paro_out"
    molecule_file: str = ""
    n_orbitals: int = 1
    augment: int = 0
    marking: str = "dorfler"
    theta: float = 0.5
    cg_tol_start: float = 1e-8
    cg_tol: float = 1e-12
    cg_max_iter: int = 100000
    max_outer: int = 200
    mixing_alpha: float = 0.3
    tol_energy: float = 1e-6
    tol_estimator: float = 0.0
    adaptive: bool = True
    max_dofs: int = 100000
    drop_tol: float = 1e-8
    workers: int = 1
    seed: int = 1
    xc: str = "lda81"
    vext_smoothing: float = 0.0
    timers: bool = True
    extra: dict = field(default_factory=dict)


def builtin_config(problem: str) -> RunConfig:
    """builtin_config (runconfig.cpp:39-88)."""
    c = RunConfig(problem=problem)
    d = {
        "laplace-square": dict(box_lo=0.0, box_hi=1.0, subdivisions=8, n_orbitals=5, augment=2, max_dofs=50000,
                               tol_energy=1e-8),
        "laplace-cube": dict(box_lo=0.0, box_hi=1.0, subdivisions=4, n_orbitals=1, augment=3, max_dofs=40000,
                             tol_energy=1e-7),
        "oscillator": dict(box_lo=-8.0, box_hi=8.0, subdivisions=16, n_orbitals=6, augment=2, max_dofs=40000,
                           tol_energy=1e-8),
        "hydrogen": dict(box_lo=-10.0, box_hi=10.0, subdivisions=4, n_orbitals=1, augment=2, max_dofs=40000,
                         tol_energy=1e-7),
        "molecule": dict(box_lo=-8.0, box_hi=8.0, subdivisions=4, augment=2, max_dofs=30000, tol_energy=1e-6),
    }[problem]
    for k, v in d.items():
        setattr(c, k, v)
    return c


def _bool(v: str, no: int) -> bool:
    if v in ("on", "true", "1"):
        return True
    if v in ("off", "false", "0"):
        return False
    raise N.ParseError(f"line {no}: expected on/off, got '{v}'")


def _num(v: str, no: int) -> float:
    try:
        return float(v)
    except ValueError:
        raise N.ParseError(f"line {no}: expected a number, got '{v}'") from None


def _int(v: str, no: int) -> int:
    try:
        return int(v, 10)
    except ValueError:
        raise N.ParseError(f"line {no}: expected an integer, got '{v}'") from None


_DOUBLE = ("box_lo", "box_hi", "theta", "cg_tol", "cg_tol_start", "mixing_alpha", "tol_energy", "tol_estimator",
           "drop_tol", "vext_smoothing")
_INT = ("subdivisions", "n_orbitals", "augment", "cg_max_iter", "max_outer", "max_dofs", "workers", "seed")


def parse_run_config(text: str) -> RunConfig:
    """parse_run_config (runconfig.cpp:133-235)."""
    entries, problem = [], "laplace-square"
    for no, line in enumerate(text.splitlines(), 1):
        line = line.split("#", 1)[0]
        if not line.strip(" \t\r"):
            continue
        if "=" not in line:
            raise N.ParseError(f"line {no}: expected 'key = value'")
        key, value = (p.strip(" \t\r") for p in line.split("=", 1))
        if not key or not value:
            raise N.ParseError(f"line {no}: empty key or value")
        if key == "problem":
            problem = value
        else:
            entries.append((no, key, value))
    if problem not in PROBLEMS:
        raise N.ParseError(f"unknown problem '{problem}'")
    c = builtin_config(problem)
    for no, key, value in entries:
        if key in ("molecule_file", "out_dir"):
            setattr(c, key, value)
        elif key in _DOUBLE:
            setattr(c, key, _num(value, no))
        elif key in _INT:
            setattr(c, key, _int(value, no))
        elif key in ("adaptive", "timers"):
            setattr(c, key, _bool(value, no))
        elif key == "marking":
            if value not in ("dorfler", "maximum"):
                raise N.ParseError(f"line {no}: marking must be dorfler or maximum")
            c.marking = value
        elif key == "xc":
            if value not in ("exchange-only", "lda81"):
                raise N.ParseError(f"line {no}: xc must be exchange-only or lda81")
            c.xc = value
        else:
            raise N.ParseError(f"line {no}: unknown key '{key}'")
    if c.problem == "molecule" and not c.molecule_file:
        raise N.ParseError("problem = molecule requires molecule_file")
    if not c.box_hi > c.box_lo:
        raise N.ParseError("box_hi must exceed box_lo")
    if c.subdivisions < 1:
        raise N.ParseError("subdivisions must be >= 1")
    if not 0.0 < c.theta < 1.0:
        raise N.ParseError("theta must lie in (0,1)")
    if not 0.0 < c.mixing_alpha <= 1.0:
        raise N.ParseError("mixing_alpha must lie in (0,1]")
    if not c.tol_energy > 0.0:
        raise N.ParseError("tol_energy must be positive")
    if not c.cg_tol > 0.0:
        raise N.ParseError("cg_tol must be positive")
    return c


def parse_molecule(text: str):
    """parse_molecule (model.cpp:97-138) -> (charges, positions [M, 3], n_electrons)."""
    Z, R, ne = [], [], None
    for no, line in enumerate(text.splitlines(), 1):
        tok = line.split("#", 1)[0].split()
        if not tok:
            continue
        if tok[0] == "electrons":
            try:
                ne = int(tok[1])
            except (IndexError, ValueError):
                raise N.ParseError(f"molecule line {no}: bad electron count") from None
            continue
        try:
            z = float(tok[0])
            xyz = [float(t) for t in tok[1:4]]
            if len(xyz) != 3:
                raise ValueError
        except ValueError:
            raise N.ParseError(f"molecule line {no}: expected 'Z x y z'") from None
        if z <= 0.0:
            raise N.ParseError(f"molecule line {no}: charge must be positive")
        Z.append(z)
        R.append(xyz)
    if not Z:
        raise N.ParseError("molecule: no nuclei")
    if ne is None:
        ne = int(round(sum(Z)))
    if ne < 1:
        raise N.ParseError("molecule: electron count must be >= 1")
    return np.array(Z), np.array(R, dtype=float), ne


def workload_of(c: RunConfig) -> Workload:
    """The fixed-mesh device workload of a run configuration."""
    if c.problem in DIM2:
        raise N.InvalidArgumentError(f"{c.problem}: 2-D problems are not part of the device path")
    if c.adaptive:
        raise N.InvalidArgumentError("adaptive refinement stays host-side in the reference; set adaptive = off")
    if c.xc != "lda81":
        raise N.InvalidArgumentError("xc = exchange-only is not part of the device path")
    common = dict(augment=c.augment, iterations=c.max_outer, cg_tol_start=c.cg_tol_start, cg_tol=c.cg_tol,
                  cg_max_iter=c.cg_max_iter, mixing_alpha=c.mixing_alpha, drop_tol=c.drop_tol, seed=c.seed,
                  tol_energy=c.tol_energy, tol_estimator=c.tol_estimator, guess="baseline")
    if c.problem == "molecule":
        path = Path(c.molecule_file)  # opened as given, like parse_molecule_file (model.cpp:140-144)
        try:
            text = path.read_text()
        except OSError:
            raise N.ParseError(f"molecule: cannot open {c.molecule_file}") from None
        Z, R, ne = parse_molecule(text)
        return Workload("molecule", "ks", c.subdivisions, c.box_lo, c.box_hi, n_orbitals=ne // 2, charges=Z,
                        positions=R, n_electrons=ne, eps=c.vext_smoothing, **common)
    if c.problem == "hydrogen":  # potential_well(0.5 I, external_potential(H atom), runner.cpp:42-45)
        return Workload("hydrogen", "linear", c.subdivisions, c.box_lo, c.box_hi, n_orbitals=c.n_orbitals,
                        potential="softwell", charges=np.array([1.0]), positions=np.zeros((1, 3)),
                        eps=c.vext_smoothing, **common)
    # laplace-cube: elliptic(I, 0)
    return Workload("laplace-cube", "linear", c.subdivisions, c.box_lo, c.box_hi, n_orbitals=c.n_orbitals,
                    potential="none", diffusion=1.0, **common)


@dataclass
class RunArtifacts:
    converged: bool
    iterations: int
    summary: str
    traces: list
    lambdas: list


def run_experiment(c: RunConfig, device: int = 0) -> RunArtifacts:
    """run_experiment (runner.cpp:67-121) on the device path."""
    from . import artifacts
    from .driver import GpuBackend, ParoRun

    w = workload_of(c)
    for attempt in range(3):
        try:
            run = ParoRun(w, GpuBackend(w, device=device), guess="baseline", timers=c.timers, estimate=True)
            traces = run.run(c.max_outer, stop=True)
            break
        except N.DegenerateSpanError as e:
            if attempt >= 2:
                raise N.Error(f"paro: run failed after 3 degenerate-span restarts: {e}") from None
            w.augment += 1  # restart with a larger candidate span (paro.cpp:384-388)
            w.seed += 1
    converged = bool(traces and traces[-1].converged)
    line = artifacts.write_run(c.out_dir, traces, list(run.lambdas), w.n_orbitals, w.kind == "ks",
                               converged=converged, mesh=(w.subdivisions, w.lo, w.hi))
    return RunArtifacts(converged, len(traces), line, traces, list(run.lambdas))


EXIT = [(N.ParseError, 2), (N.InvalidArgumentError, 2), (N.NotSpdError, 3), (N.IterationLimitError, 3),
        (N.CapacityError, 4), (N.ScfDivergenceError, 5)]


def main(argv=None) -> int:
    """tools/main.cpp:46-67 (the --suite verification runs are out of scope)."""
    ap = argparse.ArgumentParser(prog="paro_b200", description="fixed-mesh ParO on the B200 device path")
    ap.add_argument("-c", "--config", default="")
    ap.add_argument("-w", "--workers", type=int, default=0)
    ap.add_argument("-o", "--out", default="")
    a = ap.parse_args(argv)
    if not a.config:
        print("error: provide --config (see --help)", file=sys.stderr)
        return 2
    try:
        path = Path(a.config)
        try:
            text = path.read_text()
        except OSError:
            raise N.ParseError(f"cannot open config file {a.config}") from None
        c = parse_run_config(text)
        if a.workers > 0:
            c.workers = a.workers
        if a.out:
            c.out_dir = a.out
        res = run_experiment(c)
        print(res.summary)
        return 0 if res.converged else 1
    except Exception as e:  # noqa: BLE001 - the CLI maps every failure to an exit code
        for cls, code in EXIT:
            if isinstance(e, cls):
                label = {2: "config error" if isinstance(e, N.ParseError) else "error", 3: "solver error",
                         4: "capacity error", 5: "divergence"}[code]
                print(f"{label}: {e}", file=sys.stderr)
                return code
        print(f"error: {e}", file=sys.stderr)
        return 6
