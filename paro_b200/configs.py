"""Synthetic BASELINE.json workloads, shared by the GPU path,
the reference harness and the tests so both sides see identical inputs.

Portable RNG: SplitMix64; uniform[-1,1] = ((x >> 11) * 2^-53) * 2 - 1.
Guess vectors are evaluated at the interior nodes in the reference dof order.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_MASK = (1 << 64) - 1


class SplitMix64:
    def __init__(self, seed: int):
        self.state = seed & _MASK

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def unit(self) -> float:
        """uniform [0, 1)"""
        return (self.next() >> 11) * (1.0 / (1 << 53))

    def sym(self) -> float:
        """uniform [-1, 1)"""
        return self.unit() * 2.0 - 1.0

    def sym_array(self, count: int) -> np.ndarray:
        """`count` successive uniform[-1,1) draws, vectorised (same sequence as sym())."""
        idx = np.arange(1, count + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = np.uint64(self.state) + idx * np.uint64(0x9E3779B97F4A7C15)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        self.state = (self.state + count * 0x9E3779B97F4A7C15) & _MASK
        return (z >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53)) * 2.0 - 1.0


@dataclass
class Workload:
    name: str
    kind: str                      # "ks" | "linear"
    subdivisions: int
    lo: float
    hi: float
    n_orbitals: int                # N
    augment: int = 0               # m
    iterations: int = 1
    charges: np.ndarray = field(default_factory=lambda: np.zeros(0))
    positions: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    n_electrons: int = 0
    eps: float = 0.0               # V_ext smoothing (ks) / softening (linear well)
    potential: str = ""           # linear: "harmonic" | "softwell"
    guess: str = "gaussian"        # "gaussian-sum" | "gaussian-atoms" | "noise"
    seed: int = 1
    cg_tol_start: float = 1e-8
    cg_tol: float = 1e-12
    cg_tol_factor: float = 0.25
    cg_max_iter: int = 100000
    mixing_alpha: float = 0.3
    drop_tol: float = 1e-8
    tol_energy: float = 1e-6       # ParoConfig::tol_energy (paro.hpp:39): the stop tests' threshold
    tol_estimator: float = 0.0     # ParoConfig::tol_estimator: 0 disables the estimator stop test
    diffusion: float = 0.5         # linear: the stiffness scale (1 for laplace-cube)

    @property
    def K(self) -> int:
        return self.n_orbitals + self.augment

    @property
    def h(self) -> float:
        return (self.hi - self.lo) / self.subdivisions

    @property
    def n(self) -> int:
        return (self.subdivisions - 1) ** 3

    def cg_tol_for_iteration(self, it: int) -> float:
        """cg_tol_for_iteration (paro.cpp:212-214)."""
        return max(self.cg_tol, self.cg_tol_start * self.cg_tol_factor ** it)

    def scaled(self, subdivisions: int, iterations: int | None = None) -> "Workload":
        import copy

        w = copy.copy(self)
        w.subdivisions = subdivisions
        if iterations is not None:
            w.iterations = iterations
        w.name = f"{self.name}@s{subdivisions}"
        return w


def interior_coords(w: Workload):
    """Coordinates of the interior nodes (x fastest), as create_box_mesh computes them."""
    s = w.subdivisions
    i = np.arange(1, s, dtype=np.float64)
    c = w.lo + (w.hi - w.lo) * i / s
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    return x.reshape(-1), y.reshape(-1), z.reshape(-1)


def guess_vectors(w: Workload) -> np.ndarray:
    """Initial guess columns [K, n] (SURVEY.md §8d 'Initial-guess semantics')."""
    K, n = w.K, w.n
    if w.guess == "noise":
        rng = SplitMix64(w.seed)
        return rng.sym_array(K * n).reshape(K, n)  # column-major draw order
    x, y, z = interior_coords(w)
    if w.guess == "gaussian-sum":
        g = np.zeros(n)
        for R in w.positions:
            g += np.exp(-((x - R[0]) ** 2 + (y - R[1]) ** 2 + (z - R[2]) ** 2))
        return _flush_tails(np.stack([g] * K))
    # gaussian-atoms: per atom s, then p_x, p_y, p_z; first K
    cols = []
    for R in w.positions:
        dx, dy, dz = x - R[0], y - R[1], z - R[2]
        e = np.exp(-(dx * dx + dy * dy + dz * dz))
        cols += [e, dx * e, dy * e, dz * e]
        if len(cols) >= K:
            break
    if len(cols) < K:
        raise ValueError(f"{w.name}: only {len(cols)} Gaussian functions for K = {K}")
    return _flush_tails(np.stack(cols[:K]))


# Gaussian tails below this magnitude are set to 0. Without it, nodes ~19 bohr
# from every nucleus get densities of 1e-313 (denormal), where the reference
# LDA (model.cpp:282, rs = cbrt(3/(4 pi rho))) overflows to inf, v_xc becomes
# NaN and assemble_weighted_mass throws (fem.cpp:306-309) on both sides.
GUESS_FLUSH = 1e-100


def _flush_tails(g: np.ndarray) -> np.ndarray:
    g[np.abs(g) < GUESS_FLUSH] = 0.0
    return g


# ------------------------------------------------------------ BASELINE configs

def h2() -> Workload:
    """configs[0]: H2 LDA, 33^3 nodes, 20 iterations."""
    return Workload("h2", "ks", 32, -10.0, 10.0, n_orbitals=1, iterations=20,
                    charges=np.array([1.0, 1.0]), positions=np.array([[0.7, 0.0, 0.0], [-0.7, 0.0, 0.0]]),
                    n_electrons=2, guess="gaussian-sum")


def oscillator() -> Workload:
    """configs[1]: 3D harmonic oscillator, 65^3, N = 10 noise columns, 40 iterations."""
    return Workload("oscillator", "linear", 64, -8.0, 8.0, n_orbitals=10, iterations=40, potential="harmonic",
                    guess="noise", seed=1)


def water() -> Workload:
    """configs[2]: water-like LDA, 129^3, N = 5, 30 iterations."""
    a = math.radians(52.25)
    pos = np.array([[0.0, 0.0, 0.0], [1.809 * math.sin(a), 1.809 * math.cos(a), 0.0],
                    [-1.809 * math.sin(a), 1.809 * math.cos(a), 0.0]])
    return Workload("water", "ks", 128, -12.0, 12.0, n_orbitals=5, iterations=30,
                    charges=np.array([8.0, 1.0, 1.0]), positions=pos, n_electrons=10, guess="gaussian-atoms")


def source_bench(seed: int = 1) -> Workload:
    """configs[3]: 64 source problems on 257^3, 16 softened Coulomb centres, one Step 3 + Step 4."""
    rng = SplitMix64(seed)
    Z, R = [], []
    for _ in range(16):
        Z.append(float(1 + int(rng.unit() * 6)))
        R.append([rng.sym() * 10.0, rng.sym() * 10.0, rng.sym() * 10.0])
    return Workload("source64", "linear", 256, -16.0, 16.0, n_orbitals=64, iterations=1, potential="softwell",
                    charges=np.array(Z), positions=np.array(R), eps=math.sqrt(0.1), guess="noise", seed=seed + 1)


def cluster32(seed: int = 1) -> Workload:
    """configs[4]: 32-atom LDA cluster (24 C + 8 H), 257^3, N = 76, 15 iterations."""
    rng = SplitMix64(seed)
    Z, R = [], []
    for charge in [6.0] * 24 + [1.0] * 8:
        while True:
            p = np.array([rng.sym() * 9.0, rng.sym() * 9.0, rng.sym() * 9.0])
            if all(np.linalg.norm(p - q) >= 2.0 for q in R):
                break
        Z.append(charge)
        R.append(p)
    return Workload("cluster32", "ks", 256, -18.0, 18.0, n_orbitals=76, iterations=15, charges=np.array(Z),
                    positions=np.array(R), n_electrons=152, guess="gaussian-atoms")


WORKLOADS = {"h2": h2, "oscillator": oscillator, "water": water, "source64": source_bench, "cluster32": cluster32}


def get(name: str) -> Workload:
    base, _, sub = name.partition("@s")
    w = WORKLOADS[base]()
    return w.scaled(int(sub)) if sub else w
