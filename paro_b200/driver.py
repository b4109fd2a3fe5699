"""Fixed-mesh ParO outer iteration, orbitals sharded over ranks.

Mirrors the loop bodies of the reference drivers with the adaptive branch off
(SURVEY.md §8c "Oracle harness contract"):
  Kohn-Sham  proj/src/paro.cpp:514-638   (Step 2 estimator omitted on both sides)
  linear     proj/src/paro.cpp:340-354
Multi-GPU: rank r owns a contiguous block of orbital columns
and solves its Step-3 source problems with no communication. The half-step
orbitals are then transposed (one all-to-all) into row slabs: rank r holds
all K columns on its block of lattice planes (+ one halo plane each side),
and Step 4 runs sharded over the slabs (step4.py): the K x K Gram partials
are summed across ranks in rank order, the fix_sign pieces reduced, and
every per-dof operation stays on the slab. The densities are computed on the
slabs and all-gathered (the Hartree solve, KS form and energy stay
replicated on the full density), and the new orbitals go back to column
shards with a second all-to-all. The compute is delegated to a backend
(GpuBackend = the native sm_100a library); the orchestration is
backend-agnostic so the N > 1 path is testable with gloo on CPU.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import torch

from . import _native as N
from .configs import Workload, guess_vectors
from .step4 import RowSlab, Step4

OK, NOT_SPD, ITER_LIMIT = 0, 3, 4


def step3_outcome(first, final):
    """Exception order of source_solve_step (paro.cpp:95-117, serial worker):
    a failure inside the per-orbital retry escapes at once; otherwise the first
    failed first attempt (by orbital index) is rethrown."""
    for c, (f, g) in enumerate(zip(first, final)):
        if f == ITER_LIMIT and g != OK:
            return g, c
    for c, f in enumerate(first):
        if f not in (OK, ITER_LIMIT):
            return f, c
    return OK, -1


class Dist:
    """torch.distributed plumbing (NCCL on GPUs, gloo on CPU); world 1 = no-op."""

    def __init__(self, group=None, collectives: bool = False):
        """collectives=True runs every exchange through the process group even
        at world size 1 (a single-rank NCCL check of the N > 1 code path)."""
        import torch.distributed as td

        self.td = td if td.is_available() and td.is_initialized() else None
        self.group = group
        self.world = self.td.get_world_size(group) if self.td else 1
        self.rank = self.td.get_rank(group) if self.td else 0
        self.solo = self.world == 1 and not (collectives and self.td is not None)

    def _gather(self, out: torch.Tensor, inp: torch.Tensor):
        """all_gather_into_tensor (NCCL); list all_gather on backends without it (gloo)."""
        if self.td.get_backend(self.group) == "nccl":
            self.td.all_gather_into_tensor(out, inp, group=self.group)
        else:
            self.td.all_gather(list(out.chunk(self.world)), inp, group=self.group)

    def shard(self, K: int):
        base, rem = divmod(K, self.world)
        counts = [base + (1 if r < rem else 0) for r in range(self.world)]
        c0 = sum(counts[: self.rank])
        return c0, c0 + counts[self.rank], counts

    def allgather_columns(self, local: torch.Tensor, counts, out: torch.Tensor):
        """[k_r, n] blocks -> out[:K] in rank order (padded to max(counts))."""
        if self.solo:
            if local.data_ptr() != out.data_ptr():
                out[: local.shape[0]].copy_(local)
            return out
        kmax = max(counts)
        n = local.shape[1]
        send = local.new_zeros((kmax, n)) if local.shape[0] < kmax else local
        if local.shape[0] < kmax:
            send[: local.shape[0]].copy_(local)
        recv = local.new_empty((self.world * kmax, n))
        self._gather(recv, send.contiguous())
        row = 0
        for r, cnt in enumerate(counts):
            out[row: row + cnt].copy_(recv[r * kmax: r * kmax + cnt])
            row += cnt
        return out

    # ---- Step-4 reductions (step4.py): fixed rank order, identical on every rank
    def allsum_(self, t: torch.Tensor) -> torch.Tensor:
        """In-place sum over ranks, added in rank order (deterministic, and
        the same bits on every rank)."""
        if self.solo:
            return t
        flat = t.reshape(-1)
        buf = flat.new_empty(self.world * flat.numel())
        self._gather(buf, flat.contiguous())
        parts = buf.view(self.world, -1)
        flat.copy_(parts[0])
        for r in range(1, self.world):
            flat.add_(parts[r])
        return t

    def allmax_(self, t: torch.Tensor) -> torch.Tensor:
        if not self.solo:
            self.td.all_reduce(t, op=self.td.ReduceOp.MAX, group=self.group)
        return t

    def allmin_(self, t: torch.Tensor) -> torch.Tensor:
        if not self.solo:
            self.td.all_reduce(t, op=self.td.ReduceOp.MIN, group=self.group)
        return t

    def cols_to_slabs(self, local: torch.Tensor, counts, dst: torch.Tensor, slabs):
        """Column shards -> row slabs: this rank's columns [k_r, n] (all rows)
        go out as the extended row range of every rank's slab; dst[:K] receives
        every rank's columns on this rank's extended rows. One all-to-all."""
        me = slabs[self.rank]
        c0 = sum(counts[: self.rank])
        if self.solo:
            if local.data_ptr() != dst[c0:].data_ptr():
                dst[c0:c0 + local.shape[0], me.e0:me.e1].copy_(local[:, me.e0:me.e1])
            return dst
        k = local.shape[0]
        send = torch.cat([local[:, s.e0:s.e1].reshape(-1) for s in slabs])
        ext = me.e1 - me.e0
        recv = local.new_empty(sum(counts) * ext)
        self.td.all_to_all_single(recv, send, [c * ext for c in counts], [k * (s.e1 - s.e0) for s in slabs],
                                  group=self.group)
        off, col = 0, 0
        for cnt in counts:
            dst[col:col + cnt, me.e0:me.e1].copy_(recv[off:off + cnt * ext].view(cnt, ext))
            off += cnt * ext
            col += cnt
        return dst

    def slabs_to_cols(self, V: torch.Tensor, counts, slabs):
        """Row slabs -> column shards, in place: V[:K] holds every column on this
        rank's own rows; afterwards this rank's columns hold every row."""
        if self.solo:
            return V
        me = slabs[self.rank]
        c0 = sum(counts[: self.rank])
        k = counts[self.rank]
        starts = [sum(counts[:r]) for r in range(self.world)]
        send = torch.cat([V[starts[r]:starts[r] + counts[r], me.r0:me.r1].reshape(-1) for r in range(self.world)])
        rows = [s.r1 - s.r0 for s in slabs]
        recv = V.new_empty(k * sum(rows))
        self.td.all_to_all_single(recv, send, [k * r for r in rows], [c * (me.r1 - me.r0) for c in counts],
                                  group=self.group)
        off = 0
        for s, r in zip(slabs, rows):
            if s is not me:
                V[c0:c0 + k, s.r0:s.r1].copy_(recv[off:off + k * r].view(k, r))
            off += k * r
        return V

    def allgather_rows(self, f: torch.Tensor, slabs):
        """f (n) valid on this rank's own rows -> valid everywhere."""
        if self.solo:
            return f
        m = max(s.r1 - s.r0 for s in slabs)
        me = slabs[self.rank]
        send = f.new_zeros(m)
        send[: me.r1 - me.r0].copy_(f[me.r0:me.r1])
        buf = f.new_empty(self.world * m)
        self._gather(buf, send)
        for r, s in enumerate(slabs):
            if s is not me:
                f[s.r0:s.r1].copy_(buf[r * m: r * m + (s.r1 - s.r0)])
        return f

    def allgather_ints(self, values, counts, device):
        if self.solo:
            return list(values)
        kmax = max(counts)
        t = torch.full((kmax,), -1, dtype=torch.int64, device=device)
        if len(values):
            t[: len(values)] = torch.tensor(values, dtype=torch.int64, device=device)
        out = torch.empty(self.world * kmax, dtype=torch.int64, device=device)
        self._gather(out, t)
        out = out.cpu().tolist()
        res = []
        for r, cnt in enumerate(counts):
            res += out[r * kmax: r * kmax + cnt]
        return res


class GpuBackend:
    """The product backend: every call lands in the native sm_100a library."""

    def __init__(self, workload: Workload, device: int = 0):
        from . import core

        self.core = core
        self.w = workload
        self.ctx = core.Context(device).grid(workload.subdivisions, workload.lo, workload.hi)
        self.n = self.ctx.n
        self.device = self.ctx.device
        c = core
        self.mass = c.assemble_mass(self.ctx)
        if workload.kind == "ks":
            self.kinetic = c.assemble_stiffness(self.ctx, 0.5)
            self.poisson = c.assemble_stiffness(self.ctx, 1.0)
            self.vext = c.assemble_vext(self.ctx, workload.charges, workload.positions, workload.eps)
            self.forms = {"in": c.Operator.variable_empty(self.ctx), "half": c.Operator.variable_empty(self.ctx)}
            self.scratch = self.ctx.empty(self.n)
        else:
            # LinearProblem::elliptic / potential_well (runner.cpp:30-47): diffusion stiffness + reaction mass
            a = c.assemble_stiffness(self.ctx, workload.diffusion)
            if workload.potential == "harmonic":
                c.add_scaled(a, c.assemble_harmonic(self.ctx, 0.5))
            elif workload.potential != "none":
                c.add_scaled(a, c.assemble_vext(self.ctx, workload.charges, workload.positions, workload.eps))
            self.form = a

    # tensors
    def empty(self, *shape):
        return self.ctx.empty(*shape)

    def from_host(self, a):
        return torch.as_tensor(a, device=self.device).contiguous()

    def sync(self):
        torch.cuda.synchronize(self.device)

    # operators
    def core_hamiltonian(self):
        a0 = self.core.assemble_stiffness(self.ctx, 0.5)
        return self.core.add_scaled(a0, self.vext)

    def ks_form(self, rho, vh, slot):
        op, clamped = self.core.ks_form_matrix(self.kinetic, self.vext, rho, vh, out=self.forms[slot])
        return op, clamped

    def ks_form_slab(self, rho, vh, slot, z0, z1):
        """The KS form's coefficients on the dofs of planes [z0, z1) (the rest of forms[slot] is
        left as it is) and the clamp count of the slab's cells."""
        cl = self.core.ks_form_planes(self.kinetic, self.vext, rho, vh, z0, z1, self.forms[slot])
        return self.forms[slot], cl

    def form_slots(self, op):
        """[8, n] view of a variable operator's coefficient slots."""
        return op.coefficients()

    # steps
    def hartree(self, rho, out=None):
        return self.core.hartree_solve_with(self.poisson, self.mass, rho, 1e-11, out=out)

    def source_solve(self, a, u, lambdas, sigma, tol, max_iter, out):
        return self.core.source_solve_columns(a, self.mass, u, lambdas, tol, max_iter, sigma, out)

    def initial_guess(self, a, count, out):
        """initial_guess (paro.cpp:63-79) on the device: baseline eigenpairs of a."""
        og = self.core.initial_guess(a, self.mass, count, seed=self.w.seed)
        out[:count].copy_(og.orbitals)
        return out[:count], list(og.lambdas), og.gram_defect

    def ritz_copyout(self, stream, host, c0, c1):
        """One-shot host copy-out of the next ritz's orbital columns [c0, c1) (step_host)."""
        self.ctx.set_ritz_copyout(stream, host, c0, c1)

    def ritz(self, cands, a, min_keep, drop_tol, out):
        r = self.core.rayleigh_ritz(cands, a, self.mass, min_keep, drop_tol, out=out)
        return r.orbitals, list(r.lambdas), r.gram_defect

    def density(self, U, occ, out=None):
        return self.core.density_from_orbitals(self.ctx, U, occ, out=out)[0]

    def energy(self, lambdas, occ, rho, vh):
        return self.core.total_energy(self.ctx, lambdas, occ, rho, vh, self.w.charges, self.w.positions)

    def energy_xc_layers(self, rho, k0, k1):
        return self.core.energy_xc_layers(self.ctx, rho, k0, k1)

    def energy_with_xc(self, lambdas, occ, rho, vh, xc_term):
        return self.core.total_energy_with_xc(self.ctx, lambdas, occ, rho, vh, self.w.charges, self.w.positions,
                                              xc_term)

    def mix(self, rin, rout, alpha, out):
        return self.core.mix_density(self.ctx, rin, rout, alpha, out=out)

    def rho_residual(self, rout, rin):
        return self.core.rho_residual(self.ctx, rout, rin, self.scratch)

    def estimate(self, U, lambdas, rho=None, vh=None):
        """Step 2 (adapt.cpp:104-129): eta_total of the orbitals' residual estimators."""
        w = self.w
        if w.kind == "ks":
            return self.core.estimate_eta(self.ctx, U, lambdas, reaction="ks", charges=w.charges,
                                          positions=w.positions, eps=w.eps, rho=rho, vh=vh)
        if w.potential in ("harmonic", "none"):
            return self.core.estimate_eta(self.ctx, U, lambdas, diffusion=w.diffusion, reaction="harmonic",
                                          c=0.5 if w.potential == "harmonic" else 0.0)
        return self.core.estimate_eta(self.ctx, U, lambdas, diffusion=w.diffusion, reaction="well",
                                      charges=w.charges, positions=w.positions, eps=w.eps)

    def launches(self) -> int:
        return self.ctx.launches()

    # ---- Step 4 building blocks on row ranges (step4.py)
    @property
    def S(self) -> int:
        return self.ctx.S

    def mass_op(self):
        return self.mass

    def apply_planes(self, op, X, k, Y, z0, z1):
        self.core.apply_planes(op, X, k, Y, z0, z1)

    def gram_sym(self, X, Y, k, r0, r1):
        return self.core.gram_sym(self.ctx, X, Y, k, r0, r1)

    def gram_rect(self, X, k1, Y, k2, r0, r1):
        return self.core.gram_rect(self.ctx, X, k1, Y, k2, r0, r1)

    def rotate(self, X, k1, Cm, ldc, k2, Z, r0, r1, mode):
        self.core.rotate(self.ctx, X, k1, Cm, ldc, k2, Z, r0, r1, mode)

    def kk(self, m):
        return torch.empty(max(m, 1), dtype=torch.float64, device=self.device)

    def ritz_ortho(self, G, K, drop_tol, C1):
        return self.core.ritz_ortho(self.ctx, G, K, drop_tol, C1)

    def ritz_second_pass(self, G2, k, C2, Bt):
        return self.core.ritz_second_pass(self.ctx, G2, k, C2, Bt)

    def ritz_congruence(self, G, C1, k, Bt):
        self.core.ritz_congruence(self.ctx, G, C1, k, Bt)

    def ritz_pencil(self, GA, C2, Bt, GB, k, Y):
        return self.core.ritz_pencil(self.ctx, GA, C2, Bt, GB, k, Y)

    def gram_defect(self, G, k):
        return self.core.gram_defect_of(self.ctx, G, k)

    def sign_buffers(self, k):
        return self.core.sign_buffers(self.ctx, k)

    def colmax(self, V, k, r0, r1, amax):
        self.core.colmax(self.ctx, V, k, r0, r1, amax)

    def first_above(self, V, k, r0, r1, amax, first):
        self.core.first_above(self.ctx, V, k, r0, r1, amax, first)

    def sign_flags(self, V, k, r0, r1, amax, first, flip):
        self.core.sign_flags(self.ctx, V, k, r0, r1, amax, first, flip)

    def negate_columns(self, V, k, r0, r1, flip):
        self.core.negate_columns(self.ctx, V, k, r0, r1, flip)

    def copy_rows(self, src, dst, r0, r1):
        dst[:, r0:r1].copy_(src[:, r0:r1])

    def div_rows(self, src, d, dst, r0, r1):
        torch.div(src[:, r0:r1], d, out=dst[:, r0:r1])  # x /= nb (linalg.cpp:431)

    def to_host(self, t):
        return t.cpu().tolist()

    def density_rows(self, U, occ, r0, r1, rho):
        return self.core.density_rows(self.ctx, U, occ, r0, r1, rho)

    def density_normalize(self, total, rho):
        return self.core.density_normalize(self.ctx, total, rho)


@dataclass
class Trace:
    iter: int
    lambdas: list
    e_tot: float | None
    rho_residual: float | None
    sigma: float
    gram_defect: float
    cg_iterations: list
    t_source: float
    t_project: float
    t_total: float
    eta_total: float | None = None   # Step 2 (estimate=True): combine_max(estimate_eigen_residual).total()
    t_meshgen: float = 0.0           # Step 2 wall time (the reference's t_meshgen column)
    dofs: int = 0
    # what the reference driver's stop tests decide after this iteration
    # (fixed mesh: mesh_frozen = true), logged while the harness runs on:
    stable_count: int = 0            # KS: |dE| < tol_energy streak (paro.cpp:624); linear: lambdas_stable (:358-362)
    increase_count: int = 0          # KS: rising energy with a stalled density residual (paro.cpp:615-617)
    converged: bool = False          # the reference would stop here, converged (paro.cpp:632-635 / :365-369)
    diverged: bool = False           # the reference would throw ScfDivergenceError here (paro.cpp:618-622)


class StopTests:
    """The reference drivers' convergence control on a fixed mesh, evaluated
    on the harness's trace rows without changing the run:
      Kohn-Sham  paro.cpp:605-635  energy-stability streak >= 3 converges;
                 5 consecutive energy rises without density-residual progress
                 is an SCF divergence;
      linear     paro.cpp:358-369  lambdas_stable (:240-246) streak >= 2, or
                 eta_total <= tol_estimator when that test is enabled."""

    def __init__(self, w: Workload):
        self.w = w
        self.stable = 0
        self.increase = 0
        self.e_prev = None
        self.res_prev = None
        self.lam_prev = None

    def update(self, tr: "Trace") -> "Trace":
        w = self.w
        if w.kind == "ks":
            if self.e_prev is not None:
                rising = tr.e_tot > self.e_prev + 1e-14
                stalled = tr.rho_residual >= self.res_prev * (1.0 - 1e-12)
                self.increase = self.increase + 1 if (rising and stalled) else 0
                tr.diverged = self.increase >= 5
                self.stable = self.stable + 1 if abs(tr.e_tot - self.e_prev) < w.tol_energy else 0
            self.res_prev, self.e_prev = tr.rho_residual, tr.e_tot
            tr.converged = self.stable >= 3 and not tr.diverged
        else:
            lam = list(tr.lambdas)
            prev = self.lam_prev
            stable = prev is not None and len(prev) == len(lam) and all(
                abs(a - b) <= w.tol_energy * (1.0 + abs(a)) for a, b in zip(lam, prev))
            self.stable = self.stable + 1 if stable else 0
            self.lam_prev = lam
            est_ok = w.tol_estimator > 0.0 and tr.eta_total is not None and tr.eta_total <= w.tol_estimator
            tr.converged = self.stable >= 2 or est_ok
        tr.stable_count, tr.increase_count = self.stable, self.increase
        return tr


class ParoRun:
    """One fixed-mesh ParO run (KS or linear) on a backend, sharded by `dist`."""

    def __init__(self, w: Workload, backend, dist: Dist | None = None, guess=None, timers: bool = True,
                 estimate: bool = False):
        self.w = w
        self.estimate = estimate  # run Step 2 (eta_total) like the reference drivers; off in the bench
        self.be = backend
        self.dist = dist or Dist()
        self.timers = timers
        K = w.K
        n = backend.n
        self.half = backend.empty(K, n)
        self.orb = backend.empty(K, n)
        self._half_local = None
        # Step 4 over row slabs of the lattice planes (one slab per rank)
        self.slabs = RowSlab.all(backend.S, self.dist.world)
        self.slab = self.slabs[self.dist.rank]
        self.s4 = Step4(backend, self.dist, self.slab)
        if estimate and self.dist.world > 1:
            raise N.InvalidArgumentError("ParoRun: the Step-2 estimator needs every orbital row (world size 1)")
        self._out = None         # step_host: (copy stream, host orbitals) filled after Step 4
        self._hooked = False     # step_host: the copy-out was started inside Step 4
        # guess="baseline": the reference drivers' own start, initial_guess =
        # baseline eigenpairs of the core / linear operator (paro.cpp:278,
        # 499-505); otherwise the generator's guess columns, Ritz-projected
        baseline = isinstance(guess, str) and guess == "baseline"
        if not baseline:
            g = guess if guess is not None else guess_vectors(w)
            cands = backend.from_host(g) if not torch.is_tensor(g) else g

        def start(a):
            if baseline:  # replicated on every rank: all rows of every column
                return backend.initial_guess(a, K, self.orb)
            orb, lam, d = self.s4.ritz(cands, a, backend.mass_op(), K, w.drop_tol, self.orb)
            return orb, lam, d

        if w.kind == "ks":
            self.occ = [2.0] * (w.n_electrons // 2)
            if len(self.occ) != w.n_orbitals:
                raise N.InvalidArgumentError("kohn-sham: config.n_orbitals must equal N_e / 2")
            a0 = backend.core_hamiltonian()
            # initial guess: V_H = V_xc = 0 linearisation (paro.cpp:499-505)
            orb, lam, _ = start(a0)
            self.rho_in = self._density(orb[: w.n_orbitals], backend.empty(n))
            self.rho_half = backend.empty(n)
            self.rho_out = backend.empty(n)
            self.vh = backend.empty(n)
        else:
            orb, lam, _ = start(backend.form)
        if not baseline:
            self.dist.slabs_to_cols(self.orb, self.dist.shard(orb.shape[0])[2], self.slabs)
        self.k = orb.shape[0]
        self.lambdas = lam
        self.clamped = 0
        self._notspd_probe = []  # orbitals that met NotSpd in the last failing Step-3 attempt
        self.probe_hits = 0      # Step-3 attempts decided by the probe alone
        self._fail_attempts = 0  # NotSpd attempts of the last Step 3 (the probe runs for that many)
        self.stops = StopTests(w)  # the reference's stop decisions, logged per Trace row
        self._chunks = None      # step_host: (c0, c1, copy event) of the local Step-3 columns
        self._pieces = None      # step_host: (c0, c1, copy event) of every copied piece
        self._waited = set()     # step_host: ids of the chunk events the compute stream already waits on
        self._copy_stream = None
        # step_host(pipelined=True): copy-out stream, the previous step's copy-out events per column
        # chunk / of the density, and the compute stream's last read of the device state
        self._out_stream = None
        self._later_out = None
        self._d2h_events = []
        self._rho_out_event = None
        self._post_read = None
        self.timeline = None     # profiling: list of (label, CUDA event) marks, or None

    def _mark(self, label, stream=None):
        if self.timeline is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            self.timeline.append((label, ev))

    def _sync(self):
        if self.timers:
            self.be.sync()

    def step3(self, a, it: int):
        """shifted_source_step (paro.cpp:194-210) over the sharded columns + allgather."""
        w, be, d = self.w, self.be, self.dist
        K = self.k
        c0, c1, counts = d.shard(K)
        tol = w.cg_tol_for_iteration(it)
        sigma = max(0.0, 0.5 - self.lambdas[0])
        local = self.half[c0:c1] if d.world == 1 else self._local(c1 - c0)
        self.last_attempts = 0
        # column chunks whose inputs may still be in flight (step_host): each
        # waits for its copy, then solves; the first NotSpd ends the attempt
        # like the batch abort does (the remaining columns report OK)
        chunks = self._chunks if self._chunks is not None else [(c0, c1, None)]
        for attempt in range(5):
            self.last_attempts = attempt + 1
            # NotSpd probe: an attempt fails as soon as any orbital's CG meets
            # p'Ap <= 0, and each column's CG does not depend on the batch it
            # runs in, so the orbitals that failed the last failing attempt are
            # solved alone first; if one of them fails again the whole attempt
            # has the same outcome without solving the other columns, and if
            # none does their solutions are final and the batch skips them
            # (the last attempt always runs in full: its error is the result)
            done = {}
            # probing pays off for the attempts that failed last step; a probe
            # that passes only moves its columns out of the batch (a lone column
            # solves slower than inside the batch), so later attempts run in full
            if self._notspd_probe and attempt < min(4, self._fail_attempts):
                hit, done = self._probe(a, chunks, c0, c1, sigma, tol, attempt, local)
                if hit:
                    self.probe_hits += 1
                    sigma = 2.0 * sigma + 1.0
                    continue
            n_loc = c1 - c0
            first, final, iters = [OK] * n_loc, [OK] * n_loc, [0] * n_loc
            for c, (f, g, i) in done.items():
                first[c - c0], final[c - c0], iters[c - c0] = f, g, i
            failed = False
            for k0, k1, ev in chunks:
                self._wait_chunk(ev)
                if failed:  # the first NotSpd ends the attempt like the batch abort (other columns report OK)
                    continue
                # contiguous runs of this chunk's columns the probe has not solved
                runs, start = [], None
                for c in range(k0, k1 + 1):
                    if c < k1 and c not in done:
                        start = c if start is None else start
                    elif start is not None:
                        runs.append((start, c))
                        start = None
                for r0, r1 in runs:
                    f, g, i, _ = be.source_solve(a, self.orb[r0:r1], self.lambdas[r0:r1], sigma, tol, w.cg_max_iter,
                                                 local[r0 - c0:r1 - c0])
                    first[r0 - c0:r1 - c0], final[r0 - c0:r1 - c0], iters[r0 - c0:r1 - c0] = f, g, i
                    if NOT_SPD in f:
                        failed = True
                        break
            first = d.allgather_ints(first, counts, self._idev())
            final = d.allgather_ints(final, counts, self._idev())
            if NOT_SPD in first:
                self._notspd_probe = [c for c, f in enumerate(first) if f == NOT_SPD]
            code, col = step3_outcome(first, final)
            if code == NOT_SPD and attempt < 4:
                sigma = 2.0 * sigma + 1.0
                continue
            if code != OK:
                raise N.ERRORS.get(code, N.Error)(f"source_solve_step: orbital {col} failed")
            self._fail_attempts = attempt
            break
        # every chunk has landed before Step 4 writes the new orbitals into self.orb
        self._wait_chunks()
        all_iters = d.allgather_ints(iters, counts, self._idev())
        d.cols_to_slabs(local, counts, self.half, self.slabs)
        return sigma, all_iters

    def _probe(self, a, chunks, c0, c1, sigma, tol, attempt, local):
        """Solve this rank's probe orbitals alone at sigma. Returns (hit, done):
        hit if any rank's probe meets NotSpd (then the attempt fails like the
        full batch would); otherwise done maps each local probe column to its
        (first status, final status, iterations), its solution already in
        `local` -- the same per-column result the batch would produce."""
        w, be, d = self.w, self.be, self.dist
        mine = [c for c in self._notspd_probe if c0 <= c < c1]
        hit, done = 0, {}
        if mine:
            # step_host: the probe columns' copies must have landed (their pieces, not their whole batch)
            for k0, k1, ev in (self._pieces if self._pieces is not None else chunks):
                if any(k0 <= c < k1 for c in mine):
                    self._wait_chunk(ev)
            # device-side gather (a host->device index upload would queue on the
            # copy engine behind step_host's orbital transfer)
            u = torch.stack([self.orb[c] for c in mine])
            out = torch.empty_like(u)
            f, g, i, _ = be.source_solve(a, u, [self.lambdas[c] for c in mine], sigma, tol, w.cg_max_iter, out)
            if NOT_SPD in f:
                hit = 1
            else:
                for q, c in enumerate(mine):
                    local[c - c0].copy_(out[q])
                done = {c: (f[q], g[q], i[q]) for q, c in enumerate(mine)}
        hits = d.allgather_ints([hit], [1] * d.world, self._idev())
        return any(h == 1 for h in hits), done

    def _wait_chunk(self, ev):
        """step_host: make the compute stream wait for one column chunk's host
        copy (once per step, whichever attempt or probe first needs it)."""
        for e in (ev if isinstance(ev, (list, tuple)) else [ev]):
            if e is not None and id(e) not in self._waited:
                torch.cuda.current_stream(self.be.device).wait_event(e)
                self._waited.add(id(e))

    def _wait_chunks(self):
        for _, _, ev in self._chunks or ():
            self._wait_chunk(ev)

    def _local(self, k):
        if self._half_local is None or self._half_local.shape[0] < k:
            self._half_local = self.be.empty(max(k, 1), self.be.n)
        return self._half_local[:k]

    def _idev(self):
        """Device for the small status all-gathers: the GPU under NCCL, else CPU."""
        d = self.dist
        if not d.solo and d.td.get_backend(d.group) == "nccl":
            return self.be.device
        return torch.device("cpu")

    def step(self, it: int) -> Trace:
        tr = self._ks_step(it) if self.w.kind == "ks" else self._linear_step(it)
        return self.stops.update(tr)

    def _density(self, U, out):
        """density_from_orbitals (model.cpp:192-223): the nodal sum on this
        rank's slab rows, all-gathered, then normalised on the full density."""
        be = self.be
        total = be.density_rows(U, self.occ, self.slab.r0, self.slab.r1, out)
        self.dist.allgather_rows(out, self.slabs)
        be.density_normalize(total, out)
        return out

    def _ks_form(self, rho, vh, slot):
        """ks_form_matrix (paro.cpp:433-454). Sharded runs assemble the form on this rank's row slab
        (24 LDA evaluations per cell: the largest term that would otherwise be replicated) and
        all-gather the 8 coefficient slots; the clamp counts of the slabs' cells add up."""
        be, d = self.be, self.dist
        if d.solo or not hasattr(be, "ks_form_slab"):
            return be.ks_form(rho, vh, slot)
        op, cl = be.ks_form_slab(rho, vh, slot, self.slab.z0, self.slab.z1)
        slots = be.form_slots(op)
        for o in range(slots.shape[0]):
            d.allgather_rows(slots[o], self.slabs)
        cl = sum(d.allgather_ints([cl], [1] * d.world, self._idev()))
        return op, cl

    def _energy(self, lam, rho, vh):
        """total_energy (model.cpp:329-360). Sharded runs sum the XC term (24 LDA evaluations per
        cell) over the ranks' cell layers, added in rank order."""
        be, d = self.be, self.dist
        if d.solo or not hasattr(be, "energy_xc_layers"):
            return be.energy(lam, self.occ, rho, vh)
        # cell layers of this rank's slab; the top layer (k = S) goes with the last slab
        k1 = self.slab.z1 + 1 if self.slab.z1 == be.S else self.slab.z1
        part = torch.tensor([be.energy_xc_layers(rho, self.slab.z0, k1)], dtype=torch.float64, device=self._idev())
        d.allsum_(part)
        return be.energy_with_xc(lam, self.occ, rho, vh, float(part.item()))

    def _final_hook(self):
        """step_host at world size 1: Step 4 starts the host copy-out of the new
        orbitals as soon as they are final (before its Gram certificate)."""
        self._hooked = False
        if self._out is None or self.dist.world > 1:
            return None
        cs, h_orb = self._out[:2]
        main = torch.cuda.current_stream(self.be.device)

        def hook(V, k):
            cs.wait_stream(main)
            with torch.cuda.stream(cs):
                self._mark("d2h_start", cs)
                ev = self._copy_out_chunks(cs, h_orb, V, k)
                self._mark("d2h_end", cs)
            self._hooked = True
            return lambda: main.wait_event(ev)

        return hook

    def _copy_out_chunks(self, cs, h_orb, V, k):
        """This rank's block of the new orbitals to the host on stream cs (current),
        in the column chunks of the pipelined step_host when it set them (one
        event per chunk: the next step's copy-in of a chunk waits only for that
        chunk's copy-out). Returns the event after the last copy."""
        o0, o1, _ = self.dist.shard(k)
        pipelined = len(self._out) > 2
        ranges = self._out[2] if pipelined and self._out[2] else [(o0, o1)]
        self._d2h_events = []
        self._later_out = None
        ev = None
        for i, (k0, k1) in enumerate(ranges):
            a, b = max(k0, o0), min(k1, o1)
            if b <= a:
                continue
            if pipelined and i > 0:
                # the DMA queue is first-in first-out: the later pieces are queued at the end of
                # the step, behind the density's copy-out, which the next step needs first
                self._later_out = (V, [(max(p, o0), min(q, o1)) for p, q in ranges[i:]])
                break
            h_orb[a:b].copy_(V[a:b], non_blocking=True)
            ev = cs.record_event()
            self._d2h_events.append((a, b, ev))
        return ev if ev is not None else cs.record_event()

    def _to_columns(self):
        """Step 4's row slabs back to column shards for the next Step 3 (one
        all-to-all), and step_host's copy-out of this rank's block if Step 4
        did not start it."""
        d = self.dist
        d.slabs_to_cols(self.orb, d.shard(self.k)[2], self.slabs)
        if self._out is not None and not self._hooked:
            self._copy_out(self.orb[: self.k])

    def _copy_out(self, orb):
        """step_host: this rank's block of the new orbitals to the host (side stream)."""
        cs, h_orb = self._out[:2]
        cs.wait_stream(torch.cuda.current_stream(self.be.device))
        with torch.cuda.stream(cs):
            self._mark("d2h_start", cs)
            self._copy_out_chunks(cs, h_orb, orb, orb.shape[0])
            self._mark("d2h_end", cs)

    def step_host(self, it: int, h_orb: torch.Tensor, h_rho: torch.Tensor | None = None,
                  chunks: int = 2, pipelined: bool = False) -> Trace:
        """One outer iteration with the state in (pinned) host memory, the way
        a host caller of the reference interface holds it: the orbitals (and,
        for Kohn-Sham, the input density) are copied in, the new orbitals and
        the mixed density copied back out. The copies run on a side stream:
        the orbitals arrive in column chunks while the density-only work and
        the Step-3 solves of the earlier chunks run, and leave while the
        post-Step-4 density work runs. Returns when everything is back on the
        host side (h_orb, h_rho updated in place).

        pipelined=True makes the call stream-ordered instead: the copy-out runs
        on its own stream and the call returns without waiting for it; the next
        pipelined call's copy-in of a column chunk waits (on the device) for that
        chunk's copy-out only, so over PCIe's two directions a step's copy-out
        overlaps the next step's copy-in and first solves. The data still make
        the round trip through h_orb / h_rho every step; call host_join() before
        reading or writing them from the host."""
        be, d = self.be, self.dist
        dev = be.device
        main = torch.cuda.current_stream(dev)
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(dev)
        cs = self._copy_stream
        K = self.k
        c0, c1, _ = d.shard(K)
        if pipelined:
            if self._out_stream is None:
                self._out_stream = torch.cuda.Stream(dev)
            # the copy-in overwrites device state the previous step still read at its end
            if self._post_read is not None:
                cs.wait_event(self._post_read)
            else:
                cs.wait_stream(main)
            if self._rho_out_event is not None:
                cs.wait_event(self._rho_out_event)
        else:
            self.host_join()
            cs.wait_stream(main)
        with torch.cuda.stream(cs):
            if h_rho is not None:
                self.rho_in.copy_(h_rho, non_blocking=True)
                main.wait_event(cs.record_event())
            # the first chunk is small (a multiple of the 4-column groups) so
            # the Step-3 solves start early; the rest arrive while it runs
            kl = c1 - c0
            if chunks == 2:
                first = min(kl, max(4, (kl // 5 + 3) // 4 * 4))
                bounds = [c0, c0 + first, c1]
            elif chunks == 3:  # 8 / 24 / rest of 76: each chunk's solve covers the next one's copy
                first = min(kl, max(4, (kl // 10 + 3) // 4 * 4))
                bounds = [c0, c0 + first, min(c1, c0 + 4 * first), c1]
            else:
                bounds = [c0 + (kl * i) // chunks for i in range(chunks + 1)]
            ranges = [(bounds[i], bounds[i + 1]) for i in range(chunks) if bounds[i + 1] > bounds[i]]
            # pipelined: the copies move in finer pieces than the solves (a piece's copy-in
            # starts as soon as the previous step's copy-out of that piece is done), the
            # Step-3 batches stay the `ranges` and wait for every piece they contain
            pieces = ranges
            if pipelined:
                pieces = []
                for i0, (k0, k1) in enumerate(ranges):
                    # <= 20 columns per piece; the first batch in halves, so that its first half's
                    # copy-out (queued ahead of the density's) is short and its copy-in starts early
                    m = max(1, -(-(k1 - k0) // 20))
                    if i0 == 0 and k1 - k0 >= 8:
                        m = max(m, 2)
                    pieces += [(k0 + ((k1 - k0) * i) // m, k0 + ((k1 - k0) * (i + 1)) // m) for i in range(m)]
                # the NotSpd probe opens Step 3: the pieces that hold its columns travel first
                probe = [c for c in self._notspd_probe if c0 <= c < c1]
                pieces.sort(key=lambda r: not any(r[0] <= c < r[1] for c in probe))
            evs = []
            self._mark("h2d_start", cs)
            for k0, k1 in pieces:
                for a, b, ev in self._d2h_events:  # pipelined: the previous step's copy-out of these columns
                    if a < k1 and k0 < b:
                        cs.wait_event(ev)
                self.orb[k0:k1].copy_(h_orb[k0:k1], non_blocking=True)
                evs.append(cs.record_event())
                self._mark(f"h2d_cols_{k0}_{k1}", cs)
        self._d2h_events = []
        self._chunks = [(k0, k1, [ev for (a, b), ev in zip(pieces, evs) if a < k1 and k0 < b]) for k0, k1 in ranges]
        self._pieces = [(a, b, ev) for (a, b), ev in zip(pieces, evs)]
        self._waited = set()
        self._out = (self._out_stream, h_orb, pieces) if pipelined else (cs, h_orb)
        try:
            tr = self.step(it)
        finally:
            self._chunks, self._out, self._pieces = None, None, None
        main.wait_event(evs[-1])
        if not pipelined:
            if h_rho is not None:
                h_rho.copy_(self.rho_in, non_blocking=True)
            main.wait_stream(cs)
            self._d2h_events = []
            return tr
        self._post_read = main.record_event()  # every read of the device orbitals / densities of this step
        co = self._out_stream
        with torch.cuda.stream(co):
            if h_rho is not None:
                co.wait_event(self._post_read)
                h_rho.copy_(self.rho_in, non_blocking=True)
                self._rho_out_event = co.record_event()
            if self._later_out is not None:  # the rest of the orbitals (the first piece left inside Step 4)
                V, rest = self._later_out
                for a, b in rest:
                    if b > a:
                        h_orb[a:b].copy_(V[a:b], non_blocking=True)
                        self._d2h_events.append((a, b, co.record_event()))
                self._later_out = None
        return tr

    def host_join(self):
        """Make the current stream wait for the copy-outs of pipelined step_host
        calls (then a device synchronise makes h_orb / h_rho readable)."""
        if self._out_stream is not None:
            torch.cuda.current_stream(self.be.device).wait_stream(self._out_stream)
        self._d2h_events = []
        self._rho_out_event = None
        self._post_read = None

    def _ks_step(self, it: int) -> Trace:
        """paro.cpp:514-638 with adaptive = false; no stop tests."""
        w, be = self.w, self.be
        N_ = w.n_orbitals
        t0 = time.perf_counter()
        vh_in = be.hartree(self.rho_in, out=self.vh)
        # Step 2 on a fixed mesh: the estimator only feeds eta_total (paro.cpp:521-538)
        t2 = time.perf_counter()
        if self.estimate:
            self._wait_chunks()  # step_host: the estimator reads every orbital
        eta = be.estimate(self.orb[:N_], self.lambdas[:N_], self.rho_in, vh_in) if self.estimate else None
        t_meshgen = time.perf_counter() - t2
        a_in, cl = self._ks_form(self.rho_in, vh_in, "in")
        self.clamped += cl
        self._mark("step3_start")
        ts = time.perf_counter()
        sigma, iters = self.step3(a_in, it)
        self._mark("step3_end")
        self._sync()
        t_source = time.perf_counter() - ts
        tp = time.perf_counter()
        half = self.half[: self.k]
        rho_half = self._density(half[:N_], self.rho_half)
        vh_half = be.hartree(rho_half, out=self.vh)
        a_half, cl = self._ks_form(rho_half, vh_half, "half")
        self.clamped += cl
        orb, lam, defect = self.s4.ritz(half, a_half, be.mass_op(), N_, w.drop_tol, self.orb,
                                        on_final=self._final_hook())
        self._mark("ritz_end")
        self.k, self.lambdas = orb.shape[0], lam
        self._to_columns()
        self._sync()
        t_project = time.perf_counter() - tp
        rho_out = self._density(orb[:N_], self.rho_out)
        vh_out = be.hartree(rho_out, out=self.vh)
        e_tot = self._energy(lam, rho_out, vh_out)
        res = be.rho_residual(rho_out, self.rho_in)
        be.mix(self.rho_in, rho_out, w.mixing_alpha, out=self.rho_in)
        self._mark("step_end")
        self._sync()
        return Trace(it + 1, lam[: w.n_orbitals], e_tot, res, sigma, defect, iters, t_source, t_project,
                     time.perf_counter() - t0, eta, t_meshgen, be.n)

    def _linear_step(self, it: int) -> Trace:
        """paro.cpp:340-354."""
        w, be = self.w, self.be
        t0 = time.perf_counter()
        N_ = w.n_orbitals
        if self.estimate:
            self._wait_chunks()
        eta = be.estimate(self.orb[:N_], self.lambdas[:N_]) if self.estimate else None  # paro.cpp:306-315
        t_meshgen = time.perf_counter() - t0
        sigma, iters = self.step3(be.form, it)
        self._sync()
        t_source = time.perf_counter() - t0
        tp = time.perf_counter()
        orb, lam, defect = self.s4.ritz(self.half[: self.k], be.form, be.mass_op(), w.n_orbitals, w.drop_tol,
                                        self.orb, on_final=self._final_hook())
        self.k, self.lambdas = orb.shape[0], lam
        self._to_columns()
        self._sync()
        return Trace(it + 1, lam[: w.n_orbitals], None, None, sigma, defect, iters, t_source,
                     time.perf_counter() - tp, time.perf_counter() - t0, eta, t_meshgen, be.n)

    def run(self, iterations: int | None = None, stop: bool = False):
        """`iterations` outer iterations (default: the workload's count). With
        stop=True the reference's own control applies (max_outer = iterations):
        return at the first converged row, raise ScfDivergenceError at a
        divergent one (paro.cpp:618-635)."""
        out = []
        for i in range(iterations if iterations is not None else self.w.iterations):
            tr = self.step(i)
            out.append(tr)
            if stop and tr.diverged:
                raise N.ScfDivergenceError(
                    "kohn-sham: total energy increased for 5 consecutive iterations without density-residual "
                    "progress; consider a smaller mixing_alpha")
            if stop and tr.converged:
                break
        return out
