"""The callers of the hot path: predictor-corrector time loop.

Two drivers with the reference's semantics (fem.py:437-644):

* ``run_simulation`` — the host loop exactly as the reference structures
  it, calling ``assemble_global`` and ``solve`` through this module's
  globals (the same plug-in seam the reference has at fem.py:47-48), with
  host numpy buffers crossing the boundary every pass.  This is the
  drop-in path a reference user gets.
* ``simulate_device`` — the same loop run natively by librafem_b200
  (``rafem_simulate``): mesh, system, iterates and solver state stay in
  HBM and the host reads one small status block per corrector pass.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .assembly import (MaterialParams, PhysicsRangeError, SimConfig, SystemHandle,
                       assemble_global, device_mesh)
from .krylov import SolverError, SolverSession, solve

__all__ = [
    "CorrectorOutcome", "SimState", "SimulationSummary", "StepFailureError", "StepRecord",
    "corrector_step", "initial_state", "interleave_fields", "predictor", "run_simulation",
    "simulate_device", "split_fields",
]


class StepFailureError(RuntimeError):
    """Corrector failed with dt already at its floor (fem.py:76-82)."""

    def __init__(self, step: int, dt: float):
        self.step = step
        self.dt = dt
        super().__init__(f"step {step} failed to converge with dt already at the floor ({dt:g} s)")


@dataclass
class StepRecord:
    """One accepted step (results.py StepRecord)."""

    step: int
    time: float
    dt: float
    corrector_iters: int
    converged: bool
    T: np.ndarray
    V: np.ndarray


@dataclass
class SimState:
    step: int
    t: float
    dt: float
    dt_prev: float
    T: np.ndarray
    V: np.ndarray
    T_prev: np.ndarray
    corrector_iters_last: int = 0
    converged_last: bool = True


def initial_state(mesh, config) -> SimState:
    t0 = np.full(mesh.node_count, config.initial_temp)
    return SimState(step=0, t=0.0, dt=config.dt_init, dt_prev=config.dt_init, T=t0,
                    V=np.zeros(mesh.node_count), T_prev=t0.copy())


def interleave_fields(v, t):
    x = np.empty(2 * v.size)
    x[0::2] = v
    x[1::2] = t
    return x


def split_fields(x):
    return x[0::2].copy(), x[1::2].copy()


def predictor(state: SimState, dt: float):
    """T extrapolated through the last two accepted fields (fem.py:437-449)."""
    if state.step >= 1:
        return state.T + (dt / state.dt_prev) * (state.T - state.T_prev), state.V.copy()
    return state.T.copy(), state.V.copy()


@dataclass
class CorrectorOutcome:
    converged: bool
    iterations: int
    T: np.ndarray | None = None
    V: np.ndarray | None = None
    delta: float = np.inf
    solver_iterations: int = 0
    cause: str | None = None


def corrector_step(mesh, material, config, state, dt, start=None, session=None, tracer=None):
    """Picard loop of one time step (fem.py:463-540) over the device plug-ins."""
    t_it, v_it = predictor(state, dt) if start is None else start
    x_old = interleave_fields(v_it, t_it)
    total_inner = 0
    delta = np.inf
    for it in range(1, config.max_corrector_iters + 1):
        system = assemble_global(mesh, material, config, t_it, v_it, state.T, dt,
                                 threads=config.threads)
        rhs_staged = system.rhs.copy()
        x0_staged = x_old.copy()
        try:
            x_new, stats = solve(system.matrix, rhs_staged, x0=x0_staged, config=config.solver,
                                 session=session, tracer=tracer, trace_step=state.step,
                                 trace_corrector_iter=it)
        except SolverError as exc:
            return CorrectorOutcome(False, it, solver_iterations=total_inner, cause=f"solver: {exc}")
        total_inner += stats.iterations
        if not stats.converged:
            return CorrectorOutcome(
                False, it, solver_iterations=total_inner,
                cause=(f"solver stalled at relative residual {stats.final_relative_residual:.3e}"
                       + (" (stagnated)" if stats.stagnated else "")))
        delta = float(np.max(np.abs(x_new - x_old) / np.maximum(1.0, np.abs(x_old))))
        v_it, t_it = split_fields(x_new)
        x_old = x_new
        if delta < config.corrector_tol:
            return CorrectorOutcome(True, it, T=t_it, V=v_it, delta=delta, solver_iterations=total_inner)
    return CorrectorOutcome(False, config.max_corrector_iters, delta=delta,
                            solver_iterations=total_inner, cause="corrector iteration cap reached")


@dataclass
class SimulationSummary:
    state: SimState
    accepted_steps: int
    total_corrector_iters: int
    total_solver_iterations: int
    dt_halvings: int
    orderings_computed: int
    wall_ns: int
    passes: int = 0
    device_assemble_ms: float = 0.0
    device_solve_ms: float = 0.0


def run_simulation(mesh, material, config, sink=None, tracer=None, fault_hook=None) -> SimulationSummary:
    """Adaptive predictor-corrector loop (fem.py:554-644) on the device plug-ins."""
    t_wall = time.perf_counter_ns()
    state = initial_state(mesh, config)
    session = SolverSession()
    total_corr = total_inner = halvings = attempt = 0
    while state.t < config.total_time:
        remaining = config.total_time - state.t
        final = state.dt >= remaining
        dt = remaining if final else state.dt
        start = predictor(state, dt)
        if fault_hook is not None and fault_hook(state.step, attempt):
            outcome = CorrectorOutcome(False, 0, cause="injected fault")
        else:
            outcome = corrector_step(mesh, material, config, state, dt, start=start,
                                     session=session, tracer=tracer)
        total_corr += outcome.iterations
        total_inner += outcome.solver_iterations
        state.corrector_iters_last = outcome.iterations
        state.converged_last = outcome.converged
        if outcome.converged:
            state.T_prev = state.T
            state.T, state.V = outcome.T, outcome.V
            state.dt_prev = dt
            state.t = config.total_time if final else state.t + dt
            rec = StepRecord(state.step, state.t, dt, outcome.iterations, True, state.T, state.V)
            state.step += 1
            attempt = 0
            if sink is not None:
                sink(rec)
            if outcome.iterations <= 5:
                state.dt = min(dt * 1.5, config.dt_max)
            elif outcome.iterations >= 20:
                state.dt = max(dt * 0.75, config.dt_min)
            else:
                state.dt = dt
        else:
            if dt <= config.dt_min:
                raise StepFailureError(state.step, dt)
            state.dt = max(dt * 0.5, config.dt_min)
            halvings += 1
            attempt += 1
    return SimulationSummary(state, state.step, total_corr, total_inner, halvings,
                             session.orderings_computed, time.perf_counter_ns() - t_wall)


# ---------------------------------------------------------------------------
# native loop

def _sim_params(config, record_fields: bool, max_steps: int | None) -> nat.SimParams:
    from .krylov import _params
    s = config.solver
    if s.backend not in ("gmres", "pcg"):
        raise NotImplementedError(f"backend {s.backend!r} is not a device backend")
    p = nat.SimParams()
    p.total_time = config.total_time
    p.dt_init = config.dt_init
    p.dt_min = config.dt_min
    p.dt_max = config.dt_max
    p.corrector_tol = config.corrector_tol
    p.max_corrector_iters = config.max_corrector_iters
    p.record_fields = 1 if record_fields else 0
    p.applied_voltage = config.applied_voltage
    p.boundary_temp = config.boundary_temp
    p.initial_temp = config.initial_temp
    p.max_steps = int(max_steps or 0)
    p.solver = _params(s, nat.METHOD_PCG if s.backend == "pcg" else nat.METHOD_GMRES)
    return p


class DeviceRun:
    """Reusable native simulation on one mesh (keeps the device system)."""

    def __init__(self, mesh, material=None, cached: bool = True):
        from .assembly import DeviceMesh
        self.mesh = mesh
        self.material = material or MaterialParams.default()
        # cached=False uploads the mesh and redoes the symbolic phase (a
        # cold start: what a fresh process or a new mesh costs)
        self.dm = device_mesh(mesh, self.material) if cached else DeviceMesh(mesh, self.material)
        self.sys = SystemHandle(self.dm)

    @classmethod
    def from_device_mesh(cls, dm, material=None) -> "DeviceRun":
        """A run on a mesh that only exists in HBM (DeviceMesh.from_box)."""
        self = cls.__new__(cls)
        self.mesh = None
        self.material = material or MaterialParams.default()
        self.dm = dm
        self.sys = SystemHandle(dm)
        return self

    def run_streamed(self, config, sink, max_steps=None, ring_slots=8):
        """Like run(record_fields=True) but each accepted step's fields reach
        ``sink`` while the simulation is still running (rafem_simulate_stream:
        device ring + mapped progress counters, bounded memory)."""
        N = self.dm.node_count
        p = _sim_params(config, True, max_steps)
        out = nat.SimSummaryC()
        err = []

        def cb(_user, step, t, dt, iters, x):
            try:
                xa = np.ctypeslib.as_array(x, shape=(2 * N,))
                sink(StepRecord(int(step), float(t), float(dt), int(iters), True, xa[1::2].copy(), xa[0::2].copy()))
                return 0
            except Exception as exc:  # noqa: BLE001 - surfaced after the run
                err.append(exc)
                return 1

        fn = nat.RECORD_FN(cb)
        rc = nat.lib().rafem_simulate_stream(self.sys.handle, C.byref(p), C.byref(out), int(ring_slots),
                                             C.cast(fn, C.c_void_p), None)
        if err:
            raise err[0]
        if rc == nat.ERR_STEP_FAILURE:
            raise StepFailureError(int(out.failed_step), float(out.failed_dt))
        if rc == nat.ERR_PHYSICS:
            raise PhysicsRangeError(nat.last_error())
        nat.check(rc, "simulate_stream")
        return out

    def _run_collect(self, config, sink, max_steps, keep=True):
        """Records through run_streamed (bounded device memory, no step cap)."""
        records = []

        def take(rec):
            if keep:
                records.append(rec)
            if sink is not None:
                sink(rec)
        out = self.run_streamed(config, take, max_steps)
        self._note_mode()
        return records, out

    def _note_mode(self):
        mode, ctas = C.c_int32(), C.c_int32()
        nat.lib().rafem_last_solve_mode(nat.context(), C.byref(mode), C.byref(ctas))
        self.last_mode = {6: "cluster-simulation", 5: "cluster-pcg", 4: "kernel-per-phase-pcg",
                          3: "grid-streaming-pcg", 2: "fused-simulation", 1: "cluster", 0: "grid"}.get(mode.value, "none")
        self.last_ctas = ctas.value
        self.last_precond = nat.last_solve_precond()

    def run(self, config, sink=None, record_fields=True, max_steps=None, rec_cap=None):
        """Run the simulation; returns (records, SimSummaryC).

        Field records go to host buffers sized up front (2 x total/dt_init +
        64 steps).  When those would exceed 8 GB, or the run accepts more
        steps than they hold (dt shrinking on hard physics), the records
        are delivered through the streaming path instead (the run is
        deterministic, so a re-run reproduces it exactly)."""
        N = self.dm.node_count
        # dt only shrinks on hard steps, so 2 x total/dt_init bounds typical runs;
        # np.zeros is lazily paged, so the generous field buffer costs nothing unused
        est = rec_cap or int(2 * config.total_time / config.dt_init) + 64
        est = min(est, 200000)
        if max_steps:
            est = min(est, int(max_steps))
        if record_fields and rec_cap is None and est * 16 * max(N, 1) > 8e9:
            return self._run_collect(config, sink, max_steps)
        rec_step = np.zeros(est, dtype=np.int64)
        rec_time = np.zeros(est)
        rec_dt = np.zeros(est)
        rec_it = np.zeros(est, dtype=np.int32)
        rec_x = np.zeros((est, 2 * N)) if record_fields else None
        p = _sim_params(config, record_fields, max_steps)
        out = nat.SimSummaryC()
        rc = nat.lib().rafem_simulate(self.sys.handle, C.byref(p), C.byref(out), est, nat.ptr(rec_step),
                                      nat.ptr(rec_time), nat.ptr(rec_dt), nat.ptr(rec_it),
                                      nat.ptr(rec_x))
        self._note_mode()
        if rc == nat.ERR_STEP_FAILURE:
            raise StepFailureError(int(out.failed_step), float(out.failed_dt))
        if rc == nat.ERR_PHYSICS:
            raise PhysicsRangeError(nat.last_error())
        nat.check(rc, "simulate")
        nsteps = int(out.accepted_steps)
        if nsteps > est and rec_cap is None:
            import warnings
            warnings.warn(f"{nsteps} accepted steps exceed the {est}-record buffer; re-running through the "
                          "record stream", RuntimeWarning, stacklevel=2)
            if record_fields:
                return self._run_collect(config, sink, max_steps)
            _, out2 = self._run_collect(config, None, max_steps, keep=False)
            return [], out2
        records = []
        for k in range(min(nsteps, est)):
            if record_fields:
                x = rec_x[k]
                T, V = x[1::2].copy(), x[0::2].copy()
            else:
                T = V = None
            rec = StepRecord(int(rec_step[k]), float(rec_time[k]), float(rec_dt[k]), int(rec_it[k]),
                             True, T, V)
            records.append(rec)
            if sink is not None:
                sink(rec)
        return records, out


def simulate_device(mesh, material, config, sink=None, record_fields=True, max_steps=None, cached=True):
    """Native run_simulation; returns (records, SimSummaryC)."""
    return DeviceRun(mesh, material, cached=cached).run(config, sink=sink, record_fields=record_fields,
                                                        max_steps=max_steps)
