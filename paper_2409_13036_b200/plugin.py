"""Drop-in seam for the reference package.

``rafem.fem.corrector_step`` reaches assembly and solve through the module
globals ``rafem.fem.assemble_global`` and ``rafem.fem.solve`` (fem.py:47-48,
492, 501).  ``install()`` rebinds both to the B200 path; exceptions are
re-raised as the reference's own classes so its corrector handles them
exactly as before (SolverError -> step failure, fem.py:511-515).

Backends: the reference's iterative backend (``"gmres"``) runs on the
device GMRES(m).  Its direct backends (``"qr"``, ``"dense"``; dense n x n
storage, outside the device path) are passed through to the reference's
own ``solve`` unchanged, so a run configured for them behaves exactly as
without the seam.  ``install(solver="pcg")`` is an explicit opt-in that
serves ``"gmres"`` configurations with the device PCG instead (the FEM
systems are SPD) — never a silent substitution.
"""

from __future__ import annotations

import importlib
from dataclasses import dataclass, field

from . import assembly, krylov

_saved: dict = {}


@dataclass
class SeamCounters:
    """Calls that went through the seam (tests assert the device path ran)."""

    assemble: int = 0
    solve_device: int = 0
    solve_passthrough: int = 0
    backends: dict = field(default_factory=dict)


counters = SeamCounters()


class _Routed:
    """A SolverConfig view with the backend / preconditioner the seam chose."""

    def __init__(self, cfg, backend, precondition):
        self._cfg = cfg
        self.backend = backend
        self.precondition = precondition

    def __getattr__(self, name):
        return getattr(self._cfg, name)


def _wrap(rafem_solver, rafem_fem, orig_solve, solver, precondition):
    def assemble_global(mesh, material, config, t_iter, v_iter, t_prev, dt, apply_constraints=True,
                        equilibrate=True, threads=None):
        counters.assemble += 1
        try:
            return assembly.assemble_global(mesh, material, config, t_iter, v_iter, t_prev, dt,
                                            apply_constraints, equilibrate, threads)
        except assembly.PhysicsRangeError as exc:
            raise rafem_fem.PhysicsRangeError(str(exc)) from None

    def solve(a, b, x0=None, config=None, session=None, tracer=None, trace_step=-1,
              trace_corrector_iter=-1):
        cfg = config if config is not None else rafem_solver.SolverConfig()
        if cfg.backend not in krylov.DEVICE_BACKENDS:
            # direct solvers stay on the reference's own CPU implementation
            counters.solve_passthrough += 1
            rsparse = importlib.import_module(rafem_solver.__name__.rsplit(".", 1)[0] + ".sparse")
            if not isinstance(a, rsparse.CsrMatrix):
                a = rsparse.CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_idx, a.vals)
            return orig_solve(a, b, x0=x0, config=config,
                              session=session, tracer=tracer, trace_step=trace_step,
                              trace_corrector_iter=trace_corrector_iter)
        if solver is not None and cfg.backend == "gmres":
            cfg = _Routed(cfg, solver, precondition or cfg.precondition)
        counters.solve_device += 1
        counters.backends[cfg.backend] = counters.backends.get(cfg.backend, 0) + 1
        try:
            x, st = krylov.solve(a, b, x0=x0, config=cfg, session=session, tracer=tracer,
                                 trace_step=trace_step, trace_corrector_iter=trace_corrector_iter)
        except krylov.GmresBreakdownError as exc:
            raise rafem_solver.GmresBreakdownError(str(exc)) from None
        except krylov.SolverError as exc:
            raise rafem_solver.SolverError(str(exc)) from None
        out = rafem_solver.SolveStats(
            iterations=st.iterations, restarts=st.restarts,
            final_relative_residual=st.final_relative_residual, stagnated=st.stagnated,
            wall_ns=st.wall_ns, converged=st.converged, residual_history=st.residual_history)
        return x, out

    return assemble_global, solve


def install(module: str = "rafem.fem", solver: str | None = None, precondition: str | None = None) -> None:
    """Route the reference corrector's assembly and solve through the B200 path.

    ``solver``: None keeps the configured backend (``"gmres"`` -> device
    GMRES); ``"pcg"`` serves ``"gmres"`` configurations with the device PCG
    (``precondition`` overrides the configured preconditioner then)."""
    if solver not in (None, "gmres", "pcg"):
        raise ValueError(f"solver must be None, 'gmres' or 'pcg', got {solver!r}")
    fem = importlib.import_module(module)
    rsolver = importlib.import_module(module.rsplit(".", 1)[0] + ".solver")
    if module not in _saved:
        _saved[module] = (fem.assemble_global, fem.solve)
    fem.assemble_global, fem.solve = _wrap(rsolver, fem, _saved[module][1], solver, precondition)


def uninstall(module: str = "rafem.fem") -> None:
    fem = importlib.import_module(module)
    if module in _saved:
        fem.assemble_global, fem.solve = _saved.pop(module)
