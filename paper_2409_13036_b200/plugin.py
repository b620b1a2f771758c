"""Drop-in seam for the reference package.

``rafem.fem.corrector_step`` reaches assembly and solve through the module
globals ``rafem.fem.assemble_global`` and ``rafem.fem.solve`` (fem.py:47-48,
492, 501).  ``install()`` rebinds both to the B200 path; exceptions are
re-raised as the reference's own classes so its corrector handles them
exactly as before (SolverError -> step failure, fem.py:511-515).
"""

from __future__ import annotations

import importlib

from . import assembly, krylov

_saved: dict = {}


def _wrap(rafem_solver, rafem_fem):
    def assemble_global(mesh, material, config, t_iter, v_iter, t_prev, dt, apply_constraints=True,
                        equilibrate=True, threads=None):
        try:
            return assembly.assemble_global(mesh, material, config, t_iter, v_iter, t_prev, dt,
                                            apply_constraints, equilibrate, threads)
        except assembly.PhysicsRangeError as exc:
            raise rafem_fem.PhysicsRangeError(str(exc)) from None

    def solve(a, b, x0=None, config=None, session=None, tracer=None, trace_step=-1,
              trace_corrector_iter=-1):
        try:
            x, st = krylov.solve(a, b, x0=x0, config=config, session=session, tracer=tracer,
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


def install(module: str = "rafem.fem") -> None:
    """Route the reference corrector's assembly and solve through the B200 path."""
    fem = importlib.import_module(module)
    solver = importlib.import_module(module.rsplit(".", 1)[0] + ".solver")
    if module not in _saved:
        _saved[module] = (fem.assemble_global, fem.solve)
    fem.assemble_global, fem.solve = _wrap(solver, fem)


def uninstall(module: str = "rafem.fem") -> None:
    fem = importlib.import_module(module)
    if module in _saved:
        fem.assemble_global, fem.solve = _saved.pop(module)
