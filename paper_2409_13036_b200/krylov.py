"""Solver plug-in: the reference's ``solve`` contract on B200 Krylov kernels.

Mirrors rafem/solver.py's public surface for the iterative path:
``SolverConfig`` (solver.py:81-110), ``SolveStats`` (113-130), the error
taxonomy (57-78) and ``solve`` (580-636) with the same signature, argument
meaning and exceptions.  Backends:

* ``"gmres"``  — restarted GMRES(m) with Givens least squares and optional
  right Jacobi, the reference's algorithm (solver.py:381-531), run as ONE
  persistent cooperative kernel per solve (CGS2 Arnoldi, deterministic
  reductions).  Same stats semantics: inner iterations, restarts, per-cycle
  non-increasing residual history, true final residual, stagnation latch,
  breakdown rules.
* ``"pcg"``    — Jacobi-preconditioned CG for the SPD FEM systems (new
  backend name; never substituted for "gmres").  Converged only when the
  true residual meets the tolerance.
* ``"qr"``, ``"dense"`` — the reference's direct solvers are outside the
  device path (dense n x n storage) and raise
  NotImplementedError.

There is no CPU fallback anywhere on this path.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .csr import CsrMatrix, DeviceCsrMatrix

__all__ = [
    "BACKENDS", "GmresBreakdownError", "KrylovBreakdownError", "SizeCapError", "SolveStats",
    "SolverConfig", "SolverError", "SolverSession", "SingularMatrixError", "ReuseRejectedError",
    "gmres", "pcg", "solve",
]

BACKENDS = ("qr", "gmres", "dense", "pcg")
DEVICE_BACKENDS = ("gmres", "pcg")
PRECONDITIONERS = ("none", "jacobi", "block_jacobi")  # block_jacobi: this package (rafem_b200.h)
ORDERINGS = ("none", "rcm")


class SolverError(Exception):
    """Base class for solver failures (solver.py:57-58)."""


class SingularMatrixError(SolverError):
    def __init__(self, pivot: int, message: str | None = None):
        self.pivot = pivot
        super().__init__(message or f"matrix is singular at pivot {pivot}")


class ReuseRejectedError(SolverError):
    pass


class GmresBreakdownError(SolverError):
    """Arnoldi produced a zero vector before reaching the tolerance (solver.py:73-74)."""


class KrylovBreakdownError(SolverError):
    """CG met a non-positive curvature (the operator is not SPD under Jacobi)."""


class SizeCapError(SolverError):
    pass


@dataclass
class SolverConfig:
    """Backend selection and tuning (solver.py:81-110, plus backend "pcg").

    ``grid_ctas`` (device only) pins the persistent kernel's CTA count;
    0 lets the library size it.
    """

    backend: str = "qr"
    restart_m: int = 30
    tolerance: float = 1e-10
    max_total_iters: int | None = None
    precondition: str = "none"
    reuse_ordering: bool = False
    ordering: str = "rcm"
    grid_ctas: int = 0

    def __post_init__(self):
        if self.backend not in BACKENDS:
            raise ValueError(f"backend must be one of {BACKENDS}, got {self.backend!r}")
        if self.restart_m < 1:
            raise ValueError("restart_m must be at least 1")
        if not (0.0 < self.tolerance < 1.0):
            raise ValueError("tolerance must lie in (0, 1)")
        if self.max_total_iters is not None and self.max_total_iters < 1:
            raise ValueError("max_total_iters must be positive when given")
        if self.precondition not in PRECONDITIONERS:
            raise ValueError(f"precondition must be one of {PRECONDITIONERS}")
        if self.ordering not in ORDERINGS:
            raise ValueError(f"ordering must be one of {ORDERINGS}")


@dataclass
class SolveStats:
    """Observability record returned by every solve (solver.py:113-130)."""

    iterations: int = 0
    restarts: int = 0
    final_relative_residual: float = 0.0
    stagnated: bool = False
    factor_nnz: int = 0
    wall_ns: int = 0
    converged: bool = True
    ordering_ns: int = 0
    residual_history: list = field(default_factory=list)
    device_ms: float = 0.0
    # the preconditioner the device solve applied: "block_jacobi" requests
    # are served by point Jacobi outside the paper-scale pipelined PCG
    precondition_applied: str = "none"


@dataclass
class SolverSession:
    """Per-run cache (solver.py:165-170); the device path keeps its state in the library."""

    factors: object = None
    orderings_computed: int = 0


def _check_system(a, b) -> np.ndarray:
    if a.nrows != a.ncols:
        raise ValueError(f"matrix must be square, got {a.nrows} x {a.ncols}")
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.shape != (a.nrows,):
        raise ValueError(f"right-hand side has shape {b.shape}, expected ({a.nrows},)")
    if not np.all(np.isfinite(b)):
        raise ValueError("right-hand side contains non-finite entries")
    return b


def _check_x0(x0, n):
    if x0 is None:
        return None
    x = np.ascontiguousarray(x0, dtype=np.float64)
    if x.shape != (n,):
        raise ValueError(f"initial guess has shape {x.shape}, expected ({n},)")
    if not np.all(np.isfinite(x)):
        raise ValueError("initial guess contains non-finite entries")
    return x


def _params(cfg, method: int) -> nat.SolverParams:
    p = nat.SolverParams()
    p.method = method
    p.restart_m = int(cfg.restart_m)
    p.tolerance = float(cfg.tolerance)
    p.max_total_iters = int(cfg.max_total_iters) if cfg.max_total_iters is not None else 0
    p.precondition = {"jacobi": nat.PRECOND_JACOBI, "block_jacobi": nat.PRECOND_BLOCK_JACOBI}.get(
        cfg.precondition, nat.PRECOND_NONE)
    p.grid_ctas = int(getattr(cfg, "grid_ctas", 0) or 0)
    return p


_HIST_BUF: list = [np.empty(0), np.empty(0, dtype=np.int64)]


def _history_buffers(cap):
    """Reused host buffers for the residual history and the cycle lengths
    (their contents are copied into Python lists before a solve returns)."""
    if _HIST_BUF[0].size < cap:
        _HIST_BUF[0] = np.empty(cap)
        _HIST_BUF[1] = np.empty(cap, dtype=np.int64)
    return _HIST_BUF[0][:cap], _HIST_BUF[1][:cap]


def _device_solve(a, b, x0, cfg, method):
    n = a.nrows
    x = np.empty(n)
    st = nat.SolveStatsC()
    cap = int(cfg.max_total_iters) if cfg.max_total_iters is not None else 10 * n
    hist_cap = min(cap, 1 << 20) + 1
    hist, cyc = _history_buffers(hist_cap)
    p = _params(cfg, method)
    L = nat.lib()
    if isinstance(a, DeviceCsrMatrix):
        rc = a.device_system.solve(b, x0, p, x, st, hist, cyc)
    else:
        ctx = nat.context()
        h = C.c_void_p()
        nat.check(L.rafem_matrix_create(ctx, n, a.nnz, nat.ptr(a.row_ptr), nat.ptr(a.col_idx),
                                        nat.ptr(a.vals), C.byref(h)), "matrix upload")
        try:
            rc = L.rafem_matrix_solve(h, nat.ptr(b), nat.ptr(x0), C.byref(p), nat.ptr(x), C.byref(st),
                                      nat.ptr(hist), hist_cap, nat.ptr(cyc), hist_cap)
        finally:
            L.rafem_matrix_destroy(h)
    stats = SolveStats()
    stats.iterations = int(st.iterations)
    stats.restarts = int(st.restarts)
    stats.final_relative_residual = float(st.final_relative_residual)
    stats.converged = bool(st.converged)
    stats.stagnated = bool(st.stagnated)
    stats.device_ms = float(st.device_ms)
    stats.precondition_applied = nat.last_solve_precond()
    ncyc = min(int(st.cycles), hist_cap)
    lens = cyc[:ncyc]
    hl = min(int(st.history_len), hist_cap)
    hv = hist[:hl]
    out, pos = [], 0
    for ln in lens:
        ln = int(ln)
        out.append([float(v) for v in hv[pos:pos + ln]])
        pos += ln
    stats.residual_history = out
    if rc == nat.ERR_BREAKDOWN:
        msg = nat.last_error()
        raise (KrylovBreakdownError if method == nat.METHOD_PCG else GmresBreakdownError)(msg)
    if rc == nat.ERR_INVALID:
        raise ValueError(nat.last_error())
    nat.check(rc, "solve")
    return x, stats


def gmres(a: CsrMatrix, b: np.ndarray, x0: np.ndarray | None, config: SolverConfig):
    """Restarted GMRES(m) on the device; returns ``(x, SolveStats)`` (solver.py:381-531)."""
    b = _check_system(a, b)
    x0 = _check_x0(x0, a.nrows)
    if a.nrows == 0:
        return np.zeros(0), SolveStats()
    return _device_solve(a, b, x0, config, nat.METHOD_GMRES)


def pcg(a: CsrMatrix, b: np.ndarray, x0: np.ndarray | None, config: SolverConfig):
    """Jacobi-preconditioned CG on the device; returns ``(x, SolveStats)``."""
    b = _check_system(a, b)
    x0 = _check_x0(x0, a.nrows)
    if a.nrows == 0:
        return np.zeros(0), SolveStats()
    return _device_solve(a, b, x0, config, nat.METHOD_PCG)


def solve(a, b, x0=None, config=None, session=None, tracer=None, trace_step=-1,
          trace_corrector_iter=-1):
    """Dispatch on ``config.backend``; returns ``(x, SolveStats)`` (solver.py:580-636).

    ``config`` may be this module's SolverConfig or the reference's (any
    object with the same fields).  ``session``/``tracer`` are accepted for
    signature compatibility; device timings are in ``stats.device_ms``.
    """
    config = config if config is not None else SolverConfig()
    b = _check_system(a, b)
    backend = config.backend
    if backend not in DEVICE_BACKENDS:
        raise NotImplementedError(
            f"backend {backend!r} is a direct CPU solver outside the B200 path; "
            "use backend='gmres' (reference algorithm) or 'pcg'")
    t0 = time.perf_counter_ns()
    # b is checked above; gmres()/pcg() would check it a second time
    x0 = _check_x0(x0, a.nrows)
    if a.nrows == 0:
        x, stats = np.zeros(0), SolveStats()
    else:
        x, stats = _device_solve(a, b, x0, config, nat.METHOD_GMRES if backend == "gmres" else nat.METHOD_PCG)
    stats.wall_ns = max(time.perf_counter_ns() - t0, 1)
    return x, stats


def relative_residual(a, x, b) -> float:
    """||b - A x|| / ||b|| through the device SpMV (helper for callers and tests)."""
    from .csr import spmv
    bn = float(np.linalg.norm(b))
    return float(np.linalg.norm(b - spmv(a, x))) / bn if bn else 0.0

