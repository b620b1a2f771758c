"""ctypes binding of librafem_b200.so (include/rafem_b200.h).

The library is built in-tree by ``paper_2409_13036_b200.build``.  There is
no CPU fallback: if the shared object is missing or no CUDA device is
visible, every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RAFEM_LIB") or os.path.join(HERE, "librafem_b200.so")  # RAFEM_LIB: A/B builds

OK = 0
ERR_BREAKDOWN = 1
ERR_INVALID = 2
ERR_PHYSICS = 3
ERR_UNSUPPORTED = 4
ERR_STEP_FAILURE = 5
ERR_CUDA = -1

METHOD_GMRES = 0
METHOD_PCG = 1
PRECOND_NONE = 0
PRECOND_JACOBI = 1
PRECOND_BLOCK_JACOBI = 2

DOF_FREE = 0
DOF_APPLIED_VOLTAGE = 1
DOF_ZERO = 2
DOF_BOUNDARY_TEMP = 3

i32, i64, f64, u8 = C.c_int32, C.c_int64, C.c_double, C.c_uint8
vp = C.c_void_p


class SolverParams(C.Structure):
    _fields_ = [("method", i32), ("restart_m", i32), ("tolerance", f64),
                ("max_total_iters", i64), ("precondition", i32), ("grid_ctas", i32)]


class SolveStatsC(C.Structure):
    _fields_ = [("iterations", i64), ("restarts", i64), ("final_relative_residual", f64),
                ("converged", i32), ("stagnated", i32), ("cycles", i64),
                ("history_len", i64), ("device_ms", f64)]


class AssembleParams(C.Structure):
    _fields_ = [("dt", f64), ("applied_voltage", f64), ("boundary_temp", f64),
                ("apply_constraints", i32), ("equilibrate", i32)]


class SimParams(C.Structure):
    _fields_ = [("total_time", f64), ("dt_init", f64), ("dt_min", f64), ("dt_max", f64),
                ("corrector_tol", f64), ("max_corrector_iters", i32), ("record_fields", i32),
                ("applied_voltage", f64), ("boundary_temp", f64), ("initial_temp", f64),
                ("max_steps", i64), ("solver", SolverParams)]


class SimSummaryC(C.Structure):
    _fields_ = [("accepted_steps", i64), ("total_corrector_iters", i64),
                ("total_solver_iterations", i64), ("dt_halvings", i64), ("passes", i64),
                ("final_time", f64), ("status", i32), ("failed_step", i32), ("failed_dt", f64),
                ("wall_ms", f64), ("assemble_ms", f64), ("solve_ms", f64), ("bad_element", i64)]


P = C.POINTER
# rafem_record_fn: (user, step, time, dt, corrector_iters, x[2N]) -> status
RECORD_FN = C.CFUNCTYPE(i32, vp, i64, f64, f64, i32, P(f64))
_SIGS = {
    "rafem_ctx_create": (i32, [C.c_int, P(vp)]),
    "rafem_ctx_destroy": (None, [vp]),
    "rafem_last_error": (C.c_char_p, [vp]),
    "rafem_device_info": (i32, [vp, P(i32), P(i32), P(i32), P(i64)]),
    "rafem_kernel_launches": (i64, [vp]),
    "rafem_stream": (vp, [vp]),
    "rafem_last_solve_mode": (i32, [vp, P(i32), P(i32)]),
    "rafem_last_solve_precond": (i32, [vp, P(i32)]),
    "rafem_set_trace": (i32, [vp, i32]),
    "rafem_get_trace": (i64, [vp, vp, i64]),
    "rafem_spmv": (i32, [vp, i64, i64, i64, vp, vp, vp, vp, vp]),
    "rafem_coo_to_csr": (i32, [vp, i64, i64, i64, vp, vp, vp, vp, vp, vp, P(i64)]),
    "rafem_matrix_create": (i32, [vp, i64, i64, vp, vp, vp, P(vp)]),
    "rafem_matrix_destroy": (None, [vp]),
    "rafem_matrix_solve": (i32, [vp, vp, vp, P(SolverParams), vp, P(SolveStatsC), vp, i64, vp, i64]),
    "rafem_mesh_create": (i32, [vp, i64, vp, i64, vp, vp, i32, vp, vp, vp, vp, vp, vp, P(vp)]),
    "rafem_mesh_destroy": (None, [vp]),
    "rafem_mesh_set_geometry": (i32, [vp, vp, vp]),
    "rafem_mesh_slots": (i64, [vp]),
    "rafem_mesh_stencil_classes": (i32, [vp]),
    "rafem_mesh_pattern": (i32, [vp, vp, vp]),
    "rafem_mesh_set_shard_order": (i32, [vp, i64, i64]),
    "rafem_system_create": (i32, [vp, P(vp)]),
    "rafem_system_destroy": (None, [vp]),
    "rafem_assemble": (i32, [vp, vp, vp, vp, P(AssembleParams), P(f64), P(i64)]),
    "rafem_assemble_rhs": (i32, [vp, vp, vp, vp, P(AssembleParams), P(f64), P(i64), vp]),
    "rafem_system_download": (i32, [vp, vp, vp]),
    "rafem_system_solve": (i32, [vp, vp, vp, P(SolverParams), vp, P(SolveStatsC), vp, i64, vp, i64]),
    "rafem_system_spmv": (i32, [vp, vp, vp]),
    "rafem_system_spmv_bench": (i32, [vp, i32, i32, P(f64)]),
    "rafem_simulate": (i32, [vp, P(SimParams), P(SimSummaryC), i64, vp, vp, vp, vp, vp]),
    "rafem_mesh_create_box": (i32, [vp, i32, i32, i32, vp, vp, i64, vp, i64, f64, f64, f64, f64, f64, P(vp)]),
    "rafem_mesh_counts": (i64, [vp, P(i64)]),
    "rafem_mesh_download": (i32, [vp, vp, vp, vp]),
    "rafem_field_compare": (i32, [vp, i64, i64, vp, vp, i32, vp, vp]),
    "rafem_simulate_stream": (i32, [vp, P(SimParams), P(SimSummaryC), i32, vp, vp]),
    "rafem_assemble_partial": (i32, [vp, vp, vp, vp, P(AssembleParams), i64, vp, P(i64)]),
    "rafem_assemble_finish": (i32, [vp, P(AssembleParams), f64]),
    "rafem_kp_create": (i32, [vp, i64, i64, i32, i32, P(vp)]),
    "rafem_kp_destroy": (None, [vp]),
    "rafem_kp_set_halo": (i32, [vp, vp, i64]),
    "rafem_kp_buffers": (i32, [vp, P(vp), P(vp), P(vp), P(vp)]),
    "rafem_kp_begin": (i32, [vp, vp, vp, P(SolverParams)]),
    "rafem_kp_launch": (i32, [vp, i32]),
    "rafem_kp_iterate": (i32, [vp, i32]),
    "rafem_kp_state": (i32, [vp, P(i32), P(i64), P(f64)]),
    "rafem_kp_finish": (i32, [vp, vp, P(SolveStatsC), vp, i64, vp, i64]),
    "rafem_kp_ipc_export": (i32, [vp, vp, vp]),
    "rafem_kp_ipc_connect": (i32, [vp, vp, vp, i32, vp, vp, vp, i32, vp]),
    "rafem_sl_create": (i32, [vp, P(vp)]),
    "rafem_sl_destroy": (None, [vp]),
    "rafem_sl_buffers": (i32, [vp, P(vp), P(vp)]),
    "rafem_sl_init": (i32, [vp, f64]),
    "rafem_sl_predict": (i32, [vp, i32, f64, i32]),
    "rafem_sl_pack": (i32, [vp]),
    "rafem_sl_unpack": (i32, [vp]),
    "rafem_sl_assemble_partial": (i32, [vp, f64, vp, P(i64)]),
    "rafem_sl_solve_begin": (i32, [vp, P(SolverParams), i32]),
    "rafem_sl_solve_end": (i32, [vp, P(SolveStatsC), P(f64)]),
    "rafem_sl_accept": (i32, [vp]),
    "rafem_sl_download": (i32, [vp, vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_ctx = None
_lock = threading.Lock()


class NativeUnavailable(RuntimeError):
    """librafem_b200.so is missing or no CUDA device is usable."""


def load_library(path: str = LIB_PATH):
    """Load the shared object and declare every exported signature."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is missing; build it with `python -m paper_2409_13036_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    return load_library()


def context():
    """Process-wide device context on the current CUDA device (default 0)."""
    global _ctx
    with _lock:
        if _ctx is None:
            L = load_library()
            dev = int(os.environ.get("RAFEM_DEVICE", "0"))
            h = vp()
            rc = L.rafem_ctx_create(dev, C.byref(h))
            if rc != OK:
                msg = L.rafem_last_error(h).decode() if h else "context creation failed"
                if h:
                    L.rafem_ctx_destroy(h)
                raise NativeUnavailable(f"CUDA device {dev} unusable: {msg}")
            _ctx = h
        return _ctx


def last_error() -> str:
    return lib().rafem_last_error(context()).decode()


def kernel_launches() -> int:
    return int(lib().rafem_kernel_launches(context()))


def last_solve_mode() -> tuple[int, int]:
    """(mode, CTAs) of the last solve: 0 grid, 1 cluster, 2 fused simulation,
    3 grid-wide streaming PCG, 4 kernel-per-phase PCG (rafem_b200.h)."""
    mode, ctas = i32(), i32()
    check(lib().rafem_last_solve_mode(context(), C.byref(mode), C.byref(ctas)), "last_solve_mode")
    return mode.value, ctas.value


PRECOND_NAMES = {PRECOND_NONE: "none", PRECOND_JACOBI: "jacobi", PRECOND_BLOCK_JACOBI: "block_jacobi"}


def last_solve_precond() -> str:
    """Preconditioner the last solve actually applied ("none", "jacobi",
    "block_jacobi"; block-Jacobi only exists in the paper-scale pipelined PCG)."""
    v = i32()
    check(lib().rafem_last_solve_precond(context(), C.byref(v)), "last_solve_precond")
    return PRECOND_NAMES.get(v.value, "none")


def device_info() -> dict:
    sm, ma, mi, mem = i32(), i32(), i32(), i64()
    lib().rafem_device_info(context(), C.byref(sm), C.byref(ma), C.byref(mi), C.byref(mem))
    return {"sm_count": sm.value, "cc": (ma.value, mi.value), "total_mem": mem.value}


def ptr(a: np.ndarray | None):
    """Raw data pointer of a C-contiguous array (None -> NULL)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays crossing the C ABI must be contiguous"
    return a.ctypes.data


def check(rc: int, what: str = ""):
    """Map a status code onto a generic exception (callers refine the mapping)."""
    if rc == OK:
        return
    msg = last_error()
    if rc == ERR_INVALID:
        raise ValueError(msg)
    if rc == ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"{what}: {msg}" if what else msg)
