"""Per-step PSNR of two runs on the device — metrics.py:31-176 of the reference.

``psnr_series`` keeps the reference's contract (steps aligned by index,
peak = the reference run's global per-field max |value|, PSNR =
20 log10(peak) - 10 log10(MSE), ``inf`` for identical fields, analytic
noise controls, warnings on step-count / time mismatches) while the
O(steps x nodes) work — squared differences and peaks — runs in one
batched device reduction per field (rafem_field_compare), so 16M-64M
dof runs are compared without a host pass over every field (SURVEY.md
§8(f)4).  Fields may be numpy arrays (host) or CUDA tensors (device).
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass

import numpy as np

from . import _native as nat

__all__ = ["PsnrSeries", "noise_control", "psnr_series", "psnr_step"]

_TIME_MATCH_TOL = 1e-9


def noise_control(max_a: float, amplitude: float) -> float:
    """PSNR of a uniform noise floor of the given amplitude (metrics.py:67-76)."""
    if not max_a > 0.0 or not amplitude > 0.0:
        raise ValueError("max_a and amplitude must be positive")
    return 20.0 * (math.log10(max_a) - math.log10(amplitude))


def _from_sq(sq: float, n: int, max_a: float) -> float:
    mse = sq / n
    if mse == 0.0:
        return math.inf
    return 20.0 * math.log10(max_a) - 10.0 * math.log10(mse)


def _compare(ref, test):
    """(sum of squared differences, max |ref|) per row of two (steps, n) stacks."""
    import ctypes as C
    is_dev = hasattr(ref, "is_cuda") and ref.is_cuda
    if is_dev:
        import torch
        ref = ref.to(torch.float64).contiguous()
        test = test.to(torch.float64).contiguous()
        torch.cuda.synchronize(ref.device)
        steps, n = ref.shape
        pr, pt = ref.data_ptr(), test.data_ptr()
    else:
        ref = np.ascontiguousarray(ref, dtype=np.float64)
        test = np.ascontiguousarray(test, dtype=np.float64)
        steps, n = ref.shape
        pr, pt = ref.ctypes.data, test.ctypes.data
    sq = np.empty(steps)
    mx = np.empty(steps)
    nat.check(nat.lib().rafem_field_compare(nat.context(), n, steps, C.c_void_p(pr), C.c_void_p(pt),
                                            1 if is_dev else 0, nat.ptr(sq), nat.ptr(mx)), "field_compare")
    return sq, mx


def psnr_step(ref_field, test_field, max_a: float) -> float:
    """PSNR in dB of one field pair (metrics.py:47-64)."""
    ref_field = np.asarray(ref_field, dtype=np.float64)
    test_field = np.asarray(test_field, dtype=np.float64)
    if ref_field.shape != test_field.shape or ref_field.ndim != 1 or ref_field.size == 0:
        raise ValueError("fields must be equal-length non-empty vectors")
    if not max_a > 0.0:
        raise ValueError("max_a must be positive")
    sq, _ = _compare(ref_field[None], test_field[None])
    return _from_sq(float(sq[0]), ref_field.size, max_a)


@dataclass
class PsnrSeries:
    steps: np.ndarray
    times: np.ndarray
    psnr_t: np.ndarray
    psnr_v: np.ndarray
    control_amps: tuple
    control_t: np.ndarray
    control_v: np.ndarray
    peak_t: float
    peak_v: float
    mismatched_steps: np.ndarray

    def __len__(self) -> int:
        return self.steps.size


def _stack(run, count, attr):
    fields = [getattr(r, attr) for r in run.steps[:count]]
    if fields and hasattr(fields[0], "is_cuda"):
        import torch
        return torch.stack(fields)
    return np.stack(fields)


def psnr_series(ref, test, noise_controls=()) -> PsnrSeries:
    """Compare two runs step by step (metrics.py:98-166).  ``ref``/``test``
    carry ``node_count`` and ``steps`` (records with step, time, T, V)."""
    if ref.node_count != test.node_count:
        raise ValueError(f"node-count mismatch: reference has {ref.node_count}, test has {test.node_count}")
    if not ref.steps or not test.steps:
        raise ValueError("both runs must contain at least one step")
    count = min(len(ref.steps), len(test.steps))
    if len(ref.steps) != len(test.steps):
        warnings.warn(f"step-count mismatch ({len(ref.steps)} vs {len(test.steps)}); "
                      f"comparing the first {count} steps", stacklevel=2)
    n = ref.node_count
    sq_t, mx_t = _compare(_stack(ref, count, "T"), _stack(test, count, "T"))
    sq_v, mx_v = _compare(_stack(ref, count, "V"), _stack(test, count, "V"))
    if len(ref.steps) > count:  # the peak is over ALL reference steps (metrics.py:125-126)
        all_t, all_v = _stack(ref, len(ref.steps), "T"), _stack(ref, len(ref.steps), "V")
        mx_t, mx_v = _compare(all_t, all_t)[1], _compare(all_v, all_v)[1]
    peak_t, peak_v = float(np.max(mx_t)), float(np.max(mx_v))
    if peak_t <= 0.0 or peak_v <= 0.0:
        raise ValueError("reference run has a zero field; PSNR peak is undefined")
    steps = np.array([r.step for r in ref.steps[:count]], dtype=np.int64)
    times = np.array([r.time for r in ref.steps[:count]], dtype=np.float64)
    mism = [r.step for r, s in zip(ref.steps[:count], test.steps[:count]) if abs(r.time - s.time) > _TIME_MATCH_TOL]
    if mism:
        shown = ", ".join(str(s) for s in mism[:20])
        extra = f" (+{len(mism) - 20} more)" if len(mism) > 20 else ""
        warnings.warn(f"step times differ by more than 1e-9 s at steps {shown}{extra}", stacklevel=2)
    psnr_t = np.array([_from_sq(float(q), n, peak_t) for q in sq_t])
    psnr_v = np.array([_from_sq(float(q), n, peak_v) for q in sq_v])
    amps = tuple(float(a) for a in noise_controls)
    control_t = np.empty((len(amps), count))
    control_v = np.empty((len(amps), count))
    for j, amp in enumerate(amps):
        control_t[j, :] = noise_control(peak_t, amp)
        control_v[j, :] = noise_control(peak_v, amp)
    return PsnrSeries(steps, times, psnr_t, psnr_v, amps, control_t, control_v, peak_t, peak_v,
                      np.asarray(mism, dtype=np.int64))
