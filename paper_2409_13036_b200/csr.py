"""Sparse containers and the device SpMV / COO compression.

Mirrors the reference's sparse API (rafem/sparse.py:17-31): ``CooMatrix``
and ``CsrMatrix`` keep its validation contract (sparse.py:49-63, 87-111),
``spmv`` and ``coo_to_csr`` keep its bit-level results but run on the B200
through librafem_b200.  ``DeviceCsrMatrix`` is the CSR an assembly returns:
values stay in HBM (node-paired layout) and the host arrays are only
materialized if somebody reads them.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as nat

__all__ = ["CooMatrix", "CsrMatrix", "DeviceCsrMatrix", "coo_to_csr", "spmv"]


@dataclass
class CooMatrix:
    """Triplets; order fixes duplicate summation (sparse.py:34-67)."""

    nrows: int
    ncols: int
    rows: np.ndarray
    cols: np.ndarray
    vals: np.ndarray

    def __post_init__(self):
        self.rows = np.ascontiguousarray(self.rows, dtype=np.int64)
        self.cols = np.ascontiguousarray(self.cols, dtype=np.int64)
        self.vals = np.ascontiguousarray(self.vals, dtype=np.float64)
        if min(self.nrows, self.ncols) < 0:
            raise ValueError("matrix dimensions must be nonnegative")
        if not (self.rows.shape == self.cols.shape == self.vals.shape):
            raise ValueError("rows, cols and vals must have equal length")
        if self.rows.ndim != 1:
            raise ValueError("triplet arrays must be one-dimensional")
        if self.rows.size:
            if self.rows.min() < 0 or self.rows.max() >= self.nrows:
                raise ValueError("row index out of range")
            if self.cols.min() < 0 or self.cols.max() >= self.ncols:
                raise ValueError("column index out of range")

    @property
    def nnz(self) -> int:
        return int(self.rows.size)


def _validate_csr(nrows, ncols, row_ptr, col_idx, vals):
    if row_ptr.shape != (nrows + 1,):
        raise ValueError("row_ptr must have length nrows + 1")
    if row_ptr[0] != 0 or row_ptr[-1] != col_idx.size:
        raise ValueError("row_ptr must start at 0 and end at nnz")
    if np.any(row_ptr[1:] < row_ptr[:-1]):
        raise ValueError("row_ptr must be nondecreasing")
    if col_idx.shape != vals.shape:
        raise ValueError("col_idx and vals must have equal length")
    if col_idx.size:
        if col_idx.min() < 0 or col_idx.max() >= ncols:
            raise ValueError("column index out of range")
        # strictly increasing inside a row: every non-increase must sit on a row start
        drops = np.flatnonzero(col_idx[1:] <= col_idx[:-1]) + 1
        if drops.size:
            starts = np.zeros(col_idx.size + 1, dtype=bool)
            starts[row_ptr] = True
            if not np.all(starts[drops]):
                raise ValueError("column indices must be strictly increasing within a row")


class CsrMatrix:
    """Host CSR with the reference's invariants (sparse.py:70-133)."""

    def __init__(self, nrows: int, ncols: int, row_ptr, col_idx, vals):
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int64)
        self.vals = np.ascontiguousarray(vals, dtype=np.float64)
        _validate_csr(self.nrows, self.ncols, self.row_ptr, self.col_idx, self.vals)

    def __repr__(self):
        return f"CsrMatrix({self.nrows}x{self.ncols}, nnz={self.nnz})"

    @property
    def nnz(self) -> int:
        return int(self.col_idx.size)

    def entry_rows(self) -> np.ndarray:
        return np.repeat(np.arange(self.nrows, dtype=np.int64), np.diff(self.row_ptr))

    def diagonal(self) -> np.ndarray:
        n = min(self.nrows, self.ncols)
        out = np.zeros(n)
        r = self.entry_rows()
        hit = (r == self.col_idx) & (r < n)
        out[r[hit]] = self.vals[hit]
        return out

    def toarray(self) -> np.ndarray:
        dense = np.zeros((self.nrows, self.ncols))
        dense[self.entry_rows(), self.col_idx] = self.vals
        return dense


class DeviceCsrMatrix(CsrMatrix):
    """An assembled system's matrix, resident on the B200.

    The interleaved 2N x 2N CSR of fem.py:381-387 is stored as the node
    pattern (one int32 column per node pair) with one (V, T) double2 per
    slot.  ``row_ptr``/``col_idx``/``vals`` materialize the reference's
    int64/f64 host arrays lazily (one D2H of the values); the solver uses
    the device copy directly.  Treat it as immutable: edits to the host
    arrays are not pushed back to the device.
    """

    def __init__(self, system):  # system: assembly._SystemHandle
        self._sys = system
        self.nrows = self.ncols = 2 * system.mesh.node_count
        self._vals = None

    @property
    def row_ptr(self):
        return self._sys.mesh.dof_row_ptr

    @property
    def col_idx(self):
        return self._sys.mesh.dof_col_idx

    @property
    def vals(self):
        if self._vals is None:
            self._vals = self._sys.download_vals()
        return self._vals

    @property
    def nnz(self) -> int:
        return 2 * self._sys.mesh.slots

    @property
    def device_system(self):
        return self._sys


def spmv(a: CsrMatrix, x: np.ndarray) -> np.ndarray:
    """y = A x on the device, bit-identical to sparse.py:205-219."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.shape != (a.ncols,):
        raise ValueError(f"operand has length {x.shape}, expected {a.ncols}")
    y = np.empty(a.nrows)
    if a.nrows == 0:
        return y
    if isinstance(a, DeviceCsrMatrix):
        return a.device_system.spmv(x)
    L, ctx = nat.lib(), nat.context()
    rc = L.rafem_spmv(ctx, a.nrows, a.ncols, a.nnz, nat.ptr(a.row_ptr), nat.ptr(a.col_idx),
                      nat.ptr(a.vals), nat.ptr(x), nat.ptr(y))
    nat.check(rc, "spmv")
    return y


def coo_to_csr(a: CooMatrix) -> CsrMatrix:
    """Compress triplets on the device, duplicates summed in input order (sparse.py:164-197)."""
    if a.nnz == 0:
        return CsrMatrix(a.nrows, a.ncols, np.zeros(a.nrows + 1, dtype=np.int64),
                         np.empty(0, dtype=np.int64), np.empty(0))
    rp = np.empty(a.nrows + 1, dtype=np.int64)
    ci = np.empty(a.nnz, dtype=np.int64)
    vv = np.empty(a.nnz)
    nout = C.c_int64()
    L, ctx = nat.lib(), nat.context()
    rc = L.rafem_coo_to_csr(ctx, a.nrows, a.ncols, a.nnz, nat.ptr(a.rows), nat.ptr(a.cols),
                            nat.ptr(a.vals), nat.ptr(rp), nat.ptr(ci), nat.ptr(vv), C.byref(nout))
    nat.check(rc, "coo_to_csr")
    k = nout.value
    return CsrMatrix(a.nrows, a.ncols, rp, ci[:k].copy(), vv[:k].copy())
