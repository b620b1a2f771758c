"""Result stream (.rsf) of accepted steps — results.py:1-148 of the reference.

Byte-identical to the reference's ``ResultWriter`` (magic ``RFSIM1\\0``,
version 1, u32 node count, then per accepted step ``<IddIB`` + T, V as
little-endian f64; results.py:3-16, 59-94).  ``AsyncResultWriter`` moves
the serialisation and file IO onto a background thread with a bounded
queue, so at 16M-64M dofs (128-514 MB per record) writing step k
overlaps computing step k+1; combined with
``DeviceRun.run_streamed`` the device -> host copy of each record also
overlaps the running simulation kernel.
"""

from __future__ import annotations

import queue
import struct
import threading
from dataclasses import dataclass

import numpy as np

__all__ = ["RESULT_MAGIC", "RESULT_VERSION", "AsyncResultWriter", "ResultFile", "ResultFormatError",
           "ResultWriter", "read_result_file"]

RESULT_MAGIC = b"RFSIM1\x00"
RESULT_VERSION = 1
_HEAD = struct.Struct("<IddIB")


class ResultFormatError(ValueError):
    """A file that does not parse as a result stream (results.py:49-50)."""


class ResultWriter:
    """Streams accepted steps to a result file (results.py:59-94)."""

    def __init__(self, path, node_count: int):
        if node_count <= 0:
            raise ValueError("node_count must be positive")
        self.node_count = node_count
        self._fh = open(path, "wb")
        self._fh.write(RESULT_MAGIC + bytes([RESULT_VERSION]) + struct.pack("<I", node_count))

    def _encode(self, record) -> bytes:
        T = np.ascontiguousarray(record.T, dtype="<f8")
        V = np.ascontiguousarray(record.V, dtype="<f8")
        if T.shape != (self.node_count,) or V.shape != (self.node_count,):
            raise ValueError("field length does not match the writer's node count")
        head = _HEAD.pack(record.step, record.time, record.dt, record.corrector_iters,
                          1 if record.converged else 0)
        return head + T.tobytes() + V.tobytes()

    def append(self, record) -> None:
        self._fh.write(self._encode(record))

    def close(self) -> None:
        if not self._fh.closed:
            self._fh.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc) -> None:
        self.close()


class AsyncResultWriter(ResultWriter):
    """ResultWriter whose append() returns at once: records are validated
    on the caller's thread, then serialised and written in order by a
    background thread (at most ``depth`` records queued).  Errors surface
    on the next append() or on close()."""

    def __init__(self, path, node_count: int, depth: int = 4):
        super().__init__(path, node_count)
        self._q: queue.Queue = queue.Queue(maxsize=max(1, depth))
        self._err: BaseException | None = None
        self._t = threading.Thread(target=self._drain, name="rsf-writer", daemon=True)
        self._t.start()

    def _drain(self):
        while True:
            rec = self._q.get()
            if rec is None:
                return
            try:
                if self._err is None:
                    self._fh.write(self._encode(rec))
            except BaseException as exc:  # noqa: BLE001
                self._err = exc

    def append(self, record) -> None:
        if self._err is not None:
            raise self._err
        if np.shape(record.T) != (self.node_count,) or np.shape(record.V) != (self.node_count,):
            raise ValueError("field length does not match the writer's node count")
        self._q.put(record)

    def close(self) -> None:
        if self._t.is_alive():
            self._q.put(None)
            self._t.join()
        super().close()
        if self._err is not None:
            err, self._err = self._err, None
            raise err


@dataclass
class _Rec:
    step: int
    time: float
    dt: float
    corrector_iters: int
    converged: bool
    T: np.ndarray
    V: np.ndarray


@dataclass
class ResultFile:
    node_count: int
    steps: list

    def step_index(self, step: int) -> int:
        for i, rec in enumerate(self.steps):
            if rec.step == step:
                return i
        raise KeyError(f"no record for step {step}")


def read_result_file(path) -> ResultFile:
    """Parse a result stream (results.py:110-148)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    head = len(RESULT_MAGIC) + 5
    if len(blob) < head:
        raise ResultFormatError(f"{path}: too short to be a result file")
    if blob[:len(RESULT_MAGIC)] != RESULT_MAGIC:
        raise ResultFormatError(f"{path}: bad magic")
    if blob[len(RESULT_MAGIC)] != RESULT_VERSION:
        raise ResultFormatError(f"{path}: unsupported version {blob[len(RESULT_MAGIC)]}")
    (n,) = struct.unpack_from("<I", blob, len(RESULT_MAGIC) + 1)
    if n == 0:
        raise ResultFormatError(f"{path}: node count is zero")
    size = _HEAD.size + 16 * n
    if (len(blob) - head) % size:
        raise ResultFormatError(f"{path}: truncated step record")
    steps = []
    for off in range(head, len(blob), size):
        step, t, dt, it, conv = _HEAD.unpack_from(blob, off)
        T = np.frombuffer(blob, dtype="<f8", count=n, offset=off + _HEAD.size).copy()
        V = np.frombuffer(blob, dtype="<f8", count=n, offset=off + _HEAD.size + 8 * n).copy()
        steps.append(_Rec(step, t, dt, it, bool(conv), T, V))
    return ResultFile(n, steps)
