"""results.py restatement: byte-identical .rsf against a file the reference
ResultWriter wrote (tests/golden/seeded.rsf, make_golden.py gen_results),
the asynchronous writer, and the reader's error taxonomy
(reference tests/test_results.py)."""

import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2409_13036_b200.results import (AsyncResultWriter, ResultFormatError, ResultWriter,
                                           read_result_file)
from paper_2409_13036_b200.timeloop import StepRecord


def seeded_records():
    """The records make_golden.py gen_results() wrote (same RNG call order)."""
    rng = np.random.default_rng(1729)
    n = 17
    out = []
    for k in range(5):
        time = 0.5 * (k + 1) + rng.uniform()
        dt = rng.uniform(0.1, 2.0)
        iters = int(rng.integers(1, 9))
        T = 37.0 + rng.uniform(0, 30, n)
        V = rng.uniform(0, 25, n)
        out.append(StepRecord(k, time, dt, iters, True, T, V))
    return n, out


@pytest.mark.parametrize("cls", [ResultWriter, AsyncResultWriter])
def test_writer_bytes_equal_reference_file(tmp_path, cls):
    n, recs = seeded_records()
    path = tmp_path / "out.rsf"
    with cls(path, n) as w:
        for r in recs:
            w.append(r)
    assert path.read_bytes() == open(os.path.join(GOLDEN, "seeded.rsf"), "rb").read()


def test_reader_round_trip_and_step_index():
    n, recs = seeded_records()
    f = read_result_file(os.path.join(GOLDEN, "seeded.rsf"))
    assert f.node_count == n and len(f.steps) == len(recs)
    for a, b in zip(f.steps, recs):
        assert (a.step, a.time, a.dt, a.corrector_iters, a.converged) == (b.step, b.time, b.dt, b.corrector_iters, True)
        assert np.array_equal(a.T, b.T) and np.array_equal(a.V, b.V)
    assert f.step_index(3) == 3
    with pytest.raises(KeyError):
        f.step_index(99)


def test_reader_errors(tmp_path):
    good = open(os.path.join(GOLDEN, "seeded.rsf"), "rb").read()
    cases = {"magic": b"XXSIM1\x00" + good[7:], "version": good[:7] + b"\x02" + good[8:],
             "truncated": good[:-3], "short": good[:5],
             "zero": good[:8] + struct.pack("<I", 0) + good[12:]}
    for name, blob in cases.items():
        p = tmp_path / f"{name}.rsf"
        p.write_bytes(blob)
        with pytest.raises(ResultFormatError):
            read_result_file(p)


@pytest.mark.parametrize("cls", [ResultWriter, AsyncResultWriter])
def test_writer_rejects_wrong_field_length(tmp_path, cls):
    with pytest.raises(ValueError):
        cls(tmp_path / "z.rsf", 0)
    w = cls(tmp_path / "w.rsf", 5)
    with pytest.raises(ValueError):
        w.append(StepRecord(0, 1.0, 1.0, 1, True, np.zeros(4), np.zeros(5)))
    w.close()
    assert read_result_file(tmp_path / "w.rsf").steps == []
