"""GPU parity of the SURVEY.md §8(f) rows: device box-mesh generator,
streamed records (+ asynchronous .rsf), device PSNR."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, golden
from oracle import rafem_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims", [(2, 2, 2), (3, 4, 2), (6, 5, 7), (20, 20, 21), (80, 80, 79)])
def test_device_box_mesh_is_bitwise_host_generator(dims):
    from paper_2409_13036_b200 import MaterialParams, generate_box_mesh
    from paper_2409_13036_b200.assembly import DeviceMesh, _dof_kinds
    host = generate_box_mesh(*dims)
    dm = DeviceMesh.from_box(*dims)
    nodes, tets, kind = dm.download()
    assert np.array_equal(nodes, host.nodes)  # bit-identical linspace coordinates
    assert np.array_equal(tets, host.tets)
    assert np.array_equal(kind, _dof_kinds(host))
    ref = DeviceMesh(host, MaterialParams.default())
    assert dm.slots == ref.slots
    rp, col = dm.node_pattern()
    rp2, col2 = ref.node_pattern()
    assert np.array_equal(rp, rp2) and np.array_equal(col, col2)


def test_device_mesh_simulation_equals_host_mesh_simulation():
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
    from paper_2409_13036_b200.assembly import DeviceMesh
    from paper_2409_13036_b200.timeloop import DeviceRun
    cfg = SimConfig(total_time=40.0, solver=SolverConfig(backend="pcg", precondition="jacobi"))
    a, sa = DeviceRun(generate_box_mesh(15, 15, 16)).run(cfg)
    b, sb = DeviceRun.from_device_mesh(DeviceMesh.from_box(15, 15, 16)).run(cfg)
    assert len(a) == len(b) and sa.total_solver_iterations == sb.total_solver_iterations
    for x, y in zip(a, b):
        assert (x.time, x.dt, x.corrector_iters) == (y.time, y.dt, y.corrector_iters)
        assert np.array_equal(x.T, y.T) and np.array_equal(x.V, y.V)


@pytest.mark.parametrize("slots", [1, 3, 16])
def test_streamed_records_equal_batch_records_and_rsf(tmp_path, slots):
    """rafem_simulate_stream delivers every accepted step while the kernel
    runs (ring of `slots` device slots); same bits as the batch copy, and
    the asynchronous writer produces the synchronous writer's file."""
    from paper_2409_13036_b200 import SimConfig, SolverConfig, generate_box_mesh
    from paper_2409_13036_b200.results import AsyncResultWriter, ResultWriter, read_result_file
    from paper_2409_13036_b200.timeloop import DeviceRun
    mesh = generate_box_mesh(20, 20, 21)
    cfg = SimConfig(total_time=900.0, solver=SolverConfig(backend="pcg", precondition="jacobi"))
    run = DeviceRun(mesh)
    batch, sb = run.run(cfg)
    got = []
    with AsyncResultWriter(tmp_path / "a.rsf", mesh.node_count) as w:
        def sink(r):
            got.append(r)
            w.append(r)
        ss = run.run_streamed(cfg, sink, ring_slots=slots)
    assert int(ss.accepted_steps) == len(batch) == len(got) == 96
    for x, y in zip(batch, got):
        assert (x.step, x.time, x.dt, x.corrector_iters) == (y.step, y.time, y.dt, y.corrector_iters)
        assert np.array_equal(x.T, y.T) and np.array_equal(x.V, y.V)
    with ResultWriter(tmp_path / "s.rsf", mesh.node_count) as w:
        for r in batch:
            w.append(r)
    assert (tmp_path / "a.rsf").read_bytes() == (tmp_path / "s.rsf").read_bytes()
    assert len(read_result_file(tmp_path / "a.rsf").steps) == 96


def test_streamed_sink_error_surfaces():
    from paper_2409_13036_b200 import SimConfig, SolverConfig, generate_box_mesh
    from paper_2409_13036_b200.timeloop import DeviceRun
    cfg = SimConfig(total_time=40.0, solver=SolverConfig(backend="pcg", precondition="jacobi"))
    seen = []

    def sink(r):
        seen.append(r.step)
        if r.step == 2:
            raise RuntimeError("disk full")

    with pytest.raises(RuntimeError, match="disk full"):
        DeviceRun(generate_box_mesh(6, 6, 6)).run_streamed(cfg, sink, ring_slots=2)
    assert seen == [0, 1, 2]


def test_device_psnr_matches_reference_psnr_series():
    """psnr_series on the device vs the reference's own psnr_series output
    (tests/golden/psnr.npz, two reference runs at 1e-10 / 1e-6)."""
    from types import SimpleNamespace
    from paper_2409_13036_b200.metrics import psnr_series, psnr_step
    d = golden("psnr")

    def run(tag):
        steps = [SimpleNamespace(step=int(s), time=float(t), T=T, V=V)
                 for s, t, T, V in zip(d[f"{tag}_step"], d[f"{tag}_time"], d[f"{tag}_T"], d[f"{tag}_V"])]
        return SimpleNamespace(node_count=d[f"{tag}_T"].shape[1], steps=steps)

    ser = psnr_series(run("ref"), run("test"), (1e-5, 1e-12))
    assert ser.peak_t == d["peak_t"] and ser.peak_v == d["peak_v"]
    assert np.allclose(ser.psnr_t, d["psnr_t"], rtol=0, atol=1e-9)
    assert np.allclose(ser.psnr_v, d["psnr_v"], rtol=0, atol=1e-9)
    assert np.array_equal(ser.control_t, d["control_t"]) and np.array_equal(ser.control_v, d["control_v"])
    assert np.array_equal(ser.steps, d["steps"]) and np.array_equal(ser.times, d["times"])
    # identical fields: inf; a uniform 1e-5 offset at unit peak: 100 dB (metrics.py:52-56)
    f = np.linspace(0.0, 1.0, 1001)
    assert psnr_step(f, f, 1.0) == np.inf
    assert abs(psnr_step(f, f + 1e-5, 1.0) - 100.0) < 1e-9
    # CUDA tensors stay on the device
    import torch
    r, t = run("ref"), run("test")
    for rr, tt in zip(r.steps, t.steps):
        rr.T, rr.V = torch.tensor(rr.T, device="cuda"), torch.tensor(rr.V, device="cuda")
        tt.T, tt.V = torch.tensor(tt.T, device="cuda"), torch.tensor(tt.V, device="cuda")
    ser2 = psnr_series(r, t)
    assert np.array_equal(ser2.psnr_t, ser.psnr_t) and np.array_equal(ser2.psnr_v, ser.psnr_v)
