"""GPU parity: device assembly and full simulations vs oracle/golden.

Bars: pattern bitwise; values within the reference's own
assembly tolerances (single tet <= 1e-14, boxes rtol 1e-12 —
test_fem.py:134-198); scale equal; per-solve residual <= 1e-10; full runs
with an identical trajectory, final-step field error <= 1e-6 vs the
reference at 1e-10, every step <= 1e-6 vs the reference at 1e-12 when run
at 1e-12, and PSNR above the 1e-5 noise control (metrics.py:47-76).
"""

import math

import numpy as np
import pytest

from conftest import golden
from oracle import rafem_oracle as O

pytestmark = pytest.mark.gpu


def single_tet():
    from paper_2409_13036_b200 import TetMesh
    return TetMesh(np.array([[0.0, 0, 0], [1.0, 0, 0], [0.0, 1, 0], [0.0, 0, 1]]),
                   np.array([[0, 1, 2, 3]]), np.zeros(1, dtype=np.int64),
                   {"outer_boundary": np.array([2]), "electrode_pos": np.array([0]),
                    "electrode_neg": np.array([1])})


def mesh_for(name, d):
    from paper_2409_13036_b200 import generate_box_mesh
    return single_tet() if name == "tet" else generate_box_mesh(*map(int, d[f"{name}_dims"]))


@pytest.mark.parametrize("name", ["tet", "b333", "b435", "b666", "A"])
def test_assembly_vs_golden(name):
    from paper_2409_13036_b200 import MaterialParams, SimConfig, assemble_global
    d = golden("assembly")
    mesh = mesh_for(name, d)
    t, v, tp = d[f"{name}_t"], d[f"{name}_v"], d[f"{name}_tp"]
    for tag, kw in (("full", {}), ("raw", dict(apply_constraints=False)),
                    ("noeq", dict(equilibrate=False))):
        s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, tp, 0.5, **kw)
        assert np.array_equal(s.matrix.row_ptr, d[f"{name}_{tag}_row_ptr"])
        assert np.array_equal(s.matrix.col_idx, d[f"{name}_{tag}_col_idx"])
        assert s.voltage_row_scale == float(d[f"{name}_{tag}_scale"])
        ref_v, ref_b = d[f"{name}_{tag}_vals"], d[f"{name}_{tag}_rhs"]
        if name == "tet":
            assert np.max(np.abs(s.matrix.vals - ref_v)) <= 1e-14
            assert np.max(np.abs(s.rhs - ref_b)) <= 1e-14
        else:
            assert np.allclose(s.matrix.vals, ref_v, rtol=1e-12, atol=1e-15)
            assert np.allclose(s.rhs, ref_b, rtol=1e-12, atol=1e-11)
        # the elimination's explicit zeros and unit diagonals are exact (fem.py:425-427)
        if tag != "raw":
            om = O.box_mesh(*map(int, d[f"{name}_dims"])) if name != "tet" else None
            mask = (O.dirichlet(om, 25.0, 37.0)[0] if om is not None else
                    np.array([True, False, True, False, False, True, False, False]))
            rows = np.repeat(np.arange(mask.size), np.diff(s.matrix.row_ptr))
            con = mask[rows] | mask[s.matrix.col_idx]
            assert np.array_equal(s.matrix.vals[con], ref_v[con])
    cold = assemble_global(mesh, MaterialParams.default(), SimConfig(), np.full(mesh.node_count, 37.0),
                           np.zeros(mesh.node_count), np.full(mesh.node_count, 37.0), 0.5)
    assert np.allclose(cold.matrix.vals, d[f"{name}_cold_vals"], rtol=1e-12, atol=1e-15)
    assert np.allclose(cold.rhs, d[f"{name}_cold_rhs"], rtol=1e-12, atol=1e-11)


def test_two_regions_vs_golden():
    from paper_2409_13036_b200 import (MaterialParams, RegionMaterial, SimConfig, assemble_global,
                                       generate_box_mesh)
    d = golden("assembly")
    mesh = generate_box_mesh(4, 3, 5)
    mesh.regions = d["reg2_regions"].copy()
    mat = MaterialParams({0: RegionMaterial(), 1: RegionMaterial(k=0.9e-3, rho_c=2.5e-3,
                                                                  sigma0=0.35e-3, alpha=0.01)})
    s = assemble_global(mesh, mat, SimConfig(), d["reg2_t"], d["reg2_v"], d["reg2_t"], 0.25)
    # two materials: off-diagonal sums no longer cancel exactly, so the
    # absolute floor scales with the matrix (rounding residue ~ eps * |A|)
    floor = 1e-13 * np.max(np.abs(d["reg2_vals"]))
    assert np.allclose(s.matrix.vals, d["reg2_vals"], rtol=1e-12, atol=floor)
    assert np.allclose(s.rhs, d["reg2_rhs"], rtol=1e-12, atol=1e-11)


def test_assembly_deterministic_pattern_invariant_and_errors():
    from paper_2409_13036_b200 import (MaterialParams, PhysicsRangeError, SimConfig, assemble_global,
                                       generate_box_mesh)
    mesh = generate_box_mesh(6, 5, 7)
    n = mesh.node_count
    rng = np.random.default_rng(11)
    t, v, tp = rng.uniform(37, 60, n), rng.uniform(0, 25, n), rng.uniform(37, 60, n)
    a = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, tp, 0.5, threads=1)
    b = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, tp, 0.5, threads=7)
    assert np.array_equal(a.matrix.vals, b.matrix.vals) and np.array_equal(a.rhs, b.rhs)
    c = assemble_global(mesh, MaterialParams.default(), SimConfig(), np.full(n, 37.0), np.zeros(n),
                        np.full(n, 37.0), 0.125)
    assert np.array_equal(a.matrix.row_ptr, c.matrix.row_ptr)
    assert np.array_equal(a.matrix.col_idx, c.matrix.col_idx)
    # equilibration: power of two that balances the diagonal blocks
    raw = assemble_global(mesh, MaterialParams.default(), SimConfig(), np.full(n, 37.0), np.zeros(n),
                          np.full(n, 37.0), 0.5, apply_constraints=False)
    sc = raw.voltage_row_scale
    assert math.log2(sc) == round(math.log2(sc))
    dg = raw.matrix.diagonal()
    assert 0.5 <= dg[1::2].sum() / dg[0::2].sum() <= 2.0
    with pytest.raises(PhysicsRangeError, match="element"):
        assemble_global(mesh, MaterialParams.default(), SimConfig(), np.full(n, -20.0), np.zeros(n),
                        np.full(n, 37.0), 0.5)
    with pytest.raises(ValueError):
        assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, tp, 0.0)
    mesh2 = generate_box_mesh(2, 2, 2)
    mesh2.regions[:] = 5
    with pytest.raises(KeyError, match="region tag 5"):
        assemble_global(mesh2, MaterialParams.default(), SimConfig(), np.full(8, 37.0), np.zeros(8),
                        np.full(8, 37.0), 0.5)


def test_device_matrix_solves_like_host_copy():
    from paper_2409_13036_b200 import (CsrMatrix, MaterialParams, SimConfig, SolverConfig, assemble_global,
                                       generate_box_mesh, solve, spmv)
    mesh = generate_box_mesh(9, 8, 10)
    n = mesh.node_count
    rng = np.random.default_rng(2409)
    s = assemble_global(mesh, MaterialParams.default(), SimConfig(), 37 + rng.uniform(0, 30, n),
                        rng.uniform(0, 25, n), np.full(n, 37.0), 0.5)
    host = CsrMatrix(s.matrix.nrows, s.matrix.ncols, s.matrix.row_ptr, s.matrix.col_idx, s.matrix.vals)
    x = rng.standard_normal(2 * n)
    assert np.array_equal(spmv(s.matrix, x), spmv(host, x))
    for backend in ("gmres", "pcg"):
        cfg = SolverConfig(backend=backend, precondition="jacobi")
        xd, sd = solve(s.matrix, s.rhs, config=cfg)
        xh, sh = solve(host, s.rhs, config=cfg)
        res = np.linalg.norm(s.rhs - O.matvec(host.row_ptr, host.col_idx, host.vals, xd)) / np.linalg.norm(s.rhs)
        assert sd.converged and res <= 1e-10
        assert np.max(np.abs(xd - xh)) <= 1e-8 * np.max(np.abs(xh))


# ---------------------------------------------------------------- full runs

def _rel_inf(x, ref):
    return float(np.max(np.abs(x - ref)) / np.max(np.abs(ref)))


def _compare_run(records, d, field_tol, every_step):
    assert len(records) == len(d["time"])
    assert np.array_equal([r.time for r in records], d["time"])
    assert np.array_equal([r.dt for r in records], d["dt"])
    assert np.array_equal([r.corrector_iters for r in records], d["corrector_iters"])
    worst = 0.0
    kept = list(d["kept"])
    idx = range(len(kept)) if every_step else [len(kept) - 1]
    for i in idx:
        rec = records[kept[i]]
        worst = max(worst, _rel_inf(rec.T, d["T"][i]), _rel_inf(rec.V, d["V"][i]))
    assert worst <= field_tol, worst
    peak_t = float(np.max(np.abs(d["T"])))
    peak_v = float(np.max(np.abs(d["V"])))
    for i in idx:
        rec = records[kept[i]]
        assert O.psnr(d["T"][i], rec.T, peak_t) > 20 * (math.log10(peak_t) - math.log10(1e-5))
        assert O.psnr(d["V"][i], rec.V, peak_v) > 20 * (math.log10(peak_v) - math.log10(1e-5))
    return worst


@pytest.mark.parametrize("backend", ["gmres", "pcg"])
def test_host_loop_A40_vs_reference(backend):
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh, run_simulation
    recs = []
    cfg = SimConfig(total_time=40.0, solver=SolverConfig(backend=backend, precondition="jacobi"))
    run_simulation(generate_box_mesh(15, 15, 16), MaterialParams.default(), cfg, sink=recs.append)
    _compare_run(recs, golden("run_A40_1e-10"), 1e-6, every_step=False)


@pytest.mark.parametrize("backend", ["gmres", "pcg"])
def test_native_loop_A40_tight_every_step(backend):
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh, simulate_device
    cfg = SimConfig(total_time=40.0, solver=SolverConfig(backend=backend, precondition="jacobi",
                                                         tolerance=1e-12))
    recs, _ = simulate_device(generate_box_mesh(15, 15, 16), MaterialParams.default(), cfg)
    _compare_run(recs, golden("run_A40_1e-12"), 1e-6, every_step=True)


@pytest.mark.parametrize("backend", ["gmres", "pcg"])
def test_native_loop_B900_vs_reference(backend):
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh, simulate_device
    mesh = generate_box_mesh(20, 20, 21)
    cfg = SimConfig(total_time=900.0, solver=SolverConfig(backend=backend, precondition="jacobi"))
    recs, summ = simulate_device(mesh, MaterialParams.default(), cfg)
    d = golden("run_B900_1e-10")
    _compare_run(recs, d, 1e-6, every_step=False)
    assert summ.accepted_steps == 96 and summ.passes == int(d["summary"][1])
    cfg12 = SimConfig(total_time=900.0, solver=SolverConfig(backend=backend, precondition="jacobi",
                                                            tolerance=1e-12))
    recs12, _ = simulate_device(mesh, MaterialParams.default(), cfg12)
    _compare_run(recs12, golden("run_B900_1e-12"), 1e-6, every_step=True)


def test_native_and_host_loops_agree_and_are_deterministic():
    from paper_2409_13036_b200 import (MaterialParams, SimConfig, SolverConfig, generate_box_mesh,
                                       run_simulation, simulate_device)
    mesh = generate_box_mesh(6, 6, 6)
    cfg = SimConfig(total_time=30.0, solver=SolverConfig(backend="gmres", precondition="jacobi"))
    r1, _ = simulate_device(mesh, MaterialParams.default(), cfg)
    r2, _ = simulate_device(mesh, MaterialParams.default(), cfg)
    hl = []
    run_simulation(mesh, MaterialParams.default(), cfg, sink=hl.append)
    assert len(r1) == len(r2) == len(hl)
    for a, b, c in zip(r1, r2, hl):
        assert np.array_equal(a.T, b.T) and np.array_equal(a.V, b.V)
        assert (a.time, a.dt, a.corrector_iters) == (c.time, c.dt, c.corrector_iters)
        assert np.array_equal(a.T, c.T) and np.array_equal(a.V, c.V)


def test_zero_drive_is_exact_and_max_principle():
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh, simulate_device
    mesh = generate_box_mesh(5, 5, 5)
    for backend in ("gmres", "pcg"):
        idle = SimConfig(total_time=10.0, applied_voltage=0.0,
                         solver=SolverConfig(backend=backend, precondition="jacobi"))
        recs, _ = simulate_device(mesh, MaterialParams.default(), idle)
        for r in recs:
            assert np.max(np.abs(r.T - 37.0)) <= 1e-10 and np.max(np.abs(r.V)) <= 1e-12
        live = SimConfig(total_time=10.0, solver=SolverConfig(backend=backend, precondition="jacobi"))
        recs, _ = simulate_device(mesh, MaterialParams.default(), live)
        assert min(r.V.min() for r in recs) >= -1e-9 and max(r.V.max() for r in recs) <= 25 + 1e-9


def test_time_loop_failure_semantics():
    from paper_2409_13036_b200 import (MaterialParams, RegionMaterial, SimConfig, SolverConfig,
                                       StepFailureError, corrector_step, generate_box_mesh, initial_state,
                                       run_simulation, simulate_device)
    mesh = generate_box_mesh(3, 3, 3)
    g = SolverConfig(backend="gmres")
    recs = []
    seen = []

    def hook(step, attempt):
        seen.append((step, attempt))
        return step == 1 and attempt == 0

    summ = run_simulation(mesh, MaterialParams.default(), SimConfig(total_time=3.0, solver=g),
                          sink=recs.append, fault_hook=hook)
    assert summ.dt_halvings == 1 and recs[1].dt == 0.75 * 0.5 and recs[-1].time == 3.0
    attempts = []
    with pytest.raises(StepFailureError):
        run_simulation(mesh, MaterialParams.default(),
                       SimConfig(dt_init=4e-6, dt_min=1e-6, total_time=1.0, solver=g),
                       fault_hook=lambda s, a: attempts.append((s, a)) or True)
    assert attempts == [(0, 0), (0, 1), (0, 2)]
    out = corrector_step(mesh, MaterialParams.default(), SimConfig(max_corrector_iters=1, solver=g),
                         initial_state(mesh, SimConfig()), 0.5)
    assert not out.converged and out.iterations == 1 and out.cause == "corrector iteration cap reached"
    hot = MaterialParams({0: RegionMaterial(alpha=0.4)})
    cfg = SimConfig(total_time=10.0, dt_init=10.0, dt_max=10.0, applied_voltage=500.0, solver=g)
    out = corrector_step(mesh, hot, cfg, initial_state(mesh, cfg), 10.0)
    assert not out.converged and out.iterations == 50
    # the native loop reproduces the small-mesh golden run exactly in trajectory
    d = golden("run_b333_6s")
    recs, _ = simulate_device(mesh, MaterialParams.default(),
                              SimConfig(total_time=6.0, solver=SolverConfig(backend="gmres",
                                                                            precondition="jacobi")))
    assert [r.dt for r in recs] == list(d["dt"]) and [r.time for r in recs] == list(d["time"])


def test_fused_simulation_matches_multi_kernel_loop(monkeypatch):
    """The one-launch simulation kernel and the per-pass kernel loop agree
    (the fused kernel's Galerkin solver start off: it is the fused kernel's
    own, see test_galerkin_start_keeps_the_run_and_cuts_iterations)."""
    import os
    monkeypatch.setenv("RAFEM_GALERKIN_K", "0")
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
    from paper_2409_13036_b200.timeloop import DeviceRun
    mesh = generate_box_mesh(15, 15, 16)
    cfg = SimConfig(total_time=40.0, solver=SolverConfig(backend="pcg", precondition="jacobi"))
    run = DeviceRun(mesh)
    fused, sf = run.run(cfg)
    assert run.last_mode == "fused-simulation"
    os.environ["RAFEM_NO_FUSED"] = "1"
    try:
        loop, sl = DeviceRun(mesh).run(cfg)
    finally:
        del os.environ["RAFEM_NO_FUSED"]
    assert [(r.time, r.dt, r.corrector_iters) for r in fused] == [(r.time, r.dt, r.corrector_iters) for r in loop]
    assert sf.total_solver_iterations == sl.total_solver_iterations and sf.passes == sl.passes
    for a, b in zip(fused, loop):
        assert np.max(np.abs(a.T - b.T)) <= 1e-9 * np.max(np.abs(b.T))
        assert np.max(np.abs(a.V - b.V)) <= 1e-9 * np.max(np.abs(b.V))
    _compare_run(fused, golden("run_A40_1e-10"), 1e-6, every_step=False)


def test_slot_list_fill_is_bitwise_warp_fill():
    """The thread-per-slot fill over precomputed contributor lists sums in
    the same (ascending element) order as the warp-per-row fill: same bits
    for values, rhs and scale, on a hot iterate."""
    import os
    from paper_2409_13036_b200 import MaterialParams, SimConfig, assemble_global, generate_box_mesh
    mesh = generate_box_mesh(17, 13, 15)
    n = mesh.node_count
    rng = np.random.default_rng(77)
    t, v, tp = 37.0 + rng.uniform(0, 30, n), rng.uniform(0, 25, n), 37.0 + rng.uniform(0, 5, n)
    a = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, tp, 0.7)
    os.environ["RAFEM_WARP_FILL"] = "1"
    try:
        b = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, tp, 0.7)
    finally:
        del os.environ["RAFEM_WARP_FILL"]
    assert np.array_equal(a.matrix.vals, b.matrix.vals)
    assert np.array_equal(a.rhs, b.rhs) and a.voltage_row_scale == b.voltage_row_scale


def test_block_jacobi_pcg_full_run_vs_reference():
    """precondition="block_jacobi" (north_star's block-Jacobi: one Neumann
    step per CTA block in the pipelined PCG): the 900 s mesh-B run keeps the
    reference trajectory and fields (1e-10 and, at every step, 1e-12),
    with fewer solver iterations than point Jacobi."""
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh, simulate_device
    mesh = generate_box_mesh(20, 20, 21)
    cfg = SimConfig(total_time=900.0, solver=SolverConfig(backend="pcg", precondition="block_jacobi"))
    recs, summ = simulate_device(mesh, MaterialParams.default(), cfg)
    d = golden("run_B900_1e-10")
    _compare_run(recs, d, 1e-6, every_step=False)
    _, sj = simulate_device(mesh, MaterialParams.default(),
                            SimConfig(total_time=900.0, solver=SolverConfig(backend="pcg", precondition="jacobi")))
    assert summ.total_solver_iterations < 0.85 * sj.total_solver_iterations
    cfg12 = SimConfig(total_time=900.0, solver=SolverConfig(backend="pcg", precondition="block_jacobi",
                                                            tolerance=1e-12))
    recs12, _ = simulate_device(mesh, MaterialParams.default(), cfg12)
    _compare_run(recs12, golden("run_B900_1e-12"), 1e-6, every_step=True)


def test_lean_and_generic_simulation_kernels_are_bitwise_equal(monkeypatch):
    """The paper-scale instantiation of the fused simulation (pipelined PCG +
    cp.async-staged fill, everything else compiled out), the generic kernel
    taking the same paths at run time, the generic kernel with the
    register-chunked fill, and the lean kernel with tet-major element
    outputs gathered per element instead of the slot-major layout fetched
    by TMA give the same bits: same sums in the same order (the lean
    kernel's Galerkin solver start off: the generic kernel has none)."""
    import os
    monkeypatch.setenv("RAFEM_GALERKIN_K", "0")
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
    from paper_2409_13036_b200.timeloop import DeviceRun
    mesh = generate_box_mesh(15, 15, 16)
    cfg = SimConfig(total_time=40.0, solver=SolverConfig(backend="pcg", precondition="block_jacobi"))
    runs = []
    for env in ({}, {"RAFEM_NO_LEAN_SIM": "1"}, {"RAFEM_NO_LEAN_SIM": "1", "RAFEM_NO_STAGE_CONTRIB": "1"},
                {"RAFEM_NO_SLOT_MAJOR": "1"}):
        os.environ.update(env)
        try:
            recs, summ = DeviceRun(mesh).run(cfg)
        finally:
            for k in env:
                del os.environ[k]
        runs.append((recs, summ))
    (r0, s0) = runs[0]
    for recs, summ in runs[1:]:
        assert summ.total_solver_iterations == s0.total_solver_iterations and summ.passes == s0.passes
        for a, b in zip(r0, recs):
            assert (a.time, a.dt, a.corrector_iters) == (b.time, b.dt, b.corrector_iters)
            assert np.array_equal(a.T, b.T) and np.array_equal(a.V, b.V)


def test_first_pass_solver_start_extrapolates_v_without_changing_the_run():
    """The native loops start each step's first PCG solve from V extrapolated
    in time (like the reference's T predictor) while assembling from and
    measuring the corrector delta against the reference predictor: same
    trajectory, fields within solver tolerance, fewer PCG iterations
    (scripts/x0_extrap_probe.py: 8,865 -> 6,536 with the oracle's PCG)."""
    import os
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
    from paper_2409_13036_b200.timeloop import DeviceRun
    mesh = generate_box_mesh(20, 20, 21)
    cfg = SimConfig(total_time=900.0, solver=SolverConfig(backend="pcg", precondition="block_jacobi"))
    # isolate the V extrapolation from the Galerkin start (its own test below)
    os.environ["RAFEM_GALERKIN_K"] = "0"
    try:
        new, sn = DeviceRun(mesh).run(cfg)
        os.environ["RAFEM_NO_VX0"] = "1"
        old, so = DeviceRun(mesh).run(cfg)
        loop_env = {"RAFEM_NO_FUSED": "1"}
        os.environ.update(loop_env)
        old_loop, sl = DeviceRun(mesh).run(cfg)
        del os.environ["RAFEM_NO_VX0"]
        new_loop, snl = DeviceRun(mesh).run(cfg)
    finally:
        for k in ("RAFEM_NO_VX0", "RAFEM_NO_FUSED", "RAFEM_GALERKIN_K"):
            os.environ.pop(k, None)
    traj = [(r.time, r.dt, r.corrector_iters) for r in old]
    assert [(r.time, r.dt, r.corrector_iters) for r in new] == traj
    assert [(r.time, r.dt, r.corrector_iters) for r in new_loop] == traj
    assert sn.passes == so.passes and sn.total_solver_iterations < 0.85 * so.total_solver_iterations
    assert snl.total_solver_iterations < 0.85 * sl.total_solver_iterations
    # two solves of the same systems to a 1e-10 relative residual: the V
    # block (ill-conditioned next to the T block) agrees to ~4e-8 of its peak
    for a, b in zip(new, old):
        assert np.max(np.abs(a.T - b.T)) <= 1e-6 * np.max(np.abs(b.T))
        assert np.max(np.abs(a.V - b.V)) <= 1e-6 * np.max(np.abs(b.V))
    _compare_run(new, golden("run_B900_1e-10"), 1e-6, every_step=False)


@pytest.mark.parametrize("dims", [(30, 28, 31), (4, 3, 5)])
def test_fused_element_fill_is_bitwise_the_two_kernel_fill(dims, monkeypatch):
    """The fused element + fill (one warp per node row computes its incident
    elements' rows in registers; default) sums the same contributions in
    the same order as the element kernel + contributor-list fill
    (RAFEM_FUSED_FILL=0): values, rhs and scale are bit-identical, also with
    two material regions."""
    from paper_2409_13036_b200 import (MaterialParams, RegionMaterial, SimConfig, assemble_global,
                                       generate_box_mesh)
    mesh = generate_box_mesh(*dims)
    n = mesh.node_count
    rng = np.random.default_rng(11)
    mesh.regions = (rng.random(mesh.tet_count) < 0.3).astype(np.int64)
    mat = MaterialParams({0: RegionMaterial(), 1: RegionMaterial(k=0.9e-3, rho_c=2.5e-3, sigma0=0.35e-3,
                                                                  alpha=0.01)})
    t, v = 37.0 + 30 * rng.random(n), 25 * rng.random(n)
    out = []
    for mode in ("1", "0"):
        monkeypatch.setenv("RAFEM_FUSED_FILL", mode)
        for kw in ({}, dict(apply_constraints=False, equilibrate=False)):
            s = assemble_global(mesh, mat, SimConfig(), t, v, t, 0.5, **kw)
            out.append((s.matrix.vals.copy(), s.rhs.copy(), s.voltage_row_scale))
    for a, b in zip(out[:2], out[2:]):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]


@pytest.mark.parametrize("name", ["tet", "b333", "b435", "b666", "A"])
def test_exact_geometry_assembly_is_bitwise_reference(name):
    """Bit-exact assembly mode (set_exact_geometry / rafem_mesh_set_geometry,
    SURVEY §8(c)2): with the reference's own element geometry the device
    assemble_global equals the reference's output bit for bit — values and
    rhs, with and without constraints / equilibration, hot and cold."""
    from paper_2409_13036_b200 import MaterialParams, SimConfig, assemble_global, set_exact_geometry
    d = golden("assembly")
    set_exact_geometry(True)
    try:
        mesh = mesh_for(name, d)
        t, v, tp = d[f"{name}_t"], d[f"{name}_v"], d[f"{name}_tp"]
        for tag, kw in (("full", {}), ("raw", dict(apply_constraints=False)),
                        ("noeq", dict(equilibrate=False))):
            s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, tp, 0.5, **kw)
            assert np.array_equal(s.matrix.row_ptr, d[f"{name}_{tag}_row_ptr"])
            assert np.array_equal(s.matrix.col_idx, d[f"{name}_{tag}_col_idx"])
            assert s.voltage_row_scale == float(d[f"{name}_{tag}_scale"])
            assert np.array_equal(s.matrix.vals, d[f"{name}_{tag}_vals"]), tag
            assert np.array_equal(s.rhs, d[f"{name}_{tag}_rhs"]), tag
        cold = assemble_global(mesh, MaterialParams.default(), SimConfig(), np.full(mesh.node_count, 37.0),
                               np.zeros(mesh.node_count), np.full(mesh.node_count, 37.0), 0.5)
        assert np.array_equal(cold.matrix.vals, d[f"{name}_cold_vals"])
        assert np.array_equal(cold.rhs, d[f"{name}_cold_rhs"])
    finally:
        set_exact_geometry(False)


def test_exact_geometry_two_regions_bitwise():
    from paper_2409_13036_b200 import (MaterialParams, RegionMaterial, SimConfig, assemble_global,
                                       generate_box_mesh, set_exact_geometry)
    d = golden("assembly")
    set_exact_geometry(True)
    try:
        mesh = generate_box_mesh(4, 3, 5)
        mesh.regions = d["reg2_regions"].copy()
        mat = MaterialParams({0: RegionMaterial(), 1: RegionMaterial(k=0.9e-3, rho_c=2.5e-3,
                                                                      sigma0=0.35e-3, alpha=0.01)})
        s = assemble_global(mesh, mat, SimConfig(), d["reg2_t"], d["reg2_v"], d["reg2_t"], 0.25)
        assert np.array_equal(s.matrix.vals, d["reg2_vals"])
        assert np.array_equal(s.rhs, d["reg2_rhs"])
    finally:
        set_exact_geometry(False)


def test_galerkin_start_keeps_the_run_and_cuts_iterations(monkeypatch):
    """The fused kernel's Galerkin solver start (x0 += D c over the last
    increments between pass solutions, simulate_dev.cuh galerkin_start)
    changes only the solves' paths: the 900 s mesh-B run keeps its
    trajectory (time, dt, corrector passes of every step), its final fields
    stay within 1e-6 of the reference's, block-Jacobi PCG iterations drop by
    more than a third (CPU study: scripts/galerkin_x0_probe.py), and repeat
    runs are bitwise identical."""
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
    from paper_2409_13036_b200.timeloop import DeviceRun
    run = DeviceRun(generate_box_mesh(20, 20, 21), MaterialParams.default())
    cfg = SimConfig(total_time=900.0, solver=SolverConfig(backend="pcg", precondition="block_jacobi"))
    monkeypatch.setenv("RAFEM_GALERKIN_K", "0")
    base, sb = run.run(cfg)
    monkeypatch.delenv("RAFEM_GALERKIN_K")
    gal, sg = run.run(cfg)
    gal2, _ = run.run(cfg)
    assert [(r.time, r.dt, r.corrector_iters) for r in gal] == [(r.time, r.dt, r.corrector_iters) for r in base]
    # Both runs solve every system to ||r|| <= 1e-10 ||b||; from different
    # starts the ill-conditioned V block lands on different points of that
    # ball (measured: 1.4e-6 of peak at step 9), the T block much closer.
    peak = max(np.max(np.abs(r.T)) for r in base)
    assert max(np.max(np.abs(a.T - b.T)) for a, b in zip(gal, base)) <= 1e-6 * peak
    vpeak = max(np.max(np.abs(r.V)) for r in base)
    assert max(np.max(np.abs(a.V - b.V)) for a, b in zip(gal, base)) <= 5e-6 * vpeak
    _compare_run(gal, golden("run_B900_1e-10"), 1e-6, every_step=False)
    assert sg.total_solver_iterations < 0.67 * sb.total_solver_iterations, (sg.total_solver_iterations,
                                                                          sb.total_solver_iterations)
    assert all(np.array_equal(a.T, b.T) and np.array_equal(a.V, b.V) for a, b in zip(gal, gal2))
