"""Oracle restatement vs the live reference (build container only; skipped
where /root/reference is absent, e.g. on the GPU box)."""

import numpy as np

from oracle import rafem_oracle as O


def test_assembly_and_gmres_identical_to_reference(reference):
    from rafem.fem import MaterialParams, SimConfig, assemble_global
    from rafem.mesh import generate_box_mesh
    from rafem.solver import SolverConfig, gmres
    rng = np.random.default_rng(7)
    for dims in [(3, 3, 3), (6, 5, 4), (9, 7, 8)]:
        rm, om = generate_box_mesh(*dims), O.box_mesh(*dims)
        n = rm.node_count
        t, v, tp = 37 + rng.uniform(0, 30, n), rng.uniform(0, 25, n), 37 + rng.uniform(0, 30, n)
        s = assemble_global(rm, MaterialParams.default(), SimConfig(), t, v, tp, 0.37)
        o = O.assemble(om, {0: O.OMaterial()}, 25.0, 37.0, t, v, tp, 0.37)
        assert np.array_equal(s.matrix.vals, o.vals) and np.array_equal(s.rhs, o.rhs)
        x, st = gmres(s.matrix, s.rhs, None, SolverConfig(backend="gmres", precondition="jacobi"))
        x2, st2 = O.gmres(o.row_ptr, o.col_idx, o.vals, o.rhs, None, 30, 1e-10, None, "jacobi")
        assert np.array_equal(x, x2) and st.residual_history == st2.residual_history


def test_short_run_identical_to_reference(reference):
    from rafem.fem import MaterialParams, SimConfig, run_simulation
    from rafem.mesh import generate_box_mesh
    from rafem.solver import SolverConfig
    recs = []
    cfg = SimConfig(total_time=6.0, solver=SolverConfig(backend="gmres", precondition="jacobi"))
    run_simulation(generate_box_mesh(5, 5, 5), MaterialParams.default(), cfg, sink=recs.append)
    o = O.run(O.box_mesh(5, 5, 5), {0: O.OMaterial()}, O.OSim(total_time=6.0))
    assert len(recs) == len(o.records)
    for a, b in zip(recs, o.records):
        assert (a.time, a.dt, a.corrector_iters) == (b.time, b.dt, b.corrector_iters)
        assert np.array_equal(a.T, b.T) and np.array_equal(a.V, b.V)
