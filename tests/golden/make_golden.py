"""Generate golden fixtures from the REFERENCE package (run in the build container).

Usage:  PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py [--full]

Every array in tests/golden/*.npz is produced by the unmodified reference
``rafem`` 0.1.0 (/root/reference/pkg/src/rafem) through its public API, on
seeded inputs.  The GPU box has no /root/reference, so these committed
vectors are what pins the oracle and the device path there.

--full also regenerates the slow mesh-B 900 s runs (~4 min of CPU).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from rafem.fem import MaterialParams, RegionMaterial, SimConfig, assemble_global, run_simulation  # noqa: E402
from rafem.mesh import TetMesh, generate_box_mesh  # noqa: E402
from rafem.solver import SolverConfig, gmres  # noqa: E402
from rafem.sparse import CooMatrix, coo_to_csr, spmv  # noqa: E402
from oracles import random_sparse_system  # noqa: E402  (reference tests/oracles.py)


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def mesh_digest(m) -> dict:
    return {
        "nodes": digest(m.nodes.astype("<f8")),
        "tets": digest(m.tets.astype("<i8")),
        "sets": {k: digest(v.astype("<i8")) for k, v in sorted(m.node_sets.items())},
        "N": int(m.node_count),
        "M": int(m.tet_count),
    }


def gen_meshes():
    out = {}
    for dims in [(2, 2, 2), (3, 3, 3), (3, 4, 2), (4, 3, 5), (5, 5, 5), (6, 6, 6), (8, 8, 8),
                 (15, 15, 16), (20, 20, 21), (80, 80, 79)]:
        out["x".join(map(str, dims))] = mesh_digest(generate_box_mesh(*dims))
    with open(os.path.join(HERE, "meshes.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


def gen_sparse():
    rng = np.random.default_rng(20240811)
    d = {}
    for c in range(12):
        nrows = int(rng.integers(1, 40))
        ncols = int(rng.integers(1, 40))
        nnz = int(rng.integers(0, 200))
        rows = rng.integers(0, nrows, size=nnz)
        cols = rng.integers(0, ncols, size=nnz)
        if nnz > 4:
            rows[: nnz // 4] = rows[nnz // 2: nnz // 2 + nnz // 4]
            cols[: nnz // 4] = cols[nnz // 2: nnz // 2 + nnz // 4]
        vals = rng.standard_normal(nnz)
        a = coo_to_csr(CooMatrix(nrows, ncols, rows, cols, vals))
        x = rng.standard_normal(ncols)
        y = spmv(a, x)
        for k, v in dict(shape=np.array([nrows, ncols]), rows=rows, cols=cols, vals=vals,
                         row_ptr=a.row_ptr, col_idx=a.col_idx, csr_vals=a.vals, x=x, y=y).items():
            d[f"c{c}_{k}"] = v
    d["ncases"] = np.array(12)
    np.savez_compressed(os.path.join(HERE, "sparse.npz"), **d)


def single_tet():
    return TetMesh(
        nodes=np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]]),
        tets=np.array([[0, 1, 2, 3]]), regions=np.zeros(1, dtype=np.int64),
        node_sets={"outer_boundary": np.array([2]), "electrode_pos": np.array([0]),
                   "electrode_neg": np.array([1])})


def gen_assembly():
    """Assembled systems at seeded iterates (hot system recipe of SURVEY §8(d))."""
    d = {}
    cases = [("tet", None), ("b333", (3, 3, 3)), ("b435", (4, 3, 5)), ("b666", (6, 6, 6)),
             ("A", (15, 15, 16))]
    for name, dims in cases:
        mesh = single_tet() if dims is None else generate_box_mesh(*dims)
        n = mesh.node_count
        rng = np.random.default_rng(2409)
        t = 37.0 + rng.uniform(0.0, 30.0, n)
        v = rng.uniform(0.0, 25.0, n)
        tp = 37.0 + rng.uniform(0.0, 30.0, n)
        for tag, kw in (("full", {}), ("raw", dict(apply_constraints=False)),
                        ("noeq", dict(equilibrate=False))):
            s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, tp, 0.5, **kw)
            d[f"{name}_{tag}_row_ptr"] = s.matrix.row_ptr
            d[f"{name}_{tag}_col_idx"] = s.matrix.col_idx
            d[f"{name}_{tag}_vals"] = s.matrix.vals
            d[f"{name}_{tag}_rhs"] = s.rhs
            d[f"{name}_{tag}_scale"] = np.array(s.voltage_row_scale)
        d[f"{name}_t"], d[f"{name}_v"], d[f"{name}_tp"] = t, v, tp
        if dims is not None:
            d[f"{name}_dims"] = np.array(dims)
        # cold system (T = 37, V = 0, T_prev = T)
        tc = np.full(n, 37.0)
        s = assemble_global(mesh, MaterialParams.default(), SimConfig(), tc, np.zeros(n), tc, 0.5)
        d[f"{name}_cold_vals"] = s.matrix.vals
        d[f"{name}_cold_rhs"] = s.rhs
        d[f"{name}_cold_scale"] = np.array(s.voltage_row_scale)
    # a two-region material case (region tags 0/1) on 4x3x5
    mesh = generate_box_mesh(4, 3, 5)
    mesh.regions[::3] = 1
    mat = MaterialParams({0: RegionMaterial(), 1: RegionMaterial(k=0.9e-3, rho_c=2.5e-3,
                                                                  sigma0=0.35e-3, alpha=0.01)})
    rng = np.random.default_rng(77)
    n = mesh.node_count
    t = 37.0 + rng.uniform(0.0, 30.0, n)
    v = rng.uniform(0.0, 25.0, n)
    s = assemble_global(mesh, mat, SimConfig(), t, v, t, 0.25)
    d["reg2_regions"] = mesh.regions
    d["reg2_vals"], d["reg2_rhs"], d["reg2_scale"] = s.matrix.vals, s.rhs, np.array(s.voltage_row_scale)
    d["reg2_t"], d["reg2_v"] = t, v
    np.savez_compressed(os.path.join(HERE, "assembly.npz"), **d)


def gen_gmres():
    d = {}
    rng = np.random.default_rng(201)
    for c in range(8):
        n = int(rng.integers(2, 120))
        rows, cols, vals, dense, b = random_sparse_system(rng, n)
        a = coo_to_csr(CooMatrix(n, n, rows, cols, vals))
        m = int(rng.integers(3, 40))
        pre = ("none", "jacobi")[c % 2]
        tol = (1e-6, 1e-8, 1e-10, 1e-12)[c % 4]
        x, st = gmres(a, b, None, SolverConfig(backend="gmres", tolerance=tol, restart_m=m,
                                               precondition=pre))
        for k, v in dict(row_ptr=a.row_ptr, col_idx=a.col_idx, vals=a.vals, b=b, x=x,
                         x_dense=np.linalg.solve(dense, b),
                         params=np.array([m, tol, c % 2]),
                         stats=np.array([st.iterations, st.restarts, st.final_relative_residual,
                                         float(st.converged)]),
                         hist=np.concatenate([np.asarray(h, dtype=float) for h in st.residual_history]),
                         hist_lens=np.array([len(h) for h in st.residual_history])).items():
            d[f"c{c}_{k}"] = v
    d["ncases"] = np.array(8)
    # FEM cold/hot systems on the A analog, solved by reference GMRES(30)+Jacobi at 1e-10
    mesh = generate_box_mesh(15, 15, 16)
    n = mesh.node_count
    tc = np.full(n, 37.0)
    s = assemble_global(mesh, MaterialParams.default(), SimConfig(), tc, np.zeros(n), tc, 0.5)
    x0 = np.empty(2 * n)
    x0[0::2], x0[1::2] = 0.0, 37.0
    x, st = gmres(s.matrix, s.rhs, x0, SolverConfig(backend="gmres", precondition="jacobi"))
    d["femA_x"], d["femA_x0"] = x, x0
    d["femA_stats"] = np.array([st.iterations, st.restarts, st.final_relative_residual])
    np.savez_compressed(os.path.join(HERE, "gmres.npz"), **d)


def run_case(dims, total_time, tol, keep_every=1):
    mesh = generate_box_mesh(*dims)
    recs = []
    t0 = time.perf_counter()
    summ = run_simulation(mesh, MaterialParams.default(),
                          SimConfig(total_time=total_time,
                                    solver=SolverConfig(backend="gmres", precondition="jacobi",
                                                        tolerance=tol)),
                          sink=recs.append)
    wall = time.perf_counter() - t0
    keep = [i for i in range(len(recs)) if i % keep_every == 0 or i == len(recs) - 1]
    return dict(
        time=np.array([r.time for r in recs]), dt=np.array([r.dt for r in recs]),
        corrector_iters=np.array([r.corrector_iters for r in recs]),
        kept=np.array(keep), T=np.stack([recs[i].T for i in keep]),
        V=np.stack([recs[i].V for i in keep]),
        summary=np.array([summ.accepted_steps, summ.total_corrector_iters,
                          summ.total_solver_iterations, summ.dt_halvings]),
        wall_s=np.array(wall), dims=np.array(dims))


def gen_runs(full: bool):
    for tol, tag in ((1e-10, "1e-10"), (1e-12, "1e-12")):
        np.savez_compressed(os.path.join(HERE, f"run_A40_{tag}.npz"),
                            **run_case((15, 15, 16), 40.0, tol))
    if full:
        np.savez_compressed(os.path.join(HERE, "run_B900_1e-10.npz"),
                            **run_case((20, 20, 21), 900.0, 1e-10, keep_every=8))
        np.savez_compressed(os.path.join(HERE, "run_B900_1e-12.npz"),
                            **run_case((20, 20, 21), 900.0, 1e-12, keep_every=8))
        np.savez_compressed(os.path.join(HERE, "run_A900_1e-10.npz"),
                            **run_case((15, 15, 16), 900.0, 1e-10, keep_every=8))
    # small-mesh semantics cases (reference tests test_fem.py:330-420)
    np.savez_compressed(os.path.join(HERE, "run_b333_6s.npz"), **run_case((3, 3, 3), 6.0, 1e-10))


def gen_results():
    """results.py / metrics.py fixtures: a .rsf written by the reference
    ResultWriter from seeded records, and psnr_series of two reference
    runs of the same mesh at different solver tolerances."""
    from rafem.metrics import psnr_series
    from rafem.results import ResultWriter, StepRecord, read_result_file
    rng = np.random.default_rng(1729)
    n = 17
    recs = [StepRecord(step=k, time=0.5 * (k + 1) + rng.uniform(), dt=rng.uniform(0.1, 2.0),
                       corrector_iters=int(rng.integers(1, 9)), converged=True,
                       T=37.0 + rng.uniform(0, 30, n), V=rng.uniform(0, 25, n)) for k in range(5)]
    path = os.path.join(HERE, "seeded.rsf")
    with ResultWriter(path, n) as w:
        for r in recs:
            w.append(r)
    runs = {}
    for tol in (1e-10, 1e-6):
        out = os.path.join("/tmp", f"golden_psnr_{tol}.rsf")
        mesh = generate_box_mesh(5, 4, 6)
        cfg = SimConfig(total_time=20.0, solver=SolverConfig(backend="gmres", precondition="jacobi", tolerance=tol))
        with ResultWriter(out, mesh.node_count) as w:
            run_simulation(mesh, MaterialParams.default(), cfg, sink=w.append)
        runs[tol] = read_result_file(out)
    ser = psnr_series(runs[1e-10], runs[1e-6], (1e-5, 1e-12))
    d = {"psnr_t": ser.psnr_t, "psnr_v": ser.psnr_v, "peak_t": ser.peak_t, "peak_v": ser.peak_v,
         "control_t": ser.control_t, "control_v": ser.control_v, "steps": ser.steps, "times": ser.times}
    for tag, run in (("ref", runs[1e-10]), ("test", runs[1e-6])):
        d[f"{tag}_T"] = np.stack([r.T for r in run.steps])
        d[f"{tag}_V"] = np.stack([r.V for r in run.steps])
        d[f"{tag}_time"] = np.array([r.time for r in run.steps])
        d[f"{tag}_step"] = np.array([r.step for r in run.steps])
    np.savez_compressed(os.path.join(HERE, "psnr.npz"), **d)


if __name__ == "__main__":
    if "--only-results" in sys.argv:
        gen_results()
        sys.exit(0)
    full = "--full" in sys.argv
    gen_results()
    gen_meshes()
    gen_sparse()
    gen_assembly()
    gen_gmres()
    gen_runs(full)
    print("golden fixtures written to", HERE)
