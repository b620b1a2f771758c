"""GPU parity: SpMV, COO compression and the Krylov solvers vs oracle/golden.

Bars: SpMV and coo_to_csr bit-exact (integer/ordering work and the
reference's own per-row summation order); solves against dense truth and
the reference's stats contract (test_solver.py:137-236, acceptance C01/C02).
"""

import numpy as np
import pytest

from conftest import golden
from oracle import rafem_oracle as O

pytestmark = pytest.mark.gpu


def random_system(rng, n, extra_per_row=4, symmetric_pattern=True):
    """Diagonally dominant nonsymmetric values on a symmetric pattern
    (the generator of the reference tests, oracles.py:133-167, restated)."""
    dense = np.zeros((n, n))
    seen = set()
    for i in range(n):
        for _ in range(extra_per_row):
            j = int(rng.integers(0, n))
            if i == j or (i, j) in seen:
                continue
            seen.add((i, j))
            dense[i, j] = rng.uniform(-1.0, 1.0)
            if symmetric_pattern and (j, i) not in seen:
                seen.add((j, i))
                dense[j, i] = rng.uniform(-1.0, 1.0)
    off = np.abs(dense).sum(axis=1)
    dense[np.arange(n), np.arange(n)] = off + rng.uniform(1.0, 2.0, n)
    rows, cols = np.nonzero(dense)
    from paper_2409_13036_b200 import CsrMatrix
    ptr = np.concatenate(([0], np.cumsum(np.bincount(rows, minlength=n))))
    a = CsrMatrix(n, n, ptr, cols, dense[rows, cols])
    return a, dense, rng.standard_normal(n)


def rel_err(x, ref):
    return np.max(np.abs(x - ref)) / max(1.0, np.max(np.abs(ref)))


# ---------------------------------------------------------------- sparse

def test_spmv_bitwise_vs_golden():
    from paper_2409_13036_b200 import CsrMatrix, spmv
    d = golden("sparse")
    for c in range(int(d["ncases"])):
        nrows, ncols = map(int, d[f"c{c}_shape"])
        a = CsrMatrix(nrows, ncols, d[f"c{c}_row_ptr"], d[f"c{c}_col_idx"], d[f"c{c}_csr_vals"])
        assert np.array_equal(spmv(a, d[f"c{c}_x"]), d[f"c{c}_y"])


def test_spmv_bitwise_on_fem_matrix():
    from paper_2409_13036_b200 import CsrMatrix, spmv
    d = golden("assembly")
    a = CsrMatrix(d["A_full_rhs"].size, d["A_full_rhs"].size, d["A_full_row_ptr"],
                  d["A_full_col_idx"], d["A_full_vals"])
    x = np.random.default_rng(3).standard_normal(a.ncols)
    assert np.array_equal(spmv(a, x), O.matvec(a.row_ptr, a.col_idx, a.vals, x))


def test_spmv_identity_and_shape_check():
    from paper_2409_13036_b200 import CooMatrix, coo_to_csr, spmv
    eye = coo_to_csr(CooMatrix(4, 4, range(4), range(4), np.ones(4)))
    x = np.array([3.0, -1.0, 0.5, 2.0])
    assert np.array_equal(spmv(eye, x), x)
    with pytest.raises(ValueError):
        spmv(eye, np.ones(5))


def test_coo_to_csr_bitwise_vs_golden():
    from paper_2409_13036_b200 import CooMatrix, coo_to_csr
    d = golden("sparse")
    for c in range(int(d["ncases"])):
        nrows, ncols = map(int, d[f"c{c}_shape"])
        a = coo_to_csr(CooMatrix(nrows, ncols, d[f"c{c}_rows"], d[f"c{c}_cols"], d[f"c{c}_vals"]))
        assert np.array_equal(a.row_ptr, d[f"c{c}_row_ptr"])
        assert np.array_equal(a.col_idx, d[f"c{c}_col_idx"])
        assert np.array_equal(a.vals, d[f"c{c}_csr_vals"])


def test_coo_to_csr_long_rows_and_duplicates_vs_oracle():
    from paper_2409_13036_b200 import CooMatrix, coo_to_csr
    rng = np.random.default_rng(11)
    rows = np.concatenate([np.zeros(3000, dtype=np.int64), rng.integers(0, 50, 5000)])
    cols = rng.integers(0, 40, rows.size)
    vals = rng.standard_normal(rows.size)
    a = coo_to_csr(CooMatrix(50, 40, rows, cols, vals))
    ptr, col, v = O.compress(50, rows, cols, vals)
    assert np.array_equal(a.row_ptr, ptr) and np.array_equal(a.col_idx, col)
    assert np.array_equal(a.vals, v)
    empty = coo_to_csr(CooMatrix(3, 5, [], [], []))
    assert empty.nnz == 0 and np.array_equal(empty.row_ptr, np.zeros(4))


# ---------------------------------------------------------------- GMRES

def test_gmres_matches_dense_on_golden_systems():
    from paper_2409_13036_b200 import CsrMatrix, SolverConfig, gmres
    d = golden("gmres")
    for c in range(int(d["ncases"])):
        n = d[f"c{c}_b"].size
        a = CsrMatrix(n, n, d[f"c{c}_row_ptr"], d[f"c{c}_col_idx"], d[f"c{c}_vals"])
        m, tol, pre = d[f"c{c}_params"]
        x, st = gmres(a, d[f"c{c}_b"], None, SolverConfig(backend="gmres", tolerance=float(tol),
                                                           restart_m=int(m),
                                                           precondition="jacobi" if pre else "none"))
        assert st.converged
        res = np.linalg.norm(d[f"c{c}_b"] - O.matvec(a.row_ptr, a.col_idx, a.vals, x)) / np.linalg.norm(d[f"c{c}_b"])
        assert res <= 10 * float(tol)
        assert abs(st.final_relative_residual - res) < 1e-12
        if float(tol) <= 1e-10:
            assert rel_err(x, d[f"c{c}_x_dense"]) < 1e-8
        # same algorithm: inner steps and restarts equal the reference's MGS
        # run on every golden case (one-reduce Arnoldi vs MGS: the same
        # Krylov basis to working precision)
        it_ref, rs_ref = int(d[f"c{c}_stats"][0]), int(d[f"c{c}_stats"][1])
        assert (st.iterations, st.restarts) == (it_ref, rs_ref)


@pytest.mark.parametrize("seed", [201, 202, 401])
def test_gmres_random_systems_residual_contract(seed):
    from paper_2409_13036_b200 import SolverConfig, gmres, solve
    rng = np.random.default_rng(seed)
    for i in range(12):
        n = int(rng.integers(10, 151))
        a, dense, b = random_system(rng, n)
        tol = (1e-6, 1e-8, 1e-10)[i % 3]
        cfg = SolverConfig(backend="gmres", tolerance=tol, restart_m=int(rng.integers(5, 41)),
                           precondition=("none", "jacobi")[i % 2])
        x, st = solve(a, b, config=cfg)
        rel = np.linalg.norm(b - dense @ x) / np.linalg.norm(b)
        assert st.converged and rel <= 10 * tol
        assert abs(st.final_relative_residual - rel) < 1e-12
        assert st.wall_ns > 0
        for cyc in st.residual_history:
            assert np.all(np.diff(np.asarray(cyc)) <= 0.0)
        assert st.restarts == len(st.residual_history) - 1


def test_gmres_exact_guess_zero_rhs_and_breakdowns():
    from paper_2409_13036_b200 import (CooMatrix, GmresBreakdownError, SolverConfig, coo_to_csr,
                                       gmres)
    rng = np.random.default_rng(205)
    a, dense, b = random_system(rng, 30)
    x_exact = np.linalg.solve(dense, b)
    x, st = gmres(a, b, x_exact, SolverConfig(backend="gmres", tolerance=1e-8))
    assert st.converged and st.iterations == 0 and np.array_equal(x, x_exact)
    x, st = gmres(a, np.zeros(30), None, SolverConfig(backend="gmres"))
    assert st.converged and np.array_equal(x, np.zeros(30))
    # GMRES(1) on a 90-degree rotation stagnates (test_solver.py:214-222)
    rot = coo_to_csr(CooMatrix(2, 2, [0, 1], [1, 0], [-1.0, 1.0]))
    x, st = gmres(rot, np.array([1.0, 0.0]), None,
                  SolverConfig(backend="gmres", tolerance=1e-10, restart_m=1, max_total_iters=12))
    assert not st.converged and st.stagnated
    sing = coo_to_csr(CooMatrix(3, 3, [0, 1], [0, 1], [1.0, 1.0]))
    with pytest.raises(GmresBreakdownError):
        gmres(sing, np.array([0.0, 0.0, 1.0]), None, SolverConfig(backend="gmres", tolerance=1e-10))
    eye = coo_to_csr(CooMatrix(4, 4, range(4), range(4), np.ones(4)))
    x, st = gmres(eye, np.array([1.0, 2.0, 3.0, 4.0]), None, SolverConfig(backend="gmres", tolerance=1e-12))
    assert st.converged and np.allclose(x, [1, 2, 3, 4], atol=1e-14)


def test_jacobi_zero_diagonal_is_value_error_and_scaled_system():
    from paper_2409_13036_b200 import CooMatrix, CsrMatrix, SolverConfig, coo_to_csr, gmres
    a = coo_to_csr(CooMatrix(2, 2, [0, 1, 1], [1, 0, 1], [1.0, 1.0, 1.0]))
    with pytest.raises(ValueError):
        gmres(a, np.ones(2), None, SolverConfig(backend="gmres", precondition="jacobi"))
    rng = np.random.default_rng(207)
    a, dense, b = random_system(rng, 80)
    s = 10.0 ** rng.uniform(-3, 3, size=80)
    rows = np.repeat(np.arange(80), np.diff(a.row_ptr))
    a2 = CsrMatrix(80, 80, a.row_ptr, a.col_idx, a.vals * s[rows])
    x_pre, st_pre = gmres(a2, b * s, None, SolverConfig(backend="gmres", tolerance=1e-10, restart_m=40,
                                                         precondition="jacobi"))
    assert st_pre.converged and rel_err(x_pre, np.linalg.solve(dense * s[:, None], b * s)) < 1e-8
    _, st_plain = gmres(a2, b * s, None, SolverConfig(backend="gmres", tolerance=1e-10, restart_m=40))
    if st_plain.converged:
        assert st_pre.iterations <= st_plain.iterations


def test_direct_backends_are_out_of_scope():
    from paper_2409_13036_b200 import CooMatrix, SolverConfig, coo_to_csr, solve
    eye = coo_to_csr(CooMatrix(3, 3, range(3), range(3), np.ones(3)))
    with pytest.raises(NotImplementedError):
        solve(eye, np.ones(3), config=SolverConfig(backend="qr"))
    with pytest.raises(ValueError):
        solve(eye, np.ones(4), config=SolverConfig(backend="gmres"))


def test_solves_are_bitwise_deterministic():
    from paper_2409_13036_b200 import CsrMatrix, SolverConfig, solve
    d = golden("assembly")
    n = d["A_full_rhs"].size
    a = CsrMatrix(n, n, d["A_full_row_ptr"], d["A_full_col_idx"], d["A_full_vals"])
    for backend in ("gmres", "pcg"):
        cfg = SolverConfig(backend=backend, precondition="jacobi")
        x1, s1 = solve(a, d["A_full_rhs"], config=cfg)
        x2, s2 = solve(a, d["A_full_rhs"], config=cfg)
        assert np.array_equal(x1, x2) and s1.iterations == s2.iterations


# ---------------------------------------------------------------- PCG

def test_pcg_on_fem_systems_vs_oracle():
    from paper_2409_13036_b200 import CsrMatrix, SolverConfig, solve
    d = golden("assembly")
    for name in ("b666", "A"):
        n = d[f"{name}_full_rhs"].size
        a = CsrMatrix(n, n, d[f"{name}_full_row_ptr"], d[f"{name}_full_col_idx"], d[f"{name}_full_vals"])
        b = d[f"{name}_full_rhs"]
        x, st = solve(a, b, config=SolverConfig(backend="pcg", precondition="jacobi", tolerance=1e-10))
        res = np.linalg.norm(b - O.matvec(a.row_ptr, a.col_idx, a.vals, x)) / np.linalg.norm(b)
        assert st.converged and res <= 1e-10
        assert abs(st.final_relative_residual - res) < 1e-12
        xo, so = O.pcg(a.row_ptr, a.col_idx, a.vals, b, tol=1e-10)
        assert abs(st.iterations - so.iterations) <= max(3, 0.05 * so.iterations)
        assert rel_err(x, xo) < 1e-8


def test_tma_spmv_bitwise_at_1M_dofs():
    """configs[2] (1,011,200 dofs): the TMA-staged streaming SpMV is bit-exact."""
    import os
    from paper_2409_13036_b200 import (CsrMatrix, MaterialParams, SimConfig, assemble_global,
                                       generate_box_mesh, spmv)
    mesh = generate_box_mesh(80, 80, 79)
    n = mesh.node_count
    t = np.full(n, 37.0)
    s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, np.zeros(n), t, 0.5)
    x = np.random.default_rng(5).standard_normal(2 * n)
    y_dev = spmv(s.matrix, x)                       # streaming TMA kernel (matrix > 48 MB)
    os.environ["RAFEM_NO_TMA_SPMV"] = "1"
    try:
        y_plain = spmv(s.matrix, x)                 # thread-per-row kernel
    finally:
        del os.environ["RAFEM_NO_TMA_SPMV"]
    a = s.matrix
    assert np.array_equal(y_dev, y_plain)
    assert np.array_equal(y_dev, O.matvec(a.row_ptr, a.col_idx, a.vals, x))


def _c3_system(hot: bool):
    from paper_2409_13036_b200 import MaterialParams, SimConfig, assemble_global, generate_box_mesh
    mesh = generate_box_mesh(80, 80, 79)
    n = mesh.node_count
    if hot:
        rng = np.random.default_rng(2409)
        t, v = 37.0 + rng.uniform(0, 30, n), rng.uniform(0, 25, n)
    else:
        t, v = np.full(n, 37.0), np.zeros(n)
    s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
    x0 = np.empty(2 * n)
    x0[0::2], x0[1::2] = v, t
    return s, x0


def test_tma_spmv_pipeline_configs_bitwise_at_1M_dofs():
    """Every pipelined streaming-SpMV configuration sums rows left to right."""
    import os
    from paper_2409_13036_b200 import spmv
    s, _ = _c3_system(hot=True)
    x = np.random.default_rng(6).standard_normal(s.rhs.size)
    ref = O.matvec(s.matrix.row_ptr, s.matrix.col_idx, s.matrix.vals, x)
    # NT,ST,HINT[,CTAs per SM]; 1,1,1: the two-stage kernel
    for cfg in ("256,2,1", "128,4,1", "192,3,1", "192,2,1,2", "128,2,1,3", "1,1,1"):
        for classes in ("0", "1"):  # stencil-class columns on / off
            os.environ["RAFEM_SPMV_CFG"] = cfg
            os.environ["RAFEM_NO_CLASSES"] = classes
            try:
                assert np.array_equal(spmv(s.matrix, x), ref), (cfg, classes)
            finally:
                del os.environ["RAFEM_SPMV_CFG"], os.environ["RAFEM_NO_CLASSES"]


@pytest.mark.parametrize("hot", [False, True])
def test_streaming_pcg_at_1M_dofs(hot):
    """configs[2]: the TMA-streaming PCG (matrix >> L2) meets the residual
    contract, agrees with the single-barrier grid PCG and with the default
    (kernel-per-phase, stencil classes) engine, and is bit-reproducible."""
    import os
    from paper_2409_13036_b200 import SolverConfig, solve
    from paper_2409_13036_b200 import _native as nat
    s, x0 = _c3_system(hot)
    a, b = s.matrix, s.rhs
    cfg = SolverConfig(backend="pcg", precondition="jacobi", tolerance=1e-10)
    xk, sk = solve(a, b, x0=x0, config=cfg)
    assert nat.last_solve_mode()[0] == 4  # default here: kernel-per-phase
    rk = np.linalg.norm(b - O.matvec(a.row_ptr, a.col_idx, a.vals, xk)) / np.linalg.norm(b)
    assert sk.converged and rk <= 1e-10
    os.environ["RAFEM_KP"] = "0"
    try:
        x, st = solve(a, b, x0=x0, config=cfg)
        assert nat.last_solve_mode()[0] == 3  # grid-wide streaming PCG
    finally:
        del os.environ["RAFEM_KP"]
    assert abs(st.iterations - sk.iterations) <= max(3, 0.03 * sk.iterations)
    assert rel_err(x, xk) < 1e-7
    res = np.linalg.norm(b - O.matvec(a.row_ptr, a.col_idx, a.vals, x)) / np.linalg.norm(b)
    assert st.converged and res <= 1e-10
    assert abs(st.final_relative_residual - res) < 1e-12
    os.environ["RAFEM_KP"] = "0"
    try:
        x2, st2 = solve(a, b, x0=x0, config=cfg)
    finally:
        del os.environ["RAFEM_KP"]
    assert np.array_equal(x, x2) and st.iterations == st2.iterations
    os.environ["RAFEM_KP"] = "0"
    os.environ["RAFEM_NO_STREAM_PCG"] = "1"
    try:
        xg, sg = solve(a, b, x0=x0, config=cfg)
    finally:
        del os.environ["RAFEM_NO_STREAM_PCG"], os.environ["RAFEM_KP"]
    assert nat.last_solve_mode()[0] == 0
    assert abs(st.iterations - sg.iterations) <= max(3, 0.03 * sg.iterations)
    assert rel_err(x, xg) < 1e-7


@pytest.mark.parametrize("dims", [(6, 6, 6), (15, 15, 16), (20, 20, 21)])
def test_block_jacobi_pcg_on_fem_systems(dims):
    """Block-Jacobi PCG on device-assembled FEM systems: true residual <= tol,
    the stats contract, the point-Jacobi solution, fewer iterations on the
    paper-scale meshes; bit-reproducible."""
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
    mesh = generate_box_mesh(*dims)
    n = mesh.node_count
    rng = np.random.default_rng(31)
    t, v = 37.0 + rng.uniform(0, 30, n), rng.uniform(0, 25, n)
    s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
    a, b = s.matrix, s.rhs
    x0 = np.empty(2 * n)
    x0[0::2], x0[1::2] = v, t
    x, st = solve(a, b, x0=x0, config=SolverConfig(backend="pcg", precondition="block_jacobi", tolerance=1e-10))
    res = np.linalg.norm(b - O.matvec(a.row_ptr, a.col_idx, a.vals, x)) / np.linalg.norm(b)
    assert st.converged and res <= 1e-10 and abs(st.final_relative_residual - res) < 1e-12
    xj, sj = solve(a, b, x0=x0, config=SolverConfig(backend="pcg", precondition="jacobi", tolerance=1e-10))
    assert rel_err(x, xj) < 1e-7  # two solutions at residual 1e-10 (kappa ~ 1e3)
    if n > 3000:
        assert st.iterations < 0.85 * sj.iterations
    x2, st2 = solve(a, b, x0=x0, config=SolverConfig(backend="pcg", precondition="block_jacobi", tolerance=1e-10))
    assert np.array_equal(x, x2) and st.iterations == st2.iterations


@pytest.mark.parametrize("dims", [(6, 5, 7), (15, 15, 16), (20, 20, 21)])
def test_cluster_resident_pcg_vs_grid_pcg(dims):
    """Cluster-resident PCG (cluster.cu: one 16-CTA cluster, DSMEM halos and
    partials over st.async + mbarriers) against the 148-CTA grid PCG on the
    same device-assembled system: same iteration count within 3 %, true
    residual <= tol, solutions within 1e-7, bit-reproducible, stats contract;
    exact x0 comes back bitwise and b = 0 gives x = 0."""
    import os
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
    from paper_2409_13036_b200 import _native as nat
    mesh = generate_box_mesh(*dims)
    n = mesh.node_count
    rng = np.random.default_rng(77)
    t, v = 37.0 + rng.uniform(0, 30, n), rng.uniform(0, 25, n)
    s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
    a, b = s.matrix, s.rhs
    x0 = np.empty(2 * n)
    x0[0::2], x0[1::2] = v, t
    for prec in ("jacobi", "none"):
        cfg = SolverConfig(backend="pcg", precondition=prec, tolerance=1e-10)
        x, st = solve(a, b, x0=x0, config=cfg)
        assert nat.last_solve_mode()[0] == 5, nat.last_solve_mode()
        res = np.linalg.norm(b - O.matvec(a.row_ptr, a.col_idx, a.vals, x)) / np.linalg.norm(b)
        assert st.converged and res <= 1e-10 and abs(st.final_relative_residual - res) < 1e-12
        hist = [h for cyc in st.residual_history for h in cyc]
        assert len(hist) == st.iterations and st.restarts == len(st.residual_history) - 1
        assert hist[-1] <= 1e-10 * (1 + 1e-9)  # the recursive estimate that ended the last cycle
        x2, st2 = solve(a, b, x0=x0, config=cfg)
        assert np.array_equal(x, x2) and st.iterations == st2.iterations
        os.environ["RAFEM_CLUSTER"] = "0"
        try:
            xg, sg = solve(a, b, x0=x0, config=cfg)
        finally:
            del os.environ["RAFEM_CLUSTER"]
        assert nat.last_solve_mode()[0] == 0
        assert abs(st.iterations - sg.iterations) <= max(3, 0.03 * sg.iterations)
        assert rel_err(x, xg) < 1e-7
    # exact guess: returned bitwise with zero iterations; zero data: zero solution
    xe, se = solve(a, b, x0=x, config=SolverConfig(backend="pcg", precondition="jacobi", tolerance=1e-6))
    assert se.iterations == 0 and np.array_equal(xe, x)
    xz, sz = solve(a, np.zeros_like(b), x0=x0, config=SolverConfig(backend="pcg", precondition="jacobi"))
    assert sz.converged and not np.any(xz)


@pytest.mark.parametrize("dims", [(6, 5, 7), (15, 15, 16)])
def test_cluster_gmres_matches_grid_gmres(dims):
    """The cluster GMRES(30) (opt-in RAFEM_CLUSTER_GMRES=1) follows the grid
    GMRES step for step: same inner steps and restarts, solutions within
    1e-10, the stats contract (true residual, per-cycle history)."""
    import os
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
    from paper_2409_13036_b200 import _native as nat
    mesh = generate_box_mesh(*dims)
    n = mesh.node_count
    rng = np.random.default_rng(5)
    t, v = 37.0 + rng.uniform(0, 30, n), rng.uniform(0, 25, n)
    s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
    a, b = s.matrix, s.rhs
    cfg = SolverConfig(backend="gmres", precondition="jacobi", tolerance=1e-10)
    xg, sg = solve(a, b, config=cfg)
    assert nat.last_solve_mode()[0] == 0
    os.environ["RAFEM_CLUSTER_GMRES"] = "1"
    try:
        x, st = solve(a, b, config=cfg)
        assert nat.last_solve_mode()[0] == 5
    finally:
        del os.environ["RAFEM_CLUSTER_GMRES"]
    res = np.linalg.norm(b - O.matvec(a.row_ptr, a.col_idx, a.vals, x)) / np.linalg.norm(b)
    assert st.converged and res <= 1e-10 and abs(st.final_relative_residual - res) < 1e-12
    assert st.iterations == sg.iterations and st.restarts == sg.restarts
    assert [len(c) for c in st.residual_history] == [len(c) for c in sg.residual_history]
    assert rel_err(x, xg) < 1e-10


@pytest.mark.parametrize("dims", [(6, 5, 7), (15, 15, 16), (20, 20, 21)])
def test_one_reduce_gmres_matches_cgs2(dims, monkeypatch):
    """The one-reduce Arnoldi step (gmres_1r_body: the second Gram-Schmidt
    pass of each basis vector delayed into the next step's single reduction)
    builds the same Krylov basis as the three-synchronisation CGS2 step
    (RAFEM_GMRES_CGS2=1) to working precision: same inner steps, restarts and
    per-cycle history lengths, residual estimates within 1e-5 relative
    (their last digits at the 1e-10 level are rounding),
    solutions within 1e-12, and the true residual meets the tolerance."""
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
    mesh = generate_box_mesh(*dims)
    n = mesh.node_count
    rng = np.random.default_rng(11)
    t, v = 37.0 + rng.uniform(0, 30, n), rng.uniform(0, 25, n)
    s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
    a, b = s.matrix, s.rhs
    x0 = np.empty(2 * n)
    x0[0::2], x0[1::2] = v, t
    for start in (None, x0):
        cfg = SolverConfig(backend="gmres", precondition="jacobi", tolerance=1e-10)
        x1, s1 = solve(a, b, x0=start, config=cfg)
        monkeypatch.setenv("RAFEM_GMRES_CGS2", "1")
        x2, s2 = solve(a, b, x0=start, config=cfg)
        monkeypatch.delenv("RAFEM_GMRES_CGS2")
        res = np.linalg.norm(b - O.matvec(a.row_ptr, a.col_idx, a.vals, x1)) / np.linalg.norm(b)
        assert s1.converged and res <= 1e-10 and abs(s1.final_relative_residual - res) < 1e-12
        assert (s1.iterations, s1.restarts) == (s2.iterations, s2.restarts)
        assert [len(c) for c in s1.residual_history] == [len(c) for c in s2.residual_history]
        h1 = np.concatenate([np.asarray(c) for c in s1.residual_history])
        h2 = np.concatenate([np.asarray(c) for c in s2.residual_history])
        assert np.all(np.abs(h1 - h2) <= 1e-5 * h2 + 1e-15)
        assert rel_err(x1, x2) < 1e-12


@pytest.mark.parametrize("m,cap", [(1, 40), (2, 0), (5, 0), (30, 37)])
def test_one_reduce_gmres_restart_lengths_and_cap(m, cap, monkeypatch):
    """Short restart cycles (the column of step k is final one step later,
    so m = 1 exercises a cycle of one SpMV and two reductions) and an
    iteration cap that lands mid-cycle: the one-reduce step and the CGS2
    step agree on inner steps, restarts, convergence and the solution."""
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
    mesh = generate_box_mesh(6, 5, 7)
    n = mesh.node_count
    rng = np.random.default_rng(29 + m)
    t, v = 37.0 + rng.uniform(0, 30, n), rng.uniform(0, 25, n)
    s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
    a, b = s.matrix, s.rhs
    kw = dict(backend="gmres", precondition="jacobi", tolerance=1e-10, restart_m=m)
    if cap:
        kw["max_total_iters"] = cap
    cfg = SolverConfig(**kw)
    x1, s1 = solve(a, b, config=cfg)
    monkeypatch.setenv("RAFEM_GMRES_CGS2", "1")
    x2, s2 = solve(a, b, config=cfg)
    monkeypatch.delenv("RAFEM_GMRES_CGS2")
    assert (s1.iterations, s1.restarts, s1.converged) == (s2.iterations, s2.restarts, s2.converged)
    if cap:
        assert s1.iterations == cap and not s1.converged
    else:
        res = np.linalg.norm(b - O.matvec(a.row_ptr, a.col_idx, a.vals, x1)) / np.linalg.norm(b)
        assert s1.converged and res <= 1e-10
    assert rel_err(x1, x2) < 1e-10
