"""The CPU oracle against golden vectors made by the reference (CPU only).

Pins oracle/rafem_oracle.py bit-for-bit to the reference outputs stored in
tests/golden (tests/golden/make_golden.py generated them from rafem 0.1.0).
"""

import hashlib

import numpy as np
import pytest

from conftest import golden, golden_meshes
from oracle import rafem_oracle as O


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("dims", ["2x2x2", "3x3x3", "3x4x2", "4x3x5", "5x5x5", "6x6x6", "8x8x8",
                                  "15x15x16", "20x20x21"])
def test_box_mesh_digest(dims):
    ref = golden_meshes()[dims]
    m = O.box_mesh(*map(int, dims.split("x")))
    assert _digest(m.nodes.astype("<f8")) == ref["nodes"]
    assert _digest(m.tets.astype("<i8")) == ref["tets"]
    for k, v in ref["sets"].items():
        assert _digest(m.node_sets[k].astype("<i8")) == v


def test_compress_and_matvec_bitwise():
    d = golden("sparse")
    for c in range(int(d["ncases"])):
        nrows, ncols = d[f"c{c}_shape"]
        ptr, col, vals = O.compress(int(nrows), d[f"c{c}_rows"], d[f"c{c}_cols"], d[f"c{c}_vals"])
        assert np.array_equal(ptr, d[f"c{c}_row_ptr"])
        assert np.array_equal(col, d[f"c{c}_col_idx"])
        assert np.array_equal(vals, d[f"c{c}_csr_vals"])
        y = O.matvec(ptr, col, vals, d[f"c{c}_x"])
        assert np.array_equal(y, d[f"c{c}_y"])


def _single_tet():
    return O.OMesh(np.array([[0.0, 0, 0], [1.0, 0, 0], [0.0, 1, 0], [0.0, 0, 1]]),
                   np.array([[0, 1, 2, 3]]), np.zeros(1, dtype=np.int64),
                   {"outer_boundary": np.array([2]), "electrode_pos": np.array([0]),
                    "electrode_neg": np.array([1])})


@pytest.mark.parametrize("name", ["tet", "b333", "b435", "b666", "A"])
def test_assembly_bitwise(name):
    d = golden("assembly")
    mesh = _single_tet() if name == "tet" else O.box_mesh(*map(int, d[f"{name}_dims"]))
    t, v, tp = d[f"{name}_t"], d[f"{name}_v"], d[f"{name}_tp"]
    for tag, kw in (("full", {}), ("raw", dict(apply_constraints=False)),
                    ("noeq", dict(equilibrate=False))):
        s = O.assemble(mesh, {0: O.OMaterial()}, 25.0, 37.0, t, v, tp, 0.5, **kw)
        assert np.array_equal(s.row_ptr, d[f"{name}_{tag}_row_ptr"])
        assert np.array_equal(s.col_idx, d[f"{name}_{tag}_col_idx"])
        assert np.array_equal(s.vals, d[f"{name}_{tag}_vals"])
        assert np.array_equal(s.rhs, d[f"{name}_{tag}_rhs"])
        assert s.scale == float(d[f"{name}_{tag}_scale"])


def test_two_region_assembly_bitwise():
    d = golden("assembly")
    mesh = O.box_mesh(4, 3, 5)
    mesh.regions = d["reg2_regions"]
    mats = {0: O.OMaterial(), 1: O.OMaterial(k=0.9e-3, rho_c=2.5e-3, sigma0=0.35e-3, alpha=0.01)}
    s = O.assemble(mesh, mats, 25.0, 37.0, d["reg2_t"], d["reg2_v"], d["reg2_t"], 0.25)
    assert np.array_equal(s.vals, d["reg2_vals"]) and np.array_equal(s.rhs, d["reg2_rhs"])


def test_gmres_bitwise():
    d = golden("gmres")
    for c in range(int(d["ncases"])):
        m, tol, pre = d[f"c{c}_params"]
        x, st = O.gmres(d[f"c{c}_row_ptr"], d[f"c{c}_col_idx"], d[f"c{c}_vals"], d[f"c{c}_b"], None,
                        int(m), float(tol), None, "jacobi" if pre else "none")
        assert np.array_equal(x, d[f"c{c}_x"])
        it, rs, fr, conv = d[f"c{c}_stats"]
        assert (st.iterations, st.restarts, st.final_relative_residual, st.converged) == \
            (int(it), int(rs), float(fr), bool(conv))
        flat = np.concatenate([np.asarray(h, dtype=float) for h in st.residual_history])
        assert np.array_equal(flat, d[f"c{c}_hist"])


@pytest.mark.parametrize("tag", ["1e-10", "1e-12"])
def test_run_A40_bitwise(tag):
    d = golden(f"run_A40_{tag}")
    run = O.run(O.box_mesh(15, 15, 16), {0: O.OMaterial()},
                O.OSim(total_time=40.0, tolerance=float(tag)))
    assert np.array_equal([r.time for r in run.records], d["time"])
    assert np.array_equal([r.dt for r in run.records], d["dt"])
    assert np.array_equal([r.corrector_iters for r in run.records], d["corrector_iters"])
    for i, k in enumerate(d["kept"]):
        assert np.array_equal(run.records[k].T, d["T"][i])
        assert np.array_equal(run.records[k].V, d["V"][i])
    assert [run.accepted_steps, run.corrector_passes, run.solver_iterations, run.dt_halvings] == \
        list(d["summary"])


def test_pcg_oracle_solves_fem_system():
    d = golden("assembly")
    ptr, col, vals, rhs = (d["A_full_row_ptr"], d["A_full_col_idx"], d["A_full_vals"], d["A_full_rhs"])
    x, st = O.pcg(ptr, col, vals, rhs, None, tol=1e-10)
    assert st.converged
    assert np.linalg.norm(rhs - O.matvec(ptr, col, vals, x)) / np.linalg.norm(rhs) <= 1e-10
