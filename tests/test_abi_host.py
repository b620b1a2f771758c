"""CPU-side checks: the C-ABI library loads and exports every declared
symbol, and the host-side mirror of the reference interface behaves like
the reference (config validation, box mesh, dof bookkeeping)."""

import hashlib
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_meshes

HEADER = os.path.join(ROOT, "include", "rafem_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rafem_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2409_13036_b200 import _native as nat
    lib = nat.load_library()
    names = declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), f"{name} declared in include/rafem_b200.h but not exported"
    assert set(names) == set(nat.EXPORTED), "ctypes signatures must cover the header exactly"


def test_library_is_sm100a():
    from paper_2409_13036_b200 import _native as nat
    blob = open(nat.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob


def test_no_gpu_raises_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2409_13036_b200 import _native as nat
    with pytest.raises(nat.NativeUnavailable):
        nat.context()


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("dims", ["2x2x2", "3x4x2", "4x3x5", "15x15x16", "20x20x21", "80x80x79"])
def test_generate_box_mesh_matches_reference_digest(dims):
    from paper_2409_13036_b200 import generate_box_mesh
    ref = golden_meshes()[dims]
    m = generate_box_mesh(*map(int, dims.split("x")))
    assert m.node_count == ref["N"] and m.tet_count == ref["M"]
    assert _digest(m.nodes.astype("<f8")) == ref["nodes"]
    assert _digest(m.tets.astype("<i8")) == ref["tets"]
    for k, v in ref["sets"].items():
        assert _digest(m.node_sets[k].astype("<i8")) == v


def test_tetmesh_orientation_fixup_and_validation():
    from paper_2409_13036_b200 import TetMesh
    from paper_2409_13036_b200.boxmesh import MeshValidationError
    nodes = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.0, 1, 0], [0.0, 0, 1]])
    sets = {"outer_boundary": [2], "electrode_pos": [0], "electrode_neg": [1]}
    m = TetMesh(nodes, np.array([[0, 2, 1, 3]]), np.zeros(1), sets)
    assert m.tets.tolist() == [[0, 1, 2, 3]]
    with pytest.raises(MeshValidationError):
        TetMesh(nodes, np.array([[0, 1, 2, 4]]), np.zeros(1), sets)
    with pytest.raises(MeshValidationError):
        TetMesh(nodes, np.array([[0, 1, 2, 3]]), np.zeros(1),
                {"outer_boundary": [2], "electrode_pos": [0], "electrode_neg": [0]})


def test_solver_config_validation_matches_reference():
    from paper_2409_13036_b200 import SolverConfig
    for bad in (dict(backend="cg"), dict(backend="cholesky"), dict(backend="magma"),
                dict(tolerance=2.0), dict(tolerance=0.0), dict(restart_m=0),
                dict(precondition="ilu"), dict(ordering="amd"), dict(max_total_iters=0)):
        with pytest.raises(ValueError):
            SolverConfig(**bad)
    SolverConfig(backend="pcg", precondition="jacobi")


def test_sim_config_and_material_validation():
    from paper_2409_13036_b200 import RegionMaterial, SimConfig
    for bad in (dict(total_time=0.0), dict(dt_init=0.1, dt_min=0.5), dict(dt_init=20.0, dt_max=10.0),
                dict(corrector_tol=0.0), dict(max_corrector_iters=0), dict(threads=0)):
        with pytest.raises(ValueError):
            SimConfig(**bad)
    for bad in (dict(k=0.0), dict(sigma0=-1.0), dict(rho_c=0.0)):
        with pytest.raises(ValueError):
            RegionMaterial(**bad)


def test_csr_validation_matches_reference():
    from paper_2409_13036_b200 import CooMatrix, CsrMatrix
    with pytest.raises(ValueError):
        CooMatrix(2, 2, [0, 2], [0, 0], [1.0, 1.0])
    with pytest.raises(ValueError):
        CooMatrix(2, 2, [0, 1], [0], [1.0, 2.0])
    with pytest.raises(ValueError):
        CsrMatrix(2, 3, np.array([0, 2, 2]), np.array([2, 0]), np.array([1.0, 1.0]))
    with pytest.raises(ValueError):
        CsrMatrix(1, 3, np.array([0, 2]), np.array([1, 1]), np.array([1.0, 1.0]))
    with pytest.raises(ValueError):
        CsrMatrix(2, 2, np.array([0, 3, 2]), np.array([0, 1, 0]), np.ones(3))
    a = CsrMatrix(3, 3, np.array([0, 2, 2, 3]), np.array([0, 2, 1]), np.array([1.0, 2.0, 3.0]))
    assert a.diagonal().tolist() == [1.0, 0.0, 0.0]
    assert a.toarray()[0, 2] == 2.0


def test_dof_kinds_follow_reference_constraints():
    from oracle import rafem_oracle as O
    from paper_2409_13036_b200 import _native as nat
    from paper_2409_13036_b200 import generate_box_mesh
    from paper_2409_13036_b200.assembly import _dof_kinds
    mesh = generate_box_mesh(5, 4, 6)
    kind = _dof_kinds(mesh)
    mask, val = O.dirichlet(O.box_mesh(5, 4, 6), 25.0, 37.0)
    assert np.array_equal(kind != nat.DOF_FREE, mask)
    vals = np.where(kind == nat.DOF_APPLIED_VOLTAGE, 25.0,
                    np.where(kind == nat.DOF_BOUNDARY_TEMP, 37.0, 0.0))
    assert np.array_equal(vals[mask], val[mask])


def test_plugin_install_rebinds_reference_seam(reference):
    from paper_2409_13036_b200 import plugin
    import rafem.fem as fem
    orig = (fem.assemble_global, fem.solve)
    plugin.install()
    try:
        assert fem.assemble_global is not orig[0] and fem.solve is not orig[1]
        assert fem.solve.__module__.startswith("paper_2409_13036_b200")
    finally:
        plugin.uninstall()
    assert (fem.assemble_global, fem.solve) == orig
