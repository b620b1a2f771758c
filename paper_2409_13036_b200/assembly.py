"""Assembly plug-in: ``assemble_global`` on the B200.

Mirrors rafem/fem.py's configuration types (``RegionMaterial``,
``MaterialParams``, ``SimConfig``: fem.py:85-147), ``PhysicsRangeError``
(fem.py:72-73), ``AssembledSystem`` (fem.py:299-303) and the signature and
semantics of ``assemble_global`` (fem.py:325-430).  The symbolic work
(pattern, incidence lists, slot map, geometry) happens once per mesh on
the device and is cached; each call is one H2D of the three fields plus
four kernels, and the returned matrix stays in HBM.
"""

from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .csr import DeviceCsrMatrix
from .krylov import SolverConfig

__all__ = [
    "AssembledSystem", "DeviceMesh", "MaterialParams", "PhysicsRangeError", "RegionMaterial", "SimConfig",
    "assemble_global", "device_mesh",
]


class PhysicsRangeError(RuntimeError):
    """A material law left its admissible range (fem.py:72-73)."""


@dataclass
class RegionMaterial:
    k: float = 0.5e-3
    rho_c: float = 3.6e-3
    sigma0: float = 0.2e-3
    alpha: float = 0.02
    t_ref: float = 37.0

    def __post_init__(self):
        if self.k <= 0.0 or self.rho_c <= 0.0 or self.sigma0 <= 0.0:
            raise ValueError("k, rho_c and sigma0 must be positive")


@dataclass
class MaterialParams:
    regions: dict = field(default_factory=lambda: {0: RegionMaterial()})

    @classmethod
    def default(cls) -> "MaterialParams":
        return cls()

    def for_region(self, tag: int) -> RegionMaterial:
        try:
            return self.regions[tag]
        except KeyError:
            raise KeyError(f"no material defined for region tag {tag}") from None


@dataclass
class SimConfig:
    total_time: float = 900.0
    dt_init: float = 0.5
    dt_min: float = 1e-6
    dt_max: float = 10.0
    corrector_tol: float = 1e-4
    max_corrector_iters: int = 50
    applied_voltage: float = 25.0
    boundary_temp: float = 37.0
    initial_temp: float = 37.0
    threads: int = 1
    solver: SolverConfig = field(default_factory=SolverConfig)

    def __post_init__(self):
        if self.total_time <= 0.0:
            raise ValueError("total_time must be positive")
        if not (0.0 < self.dt_min <= self.dt_init <= self.dt_max):
            raise ValueError("need 0 < dt_min <= dt_init <= dt_max")
        if self.corrector_tol <= 0.0:
            raise ValueError("corrector_tol must be positive")
        if self.max_corrector_iters < 1:
            raise ValueError("max_corrector_iters must be at least 1")
        if self.threads < 1:
            raise ValueError("threads must be at least 1")


# ---------------------------------------------------------------------------
# device handles

def _region_tables(mesh, material):
    """Region tag -> row index and per-region coefficient tables (fem.py:212-226)."""
    reg = np.asarray(mesh.regions)
    lo = int(reg.min()) if reg.size else 0
    if reg.size and lo == int(reg.max()):  # one region (the common case): no sort
        tags, index = np.array([lo]), np.zeros(reg.shape, dtype=np.int32)
    else:
        tags, index = np.unique(reg, return_inverse=True)
    mats = [material.for_region(int(t)) for t in tags]  # KeyError like the reference
    tab = {name: np.ascontiguousarray([getattr(m, name) for m in mats], dtype=np.float64)
           for name in ("k", "rho_c", "sigma0", "alpha", "t_ref")}
    return np.ascontiguousarray(index, dtype=np.int32), tab


def _dof_kinds(mesh):
    """Dirichlet kind per interleaved dof (fem.py:403-413)."""
    kind = np.zeros(2 * mesh.node_count, dtype=np.uint8)
    kind[2 * mesh.node_sets["electrode_pos"]] = nat.DOF_APPLIED_VOLTAGE
    kind[2 * mesh.node_sets["electrode_neg"]] = nat.DOF_ZERO
    kind[2 * mesh.node_sets["outer_boundary"] + 1] = nat.DOF_BOUNDARY_TEMP
    return kind


_EXACT_GEOMETRY = os.environ.get("RAFEM_EXACT_GEOMETRY", "0") == "1"


def set_exact_geometry(on: bool) -> None:
    """Bit-exact assembly mode: device meshes created afterwards take the
    reference's own element geometry (fem.py:229-240, np.linalg.det / inv,
    computed once per mesh on the host and uploaded through
    rafem_mesh_set_geometry); every assembly is then bit-identical to
    assemble_global.  Off by default: the device geometry kernel agrees to
    rtol 1e-12.  Also RAFEM_EXACT_GEOMETRY=1."""
    global _EXACT_GEOMETRY
    _EXACT_GEOMETRY = bool(on)


def reference_geometry(nodes, tets):
    """_basis_gradients (fem.py:229-240) for all tets: gradients (M, 4, 3)
    and volumes (M,), the same numpy operations in the same order."""
    corners = nodes[tets]
    edges = corners[:, 1:, :] - corners[:, :1, :]
    vol = np.linalg.det(edges) / 6.0
    inv = np.linalg.inv(edges)
    grads = np.empty((corners.shape[0], 4, 3))
    grads[:, 1:, :] = np.transpose(inv, (0, 2, 1))
    grads[:, 0, :] = -grads[:, 1:, :].sum(axis=1)
    return grads, vol


class DeviceMesh:
    """Mesh + symbolic pattern + geometry resident on the device."""

    def __init__(self, mesh, material):
        self.node_count = int(mesh.nodes.shape[0])
        self.tet_count = int(mesh.tets.shape[0])
        region_index, tab = _region_tables(mesh, material)
        self.regions_tags = _region_tags(mesh)  # memoised per regions array (np.unique costs ~0.14 ms here)
        kind = _dof_kinds(mesh)
        nodes = np.ascontiguousarray(mesh.nodes, dtype=np.float64)
        tets = np.ascontiguousarray(mesh.tets, dtype=np.int64)
        h = C.c_void_p()
        L = nat.lib()
        rc = L.rafem_mesh_create(nat.context(), self.node_count, nat.ptr(nodes), self.tet_count,
                                 nat.ptr(tets), nat.ptr(region_index), len(tab["k"]),
                                 nat.ptr(tab["k"]), nat.ptr(tab["rho_c"]), nat.ptr(tab["sigma0"]),
                                 nat.ptr(tab["alpha"]), nat.ptr(tab["t_ref"]), nat.ptr(kind),
                                 C.byref(h))
        nat.check(rc, "mesh setup")
        self._adopt(h)
        self.exact_geometry = False
        if _EXACT_GEOMETRY and self.tet_count > 0:
            grads, vol = reference_geometry(nodes, tets)
            grads = np.ascontiguousarray(grads, dtype=np.float64)
            vol = np.ascontiguousarray(vol, dtype=np.float64)
            nat.check(L.rafem_mesh_set_geometry(h, nat.ptr(grads), nat.ptr(vol)), "mesh geometry")
            self.exact_geometry = True

    def _adopt(self, h):
        L = nat.lib()
        self.handle = h
        # pooled systems reference the mesh: one finalizer frees them first
        # (also at interpreter exit, where finalizers run before __del__)
        self._pool: list = []
        self._finalizer = weakref.finalize(self, _destroy_mesh, L, h, self._pool)
        self.slots = int(L.rafem_mesh_slots(h))
        self._pattern = None

    @classmethod
    def from_box(cls, nx: int, ny: int, nz: int, material=None, extent=None) -> "DeviceMesh":
        """generate_box_mesh (mesh.py:306-375) built directly in HBM
        (rafem_mesh_create_box): no host mesh, no host validation pass."""
        from .boxmesh import DEFAULT_EXTENT, electrode_nodes
        material = material or MaterialParams.default()
        extent = extent or DEFAULT_EXTENT
        rm = material.for_region(0)
        pos, neg = electrode_nodes(nx, ny, nz, extent)
        ext = np.ascontiguousarray([v for ab in extent for v in ab], dtype=np.float64)
        pos = np.ascontiguousarray(pos, dtype=np.int64)
        neg = np.ascontiguousarray(neg, dtype=np.int64)
        h = C.c_void_p()
        rc = nat.lib().rafem_mesh_create_box(nat.context(), int(nx), int(ny), int(nz), nat.ptr(ext), nat.ptr(pos),
                                             pos.size, nat.ptr(neg), neg.size, rm.k, rm.rho_c, rm.sigma0, rm.alpha,
                                             rm.t_ref, C.byref(h))
        nat.check(rc, "box mesh setup")
        self = cls.__new__(cls)
        nt = C.c_int64()
        self.node_count = int(nat.lib().rafem_mesh_counts(h, C.byref(nt)))
        self.tet_count = int(nt.value)
        self.regions_tags = np.zeros(1, dtype=np.int64)
        self._adopt(h)
        return self

    def download(self):
        """(nodes (N, 3) f64, tets (M, 4) int64, dof kinds (2N,) u8) from HBM."""
        nodes = np.empty((self.node_count, 3))
        tets = np.empty((self.tet_count, 4), dtype=np.int32)
        kind = np.empty(2 * self.node_count, dtype=np.uint8)
        nat.check(nat.lib().rafem_mesh_download(self.handle, nat.ptr(nodes), nat.ptr(tets), nat.ptr(kind)), "download")
        return nodes, tets.astype(np.int64), kind

    def node_pattern(self):
        if self._pattern is None:
            rp = np.empty(self.node_count + 1, dtype=np.int64)
            col = np.empty(max(self.slots, 1), dtype=np.int32)
            nat.check(nat.lib().rafem_mesh_pattern(self.handle, nat.ptr(rp), nat.ptr(col)), "pattern")
            self._pattern = (rp, col[: self.slots].astype(np.int64))
        return self._pattern

    @property
    def dof_row_ptr(self):
        if not hasattr(self, "_dof_rp"):
            rp, _ = self.node_pattern()
            deg = np.diff(rp)
            out = np.empty(2 * self.node_count + 1, dtype=np.int64)
            out[0] = 0
            out[1::2] = 2 * rp[:-1] + deg      # end of row 2i
            out[2::2] = 2 * rp[1:]             # end of row 2i+1
            self._dof_rp = out
        return self._dof_rp

    @property
    def dof_col_idx(self):
        if not hasattr(self, "_dof_ci"):
            rp, col = self.node_pattern()
            deg = np.diff(rp)
            node = np.repeat(np.arange(self.node_count), deg)
            pos = np.arange(self.slots) - rp[node]                 # offset within the node row
            out = np.empty(2 * self.slots, dtype=np.int64)
            out[2 * rp[node] + pos] = 2 * col                       # V row: cols 2j
            out[2 * rp[node] + deg[node] + pos] = 2 * col + 1       # T row: cols 2j+1
            self._dof_ci = out
        return self._dof_ci

    def acquire_system(self):
        if self._pool:
            return self._pool.pop()
        h = C.c_void_p()
        nat.check(nat.lib().rafem_system_create(self.handle, C.byref(h)), "system alloc")
        return h

    def release_system(self, h):
        if not self._finalizer.alive:  # mesh already freed (interpreter exit): nothing to return to
            return
        if len(self._pool) < 4:
            self._pool.append(h)
        else:
            nat.lib().rafem_system_destroy(h)



def _destroy_mesh(L, h, pool):
    for s in pool:
        L.rafem_system_destroy(s)
    pool.clear()
    L.rafem_mesh_destroy(h)


class SystemHandle:
    """One assembled system in HBM; returned to its mesh's pool when dropped."""

    def __init__(self, mesh: DeviceMesh):
        self.mesh = mesh
        self.handle = mesh.acquire_system()
        self.scale = 1.0
        self._rhs = None

    def __del__(self):
        try:
            self.mesh.release_system(self.handle)
        except Exception:
            pass

    def download_vals(self):
        out = np.empty(2 * self.mesh.slots)
        nat.check(nat.lib().rafem_system_download(self.handle, nat.ptr(out), None), "download")
        return out

    def rhs(self):
        if self._rhs is None:
            out = np.empty(2 * self.mesh.node_count)
            nat.check(nat.lib().rafem_system_download(self.handle, None, nat.ptr(out)), "download")
            self._rhs = out
        return self._rhs

    def spmv(self, x):
        y = np.empty(2 * self.mesh.node_count)
        nat.check(nat.lib().rafem_system_spmv(self.handle, nat.ptr(x), nat.ptr(y)), "spmv")
        return y

    def solve(self, b, x0, params, x_out, st, hist, cyc):
        return nat.lib().rafem_system_solve(self.handle, nat.ptr(b), nat.ptr(x0), C.byref(params),
                                            nat.ptr(x_out), C.byref(st), nat.ptr(hist), hist.size,
                                            nat.ptr(cyc), cyc.size)


_MESH_CACHE: dict = {}


_TAGS_CACHE: dict = {}


def _region_tags(mesh):
    """np.unique(mesh.regions), memoised per regions array (the plug-in seam
    asks for it on every corrector pass; a 43K-tet unique costs ~0.1 ms)."""
    key = id(mesh.regions)
    hit = _TAGS_CACHE.get(key)
    if hit is not None and hit[0] is mesh.regions:
        return hit[1]
    reg = np.asarray(mesh.regions)
    if reg.size and reg.min() == reg.max():  # one region (the common case): no sort
        tags = reg.reshape(-1)[:1].copy()
    else:
        tags = np.unique(reg)
    if len(_TAGS_CACHE) > 64:
        _TAGS_CACHE.clear()
    _TAGS_CACHE[key] = (mesh.regions, tags)
    return tags


def _material_key(mesh, material):
    tags = _region_tags(mesh)
    rows = []
    for t in tags:
        m = material.for_region(int(t))
        rows.append((int(t), m.k, m.rho_c, m.sigma0, m.alpha, m.t_ref))
    return tuple(rows)


def device_mesh(mesh, material) -> DeviceMesh:
    """Cached device mesh for (mesh object, material values)."""
    key = (id(mesh), _material_key(mesh, material), _EXACT_GEOMETRY)
    hit = _MESH_CACHE.get(key)
    if hit is not None:
        ref, nodes_id, tets_id, dm = hit
        if ref() is mesh and nodes_id == id(mesh.nodes) and tets_id == id(mesh.tets):
            return dm
    dm = DeviceMesh(mesh, material)
    try:
        ref = weakref.ref(mesh, lambda _r, k=key: _MESH_CACHE.pop(k, None))
    except TypeError:  # not weak-referenceable: keep a strong ref
        ref = (lambda m=mesh: m)
    _MESH_CACHE[key] = (ref, id(mesh.nodes), id(mesh.tets), dm)
    return dm


class AssembledSystem:
    """(matrix, rhs, voltage_row_scale) of fem.py:299-303; rhs is read from HBM on first use."""

    def __init__(self, handle: SystemHandle):
        self._h = handle
        self.matrix = DeviceCsrMatrix(handle)
        self.voltage_row_scale = handle.scale

    @property
    def rhs(self):
        return self._h.rhs()

    @property
    def device(self) -> SystemHandle:
        return self._h


def assemble_global(mesh, material, config, t_iter, v_iter, t_prev, dt, apply_constraints=True,
                    equilibrate=True, threads=None) -> AssembledSystem:
    """Interleaved 2N x 2N system for one corrector pass (fem.py:325-430).

    ``threads`` is validated and otherwise ignored: the device fill is
    bit-identical for any launch configuration, which is the property the
    reference's thread count guarantees (fem.py:343-346).
    """
    if dt <= 0.0:
        raise ValueError("dt must be positive")
    threads = config.threads if threads is None else threads
    if threads < 1:
        raise ValueError("threads must be at least 1")
    n = int(mesh.nodes.shape[0])
    t_iter = np.ascontiguousarray(t_iter, dtype=np.float64)
    v_iter = np.ascontiguousarray(v_iter, dtype=np.float64)
    t_prev = np.ascontiguousarray(t_prev, dtype=np.float64)
    for arr in (t_iter, v_iter, t_prev):
        if arr.shape != (n,):
            raise ValueError("field length does not match the mesh node count")
    dm = device_mesh(mesh, material)
    h = SystemHandle(dm)
    p = nat.AssembleParams()
    p.dt = float(dt)
    p.applied_voltage = float(config.applied_voltage)
    p.boundary_temp = float(config.boundary_temp)
    p.apply_constraints = 1 if apply_constraints else 0
    p.equilibrate = 1 if equilibrate else 0
    scale = C.c_double()
    bad = C.c_int64(-1)
    # the rhs comes back with the same stream synchronisation: every caller
    # of assemble_global reads it (fem.py:495)
    rhs = np.empty(2 * n)
    rc = nat.lib().rafem_assemble_rhs(h.handle, nat.ptr(t_iter), nat.ptr(v_iter), nat.ptr(t_prev),
                                      C.byref(p), C.byref(scale), C.byref(bad), nat.ptr(rhs))
    if rc == nat.ERR_PHYSICS:
        e = int(bad.value)
        tets = mesh.tets[e]
        tbar = float(np.mean(t_iter[tets]))
        rm = material.for_region(int(mesh.regions[e]))
        sigma = rm.sigma0 * (1.0 + rm.alpha * (tbar - rm.t_ref))
        raise PhysicsRangeError(
            f"sigma(T) = {sigma:.3g} S/mm <= 0 in element {e} (mean T {tbar:.3g})")
    nat.check(rc, "assemble")
    h.scale = float(scale.value)
    h._rhs = rhs
    return AssembledSystem(h)
