"""Tet mesh container and the structured Kuhn box generator (input side).

Mirrors rafem/mesh.py's ``TetMesh`` contract (mesh.py:66-134: index
validation, required node sets, positive orientation by swapping local
vertices 1 and 2) and ``generate_box_mesh`` (mesh.py:306-375: node id
``(i*ny + j)*nz + k``, six Kuhn tets per cell in lexicographic axis-order,
outer surface and two electrode columns).  The box generator knows each
Kuhn tet's orientation from its axis permutation's parity, so it skips the
per-tet determinant pass for big meshes (the device geometry kernel
re-derives every volume anyway).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["MeshValidationError", "TetMesh", "electrode_nodes", "generate_box_mesh", "REQUIRED_SETS"]

GEOM_EPS = 1e-12
REQUIRED_SETS = ("outer_boundary", "electrode_pos", "electrode_neg")
DEFAULT_EXTENT = ((-50.0, 50.0), (-50.0, 50.0), (0.0, 100.0))
ELECTRODE_X = (15.0, -15.0)
ELECTRODE_Y = 0.0
ELECTRODE_Z = (40.0, 60.0)
# axis orders of the Kuhn split (lexicographic) and their parities
_ORDERS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))
_ODD = (False, True, True, False, False, True)


class MeshValidationError(ValueError):
    pass


def signed_volumes(nodes, tets):
    c = nodes[tets]
    return np.linalg.det(c[:, 1:, :] - c[:, :1, :]) / 6.0


@dataclass
class TetMesh:
    nodes: np.ndarray
    tets: np.ndarray
    regions: np.ndarray
    node_sets: dict = field(default_factory=dict)
    trusted: bool = field(default=False, repr=False, compare=False)

    def __post_init__(self):
        self.nodes = np.ascontiguousarray(self.nodes, dtype=np.float64)
        self.tets = np.ascontiguousarray(self.tets, dtype=np.int64)
        self.regions = np.ascontiguousarray(self.regions, dtype=np.int64)
        if self.nodes.ndim != 2 or self.nodes.shape[1] != 3:
            raise MeshValidationError("nodes must be an (N, 3) array")
        if self.tets.ndim != 2 or self.tets.shape[1] != 4:
            raise MeshValidationError("tets must be an (M, 4) array")
        if self.regions.shape != (self.tets.shape[0],):
            raise MeshValidationError("regions must hold one tag per tet")
        n = self.node_count
        self.node_sets = {k: np.unique(np.ascontiguousarray(v, dtype=np.int64))
                          for k, v in self.node_sets.items()}
        for name in REQUIRED_SETS:
            if name not in self.node_sets:
                raise MeshValidationError(f"required node set {name!r} is missing")
        if self.trusted:
            return
        if not np.all(np.isfinite(self.nodes)):
            raise MeshValidationError("node coordinates must be finite")
        if self.tets.size and (self.tets.min() < 0 or self.tets.max() >= n):
            bad = int(np.flatnonzero(((self.tets < 0) | (self.tets >= n)).any(axis=1))[0])
            raise MeshValidationError(f"tet {bad} references a node outside 0..{n - 1}")
        for name, ids in self.node_sets.items():
            if ids.size and (ids[0] < 0 or ids[-1] >= n):
                raise MeshValidationError(f"node set {name!r} references a node outside 0..{n - 1}")
        pos, neg = self.node_sets["electrode_pos"], self.node_sets["electrode_neg"]
        if pos.size == 0 or neg.size == 0:
            raise MeshValidationError("electrode node sets must be non-empty")
        if np.intersect1d(pos, neg).size:
            raise MeshValidationError("electrode_pos and electrode_neg must be disjoint")
        vol = signed_volumes(self.nodes, self.tets)
        neg_or = vol < 0.0
        if neg_or.any():
            self.tets[neg_or, 1], self.tets[neg_or, 2] = (self.tets[neg_or, 2].copy(),
                                                         self.tets[neg_or, 1].copy())
            vol = signed_volumes(self.nodes, self.tets)
        small = vol <= GEOM_EPS
        if small.any():
            bad = int(np.flatnonzero(small)[0])
            raise MeshValidationError(f"tet {bad} is degenerate (volume {vol[bad]:.3g} mm^3 <= {GEOM_EPS:g})")

    @property
    def node_count(self) -> int:
        return int(self.nodes.shape[0])

    @property
    def tet_count(self) -> int:
        return int(self.tets.shape[0])


def _nearest(coords, target, high):
    d = np.abs(coords - target)
    hits = np.flatnonzero(d == d.min())
    return int(hits[-1] if high else hits[0])


def electrode_nodes(nx: int, ny: int, nz: int, extent=DEFAULT_EXTENT):
    """Node ids of the two electrode columns (mesh.py:350-375): nearest grid
    column to each electrode's (x, y), z within the electrode span."""
    (x0, x1), (y0, y1), (z0, z1) = extent
    xs, ys, zs = np.linspace(x0, x1, nx), np.linspace(y0, y1, ny), np.linspace(z0, z1, nz)

    def column(xt):
        ci = _nearest(xs, xt, xt >= 0.0)
        cj = _nearest(ys, ELECTRODE_Y, False)
        ks = np.flatnonzero((zs >= ELECTRODE_Z[0]) & (zs <= ELECTRODE_Z[1]))
        if ks.size == 0:
            ks = np.array([_nearest(zs, 0.5 * (ELECTRODE_Z[0] + ELECTRODE_Z[1]), False)])
        return ci, cj, ks

    ip, jp, kp = column(ELECTRODE_X[0])
    im, jm, km = column(ELECTRODE_X[1])
    if ip == im and jp == jm:
        if ip + 1 < nx:
            ip += 1
        else:
            im -= 1
    pos = ((ip * ny + jp) * nz + np.asarray(kp)).astype(np.int64)
    neg = ((im * ny + jm) * nz + np.asarray(km)).astype(np.int64)
    return pos, neg


def generate_box_mesh(nx: int, ny: int, nz: int, extent=DEFAULT_EXTENT) -> TetMesh:
    """Structured box, 6 Kuhn tets per cell (mesh.py:306-375), bit-identical output."""
    if nx < 2 or ny < 2 or nz < 2:
        raise ValueError("generate_box_mesh requires nx, ny, nz >= 2")
    (x0, x1), (y0, y1), (z0, z1) = extent
    if not (x0 < x1 and y0 < y1 and z0 < z1):
        raise ValueError("extent bounds must be strictly increasing per axis")
    xs, ys, zs = np.linspace(x0, x1, nx), np.linspace(y0, y1, ny), np.linspace(z0, z1, nz)
    nodes = np.empty((nx * ny * nz, 3))
    nodes.reshape(nx, ny, nz, 3)[..., 0] = xs[:, None, None]
    nodes.reshape(nx, ny, nz, 3)[..., 1] = ys[None, :, None]
    nodes.reshape(nx, ny, nz, 3)[..., 2] = zs[None, None, :]

    # cell-corner node id and the id offsets of the axis steps
    corner = ((np.arange(nx - 1)[:, None, None] * ny + np.arange(ny - 1)[None, :, None]) * nz
              + np.arange(nz - 1)[None, None, :]).reshape(-1).astype(np.int64)
    step = (ny * nz, nz, 1)
    tets = np.empty((corner.size, 6, 4), dtype=np.int64)
    for t, (order, odd) in enumerate(zip(_ORDERS, _ODD)):
        off = [0]
        for ax in order:
            off.append(off[-1] + step[ax])
        if odd:  # negative Kuhn parity: TetMesh swaps local vertices 1 and 2
            off[1], off[2] = off[2], off[1]
        for v in range(4):
            tets[:, t, v] = corner + off[v]
    tets = tets.reshape(-1, 4)

    i, j, k = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    surf = (i == 0) | (i == nx - 1) | (j == 0) | (j == ny - 1) | (k == 0) | (k == nz - 1)
    outer = np.flatnonzero(surf.reshape(-1)).astype(np.int64)

    pos, neg = electrode_nodes(nx, ny, nz, extent)
    return TetMesh(nodes=nodes, tets=tets, regions=np.zeros(tets.shape[0], dtype=np.int64),
                   node_sets={"outer_boundary": outer, "electrode_pos": pos, "electrode_neg": neg},
                   trusted=True)
