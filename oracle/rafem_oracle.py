"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the RAFEM hot path (reference package ``rafem``
0.1.0 under /root/reference/pkg/src/rafem).  It exists to *check* the
B200 path, never to run as part of it: only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl
reference`` legs of ``bench.py`` may import it.  The product package
``paper_2409_13036_b200`` must not import anything from here.

Parity pin: the functions below are checked bit-for-bit against the
reference itself (tests/test_oracle_vs_reference.py, run wherever
/root/reference exists) and against golden vectors generated from the
reference (tests/golden/*.npz, made by tests/golden/make_golden.py).
The arithmetic order mirrors the numpy primitives the reference uses
(np.linalg.det/inv, np.einsum, np.bincount, np.linalg.norm, np.dot),
so results are bit-identical on the numpy this was pinned on (2.3.5).

Every function cites the reference file:line it restates (paths are
relative to /root/reference/pkg/src/rafem/).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# mesh: structured Kuhn box (mesh.py:306-375, TetMesh orientation fix-up
# mesh.py:115-126)

BOX_EXTENT = ((-50.0, 50.0), (-50.0, 50.0), (0.0, 100.0))  # mesh.py:39
_ELECTRODE_XS = (15.0, -15.0)                               # mesh.py:42
_ELECTRODE_Z = (40.0, 60.0)                                 # mesh.py:44


@dataclass
class OMesh:
    nodes: np.ndarray            # (N, 3) f64
    tets: np.ndarray             # (M, 4) i64, positively oriented
    regions: np.ndarray          # (M,) i64
    node_sets: dict = field(default_factory=dict)

    @property
    def node_count(self) -> int:
        return int(self.nodes.shape[0])

    @property
    def tet_count(self) -> int:
        return int(self.tets.shape[0])


def _orient(nodes, tets):
    """Swap vertices 1/2 of negatively oriented tets (mesh.py:115-120)."""
    tets = tets.copy()
    c = nodes[tets]
    det = np.linalg.det(c[:, 1:, :] - c[:, :1, :])
    neg = det < 0.0
    tets[neg, 1], tets[neg, 2] = tets[neg, 2].copy(), tets[neg, 1].copy()
    return tets


def _closest(coords, target, high):
    """Index of the grid coordinate nearest ``target`` (mesh.py:286-290)."""
    d = np.abs(coords - target)
    hits = np.nonzero(d == d.min())[0]
    return int(hits[-1]) if high else int(hits[0])


def box_mesh(nx: int, ny: int, nz: int, extent=BOX_EXTENT) -> OMesh:
    """Kuhn 6-tet box, node id (i*ny + j)*nz + k (mesh.py:306-375)."""
    if min(nx, ny, nz) < 2:
        raise ValueError("box needs at least 2 nodes per axis")
    xs = np.linspace(extent[0][0], extent[0][1], nx)
    ys = np.linspace(extent[1][0], extent[1][1], ny)
    zs = np.linspace(extent[2][0], extent[2][1], nz)
    I, J, K = np.indices((nx, ny, nz))
    I, J, K = I.reshape(-1), J.reshape(-1), K.reshape(-1)
    nodes = np.stack([xs[I], ys[J], zs[K]], axis=1)

    ci, cj, ck = (a.reshape(-1) for a in np.indices((nx - 1, ny - 1, nz - 1)))
    per_cell = []
    # the six axis orders, lexicographic (mesh.py:47-49); each tet walks
    # the cell from corner (0,0,0) to (1,1,1) one axis at a time
    for order in ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)):
        step = [0, 0, 0]
        verts = [((ci) * ny + cj) * nz + ck]
        for ax in order:
            step[ax] += 1
            verts.append(((ci + step[0]) * ny + (cj + step[1])) * nz + (ck + step[2]))
        per_cell.append(np.stack(verts, axis=1))
    tets = np.stack(per_cell, axis=1).reshape(-1, 4).astype(np.int64)
    tets = _orient(nodes, tets)

    surf = (I == 0) | (I == nx - 1) | (J == 0) | (J == ny - 1) | (K == 0) | (K == nz - 1)
    outer = np.nonzero(surf)[0].astype(np.int64)

    def electrode(xt):
        i = _closest(xs, xt, high=xt >= 0.0)
        j = _closest(ys, 0.0, high=False)
        ks = np.nonzero((zs >= _ELECTRODE_Z[0]) & (zs <= _ELECTRODE_Z[1]))[0]
        if ks.size == 0:
            ks = np.array([_closest(zs, 0.5 * sum(_ELECTRODE_Z), high=False)])
        return i, j, ks

    ip, jp, kp = electrode(_ELECTRODE_XS[0])
    im, jm, km = electrode(_ELECTRODE_XS[1])
    if (ip, jp) == (im, jm):
        if ip + 1 < nx:
            ip += 1
        else:
            im -= 1
    pos = np.array([(ip * ny + jp) * nz + k for k in kp], dtype=np.int64)
    neg = np.array([(im * ny + jm) * nz + k for k in km], dtype=np.int64)
    sets = {"outer_boundary": np.unique(outer), "electrode_pos": np.unique(pos),
            "electrode_neg": np.unique(neg)}
    return OMesh(nodes, tets, np.zeros(tets.shape[0], dtype=np.int64), sets)


# ---------------------------------------------------------------------------
# material / config (fem.py:85-147)

@dataclass
class OMaterial:
    k: float = 0.5e-3
    rho_c: float = 3.6e-3
    sigma0: float = 0.2e-3
    alpha: float = 0.02
    t_ref: float = 37.0


@dataclass
class OSim:
    total_time: float = 900.0
    dt_init: float = 0.5
    dt_min: float = 1e-6
    dt_max: float = 10.0
    corrector_tol: float = 1e-4
    max_corrector_iters: int = 50
    applied_voltage: float = 25.0
    boundary_temp: float = 37.0
    initial_temp: float = 37.0
    # solver (solver.py:81-96) — only the iterative path is restated
    method: str = "gmres"       # "gmres" or "pcg"
    restart_m: int = 30
    tolerance: float = 1e-10
    max_total_iters: int | None = None
    precondition: str = "jacobi"


def per_tet(mesh: OMesh, materials: dict):
    """Per-element coefficient arrays from region tags (fem.py:212-226)."""
    out = {name: np.empty(mesh.tet_count) for name in ("k", "rho_c", "sigma0", "alpha", "t_ref")}
    for tag in np.unique(mesh.regions):
        if int(tag) not in materials:
            raise KeyError(f"no material defined for region tag {int(tag)}")
        m = materials[int(tag)]
        sel = mesh.regions == tag
        for name in out:
            out[name][sel] = getattr(m, name)
    return out


# ---------------------------------------------------------------------------
# element geometry and coefficients (fem.py:229-292)

def geometry(mesh: OMesh):
    """P1 gradients (M,4,3) and volumes (M,) (fem.py:229-240)."""
    c = mesh.nodes[mesh.tets]
    e = c[:, 1:, :] - c[:, :1, :]
    vol = np.linalg.det(e) / 6.0
    g = np.empty((c.shape[0], 4, 3))
    g[:, 1:, :] = np.linalg.inv(e).transpose(0, 2, 1)
    g[:, 0, :] = -g[:, 1:, :].sum(axis=1)
    return g, vol


MASS_PATTERN = (np.ones((4, 4)) + np.eye(4)) / 20.0   # fem.py:244


class PhysicsRange(RuntimeError):
    """sigma(T) <= 0 in some element (fem.py:72-73, 272-278)."""

    def __init__(self, element: int, message: str):
        self.element = element
        super().__init__(message)


def element_terms(mesh, coef, grads, vol, t_field, v_field):
    """sigma, V-block, base, mass, Joule load per element (fem.py:247-292)."""
    tv = t_field[mesh.tets]
    tbar = tv.mean(axis=1)
    sigma = coef["sigma0"] * (1.0 + coef["alpha"] * (tbar - coef["t_ref"]))
    bad = np.nonzero(sigma <= 0.0)[0]
    if bad.size:
        e = int(bad[0])
        raise PhysicsRange(e, f"sigma(T) = {sigma[e]:.3g} S/mm <= 0 in element {e} "
                              f"(mean T {tbar[e]:.3g})")
    base = vol[:, None, None] * np.einsum("mid,mjd->mij", grads, grads)
    mass = vol[:, None, None] * MASS_PATTERN
    gv = np.einsum("mj,mjd->md", v_field[mesh.tets], grads)
    power = sigma * np.einsum("md,md->m", gv, gv) * vol
    return sigma, base, mass, power / 4.0


# ---------------------------------------------------------------------------
# sparse (sparse.py:164-219)

def compress(nrows, rows, cols, vals):
    """Triplets -> CSR with in-order duplicate sums (sparse.py:164-197).

    Duplicates are folded after a stable sort on (row, col), summing
    each run first to last from 0.0, exactly like a sequential
    ``bincount`` over the sorted triplets.
    """
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    if rows.size == 0:
        return np.zeros(nrows + 1, np.int64), np.empty(0, np.int64), np.empty(0)
    perm = np.lexsort((cols, rows))
    r, c, v = rows[perm], cols[perm], vals[perm]
    head = np.ones(r.size, dtype=bool)
    head[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    run = np.cumsum(head) - 1
    summed = np.bincount(run, weights=v)
    first = np.nonzero(head)[0]
    ptr = np.concatenate(([0], np.cumsum(np.bincount(r[first], minlength=nrows)))).astype(np.int64)
    return ptr, c[first].copy(), summed


def row_of_entry(row_ptr):
    n = row_ptr.size - 1
    return np.repeat(np.arange(n, dtype=np.int64), np.diff(row_ptr))


def matvec(row_ptr, col_idx, vals, x):
    """y = A x, per-row left-to-right sum of rounded products (sparse.py:205-219)."""
    n = row_ptr.size - 1
    if col_idx.size == 0:
        return np.zeros(n)
    return np.bincount(row_of_entry(row_ptr), weights=vals * x[col_idx], minlength=n)


def diag_of(row_ptr, col_idx, vals):
    """Stored diagonal, zero where absent (sparse.py:121-128)."""
    n = row_ptr.size - 1
    d = np.zeros(n)
    r = row_of_entry(row_ptr)
    hit = r == col_idx
    d[r[hit]] = vals[hit]
    return d


# ---------------------------------------------------------------------------
# global assembly (fem.py:306-430)

@dataclass
class OSystem:
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray
    rhs: np.ndarray
    scale: float


def dirichlet(mesh: OMesh, applied_voltage: float, boundary_temp: float):
    """Constraint mask and values over the interleaved dofs (fem.py:403-413)."""
    n2 = 2 * mesh.node_count
    mask = np.zeros(n2, dtype=bool)
    val = np.zeros(n2)
    pos, neg = mesh.node_sets["electrode_pos"], mesh.node_sets["electrode_neg"]
    outer = mesh.node_sets["outer_boundary"]
    mask[2 * pos] = True
    val[2 * pos] = applied_voltage
    mask[2 * neg] = True
    val[2 * neg] = 0.0
    mask[2 * outer + 1] = True
    val[2 * outer + 1] = boundary_temp
    return mask, val


def assemble(mesh: OMesh, materials: dict, applied_voltage: float, boundary_temp: float,
             t_iter, v_iter, t_prev, dt, apply_constraints=True, equilibrate=True,
             geom=None) -> OSystem:
    """Interleaved 2N x 2N corrector-pass system (fem.py:325-430)."""
    if dt <= 0.0:
        raise ValueError("dt must be positive")
    t_iter = np.asarray(t_iter, dtype=np.float64)
    v_iter = np.asarray(v_iter, dtype=np.float64)
    t_prev = np.asarray(t_prev, dtype=np.float64)
    coef = per_tet(mesh, materials)
    rcdt = coef["rho_c"] / dt
    grads, vol = geom if geom is not None else geometry(mesh)
    sigma, base, mass, fj = element_terms(mesh, coef, grads, vol, t_iter, v_iter)
    tets = mesh.tets
    m = tets.shape[0]
    r4 = np.broadcast_to(tets[:, :, None], (m, 4, 4)).reshape(-1)
    c4 = np.broadcast_to(tets[:, None, :], (m, 4, 4)).reshape(-1)
    kv = (sigma[:, None, None] * base).reshape(-1)
    mt = rcdt[:, None, None] * mass
    kt = (mt + coef["k"][:, None, None] * base).reshape(-1)
    # V triplets for every element first, then T triplets (fem.py:381-383)
    ptr, col, vals = compress(2 * mesh.node_count,
                              np.concatenate([2 * r4, 2 * r4 + 1]),
                              np.concatenate([2 * c4, 2 * c4 + 1]),
                              np.concatenate([kv, kt]))
    load = np.einsum("mij,mj->mi", mt, t_prev[tets]) + fj[:, None]
    rhs = np.bincount((2 * tets + 1).reshape(-1), weights=load.reshape(-1),
                      minlength=2 * mesh.node_count)

    scale = 1.0
    er = row_of_entry(ptr)
    if equilibrate:                                            # fem.py:390-400
        d = diag_of(ptr, col, vals)
        sv, st = float(d[0::2].sum()), float(d[1::2].sum())
        if sv > 0.0 and st > 0.0:
            scale = 2.0 ** round(np.log2(st / sv))
        vals[er % 2 == 0] *= scale
        rhs[0::2] *= scale

    if apply_constraints:                                      # fem.py:402-428
        mask, val = dirichlet(mesh, applied_voltage, boundary_temp)
        rc, cc = mask[er], mask[col]
        moving = cc & ~rc
        if moving.any():
            rhs -= np.bincount(er[moving], weights=vals[moving] * val[col[moving]],
                               minlength=rhs.size)
        vals[rc | cc] = 0.0
        vals[(er == col) & rc] = 1.0
        rhs[mask] = val[mask]
    return OSystem(ptr, col, vals, rhs, scale)


# ---------------------------------------------------------------------------
# Krylov solvers

class Breakdown(RuntimeError):
    """Arnoldi breakdown above tolerance (solver.py:73-74, 516-524)."""


@dataclass
class OStats:
    iterations: int = 0
    restarts: int = 0
    final_relative_residual: float = 0.0
    stagnated: bool = False
    converged: bool = True
    residual_history: list = field(default_factory=list)


def _jacobi(row_ptr, col_idx, vals):
    d = diag_of(row_ptr, col_idx, vals)
    if np.any(d == 0.0):
        raise ValueError("Jacobi preconditioning requires a zero-free diagonal")
    return 1.0 / d


def gmres(row_ptr, col_idx, vals, b, x0=None, restart_m=30, tol=1e-10,
          max_total_iters=None, precondition="none"):
    """Restarted GMRES(m), MGS Arnoldi, Givens LSQ, right Jacobi (solver.py:381-531)."""
    b = np.asarray(b, dtype=np.float64)
    n = b.size
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    cap = max_total_iters if max_total_iters is not None else 10 * n
    minv = _jacobi(row_ptr, col_idx, vals) if precondition == "jacobi" else None
    st = OStats()
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        return np.zeros(n), st
    done = 0
    ncycles = 0
    weak = 0
    latched = False
    last_start = None
    ok = False
    rel = math.inf
    tiny = np.finfo(np.float64).tiny
    while True:
        r = b - matvec(row_ptr, col_idx, vals, x)
        rel = float(np.linalg.norm(r)) / bn
        if last_start is not None:                             # solver.py:440-447
            weak = weak + 1 if rel > (1.0 - 1e-3) * last_start else 0
            latched = latched or weak >= 3
            last_start = None
        if rel <= tol:
            ok = True
            break
        if done >= cap:
            break
        start = rel
        beta = rel * bn
        basis = np.zeros((restart_m + 1, n))
        basis[0] = r / beta
        hess = np.zeros((restart_m + 1, restart_m))
        g = np.zeros(restart_m + 1)
        g[0] = beta
        cs = np.zeros(restart_m)
        sn = np.zeros(restart_m)
        hist = []
        used = 0
        broke = False
        dead = False
        for k in range(restart_m):
            z = basis[k] * minv if minv is not None else basis[k]
            w = matvec(row_ptr, col_idx, vals, z)
            for i in range(k + 1):                             # MGS (solver.py:471-474)
                hik = float(np.dot(basis[i], w))
                hess[i, k] = hik
                w = w - hik * basis[i]
            hk1 = float(np.linalg.norm(w))
            hess[k + 1, k] = hk1
            done += 1
            for i in range(k):                                 # old rotations
                a0 = cs[i] * hess[i, k] + sn[i] * hess[i + 1, k]
                hess[i + 1, k] = -sn[i] * hess[i, k] + cs[i] * hess[i + 1, k]
                hess[i, k] = a0
            rad = math.hypot(hess[k, k], hess[k + 1, k])
            if rad == 0.0:
                dead = True
                used = k
                break
            cs[k] = hess[k, k] / rad
            sn[k] = hess[k + 1, k] / rad
            hess[k, k] = rad
            hess[k + 1, k] = 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            used = k + 1
            est = abs(g[k + 1]) / bn
            hist.append(est)
            if hk1 < tiny:
                broke = True
                break
            basis[k + 1] = w / hk1
            if est <= tol or done >= cap:
                break
        if used > 0:                                           # solver.py:504-511
            y = np.zeros(used)
            for i in range(used - 1, -1, -1):
                y[i] = (g[i] - float(np.dot(hess[i, i + 1:used], y[i + 1:used]))) / hess[i, i]
            upd = basis[:used].T @ y
            if minv is not None:
                upd = minv * upd
            x = x + upd
        st.residual_history.append(hist)
        ncycles += 1
        last_start = start
        if broke or dead:
            rel = float(np.linalg.norm(b - matvec(row_ptr, col_idx, vals, x))) / bn
            if rel <= tol:
                ok = True
                break
            raise Breakdown(f"Arnoldi breakdown with relative residual {rel:.3e} "
                            f"above tolerance {tol:.3e}")
    st.iterations = done
    st.restarts = max(ncycles - 1, 0)
    st.final_relative_residual = rel
    st.converged = ok
    st.stagnated = latched and not ok
    return x, st


def pcg(row_ptr, col_idx, vals, b, x0=None, tol=1e-10, max_total_iters=None,
        precondition="jacobi"):
    """Jacobi-preconditioned CG with a true-residual exit check.

    Not in the reference (which only ships GMRES); this is the oracle for
    the device "pcg" backend, kept to the same stats contract as
    solver.py:113-130: converged only when the TRUE residual meets tol.
    """
    b = np.asarray(b, dtype=np.float64)
    n = b.size
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    cap = max_total_iters if max_total_iters is not None else 10 * n
    minv = _jacobi(row_ptr, col_idx, vals) if precondition == "jacobi" else np.ones(n)
    st = OStats()
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        return np.zeros(n), st
    done = 0
    restarts = 0
    while True:
        r = b - matvec(row_ptr, col_idx, vals, x)
        rel = float(np.linalg.norm(r)) / bn
        if rel <= tol:
            st.converged = True
            break
        if done >= cap:
            st.converged = False
            break
        hist = []
        z = minv * r
        p = z.copy()
        rz = float(np.dot(r, z))
        while done < cap:
            q = matvec(row_ptr, col_idx, vals, p)
            alpha = rz / float(np.dot(p, q))
            x = x + alpha * p
            r = r - alpha * q
            done += 1
            est = float(np.linalg.norm(r)) / bn
            hist.append(est)
            if est <= tol:
                break
            z = minv * r
            rz_new = float(np.dot(r, z))
            p = z + (rz_new / rz) * p
            rz = rz_new
        st.residual_history.append(hist)
        restarts += 1
    st.iterations = done
    st.restarts = max(restarts - 1, 0)
    st.final_relative_residual = rel
    return x, st


# ---------------------------------------------------------------------------
# predictor-corrector time loop (fem.py:437-644)

@dataclass
class ORecord:
    step: int
    time: float
    dt: float
    corrector_iters: int
    T: np.ndarray
    V: np.ndarray


@dataclass
class ORun:
    records: list
    accepted_steps: int
    corrector_passes: int
    solver_iterations: int
    dt_halvings: int
    wall_s: float


def run(mesh: OMesh, materials: dict, cfg: OSim, keep_fields=True, max_steps=None, on_step=None) -> ORun:
    """Adaptive predictor-corrector loop (fem.py:554-644, 463-540).

    ``max_steps`` stops after that many accepted steps (a bounded sample
    of the workload for CPU timing); ``None`` runs to ``total_time``.
    ``on_step(record)`` is called per accepted step, like the reference's
    ``sink`` (fem.py:609-610).
    """
    t0 = time.perf_counter()
    N = mesh.node_count
    geom = geometry(mesh)
    T = np.full(N, cfg.initial_temp)
    V = np.zeros(N)
    T_prev = T.copy()
    t, dt_cur, dt_prev, step = 0.0, cfg.dt_init, cfg.dt_init, 0
    recs, passes, inner, halvings = [], 0, 0, 0
    while t < cfg.total_time:
        if max_steps is not None and step >= max_steps:
            break
        remaining = cfg.total_time - t
        last = dt_cur >= remaining
        dt = remaining if last else dt_cur
        t_it = T + (dt / dt_prev) * (T - T_prev) if step >= 1 else T.copy()   # fem.py:445-449
        v_it = V.copy()
        x_old = np.empty(2 * N)
        x_old[0::2], x_old[1::2] = v_it, t_it
        ok, used = False, 0
        for it in range(1, cfg.max_corrector_iters + 1):
            used = it
            passes += 1
            sysm = assemble(mesh, materials, cfg.applied_voltage, cfg.boundary_temp,
                            t_it, v_it, T, dt, geom=geom)
            try:
                if cfg.method == "pcg":
                    x_new, stt = pcg(sysm.row_ptr, sysm.col_idx, sysm.vals, sysm.rhs.copy(),
                                     x0=x_old.copy(), tol=cfg.tolerance,
                                     max_total_iters=cfg.max_total_iters,
                                     precondition=cfg.precondition)
                else:
                    x_new, stt = gmres(sysm.row_ptr, sysm.col_idx, sysm.vals, sysm.rhs.copy(),
                                       x0=x_old.copy(), restart_m=cfg.restart_m,
                                       tol=cfg.tolerance, max_total_iters=cfg.max_total_iters,
                                       precondition=cfg.precondition)
            except Breakdown:
                break
            inner += stt.iterations
            if not stt.converged:
                break
            delta = float(np.max(np.abs(x_new - x_old) / np.maximum(1.0, np.abs(x_old))))
            v_it, t_it = x_new[0::2].copy(), x_new[1::2].copy()
            x_old = x_new
            if delta < cfg.corrector_tol:
                ok = True
                break
        if ok:
            T_prev, T, V = T, t_it, v_it
            dt_prev = dt
            t = cfg.total_time if last else t + dt
            recs.append(ORecord(step, t, dt, used, T if keep_fields else None,
                                V if keep_fields else None))
            if on_step is not None:
                on_step(recs[-1])
            step += 1
            if used <= 5:
                dt_cur = min(dt * 1.5, cfg.dt_max)
            elif used >= 20:
                dt_cur = max(dt * 0.75, cfg.dt_min)
            else:
                dt_cur = dt
        else:
            if dt <= cfg.dt_min:
                raise RuntimeError(f"step {step} failed at the dt floor ({dt:g} s)")
            dt_cur = max(dt * 0.5, cfg.dt_min)
            halvings += 1
    return ORun(recs, step, passes, inner, halvings, time.perf_counter() - t0)


def psnr(ref_field, test_field, peak):
    """20 log10(peak) - 10 log10(MSE), inf when identical (metrics.py:47-64)."""
    d = np.asarray(ref_field, dtype=np.float64) - np.asarray(test_field, dtype=np.float64)
    mse = float(np.mean(d * d))
    if mse == 0.0:
        return math.inf
    return 20.0 * math.log10(peak) - 10.0 * math.log10(mse)
