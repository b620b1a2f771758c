"""Numpy emulation of the kernel-per-phase PCG engine (csrc/shard.cu).

Test infrastructure only: it stands in for KPDeviceEngine so the host-side
orchestration of paper_2409_13036_b200.shard (ShardedPCG phase sequence,
halo exchange, scalar-slot all-gather, state polling) can run under a
multi-process gloo group on CPU.  It restates the device state machine of
kp_update_kernel step for step; the arithmetic is plain numpy.
"""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import torch

from paper_2409_13036_b200.shard import (BNORM_FINISH, FLAG_CONVERGED, FLAG_DONE, FLAG_NEED_HEAD, HEAD,
                                         PACK_U, PACK_U_AFTER_HEAD, PACK_X, SPMV, SPMV_AFTER_HEAD, UPDATE,
                                         UPDATE_FIRST)


def _state():
    return dict(done=0, converged=0, status=0, need_head=0, total=0, hlen=0, cycles=0, hstart=0,
                bnorm=0.0, alpha=0.0, beta=0.0, gamma=0.0, rel=np.inf)


class NumpyKPEngine:
    """rp/ci/va: dof-level CSR of the owned dof rows (2 n_own), columns in
    the extended dof numbering (2 * local node + component)."""

    def __init__(self, rp, ci, va, n_own, n_ext, nranks, rank, send_idx):
        self.rp, self.ci, self.va = rp, ci, va
        self.n_own, self.n_ext, self.nranks, self.rank = n_own, n_ext, nranks, rank
        self.send_idx = np.asarray(send_idx, dtype=np.int64)
        self.n_send = int(self.send_idx.size)
        self._x = np.zeros(2 * n_ext)
        self._u = np.zeros(2 * n_ext)
        self._send = np.zeros(2 * max(self.n_send, 1))
        self._slots = np.zeros(4 * nranks)
        self.x_ext = torch.from_numpy(self._x)
        self.u_ext = torch.from_numpy(self._u)
        self.send_buf = torch.from_numpy(self._send)
        self.slots = torch.from_numpy(self._slots)
        n = 2 * n_own
        self.r, self.w, self.s, self.p = (np.zeros(n) for _ in range(4))
        self.hist, self.cyc = [], []
        self.part_a = (0.0, 0.0)
        self.idx = 0
        self.st = [_state(), _state()]
        self.launches = 0

    def _matvec(self, v):
        prod = self.va * v[self.ci]
        return np.add.reduceat(prod, self.rp[:-1]) if prod.size else np.zeros(2 * self.n_own)

    def _slot(self, vals):
        self._slots[4 * self.rank:4 * self.rank + 4] = vals

    def begin(self, b, x0, params):
        n = 2 * self.n_own
        self.b = np.zeros(n) if b is None else np.array(b, dtype=np.float64)
        self._x[:n] = 0.0 if x0 is None else x0
        diag = np.zeros(n)
        rows = np.repeat(np.arange(n), np.diff(self.rp))
        on = self.ci == rows  # owned dof j sits at ext column j
        diag[rows[on]] = self.va[on]
        if params.precondition == 1:
            if np.any(diag == 0.0):
                raise ValueError("zero diagonal entry: Jacobi preconditioner undefined")
            self.minv = 1.0 / diag
        else:
            self.minv = np.ones(n)
        self.tol = params.tolerance
        self.cap = params.max_total_iters if params.max_total_iters > 0 else 10 * n
        self._slot([float(self.b @ self.b), 0.0, 0.0, 0.0])

    def _gathered(self):
        s = np.zeros(3)
        for q in range(self.nranks):
            s += self._slots[4 * q:4 * q + 3]
        return s

    def launch(self, phase):
        self.launches += 1
        S = self.st[self.idx]
        n = 2 * self.n_own
        if phase == BNORM_FINISH:
            bb = sum(self._slots[4 * q] for q in range(self.nranks))
            st = _state()
            st["bnorm"] = float(np.sqrt(bb))
            if st["bnorm"] == 0.0:
                st.update(done=1, converged=1, rel=0.0)
            self.st = [dict(st), dict(st)]
            self.idx = 0
        elif phase == HEAD:
            if S["done"]:
                return
            self.r[:] = self.b - self._matvec(self._x)
            self._u[:n] = self.minv * self.r
            self.part_a = (float(self.r @ self._u[:n]), float(self.r @ self.r))
        elif phase in (SPMV, SPMV_AFTER_HEAD):
            if S["done"] or (phase == SPMV and S["need_head"]):
                return
            self.w[:] = self._matvec(self._u)
            self._slot([self.part_a[0], float(self.w @ self._u[:n]), self.part_a[1], 0.0])
        elif phase in (UPDATE, UPDATE_FIRST):
            self._update(S, phase == UPDATE_FIRST)
        elif phase in (PACK_X, PACK_U, PACK_U_AFTER_HEAD):
            if S["done"] or (phase == PACK_U and S["need_head"]):
                return
            v = (self._x if phase == PACK_X else self._u).reshape(-1, 2)
            self._send[:2 * self.n_send] = v[self.send_idx].reshape(-1)
        else:
            raise ValueError(phase)

    def _update(self, S, first):
        S = dict(S)
        gn, dn, rrn = self._gathered()
        step = False
        stopped = S["done"] or (not first and S["need_head"])
        alpha, beta = S["alpha"], 0.0
        if not stopped:
            if first:
                S["need_head"] = 0
                S["rel"] = float(np.sqrt(rrn)) / S["bnorm"]
                if S["rel"] <= self.tol:
                    S.update(done=1, converged=1)
                elif S["total"] >= self.cap:
                    S["done"] = 1
                elif not (gn > 0 and dn > 0):
                    S.update(status=1, done=1)
                else:
                    S.update(gamma=gn, alpha=gn / dn, beta=0.0, hstart=S["hlen"])
                    alpha = S["alpha"]
                    step = True
            else:
                S["total"] += 1
                est = float(np.sqrt(rrn)) / S["bnorm"]
                self.hist.append(est)
                S["hlen"] += 1
                close = False
                if est <= self.tol or S["total"] >= self.cap:
                    S["need_head"] = 1
                    close = True
                else:
                    bnew = gn / S["gamma"]
                    den = dn - bnew * gn / S["alpha"]
                    if not (gn > 0 and den > 0):
                        S.update(status=1, done=1)
                        close = True
                    else:
                        S.update(alpha=gn / den, beta=bnew, gamma=gn)
                        alpha, beta = S["alpha"], bnew
                        step = True
                if close:
                    self.cyc.append(S["hlen"] - S["hstart"])
                    S["cycles"] += 1
        self.st[self.idx ^ 1] = S
        self.idx ^= 1
        if not step:
            return
        n = 2 * self.n_own
        u, x = self._u[:n], self._x[:n]
        if first:
            self.p[:] = u
            self.s[:] = self.w
        else:
            self.p[:] = u + beta * self.p
            self.s[:] = self.w + beta * self.s
        x += alpha * self.p
        self.r -= alpha * self.s
        u[:] = self.minv * self.r
        self.part_a = (float(self.r @ u), float(self.r @ self.r))

    def iterate(self, n):
        for _ in range(n):
            self.launch(SPMV)
            self.launch(UPDATE)

    def state(self):
        S = self.st[self.idx]
        f = (FLAG_DONE if S["done"] else 0) | (FLAG_NEED_HEAD if S["need_head"] else 0) | \
            (FLAG_CONVERGED if S["converged"] else 0)
        return f, S["total"], S["rel"]

    def finish(self, hist_cap):
        S = self.st[self.idx]
        x = self._x[:2 * self.n_own].copy()
        if S["bnorm"] == 0.0:
            x[:] = 0.0
        st = SimpleNamespace(iterations=S["total"], restarts=max(S["cycles"] - 1, 0),
                             final_relative_residual=S["rel"], converged=S["converged"], stagnated=0,
                             cycles=S["cycles"], history_len=S["hlen"], device_ms=0.0)
        hist = np.zeros(hist_cap)
        cyc = np.zeros(hist_cap, dtype=np.int64)
        h = self.hist[:hist_cap]
        hist[:len(h)] = h
        cyc[:len(self.cyc[:hist_cap])] = self.cyc[:hist_cap]
        return S["status"], x, st, hist, cyc


def local_csr(row_ptr, col_idx, vals, plan):
    """Owned dof rows of a global dof CSR with columns renumbered into the
    shard's extended numbering."""
    g2l = np.full(plan.bounds[-1], -1, dtype=np.int64)
    l2g = plan.local_to_global
    g2l[l2g] = np.arange(l2g.size)
    r0, r1 = 2 * plan.lo, 2 * plan.hi
    s0, s1 = row_ptr[r0], row_ptr[r1]
    cols = col_idx[s0:s1]
    lc = 2 * g2l[cols // 2] + cols % 2
    assert np.all(lc >= 0), "a column of an owned row is neither owned nor ghost"
    return row_ptr[r0:r1 + 1] - s0, lc, vals[s0:s1].copy()


class EmulShardSystem:
    """Stand-in for ShardedSystem on CPU: oracle assembly of the shard's
    sub-mesh, global equilibration scale from all-gathered owned-row
    diagonal sums, NumpyKPEngine + ShardedPCG for the solve."""

    def __init__(self, om, materials, plan, comm, O):
        self.O, self.om, self.mats, self.plan, self.comm = O, om, materials, plan, comm
        l2g = plan.local_to_global
        pos = np.full(om.node_count, -1, dtype=np.int64)
        pos[l2g] = np.arange(l2g.size)
        sets = {}
        for k, v in om.node_sets.items():
            loc = pos[np.asarray(v)]
            sets[k] = np.sort(loc[loc >= 0])
        self.sub = O.OMesh(nodes=om.nodes[l2g], tets=plan.local_tets, regions=om.regions[plan.tet_ids],
                           node_sets=sets)

    def assemble(self, te, ve, tpe, dt, config):
        O, p = self.O, self.plan
        n2 = 2 * p.n_own
        raw = O.assemble(self.sub, self.mats, config.applied_voltage, config.boundary_temp, te, ve, tpe, dt,
                         equilibrate=False, apply_constraints=False)
        d = O.diag_of(raw.row_ptr, raw.col_idx, raw.vals)[:n2]
        rows = self.comm.allgather_host(np.array([d[0::2].sum(), d[1::2].sum()])) if self.comm else \
            np.array([[d[0::2].sum(), d[1::2].sum()]])
        sv, st = 0.0, 0.0
        for r in range(rows.shape[0]):
            sv += rows[r, 0]
            st += rows[r, 1]
        scale = 2.0 ** round(np.log2(st / sv)) if sv > 0 and st > 0 else 1.0
        loc = O.assemble(self.sub, self.mats, config.applied_voltage, config.boundary_temp, te, ve, tpe, dt,
                         equilibrate=False)
        # scaling by a power of two commutes exactly with the elimination
        mask, _ = O.dirichlet(self.sub, config.applied_voltage, config.boundary_temp)
        er = O.row_of_entry(loc.row_ptr)
        vrow = (er % 2 == 0) & ~mask[er]
        vals = loc.vals.copy()
        vals[vrow] *= scale
        rhs = loc.rhs.copy()
        rsel = np.zeros(rhs.size, dtype=bool)
        rsel[0::2] = True
        rhs[rsel & ~mask] *= scale
        end = loc.row_ptr[n2]
        self.rp, self.ci, self.va = loc.row_ptr[:n2 + 1].copy(), loc.col_idx[:end].copy(), vals[:end]
        self.b = rhs[:n2].copy()
        return scale

    def solve(self, b=None, x0=None, config=None):
        from paper_2409_13036_b200 import _native as nat
        from paper_2409_13036_b200.shard import ShardedPCG
        p = self.plan
        eng = NumpyKPEngine(self.rp, self.ci, self.va, p.n_own, p.n_ext, p.nranks, p.rank, p.send_index())
        prm = nat.SolverParams()
        prm.method, prm.restart_m, prm.tolerance = 1, 30, config.tolerance
        prm.max_total_iters = int(config.max_total_iters or 0)
        prm.precondition = 1 if config.precondition == "jacobi" else 0
        return ShardedPCG(eng, self.comm, p, batch=8).solve(self.b if b is None else b, x0, prm, 1 << 14)
