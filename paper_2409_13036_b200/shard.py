"""Row-block sharding of the corrector-pass system across GPUs.

The reference is single-process (its only parallelism is the assembly
thread pool, fem.py:368-379); this module adds the one decomposition the
B200 build needs for meshes that outgrow one GPU: contiguous blocks of
node rows (a node's V and T rows never split; for Kuhn boxes a block is an
x-slab, mesh.py:334-335), one shard per rank, one process per GPU.

Per shard:
  * ``ShardPlan``   — owned node block, ghost nodes (non-owned vertices of
    the tets touching the block, ordered by owner then global id), the
    sub-mesh of those tets in ascending global tet order (so every owned
    row is assembled from the same contributions in the same order as the
    global system: owned rows are bit-identical to assemble_global's), and
    the halo send lists.
  * ``ShardComm``   — the collectives: per-shard scalar slots all-gathered
    (the PCG dot products and the equilibration sums, reduced in rank order
    on the device so every rank takes identical decisions), and the halo
    exchange of ghost node values.  NCCL on device buffers (one process per
    GPU over NVLink) or host-staged (gloo; ranks sharing a GPU, CPU tests).
  * ``ShardedPCG``  — the host side of the kernel-per-phase PCG in
    csrc/shard.cu: launches the phases, puts the collectives between them,
    and reads the solver state only every ``batch`` iterations.
  * ``ShardedSystem`` — assemble_global (fem.py:325-430) split at its one
    global reduction (equilibration, fem.py:390-400) and solve
    (solver.py:580-636) for one shard.
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .krylov import KrylovBreakdownError, SolveStats

__all__ = ["ShardPlan", "partition_rows", "build_plan", "ShardComm", "ShardedPCG", "ShardedSystem",
           "KPDeviceEngine", "ShardedSimulation", "DeviceShardedSimulation", "connect_ipc"]

# phases of rafem_kp_launch (include/rafem_b200.h)
BNORM_FINISH, HEAD, SPMV_AFTER_HEAD, SPMV, UPDATE_FIRST, UPDATE, PACK_X, PACK_U_AFTER_HEAD, PACK_U = range(9)
FLAG_DONE, FLAG_NEED_HEAD, FLAG_CONVERGED = 1, 2, 4


# ---------------------------------------------------------------------------
# partition and plan (pure numpy; identical on every rank)

def partition_rows(tets: np.ndarray, n_nodes: int, nranks: int) -> np.ndarray:
    """Contiguous node-row blocks balanced by incident-tet count (a proxy
    for a row's slots and its share of the element work); returns the
    nranks + 1 block boundaries."""
    if nranks < 1 or nranks > max(n_nodes, 1):
        raise ValueError("need 1 <= nranks <= node count")
    w = np.bincount(np.asarray(tets, dtype=np.int64).reshape(-1), minlength=n_nodes).astype(np.float64) + 1.0
    cum = np.concatenate(([0.0], np.cumsum(w)))
    targets = cum[-1] * np.arange(1, nranks) / nranks
    cuts = np.searchsorted(cum, targets, side="left")
    bounds = np.concatenate(([0], cuts, [n_nodes])).astype(np.int64)
    # strictly increasing (every shard owns at least one node)
    for r in range(1, nranks + 1):
        bounds[r] = max(bounds[r], bounds[r - 1] + 1)
    for r in range(nranks - 1, -1, -1):
        bounds[r] = min(bounds[r], bounds[r + 1] - 1)
    if bounds[0] != 0:
        raise ValueError("mesh too small for this many shards")
    return bounds


@dataclass
class ShardPlan:
    rank: int
    nranks: int
    bounds: np.ndarray        # nranks + 1 node boundaries
    n_own: int
    ghosts: np.ndarray        # global ids of ghost nodes, ordered by (owner, id)
    tet_ids: np.ndarray       # global ids of the sub-mesh tets, ascending
    local_tets: np.ndarray    # (m, 4) local node ids
    recv: dict = field(default_factory=dict)   # q -> (start, count) in the ghost block
    send: dict = field(default_factory=dict)   # q -> local owned ids q needs, ascending global id

    @property
    def lo(self) -> int:
        return int(self.bounds[self.rank])

    @property
    def hi(self) -> int:
        return int(self.bounds[self.rank + 1])

    @property
    def n_ext(self) -> int:
        return self.n_own + int(self.ghosts.size)

    @property
    def local_to_global(self) -> np.ndarray:
        return np.concatenate([np.arange(self.lo, self.hi, dtype=np.int64), self.ghosts])

    @property
    def neighbours(self) -> list:
        return sorted(set(self.recv) | set(self.send))

    def send_index(self) -> np.ndarray:
        """Concatenated send lists in neighbour order (the packed buffer layout)."""
        parts = [self.send[q] for q in self.neighbours if q in self.send]
        return np.concatenate(parts).astype(np.int32) if parts else np.zeros(0, dtype=np.int32)

    def send_offsets(self) -> dict:
        off, out = 0, {}
        for q in self.neighbours:
            n = int(self.send[q].size) if q in self.send else 0
            out[q] = (off, n)
            off += n
        return out

    def extend(self, global_field: np.ndarray) -> np.ndarray:
        """Owned + ghost values of a global node field (helper for callers
        that hold the whole field, e.g. tests and single-host drivers)."""
        return np.ascontiguousarray(np.asarray(global_field)[self.local_to_global])


def build_plan(tets: np.ndarray, n_nodes: int, bounds: np.ndarray, rank: int) -> ShardPlan:
    """Shard `rank`'s sub-mesh, ghosts and halo lists from the global tets."""
    tets = np.asarray(tets, dtype=np.int64)
    nranks = len(bounds) - 1
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    owner = np.searchsorted(bounds, tets, side="right") - 1
    mine = owner == rank
    touching = np.flatnonzero(mine.any(axis=1))
    sub = tets[touching]
    sub_owner = owner[touching]
    verts = np.unique(sub)
    ghosts = verts[(verts < lo) | (verts >= hi)]  # ascending id == ordered by (owner, id)
    n_own = hi - lo
    g2l = np.full(n_nodes, -1, dtype=np.int64)
    g2l[lo:hi] = np.arange(n_own)
    g2l[ghosts] = n_own + np.arange(ghosts.size)
    local_tets = g2l[sub]
    recv, send = {}, {}
    gown = np.searchsorted(bounds, ghosts, side="right") - 1
    for q in np.unique(gown):
        idx = np.flatnonzero(gown == q)
        recv[int(q)] = (int(idx[0]), int(idx.size))
    sub_mine = sub_owner == rank
    for q in np.unique(sub_owner[~sub_mine]):
        rows = (sub_owner == q).any(axis=1)
        need = np.unique(sub[rows][sub_mine[rows]])
        send[int(q)] = (need - lo).astype(np.int64)
    return ShardPlan(rank=rank, nranks=nranks, bounds=np.asarray(bounds, dtype=np.int64), n_own=n_own,
                     ghosts=ghosts, tet_ids=touching, local_tets=local_tets, recv=recv, send=send)


def local_mesh(mesh, plan: ShardPlan):
    """The shard's sub-mesh as a TetMesh (local ids; node sets restricted)."""
    from .boxmesh import TetMesh
    l2g = plan.local_to_global
    g2l = {}
    pos = np.full(mesh.node_count, -1, dtype=np.int64)
    pos[l2g] = np.arange(l2g.size)
    for name, ids in mesh.node_sets.items():
        ids = np.asarray(ids, dtype=np.int64)
        loc = pos[ids]
        g2l[name] = np.sort(loc[loc >= 0])
    return TetMesh(nodes=mesh.nodes[l2g], tets=plan.local_tets, regions=mesh.regions[plan.tet_ids],
                   node_sets=g2l, trusted=True)


# ---------------------------------------------------------------------------
# collectives

class ShardComm:
    """Scalar-slot all-gather and halo exchange for one shard.

    ``device_collectives`` (NCCL, one GPU per rank): collectives run on the
    library's CUDA stream directly on device buffers.  Otherwise buffers
    are staged through host memory and exchanged with the process group's
    CPU collectives (gloo): ranks sharing one GPU, and the CPU tests.
    """

    def __init__(self, group=None, device_collectives: bool | None = None, stream=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        if device_collectives is None:
            device_collectives = dist.get_backend(group) == "nccl"
        self.device = device_collectives
        # torch stream the device collectives are ordered on.  The library
        # enqueues its phase kernels (pack, SpMV, update) on its own
        # non-blocking stream, so device collectives must run on THAT stream
        # to be ordered after the pack and before the SpMV: default to it.
        if self.device and stream is None:
            import torch
            from . import _native as nat
            stream = torch.cuda.ExternalStream(nat.lib().rafem_stream(nat.context()))
        self.stream = stream

    def _ctx(self):
        import contextlib
        import torch
        if self.device and self.stream is not None:
            return torch.cuda.stream(self.stream)
        return contextlib.nullcontext()

    def _sync(self, t):
        import torch
        if t.is_cuda:
            torch.cuda.synchronize(t.device)

    def allgather_slots(self, slots, width: int = 4):
        """slots: tensor of size * width doubles; slot `rank` is this shard's."""
        r, w = self.rank, width
        if self.size == 1:
            return
        if self.device:
            with self._ctx():
                # a separate input buffer (not a view of the output) keeps NCCL's
                # in-place rules out of the picture
                mine = slots[r * w:(r + 1) * w].clone()
                self.dist.all_gather_into_tensor(slots, mine, group=self.group)
            return
        self._sync(slots)
        mine = slots[r * w:(r + 1) * w].cpu().clone()
        out = [mine.new_empty(w) for _ in range(self.size)]
        self.dist.all_gather(out, mine, group=self.group)
        slots.copy_(self._torch().cat(out).to(slots.device))
        self._sync(slots)

    def allgather_host(self, arr: np.ndarray) -> np.ndarray:
        """(size, *arr.shape) gather of a small host array (rank order)."""
        import torch
        t = torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64))
        if self.size == 1:
            return t.numpy()[None]
        if self.device:
            dev = torch.device("cuda", torch.cuda.current_device())
            src = t.to(dev)
            out = torch.empty((self.size,) + tuple(t.shape), dtype=t.dtype, device=dev)
            self.dist.all_gather_into_tensor(out, src, group=self.group)
            return out.cpu().numpy()
        out = [torch.empty_like(t) for _ in range(self.size)]
        self.dist.all_gather(out, t, group=self.group)
        return torch.stack(out).numpy()

    def halo(self, plan: ShardPlan, send_buf, ext, n_send: int, width: int = 2, base: int | None = None):
        """ext[width * (base + recv[q])] <- neighbour q's packed values for
        this shard.  send_buf / ext: tensors of doubles, `width` per node;
        base = n_own for an extended vector (the default), 0 for a
        ghost-only buffer."""
        if self.size == 1 or not plan.neighbours:
            return
        offs = plan.send_offsets()
        n0 = plan.n_own if base is None else base
        w = width
        P2P = self.dist.P2POp
        if self.device:
            with self._ctx():
                ops = []
                for q in plan.neighbours:
                    so, sn = offs[q]
                    if sn:
                        ops.append(P2P(self.dist.isend, send_buf[w * so:w * (so + sn)], q, group=self.group))
                    if q in plan.recv:
                        rs, rn = plan.recv[q]
                        ops.append(P2P(self.dist.irecv, ext[w * (n0 + rs):w * (n0 + rs + rn)], q, group=self.group))
                if ops:
                    for req in self.dist.batch_isend_irecv(ops):
                        req.wait()
            return
        self._sync(ext)
        sb = send_buf[:w * n_send].cpu().clone() if n_send else None
        bufs, reqs = {}, []
        for q in plan.neighbours:
            so, sn = offs[q]
            if sn:
                reqs.append(self.dist.isend(sb[w * so:w * (so + sn)].clone(), q, group=self.group))
            if q in plan.recv:
                rs, rn = plan.recv[q]
                bufs[q] = ext.new_empty(w * rn, device="cpu")
                reqs.append(self.dist.irecv(bufs[q], q, group=self.group))
        for req in reqs:
            req.wait()
        for q, b in bufs.items():
            rs, rn = plan.recv[q]
            ext[w * (n0 + rs):w * (n0 + rs + rn)].copy_(b.to(ext.device))
        self._sync(ext)

    def exchange_fields(self, plan: ShardPlan, own: np.ndarray) -> np.ndarray:
        """Owned node values (n_own, k) -> extended (n_ext, k): ghost rows
        filled from their owners (host arrays; device-staged under NCCL)."""
        import torch
        own = np.ascontiguousarray(own, dtype=np.float64)
        k = own.shape[1] if own.ndim == 2 else 1
        flat = own.reshape(plan.n_own, k)
        ext = np.empty((plan.n_ext, k))
        ext[:plan.n_own] = flat
        if self.size == 1 or not plan.neighbours:
            return ext.reshape((plan.n_ext,) + own.shape[1:])
        dev = torch.device("cuda", torch.cuda.current_device()) if self.device else torch.device("cpu")
        sends, recvs, ops = [], {}, []
        for q in plan.neighbours:
            if q in plan.send and plan.send[q].size:
                t = torch.from_numpy(np.ascontiguousarray(flat[plan.send[q]])).to(dev)
                sends.append(t)
                ops.append(self.dist.P2POp(self.dist.isend, t, q, group=self.group))
            if q in plan.recv:
                rs, rn = plan.recv[q]
                recvs[q] = torch.empty((rn, k), dtype=torch.float64, device=dev)
                ops.append(self.dist.P2POp(self.dist.irecv, recvs[q], q, group=self.group))
        if self.device:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        else:
            reqs = [(self.dist.isend if op.op is self.dist.isend else self.dist.irecv)(op.tensor, op.peer,
                                                                                       group=self.group)
                    for op in ops]
            for req in reqs:
                req.wait()
        for q, t in recvs.items():
            rs, rn = plan.recv[q]
            ext[plan.n_own + rs:plan.n_own + rs + rn] = t.cpu().numpy()
        return ext.reshape((plan.n_ext,) + own.shape[1:])

    def allreduce_max(self, v: float) -> float:
        return float(np.max(self.allgather_host(np.array([v]))[:, 0])) if self.size > 1 else float(v)

    @staticmethod
    def _torch():
        import torch
        return torch


# ---------------------------------------------------------------------------
# device engine (ctypes over rafem_kp_*)

class _CudaArray:
    """Zero-copy view of library-owned device memory for torch."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None, "stream": None}


class KPDeviceEngine:
    """The kernel-per-phase PCG of csrc/shard.cu for one shard's system."""

    def __init__(self, system_handle, n_own: int, n_ext: int, nranks: int, rank: int,
                 send_idx: np.ndarray | None = None):
        import torch
        self.L = nat.lib()
        self.n_own, self.n_ext, self.nranks, self.rank = n_own, n_ext, nranks, rank
        h = C.c_void_p()
        nat.check(self.L.rafem_kp_create(system_handle, n_own, n_ext, nranks, rank, C.byref(h)), "kp_create")
        self.h = h
        idx = np.ascontiguousarray(send_idx if send_idx is not None else np.zeros(0), dtype=np.int32)
        nat.check(self.L.rafem_kp_set_halo(h, nat.ptr(idx), idx.size), "kp_set_halo")
        self.n_send = int(idx.size)
        px, pu, ps, pr = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        nat.check(self.L.rafem_kp_buffers(h, C.byref(px), C.byref(pu), C.byref(ps), C.byref(pr)), "kp_buffers")
        dev = torch.device("cuda", torch.cuda.current_device())
        self.x_ext = torch.as_tensor(_CudaArray(px.value, 2 * n_ext), device=dev)
        self.u_ext = torch.as_tensor(_CudaArray(pu.value, 2 * n_ext), device=dev)
        self.send_buf = torch.as_tensor(_CudaArray(ps.value, 2 * max(self.n_send, 1)), device=dev)
        self.slots = torch.as_tensor(_CudaArray(pr.value, 4 * nranks), device=dev)

    def close(self):
        if self.h:
            self.L.rafem_kp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def begin(self, b, x0, params):
        rc = self.L.rafem_kp_begin(self.h, nat.ptr(b), nat.ptr(x0), C.byref(params))
        if rc == nat.ERR_INVALID:
            raise ValueError(nat.last_error())
        nat.check(rc, "kp_begin")

    def launch(self, phase: int):
        nat.check(self.L.rafem_kp_launch(self.h, phase), "kp_launch")

    def iterate(self, n: int):
        nat.check(self.L.rafem_kp_iterate(self.h, n), "kp_iterate")

    def state(self):
        f, it, rel = C.c_int32(), C.c_int64(), C.c_double()
        nat.check(self.L.rafem_kp_state(self.h, C.byref(f), C.byref(it), C.byref(rel)), "kp_state")
        return int(f.value), int(it.value), float(rel.value)

    def finish(self, hist_cap: int):
        x = np.empty(2 * self.n_own)
        st = nat.SolveStatsC()
        hist = np.empty(hist_cap)
        cyc = np.empty(hist_cap, dtype=np.int64)
        rc = self.L.rafem_kp_finish(self.h, nat.ptr(x), C.byref(st), nat.ptr(hist), hist_cap, nat.ptr(cyc),
                                    hist_cap)
        return rc, x, st, hist, cyc


# ---------------------------------------------------------------------------
# orchestration

class ShardedPCG:
    """Host side of one shard's PCG: phases, collectives, state polling.

    The same sequence runs on every rank, so the collectives pair up; all
    decisions come from the device state, which every rank computes from
    the same all-gathered scalars.
    """

    def __init__(self, engine, comm: ShardComm | None, plan: ShardPlan | None, batch: int = 16):
        self.e, self.comm, self.plan, self.batch = engine, comm, plan, batch
        self.multi = comm is not None and comm.size > 1
        self.ipc = False  # device-initiated halo / slots (connect_ipc)

    def _slots(self):
        if self.multi and not self.ipc:
            self.comm.allgather_slots(self.e.slots)

    def _halo(self, which):
        if self.multi and not self.ipc:
            self.comm.halo(self.plan, self.e.send_buf, self.e.u_ext if which == "u" else self.e.x_ext,
                           self.e.n_send)

    def solve(self, b, x0, params, hist_cap: int):
        e = self.e
        t0 = time.perf_counter_ns()
        e.begin(b, x0, params)
        self.run_phases()
        rc, x, st, hist, cyc = e.finish(hist_cap)
        stats = SolveStats()
        stats.iterations = int(st.iterations)
        stats.restarts = int(st.restarts)
        stats.final_relative_residual = float(st.final_relative_residual)
        stats.converged = bool(st.converged)
        stats.device_ms = float(st.device_ms)
        lens = cyc[:min(int(st.cycles), hist_cap)]
        hv = hist[:min(int(st.history_len), hist_cap)]
        out, pos = [], 0
        for ln in lens:
            out.append([float(v) for v in hv[pos:pos + int(ln)]])
            pos += int(ln)
        stats.residual_history = out
        stats.wall_ns = max(time.perf_counter_ns() - t0, 1)
        if rc == nat.ERR_BREAKDOWN:
            raise KrylovBreakdownError("PCG breakdown: system not SPD under the preconditioner")
        nat.check(rc, "kp solve")
        return x, stats

    def run_phases(self):
        """Every phase of one begun solve, up to the done flag."""
        e = self.e
        self._slots()
        e.launch(BNORM_FINISH)
        flags, _, _ = e.state()
        while not flags & FLAG_DONE:
            # true-residual head: r = b - A x, u = M r, w = A u, first step
            e.launch(PACK_X)
            self._halo("x")
            e.launch(HEAD)
            e.launch(PACK_U_AFTER_HEAD)
            self._halo("u")
            e.launch(SPMV_AFTER_HEAD)
            self._slots()
            e.launch(UPDATE_FIRST)
            flags, _, _ = e.state()
            while not flags & (FLAG_DONE | FLAG_NEED_HEAD):
                if self.multi and not self.ipc:
                    for _ in range(self.batch):
                        e.launch(PACK_U)
                        self._halo("u")
                        e.launch(SPMV)
                        self._slots()
                        e.launch(UPDATE)
                else:
                    # single shard, or the device-initiated data plane: a batch of
                    # iterations with no host collective and no host round trip
                    e.iterate(self.batch)
                flags, _, _ = e.state()


def connect_ipc(engine: "KPDeviceEngine", plan: ShardPlan, comm: ShardComm, pcg: "ShardedPCG | None" = None):
    """Switch one shard's PCG to the device-initiated data plane
    (rafem_kp_ipc_connect): every rank exports its kp block, the handles,
    layouts and ghost offsets are all-gathered once (the only host
    collective), and from then on the phase kernels push the halo into the
    neighbours' ghost ranges and the scalar slots into every peer through
    the IPC mappings themselves.  Collective over the group."""
    L = nat.lib()
    hb = (C.c_char * 64)()
    offs = np.zeros(4, dtype=np.int64)
    nat.check(L.rafem_kp_ipc_export(engine.h, hb, nat.ptr(offs)), "kp_ipc_export")
    mine = {"rank": plan.rank, "n_own": plan.n_own, "recv": dict(plan.recv), "handle": bytes(hb),
            "offs": offs.tolist()}
    allv = [None] * comm.size
    comm.dist.all_gather_object(allv, mine, group=comm.group)
    allv.sort(key=lambda d: d["rank"])
    handles = b"".join(d["handle"] for d in allv)
    aoffs = np.ascontiguousarray(np.array([d["offs"] for d in allv], dtype=np.int64).reshape(-1))
    so = plan.send_offsets()
    segs = [(q, o, n) for q, (o, n) in so.items() if n > 0]
    peer = np.array([q for q, _, _ in segs], dtype=np.int32)
    start = np.array([o for _, o, _ in segs] + [sum(n for _, _, n in segs)], dtype=np.int64)
    dst = np.array([allv[q]["n_own"] + allv[q]["recv"][plan.rank][0] for q, _, _ in segs], dtype=np.int64)
    recv = np.array(sorted(plan.recv), dtype=np.int32)
    hbuf = (C.c_char * len(handles)).from_buffer_copy(handles)
    nat.check(L.rafem_kp_ipc_connect(engine.h, hbuf, nat.ptr(aoffs), len(segs), nat.ptr(peer), nat.ptr(start),
                                     nat.ptr(dst), recv.size, nat.ptr(recv)), "kp_ipc_connect")
    comm.dist.barrier(group=comm.group)  # every peer mapped before anyone pushes
    if pcg is not None:
        pcg.ipc = True


# ---------------------------------------------------------------------------
# one shard of the corrector-pass system

class ShardedSystem:
    """assemble_global + solve for one row block of the global system."""

    def __init__(self, mesh, material, comm: ShardComm | None = None, bounds=None, batch: int = 16,
                 ipc: bool = False):
        from .assembly import DeviceMesh, SystemHandle
        self.comm = comm
        nranks = comm.size if comm is not None else 1
        rank = comm.rank if comm is not None else 0
        if bounds is None:
            bounds = partition_rows(mesh.tets, mesh.node_count, nranks)
        self.plan = build_plan(mesh.tets, mesh.node_count, bounds, rank)
        self.mesh = mesh
        self.material = material
        self.lmesh = local_mesh(mesh, self.plan)
        self.dm = DeviceMesh(self.lmesh, material)
        # below-owner ghosts precede the owned block in global order: the
        # constraint sums follow global column order (owned rhs bitwise the
        # unsharded one)
        n_below = int(np.count_nonzero(self.plan.ghosts < self.plan.lo))
        nat.check(nat.lib().rafem_mesh_set_shard_order(self.dm.handle, self.plan.n_own, n_below), "shard order")
        self.h = SystemHandle(self.dm)
        self.engine = KPDeviceEngine(self.h.handle, self.plan.n_own, self.plan.n_ext, nranks, rank,
                                     self.plan.send_index())
        self.pcg = ShardedPCG(self.engine, comm, self.plan, batch=batch)
        self.scale = 1.0
        if ipc and comm is not None and comm.size > 1:
            connect_ipc(self.engine, self.plan, comm, self.pcg)

    @classmethod
    def from_device_mesh(cls, dm, batch: int = 16) -> "ShardedSystem":
        """One shard owning every row of a device mesh (DeviceMesh.from_box:
        no host mesh at all — the 64M-dof configs[4] on one GPU)."""
        from .assembly import SystemHandle
        self = cls.__new__(cls)
        self.comm = None
        n = dm.node_count
        self.plan = ShardPlan(rank=0, nranks=1, bounds=np.array([0, n], dtype=np.int64), n_own=n,
                              ghosts=np.zeros(0, dtype=np.int64), tet_ids=None, local_tets=None)
        self.mesh = self.lmesh = None
        self.material = None
        self.dm = dm
        self.h = SystemHandle(dm)
        self.engine = KPDeviceEngine(self.h.handle, n, n, 1, 0, None)
        self.pcg = ShardedPCG(self.engine, None, self.plan, batch=batch)
        self.scale = 1.0
        return self

    @property
    def n_own(self) -> int:
        return self.plan.n_own

    def assemble(self, t_ext, v_ext, tp_ext, dt, config, apply_constraints=True, equilibrate=True):
        """Assemble this shard's rows; fields are owned + ghost node values
        (ShardPlan.extend).  Raises PhysicsRangeError on every rank if any
        shard sees sigma <= 0 (lowest global element id)."""
        if dt <= 0.0:
            raise ValueError("dt must be positive")
        n = self.plan.n_ext
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (t_ext, v_ext, tp_ext)]
        for a in arrs:
            if a.shape != (n,):
                raise ValueError("shard field length must be owned + ghost node count")
        p = self.assemble_params(dt, config, apply_constraints, equilibrate)
        sums = np.zeros(2)
        bad = C.c_int64(-1)
        rc = nat.lib().rafem_assemble_partial(self.h.handle, nat.ptr(arrs[0]), nat.ptr(arrs[1]), nat.ptr(arrs[2]),
                                              C.byref(p), self.plan.n_own, nat.ptr(sums), C.byref(bad))
        if rc not in (nat.OK, nat.ERR_PHYSICS):
            nat.check(rc, "assemble_partial")
        return self._finish(sums, bad.value, p, equilibrate)

    @staticmethod
    def assemble_params(dt, config, apply_constraints=True, equilibrate=True):
        p = nat.AssembleParams()
        p.dt = float(dt)
        p.applied_voltage = float(config.applied_voltage)
        p.boundary_temp = float(config.boundary_temp)
        p.apply_constraints = 1 if apply_constraints else 0
        p.equilibrate = 1 if equilibrate else 0
        return p

    def _finish(self, sums, bad: int, p, equilibrate: bool) -> float:
        """The one global reduction of assemble_global (fem.py:390-400) over
        the shards' owned diagonal sums, in rank order; PhysicsRangeError on
        every rank for the lowest global bad element; then the scale and
        the Dirichlet elimination (rafem_assemble_finish)."""
        from .assembly import PhysicsRangeError
        tid = self.plan.tet_ids
        gbad = (float(tid[bad]) if tid is not None else float(bad)) if bad >= 0 else -1.0
        row = np.array([sums[0], sums[1], gbad])
        allr = self.comm.allgather_host(row) if self.comm is not None else row[None]
        bads = allr[:, 2][allr[:, 2] >= 0]
        if bads.size:
            raise PhysicsRangeError(f"sigma(T) <= 0 in element {int(bads.min())}")
        sv, stt = 0.0, 0.0
        for r in range(allr.shape[0]):  # rank order
            sv += allr[r, 0]
            stt += allr[r, 1]
        scale = 1.0
        if equilibrate and sv > 0.0 and stt > 0.0:
            scale = float(np.ldexp(1.0, int(np.rint(np.log2(stt / sv)))))
        nat.check(nat.lib().rafem_assemble_finish(self.h.handle, C.byref(p), scale), "assemble_finish")
        self.scale = scale
        return scale

    def owned_rows(self):
        """(row_ptr, global col, vals) of the owned dof rows, host copies (tests)."""
        rp = self.dm.dof_row_ptr
        ci = self.dm.dof_col_idx
        vals = self.h.download_vals()
        nrow = 2 * self.plan.n_own
        end = rp[nrow]
        l2g = self.plan.local_to_global
        gcol = 2 * l2g[ci[:end] // 2] + (ci[:end] % 2)
        return rp[:nrow + 1].copy(), gcol, vals[:end].copy()

    def rhs(self):
        return self.h.rhs()[:2 * self.plan.n_own].copy()

    def solve(self, b=None, x0=None, config=None):
        """PCG over the shard's rows; b/x0 are owned dof vectors (2 n_own) or
        None (assembled rhs / zero).  Returns (x_owned, SolveStats)."""
        from .krylov import SolverConfig, _params
        config = config or SolverConfig(backend="pcg", precondition="jacobi")
        n = 2 * self.plan.n_own
        b = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
        x0 = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
        for v in (b, x0):
            if v is not None and v.shape != (n,):
                raise ValueError("owned vector has the wrong length")
        p = _params(config, nat.METHOD_PCG)
        cap = int(config.max_total_iters) if config.max_total_iters is not None else 10 * n
        return self.pcg.solve(b, x0, p, min(cap, 1 << 20) + 1)


# ---------------------------------------------------------------------------
# the time loop over shards (configs 4-5: re-assembly every corrector pass)

@dataclass
class ShardStep:
    step: int
    time: float
    dt: float
    corrector_iters: int
    T: np.ndarray | None  # owned node values
    V: np.ndarray | None


@dataclass
class ShardSummary:
    accepted_steps: int
    total_corrector_iters: int
    total_solver_iterations: int
    dt_halvings: int
    final_time: float
    assemble_s: float
    solve_s: float
    wall_s: float
    passes: int = 0
    solve_device_ms: float = 0.0


class ShardedSimulation:
    """run_simulation (fem.py:554-644) + corrector_step (fem.py:463-540) with
    the fields distributed: every rank holds its owned node values, ghosts
    arrive by halo exchange before each assembly, the corrector delta is an
    all-reduce max, and every scalar decision (acceptance, dt growth /
    shrink / halving) is taken on identical global values on all ranks.

    ``system`` is a ShardedSystem (or any object with its ``plan``,
    ``assemble`` and ``solve``); ``comm`` None means one shard.
    """

    def __init__(self, system, comm: ShardComm | None = None):
        self.sys = system
        self.comm = comm
        self.plan = system.plan

    def _ext(self, *fields):
        own = np.stack(fields, axis=1)
        if self.comm is None:
            return [own[:, i].copy() for i in range(len(fields))]
        ext = self.comm.exchange_fields(self.plan, own)
        return [np.ascontiguousarray(ext[:, i]) for i in range(len(fields))]

    def _max(self, v):
        return self.comm.allreduce_max(v) if self.comm is not None else float(v)

    def run(self, config, record_fields=False, max_steps=None, sink=None):
        from .krylov import SolverError
        from .timeloop import StepFailureError
        n = self.plan.n_own
        T = np.full(n, config.initial_temp)
        V = np.zeros(n)
        T_prev, V_prev = T.copy(), V.copy()
        # like the fused kernel: a step's first solve starts from V extrapolated
        # in time too (the pass still assembles from / compares with x_old)
        vx0 = os.environ.get("RAFEM_NO_VX0", "0") != "1"
        t, dt_cur, dt_prev, step = 0.0, config.dt_init, config.dt_init, 0
        corr = inner = halv = 0
        asm_s = sol_s = 0.0
        w0 = time.perf_counter()
        recs = []
        while t < config.total_time:
            if max_steps is not None and step >= max_steps:
                break
            remaining = config.total_time - t
            last = dt_cur >= remaining
            dt = remaining if last else dt_cur
            t_it = T + (dt / dt_prev) * (T - T_prev) if step >= 1 else T.copy()  # fem.py:445-449
            v_it = V.copy()
            x_old = np.empty(2 * n)
            x_old[0::2], x_old[1::2] = v_it, t_it
            ok, used = False, 0
            for it in range(1, config.max_corrector_iters + 1):
                used = it
                a0 = time.perf_counter()
                te, ve, tpe = self._ext(t_it, v_it, T)
                self.sys.assemble(te, ve, tpe, dt, config)
                a1 = time.perf_counter()
                x0 = x_old
                if vx0 and it == 1 and step >= 1:
                    x0 = x_old.copy()
                    x0[0::2] = V + (dt / dt_prev) * (V - V_prev)
                try:
                    x_new, st = self.sys.solve(x0=x0, config=config.solver)
                except SolverError:
                    break  # step failure (fem.py:511-515)
                finally:
                    sol_s += time.perf_counter() - a1
                    asm_s += a1 - a0
                inner += st.iterations
                if not st.converged:
                    break
                d = float(np.max(np.abs(x_new - x_old) / np.maximum(1.0, np.abs(x_old)))) if n else 0.0
                delta = self._max(d)
                v_it, t_it = x_new[0::2].copy(), x_new[1::2].copy()
                x_old = x_new
                if delta < config.corrector_tol:
                    ok = True
                    break
            corr += used
            if ok:
                T_prev, T, V_prev, V = T, t_it, V, v_it
                dt_prev = dt
                t = config.total_time if last else t + dt
                rec = ShardStep(step, t, dt, used, T.copy() if record_fields else None,
                                V.copy() if record_fields else None)
                recs.append(rec)
                if sink is not None:
                    sink(rec)
                step += 1
                if used <= 5:
                    dt_cur = min(dt * 1.5, config.dt_max)
                elif used >= 20:
                    dt_cur = max(dt * 0.75, config.dt_min)
                else:
                    dt_cur = dt
            else:
                if dt <= config.dt_min:
                    raise StepFailureError(step, dt)
                dt_cur = max(dt * 0.5, config.dt_min)
                halv += 1
        return recs, ShardSummary(step, corr, inner, halv, t, asm_s, sol_s, time.perf_counter() - w0)


class DeviceShardedSimulation:
    """ShardedSimulation with the fields in HBM (csrc/shard.cu, rafem_sl_*).

    The same control contract (run_simulation, fem.py:554-644, and
    corrector_step, fem.py:463-540): the shard's accepted / previous /
    iterate states never leave the device; per corrector pass the host
    exchanges a 4-double halo per boundary node, the equilibration sums,
    the kp solver's collectives, and ONE scalar (the corrector delta,
    all-reduced max) on which every rank takes the same decision.  Records
    (owned fields of each accepted step) are read back only on request.
    """

    def __init__(self, system: ShardedSystem, comm: ShardComm | None = None):
        import torch
        self.sys = system
        self.comm = comm
        self.plan = system.plan
        self.L = nat.lib()
        h = C.c_void_p()
        nat.check(self.L.rafem_sl_create(system.engine.h, C.byref(h)), "sl_create")
        self.h = h
        ps, pg = C.c_void_p(), C.c_void_p()
        nat.check(self.L.rafem_sl_buffers(h, C.byref(ps), C.byref(pg)), "sl_buffers")
        dev = torch.device("cuda", torch.cuda.current_device())
        n_send = system.engine.n_send
        n_ghost = self.plan.n_ext - self.plan.n_own
        self.send4 = torch.as_tensor(_CudaArray(ps.value, 4 * max(n_send, 1)), device=dev)
        self.ghost4 = torch.as_tensor(_CudaArray(pg.value, 4 * max(n_ghost, 1)), device=dev)
        self.n_send = n_send

    def close(self):
        if self.h:
            self.L.rafem_sl_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _halo(self):
        """Ghost nodes' iterate and accepted (V, T) from their owners."""
        if self.comm is None or self.comm.size == 1 or not self.plan.neighbours:
            return
        nat.check(self.L.rafem_sl_pack(self.h), "sl_pack")
        self.comm.halo(self.plan, self.send4, self.ghost4, self.n_send, width=4, base=0)
        nat.check(self.L.rafem_sl_unpack(self.h), "sl_unpack")

    def _max(self, v):
        return self.comm.allreduce_max(v) if self.comm is not None else float(v)

    def download(self):
        """(T, V) owned node values of the accepted state (host)."""
        x = np.empty(2 * self.plan.n_own)
        nat.check(self.L.rafem_sl_download(self.h, nat.ptr(x)), "sl_download")
        return x[1::2].copy(), x[0::2].copy()

    def run(self, config, record_fields=False, max_steps=None, sink=None):
        from .krylov import _params
        from .timeloop import StepFailureError
        sysm, L, h = self.sys, self.L, self.h
        params = _params(config.solver, nat.METHOD_PCG)
        if config.solver.backend != "pcg":
            raise ValueError("the sharded time loop solves with the kernel-per-phase PCG (backend='pcg')")
        vx0 = os.environ.get("RAFEM_NO_VX0", "0") != "1"
        nat.check(L.rafem_sl_init(h, float(config.initial_temp)), "sl_init")
        t, dt_cur, dt_prev, step = 0.0, config.dt_init, config.dt_init, 0
        corr = inner = halv = passes = 0
        asm_s = sol_s = 0.0
        sol_dev_ms = 0.0
        w0 = time.perf_counter()
        recs = []
        sums = np.zeros(2)
        bad = C.c_int64(-1)
        st = nat.SolveStatsC()
        delta = C.c_double()
        while t < config.total_time:
            if max_steps is not None and step >= max_steps:
                break
            remaining = config.total_time - t
            last = dt_cur >= remaining
            dt = remaining if last else dt_cur
            start = vx0 and step >= 1
            nat.check(L.rafem_sl_predict(h, step, dt / dt_prev, 1 if start else 0), "sl_predict")
            p = sysm.assemble_params(dt, config)
            ok, used = False, 0
            for it in range(1, config.max_corrector_iters + 1):
                used = it
                passes += 1
                a0 = time.perf_counter()
                self._halo()
                rc = L.rafem_sl_assemble_partial(h, float(dt), nat.ptr(sums), C.byref(bad))
                if rc not in (nat.OK, nat.ERR_PHYSICS):
                    nat.check(rc, "sl_assemble_partial")
                sysm._finish(sums, bad.value, p, True)
                a1 = time.perf_counter()
                nat.check(L.rafem_sl_solve_begin(h, C.byref(params), 1 if (start and it == 1) else 0),
                          "sl_solve_begin")
                sysm.pcg.run_phases()
                rc = L.rafem_sl_solve_end(h, C.byref(st), C.byref(delta))
                sol_s += time.perf_counter() - a1
                asm_s += a1 - a0
                sol_dev_ms += float(st.device_ms)
                if rc == nat.ERR_BREAKDOWN:
                    break  # SolverError -> step failure (fem.py:511-515)
                nat.check(rc, "sl_solve_end")
                inner += int(st.iterations)
                if not st.converged:
                    break
                d = self._max(delta.value)
                if d < config.corrector_tol:
                    ok = True
                    break
            corr += used
            if ok:
                nat.check(L.rafem_sl_accept(h), "sl_accept")
                dt_prev = dt
                t = config.total_time if last else t + dt
                T = V = None
                if record_fields:
                    T, V = self.download()
                rec = ShardStep(step, t, dt, used, T, V)
                recs.append(rec)
                if sink is not None:
                    sink(rec)
                step += 1
                if used <= 5:
                    dt_cur = min(dt * 1.5, config.dt_max)
                elif used >= 20:
                    dt_cur = max(dt * 0.75, config.dt_min)
                else:
                    dt_cur = dt
            else:
                if dt <= config.dt_min:
                    raise StepFailureError(step, dt)
                dt_cur = max(dt * 0.5, config.dt_min)
                halv += 1
        return recs, ShardSummary(step, corr, inner, halv, t, asm_s, sol_s, time.perf_counter() - w0, passes,
                                  sol_dev_ms)
