"""CPU tests of the row-block sharding host logic.

* the partition and shard plans: coverage, ghost/halo symmetry, and owned
  rows of the sub-mesh assembly equal to the global assembly's rows,
  bit for bit (oracle assembly on both);
* the full sharded PCG orchestration (ShardedPCG + ShardComm over gloo,
  world size 2 and 3) with the numpy engine of tests/kp_emul.py, against
  the single-process oracle PCG.
"""

import os

import numpy as np
import pytest

from oracle import rafem_oracle as O
from paper_2409_13036_b200.shard import ShardPlan, build_plan, partition_rows


def _hot_fields(n, seed=2409):
    rng = np.random.default_rng(seed)
    return 37.0 + rng.uniform(0, 30, n), rng.uniform(0, 25, n)


def _sub_omesh(om, plan: ShardPlan):
    l2g = plan.local_to_global
    pos = np.full(om.node_count, -1, dtype=np.int64)
    pos[l2g] = np.arange(l2g.size)
    sets = {}
    for k, v in om.node_sets.items():
        loc = pos[np.asarray(v)]
        sets[k] = np.sort(loc[loc >= 0])
    return O.OMesh(nodes=om.nodes[l2g], tets=plan.local_tets, regions=om.regions[plan.tet_ids], node_sets=sets)


@pytest.mark.parametrize("dims,nranks", [((6, 5, 7), 2), ((6, 5, 7), 3), ((5, 4, 6), 4), ((9, 3, 3), 2)])
def test_plans_cover_and_halos_are_symmetric(dims, nranks):
    om = O.box_mesh(*dims)
    n = om.node_count
    bounds = partition_rows(om.tets, n, nranks)
    assert bounds[0] == 0 and bounds[-1] == n and np.all(np.diff(bounds) > 0)
    plans = [build_plan(om.tets, n, bounds, r) for r in range(nranks)]
    # every tet lands in the sub-mesh of each shard owning one of its vertices
    for p in plans:
        owner = np.searchsorted(bounds, om.tets, side="right") - 1
        assert np.array_equal(p.tet_ids, np.flatnonzero((owner == p.rank).any(axis=1)))
    for p in plans:
        for q, (start, cnt) in p.recv.items():
            got = p.ghosts[start:start + cnt]
            sent = plans[q].send[p.rank] + plans[q].lo
            assert np.array_equal(got, sent), (p.rank, q)
            assert np.all((got >= plans[q].lo) & (got < plans[q].hi))
        assert set(p.send) == set(p.recv)  # the stencil is symmetric


@pytest.mark.parametrize("nranks", [2, 3])
def test_owned_rows_of_sub_mesh_assembly_are_bitwise_global_rows(nranks):
    """Sub-mesh assembly reproduces the owned rows of the global system bit
    for bit (values, rhs, Dirichlet elimination); the equilibration scale
    from the per-shard diagonal sums equals the global one."""
    om = O.box_mesh(6, 5, 7)
    n = om.node_count
    t, v = _hot_fields(n)
    tp = t - 0.25
    mats = {0: O.OMaterial()}
    glob = O.assemble(om, mats, 25.0, 37.0, t, v, tp, 0.5, equilibrate=False)
    scale_ref = O.assemble(om, mats, 25.0, 37.0, t, v, tp, 0.5).scale
    bounds = partition_rows(om.tets, n, nranks)
    sv = st = 0.0
    for r in range(nranks):
        p = build_plan(om.tets, n, bounds, r)
        sm = _sub_omesh(om, p)
        fields = (p.extend(t), p.extend(v), p.extend(tp))
        loc = O.assemble(sm, mats, 25.0, 37.0, *fields, 0.5, equilibrate=False)
        raw = O.assemble(sm, mats, 25.0, 37.0, *fields, 0.5, equilibrate=False, apply_constraints=False)
        d = O.diag_of(raw.row_ptr, raw.col_idx, raw.vals)[:2 * p.n_own]
        sv += d[0::2].sum()
        st += d[1::2].sum()
        l2g = p.local_to_global
        r0, r1 = 2 * p.lo, 2 * p.hi
        g_ptr = glob.row_ptr[r0:r1 + 1] - glob.row_ptr[r0]
        g_col = glob.col_idx[glob.row_ptr[r0]:glob.row_ptr[r1]]
        g_val = glob.vals[glob.row_ptr[r0]:glob.row_ptr[r1]]
        l_end = loc.row_ptr[2 * p.n_own]
        l_col = 2 * l2g[loc.col_idx[:l_end] // 2] + loc.col_idx[:l_end] % 2
        l_val = loc.vals[:l_end]
        assert np.array_equal(loc.row_ptr[:2 * p.n_own + 1], g_ptr)
        assert np.array_equal(loc.rhs[:2 * p.n_own], glob.rhs[r0:r1])
        for i in range(2 * p.n_own):  # same entries; local ids sort ghosts last inside a row
            a, b = g_ptr[i], g_ptr[i + 1]
            gk = np.argsort(g_col[a:b], kind="stable")
            lk = np.argsort(l_col[a:b], kind="stable")
            assert np.array_equal(g_col[a:b][gk], l_col[a:b][lk])
            assert np.array_equal(g_val[a:b][gk], l_val[a:b][lk]), (r, i)
    assert 2.0 ** round(np.log2(st / sv)) == scale_ref


def _worker(rank, world, port, dims, tol, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from kp_emul import NumpyKPEngine, local_csr
        from paper_2409_13036_b200 import _native as nat
        from paper_2409_13036_b200.shard import ShardComm, ShardedPCG
        om = O.box_mesh(*dims)
        n = om.node_count
        t, v = _hot_fields(n)
        glob = O.assemble(om, {0: O.OMaterial()}, 25.0, 37.0, t, v, t, 0.5)
        bounds = partition_rows(om.tets, n, world)
        plan = build_plan(om.tets, n, bounds, rank)
        rp, ci, va = local_csr(glob.row_ptr, glob.col_idx, glob.vals, plan)
        eng = NumpyKPEngine(rp, ci, va, plan.n_own, plan.n_ext, world, rank, plan.send_index())
        comm = ShardComm(device_collectives=False)
        pcg = ShardedPCG(eng, comm, plan, batch=4)
        x0 = np.empty(2 * n)
        x0[0::2], x0[1::2] = v, t
        p = nat.SolverParams()
        p.method, p.restart_m, p.tolerance, p.max_total_iters, p.precondition = 1, 30, tol, 0, 1
        b_own = glob.rhs[2 * plan.lo:2 * plan.hi]
        x, st = pcg.solve(b_own, x0[2 * plan.lo:2 * plan.hi], p, 4096)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), x=x, lo=plan.lo, it=st.iterations,
                 rel=st.final_relative_residual, conv=st.converged, hist=sum(st.residual_history, []))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_pcg_orchestration_gloo(tmp_path, world):
    import torch.multiprocessing as mp
    dims, tol = (8, 6, 7), 1e-10
    port = 29500 + (os.getpid() % 500) + 7 * world
    mp.start_processes(_worker, args=(world, port, dims, tol, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    om = O.box_mesh(*dims)
    n = om.node_count
    t, v = _hot_fields(n)
    glob = O.assemble(om, {0: O.OMaterial()}, 25.0, 37.0, t, v, t, 0.5)
    x = np.empty(2 * n)
    its = set()
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        lo = int(d["lo"])
        x[2 * lo:2 * lo + d["x"].size] = d["x"]
        assert bool(d["conv"])
        its.add(int(d["it"]))
    assert len(its) == 1  # every rank took the same decisions
    res = np.linalg.norm(glob.rhs - O.matvec(glob.row_ptr, glob.col_idx, glob.vals, x)) / np.linalg.norm(glob.rhs)
    assert res <= tol
    x0 = np.empty(2 * n)
    x0[0::2], x0[1::2] = v, t
    xo, so = O.pcg(glob.row_ptr, glob.col_idx, glob.vals, glob.rhs, x0=x0, tol=tol)
    assert abs(its.pop() - so.iterations) <= max(3, 0.05 * so.iterations)
    assert np.max(np.abs(x - xo)) <= 1e-7 * np.max(np.abs(xo))


def _sim_worker(rank, world, port, dims, total, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from kp_emul import EmulShardSystem
        from paper_2409_13036_b200 import SimConfig, SolverConfig
        from paper_2409_13036_b200.shard import ShardComm, ShardedSimulation
        om = O.box_mesh(*dims)
        n = om.node_count
        comm = ShardComm(device_collectives=False)
        plan = build_plan(om.tets, n, partition_rows(om.tets, n, world), rank)
        sysm = EmulShardSystem(om, {0: O.OMaterial()}, plan, comm, O)
        cfg = SimConfig(total_time=total, solver=SolverConfig(backend="pcg", precondition="jacobi", tolerance=1e-12))
        recs, summ = ShardedSimulation(sysm, comm).run(cfg, record_fields=True)
        np.savez(os.path.join(out_dir, f"m{rank}.npz"), lo=plan.lo,
                 traj=np.array([(r.step, r.time, r.dt, r.corrector_iters) for r in recs]),
                 T=np.array([r.T for r in recs]), V=np.array([r.V for r in recs]))
    finally:
        dist.destroy_process_group()


def test_sharded_time_loop_gloo_matches_oracle_run(tmp_path):
    """ShardedSimulation over 2 gloo ranks: same trajectory as the oracle's
    single-process run (fem.py:554-644) and fields within 1e-8 of peak."""
    import torch.multiprocessing as mp
    dims, total, world = (7, 6, 8), 12.0, 2
    port = 28600 + (os.getpid() % 500)
    mp.start_processes(_sim_worker, args=(world, port, dims, total, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    om = O.box_mesh(*dims)
    ref = O.run(om, {0: O.OMaterial()}, O.OSim(total_time=total, method="pcg", tolerance=1e-12))
    parts = [np.load(tmp_path / f"m{r}.npz") for r in range(world)]
    traj = [tuple(x) for x in parts[0]["traj"]]
    assert all([tuple(x) for x in p["traj"]] == traj for p in parts)
    assert traj == [(r.step, r.time, r.dt, r.corrector_iters) for r in ref.records]
    T = np.concatenate([p["T"] for p in parts], axis=1)
    V = np.concatenate([p["V"] for p in parts], axis=1)
    for k, r in enumerate(ref.records):
        assert np.max(np.abs(T[k] - r.T)) <= 1e-8 * np.max(np.abs(r.T))
        assert np.max(np.abs(V[k] - r.V)) <= 1e-8 * max(np.max(np.abs(r.V)), 1.0)
