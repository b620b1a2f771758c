"""Per-phase clock64 stamps of the cluster-resident PCG (rank 0, thread 0):
wait, gather+scalars, SpMV, update, push, publish+arrive.
python scripts/cluster_phase.py [nx ny nz]"""
import os, sys
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import _native as nat
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
L, ctx = nat.lib(), nat.context()
dims = tuple(int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (20, 20, 21)
mesh = generate_box_mesh(*dims)
n = mesh.node_count
rng = np.random.default_rng(2409)
t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
x0 = np.zeros(2 * n)
cfg = SolverConfig(backend="pcg", precondition="jacobi")
names = ["own-spmv", "wait", "ghost-spmv+gather+scalars", "update+push", "publish+arrive", "->loop top"]
for rep in range(3):
    L.rafem_set_trace(ctx, 1)
    x, st = solve(s.matrix, s.rhs, x0=x0, config=cfg)
    L.rafem_set_trace(ctx, 0)
    tr = np.zeros(8 * 4096, dtype=np.int64)
    L.rafem_get_trace(ctx, tr.ctypes.data, tr.size)
    tr = tr.reshape(-1, 8)[3:min(st.iterations, 4095) - 2].astype(np.float64)
    tr = tr[tr[:, 0] > 0]
    d01 = np.median(tr[:, 1] - tr[:, 0]); d12 = np.median(tr[:, 2] - tr[:, 1])
    d23 = np.median(tr[1:, 3] - tr[:-1, 2]); d34 = np.median(tr[:, 4] - tr[:, 3]); d45 = np.median(tr[:, 5] - tr[:, 4])
    d50 = np.median(tr[:, 0] - tr[:, 5])
    d = np.array([d01, d12, d23, d34, d45, d50]) / 1.965e3
    per = np.median(np.diff(tr[:, 0])) / 1.965e3
    print(f"{dims} it={st.iterations} {st.device_ms*1e3/max(st.iterations,1):.2f} us/it | " +
          " ".join(f"{nm} {x:.3f}" for nm, x in zip(names, d)) + f" | iter {per:.3f} us", flush=True)
