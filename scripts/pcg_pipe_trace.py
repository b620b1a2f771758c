"""Per-phase timing of the grid pipelined PCG iteration (pcg_pipe_core, the
fused simulation's solver) on the mesh-B system, block-Jacobi and Jacobi,
CTA 0's clock; RAFEM_CLUSTER=0 keeps the standalone solve on the grid engine."""
import os, sys
sys.path.insert(0, ".")
os.environ["RAFEM_CLUSTER"] = "0"
import numpy as np
from paper_2409_13036_b200 import _native as nat
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
L, ctx = nat.lib(), nat.context()
mesh = generate_box_mesh(20, 20, 21)
n = mesh.node_count
rng = np.random.default_rng(2409)
t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
x0 = np.empty(2 * n); x0[0::2], x0[1::2] = v, t
names = [(0, 1, "SpMV || partial fold"), (1, 6, "scalars"), (6, 7, "owner update"), (7, 2, "dot partials"),
         (2, 3, "publish || block step"), (3, 4, "-"), (4, 5, "grid barrier")]
for prec in ("block_jacobi", "jacobi"):
    cfg = SolverConfig(backend="pcg", precondition=prec)
    solve(s.matrix, s.rhs, x0=x0, config=cfg)
    L.rafem_set_trace(ctx, 1)
    x, st = solve(s.matrix, s.rhs, x0=x0, config=cfg)
    L.rafem_set_trace(ctx, 0)
    tr = np.zeros(8 * 4096, dtype=np.int64)
    L.rafem_get_trace(ctx, tr.ctypes.data, tr.size)
    rows = tr.reshape(-1, 8)[3:min(st.iterations, 4000) - 2].astype(float) / 1.965e3
    rows = rows[(rows > 0).all(axis=1)]
    print(f"{prec}: {st.iterations} its, {st.device_ms * 1e3 / st.iterations:.2f} us/it (device), mode {nat.last_solve_mode()}")
    for a, b, nm in names:
        print(f"  {nm:24s} {np.mean(rows[:, b] - rows[:, a]):6.2f} us")
    print(f"  {'iteration (0 -> 0)':24s} {np.mean(np.diff(rows[:, 0])):6.2f} us")
