"""Per-phase timing of the persistent GMRES inner step (paper scale)."""
import ctypes as C, sys
sys.path.insert(0, ".")
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
cfg = SolverConfig(backend="gmres", precondition="jacobi")
solve(s.matrix, s.rhs, x0=x0, config=cfg)
L.rafem_set_trace(ctx, 1)
x, st = solve(s.matrix, s.rhs, x0=x0, config=cfg)
L.rafem_set_trace(ctx, 0)
tr = np.zeros(8 * 4096, dtype=np.int64)
L.rafem_get_trace(ctx, tr.ctypes.data, tr.size)
tr = tr.reshape(-1, 8)[5:min(st.iterations, 4000) - 1]
ok = (tr[:, :7] > 0).all(axis=1)
tr = tr[ok]
d = np.diff(tr[:, :7], axis=1) / 1.965e3
names = ["basis row + spmv", "multidot1", "sync_gather1", "update1+multidot2", "sync_gather2", "update2+barrier"]
print(f"gmres: {st.iterations} its, {st.device_ms*1e3/st.iterations:.2f} us/it")
for i, nme in enumerate(names):
    print(f"  {nme:22s} {d[:, i].mean():6.2f} us")
print(f"  step (0->0)            {np.diff(tr[:, 0]).mean() / 1.965e3:6.2f} us")
