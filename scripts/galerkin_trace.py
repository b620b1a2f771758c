import sys
sys.path.insert(0, ".")
import numpy as np, os
from paper_2409_13036_b200 import _native as nat
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
from paper_2409_13036_b200.timeloop import DeviceRun
L, ctx = nat.lib(), nat.context()
run = DeviceRun(generate_box_mesh(20, 20, 21), MaterialParams.default())
cfg = SimConfig(total_time=900.0, solver=SolverConfig(backend="pcg", precondition="block_jacobi"))
run.run(cfg, record_fields=False)
L.rafem_set_trace(ctx, 1)
recs, out = run.run(cfg, record_fields=False)
L.rafem_set_trace(ctx, 0)
tr = np.zeros(8 * 4096, dtype=np.int64)
L.rafem_get_trace(ctx, tr.ctypes.data, tr.size)
tr = tr.reshape(-1, 8)[: int(out.passes)].astype(float)
ok = tr[:, 6] > 0
print("passes", out.passes, "with galerkin", ok.sum())
print("galerkin us: mean", np.mean((tr[ok, 6] - tr[ok, 4]) / 1e3), "median", np.median((tr[ok, 6] - tr[ok, 4]) / 1e3))
print("pcg after galerkin us mean", np.mean((tr[ok, 5] - tr[ok, 6]) / 1e3), "its", tr[ok, 7].mean())
print("pass total us mean", np.mean(np.diff(tr[:, 0])) / 1e3)
d = tr_all = np.zeros(8 * 4096, dtype=np.int64)
L.rafem_get_trace(ctx, d.ctypes.data, d.size)
g = d[8 * 4000: 8 * 4000 + 8].astype(float)
print("last galerkin phases (us): spmv", (g[1] - g[0]) / 1e3, "stage D", (g[2] - g[1]) / 1e3, "dots", (g[3] - g[2]) / 1e3,
      "barrier", (g[4] - g[3]) / 1e3, "c0 loop entry", (g[6] - g[2]) / 1e3, "c0 dot done", (g[7] - g[2]) / 1e3, "gather", (g[5] - g[4]) / 1e3, "x", 0)
