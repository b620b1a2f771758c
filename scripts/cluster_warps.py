"""Per-warp phase timeline of the cluster PCG (CTA 0): for each phase the
median over iterations of the earliest / latest warp, relative to the
earliest loop-top stamp of the iteration (clocks)."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import _native as nat
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
L, ctx = nat.lib(), nat.context()
dims = tuple(int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (20, 20, 21)
mesh = generate_box_mesh(*dims); n = mesh.node_count
rng = np.random.default_rng(2409)
t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
cfg = SolverConfig(backend="pcg", precondition="jacobi", tolerance=1e-300, max_total_iters=120)
for rep in range(2):
    L.rafem_set_trace(ctx, 1)
    x, st = solve(s.matrix, s.rhs, x0=np.zeros(2 * n), config=cfg)
    L.rafem_set_trace(ctx, 0)
tr = np.zeros(8 * 4096, dtype=np.int64)
L.rafem_get_trace(ctx, tr.ctypes.data, tr.size)
tr = tr.reshape(-1, 32, 8)[10:100].astype(np.float64)  # iterations x warps x stamps
nw = int((tr[0, :, 0] > 0).sum())
tr = tr[:, :nw, :]
t0 = tr[:, :, 0].min(axis=1, keepdims=True)
rel = tr - t0[:, :, None]
names = ["loop top", "own spmv done", "wait done", "ghost spmv+gather+scalars done", "update+push done", "publish returned", "publish BAR passed", "partials sent"]
order = [0, 1, 2, 3, 4, 6, 7, 5]
print(f"{dims}: {nw} warps, iteration {np.median(np.diff(tr[:, 0, 0])):.0f} clk")
for k in order:
    lo = np.median(rel[:, :, k].min(axis=1)); hi = np.median(rel[:, :, k].max(axis=1))
    print(f"  {names[k]:32s} first warp {lo:7.0f}  last warp {hi:7.0f}")
