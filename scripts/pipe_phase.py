"""Per-phase clock stamps of the pipelined PCG (CTA 0, thread 0) on the
mesh-B analog's hot system: SpMV + dot fold, vector update, block-Jacobi
step, publish, grid barrier.   python scripts/pipe_phase.py [jacobi|block_jacobi]"""
import os, sys
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import _native as nat
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
L, ctx = nat.lib(), nat.context()
prec = sys.argv[1] if len(sys.argv) > 1 else "block_jacobi"
mesh = generate_box_mesh(20, 20, 21)
n = mesh.node_count
rng = np.random.default_rng(2409)
t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
x0 = np.zeros(2 * n)
cfg = SolverConfig(backend="pcg", precondition=prec)
for rep in range(3):
    L.rafem_set_trace(ctx, 1)
    x, st = solve(s.matrix, s.rhs, x0=x0, config=cfg)
    L.rafem_set_trace(ctx, 0)
    tr = np.zeros(8 * 4096, dtype=np.int64)
    L.rafem_get_trace(ctx, tr.ctypes.data, tr.size)
    tr = tr.reshape(-1, 8)[5:min(st.iterations, 4095) - 1].astype(np.float64)
    ok = tr[:, 0] > 0
    tr = tr[ok]
    d = np.diff(tr[:, :6], axis=1).mean(axis=0) / 1.965e3
    per = np.diff(tr[:, 0]).mean() / 1.965e3
    # slots 2-7 are stamped after the iteration counter moved on: align them
    t1 = tr[:-1, 1]
    nx = tr[1:]
    sc = (nx[:, 6] - t1).mean() / 1.965e3, (nx[:, 7] - nx[:, 6]).mean() / 1.965e3, (nx[:, 2] - nx[:, 7]).mean() / 1.965e3
    print(f"   update split: scalars {sc[0]:.2f} loop {sc[1]:.2f} divisions+partials+bar {sc[2]:.2f} us")
    print(f"{prec}: it={st.iterations} dev={st.device_ms*1e3:.0f}us ({st.device_ms*1e3/max(st.iterations,1):.2f} us/it) | "
          f"spmv+fold {d[0]:.2f} update {d[1]:.2f} block {d[2]:.2f} publish {d[3]:.2f} barrier {d[4]:.2f} | iter {per:.2f} us")
