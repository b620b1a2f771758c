"""C4 (16M dofs) single-shard kernel-per-phase PCG, capped iterations (ncu captures)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
from paper_2409_13036_b200.shard import ShardedSystem
dims = tuple(int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (200, 200, 200)
iters = int(sys.argv[4]) if len(sys.argv) >= 5 else 20
mesh = generate_box_mesh(*dims)
n = mesh.node_count
sh = ShardedSystem(mesh, MaterialParams.default(), batch=8)
t = np.full(n, 37.0)
sh.assemble(t, np.zeros(n), t, 0.5, SimConfig())
x0 = np.empty(2 * n); x0[0::2], x0[1::2] = 0.0, 37.0
x, st = sh.solve(x0=x0, config=SolverConfig(backend="pcg", precondition="jacobi", max_total_iters=iters))
print(st.iterations, st.device_ms)
