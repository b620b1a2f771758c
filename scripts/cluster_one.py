"""One paper-scale PCG solve through the cluster engine (for ncu captures)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
dims = tuple(int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (20, 20, 21)
mesh = generate_box_mesh(*dims)
n = mesh.node_count
rng = np.random.default_rng(2409)
t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
for _ in range(2):
    x, st = solve(s.matrix, s.rhs, x0=np.zeros(2 * n), config=SolverConfig(backend="pcg", precondition="block_jacobi"))
print(st.iterations, st.device_ms)
