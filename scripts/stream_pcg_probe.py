"""One PCG solve capped at a few iterations, for ncu captures of the streaming kernel."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
dims = tuple(int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (80, 80, 79)
iters = int(sys.argv[4]) if len(sys.argv) >= 5 else 40
mesh = generate_box_mesh(*dims)
n = mesh.node_count
t = np.full(n, 37.0)
s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, np.zeros(n), t, 0.5)
x0 = np.empty(2 * n); x0[0::2], x0[1::2] = 0.0, 37.0
x, st = solve(s.matrix, s.rhs, x0=x0, config=SolverConfig(backend="pcg", precondition="jacobi", max_total_iters=iters))
print(st.iterations, st.device_ms, 1e3 * st.device_ms / st.iterations, "us/it")
