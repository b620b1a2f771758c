"""Cluster-resident PCG vs grid PCG per preconditioner and partition:
iterations, us per iteration, solve time (best of 5), true residual."""
import os, subprocess, sys
sys.path.insert(0, ".")
code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from oracle import rafem_oracle as O
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
from paper_2409_13036_b200 import _native as nat
dims = tuple(int(a) for a in sys.argv[1:4]); prec = sys.argv[4]
mesh = generate_box_mesh(*dims); n = mesh.node_count
rng = np.random.default_rng(2409)
t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
x0 = np.empty(2 * n); x0[0::2], x0[1::2] = v, t
best = 1e9
for _ in range(5):
    x, st = solve(s.matrix, s.rhs, x0=x0, config=SolverConfig(backend="pcg", precondition=prec, tolerance=1e-10))
    best = min(best, st.device_ms * 1e3)
res = np.linalg.norm(s.rhs - O.matvec(s.matrix.row_ptr, s.matrix.col_idx, s.matrix.vals, x)) / np.linalg.norm(s.rhs)
print(f"mode={nat.last_solve_mode()[0]} it={st.iterations} {best/max(st.iterations,1):.2f} us/it solve {best:.0f} us res={res:.1e}")
'''
for dims in (["20", "20", "21"], ["15", "15", "16"]):
    for prec in ("jacobi", "block_jacobi"):
        for name, extra in (("grid", {"RAFEM_CLUSTER": "0"}), ("cluster-slab", {"RAFEM_CL_RCB": "0"}),
                            ("cluster-rcb", {"RAFEM_CL_RCB": "1"}), ("cluster-rcb-nosplit", {"RAFEM_CL_RCB": "1", "RAFEM_CL_SPLIT": "0", "RAFEM_CL_SORT": "0"})):
            env = dict(os.environ, **extra)
            out = subprocess.run([sys.executable, "-c", code] + dims + [prec], env=env, capture_output=True, text=True)
            print(dims, prec, name, out.stdout.strip() or out.stderr.strip()[-300:], flush=True)
