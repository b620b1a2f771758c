"""One-reduce Arnoldi GMRES(30) (krylov.cu gmres_1r_body, the default) vs
the three-synchronisation CGS2 step (RAFEM_GMRES_CGS2=1) on paper-scale
systems: iterations, us per inner step, true residual, agreement of the
solutions."""
import os, subprocess, sys
sys.path.insert(0, ".")
code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from oracle import rafem_oracle as O
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
from paper_2409_13036_b200 import _native as nat
dims = tuple(int(a) for a in sys.argv[1:4]); hot = sys.argv[4] == "hot"
mesh = generate_box_mesh(*dims); n = mesh.node_count
rng = np.random.default_rng(2409)
t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
x0 = np.empty(2 * n); x0[0::2], x0[1::2] = v, t
if not hot: x0[:] = 0.0
best = 1e9
for _ in range(3):
    x, st = solve(s.matrix, s.rhs, x0=x0, config=SolverConfig(backend="gmres", precondition="jacobi", tolerance=1e-10))
    best = min(best, st.device_ms * 1e3)
res = np.linalg.norm(s.rhs - O.matvec(s.matrix.row_ptr, s.matrix.col_idx, s.matrix.vals, x)) / np.linalg.norm(s.rhs)
np.save(sys.argv[5], x)
print(f"mode={nat.last_solve_mode()[0]} it={st.iterations} restarts={st.restarts} {best/max(st.iterations,1):.2f} us/step solve {best:.0f} us res={res:.2e} rep={st.final_relative_residual:.2e} conv={st.converged}")
'''
import numpy as np
for dims in (["20", "20", "21"], ["15", "15", "16"], ["6", "5", "7"]):
    for hot in ("hot", "cold"):
        xs = {}
        for name, extra in (("cgs2", {"RAFEM_GMRES_CGS2": "1"}), ("one_reduce", {})):
            env = dict(os.environ, **extra)
            f = f"/tmp/g_{name}.npy"
            out = subprocess.run([sys.executable, "-c", code] + dims + [hot, f], env=env, capture_output=True, text=True)
            print(dims, hot, name, out.stdout.strip() or out.stderr.strip()[-400:], flush=True)
            xs[name] = np.load(f) if os.path.exists(f) else None
        if xs["cgs2"] is not None and xs["one_reduce"] is not None:
            a, b = xs["cgs2"], xs["one_reduce"]
            print("   rel diff", float(np.max(np.abs(a - b)) / np.max(np.abs(a))), flush=True)
