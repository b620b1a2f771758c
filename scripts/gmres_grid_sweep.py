"""One-reduce GMRES(30) on the mesh-B analog system: us per inner step over
the persistent grid's CTA count and the partial-sum gather (wide vs warp per
coefficient, RAFEM_GMRES_GATHER)."""
import os, subprocess, sys
code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
mesh = generate_box_mesh(20, 20, 21); n = mesh.node_count
rng = np.random.default_rng(2409)
t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
x0 = np.empty(2 * n); x0[0::2], x0[1::2] = v, t
G = int(sys.argv[1])
best = 1e9
for _ in range(4):
    x, st = solve(s.matrix, s.rhs, x0=x0, config=SolverConfig(backend="gmres", precondition="jacobi", tolerance=1e-10, grid_ctas=G))
    best = min(best, st.device_ms * 1e3)
print(f"G={G} it={st.iterations} {best/st.iterations:.2f} us/step")
'''
sys.path.insert(0, ".")
for gather in ("wide", "warp"):
    for G in (148, 128, 111, 96, 74, 56):
        env = dict(os.environ, RAFEM_GMRES_GATHER=gather)
        out = subprocess.run([sys.executable, "-c", code, str(G)], env=env, capture_output=True, text=True)
        print(gather, out.stdout.strip() or out.stderr.strip()[-300:], flush=True)
