"""Cost breakdown of the cluster PCG iteration by ablation (RAFEM_CL_ABL):
fixed 400 iterations, convergence tests off; each line removes one part."""
import os, subprocess, sys
sys.path.insert(0, ".")
code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
dims = tuple(int(a) for a in sys.argv[1:4])
mesh = generate_box_mesh(*dims); n = mesh.node_count
rng = np.random.default_rng(2409)
t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
best = 1e9
for _ in range(5):
    x, st = solve(s.matrix, s.rhs, x0=np.zeros(2 * n), config=SolverConfig(backend="pcg", precondition="jacobi", tolerance=1e-300, max_total_iters=400))
    best = min(best, st.device_ms * 1e3 / max(st.iterations, 1))
print(f"{best:.3f}")
'''
for dims in (["20", "20", "21"], ["15", "15", "16"]):
    for extra in ({}, {"RAFEM_CL_RCB": "0"}, {"RAFEM_CL_RCB": "0", "RAFEM_CL_SPLIT": "0", "RAFEM_CL_SORT": "0"}):
        res = []
        for abl, name in [(8, "full"), (9, "-own spmv"), (10, "-ghost spmv"), (11, "-spmv"), (12, "-halo"), (15, "-spmv-halo")]:
            env = dict(os.environ, RAFEM_CL_ABL=str(abl), **extra)
            out = subprocess.run([sys.executable, "-c", code] + dims, env=env, capture_output=True, text=True)
            res.append(f"{name} {out.stdout.strip() or out.stderr.strip()[-80:]}")
        print(dims, extra, " | ".join(res), flush=True)
