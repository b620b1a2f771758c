import sys, numpy as np
sys.path.insert(0, ".")
from paper_2409_13036_b200 import CsrMatrix, SolverConfig, gmres
sys.path.insert(0, "tests")
from test_gpu_sparse_solver import random_system
rng = np.random.default_rng(1)
for n, m in [(10, 3), (10, 30), (40, 5), (420, 30)]:
    a, dense, b = random_system(rng, n)
    x, st = gmres(a, b, None, SolverConfig(backend="gmres", tolerance=1e-10, restart_m=m))
    print(n, m, st.iterations, st.converged, np.abs(dense @ x - b).max(), flush=True)
