"""PCG us/iteration on the paper-scale systems vs persistent grid size."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
for dims in [(20, 20, 21), (15, 15, 16)]:
    mesh = generate_box_mesh(*dims)
    n = mesh.node_count
    rng = np.random.default_rng(2409)
    t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
    s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
    x0 = np.empty(2 * n); x0[0::2], x0[1::2] = v, t
    for G in [148, 128, 96, 74, 64, 48, 37, 32]:
        for team in ["", "4", "8", "16"]:
            if team:
                os.environ["RAFEM_TEAM"] = team
            cfg = SolverConfig(backend="pcg", precondition="jacobi")
            cfg.grid_ctas = G
            best = 1e9
            for _ in range(3):
                x, st = solve(s.matrix, s.rhs, x0=x0, config=cfg)
                best = min(best, st.device_ms * 1e3 / st.iterations)
            os.environ.pop("RAFEM_TEAM", None)
            print(f"{dims} G={G:3d} team={team or 'auto':4s} it={st.iterations} {best:.2f} us/it", flush=True)
