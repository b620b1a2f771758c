"""Cluster-resident PCG (cluster.cu) vs the 148-CTA grid PCG at paper scale:
iterations, us per iteration, true residual, agreement of the solutions."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
from oracle import rafem_oracle as O
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve

for dims in [(20, 20, 21), (15, 15, 16), (6, 5, 7)]:
    mesh = generate_box_mesh(*dims)
    n = mesh.node_count
    rng = np.random.default_rng(2409)
    t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
    s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
    a = s.matrix
    x0 = np.empty(2 * n); x0[0::2], x0[1::2] = v, t
    sols = {}
    for eng, prec in [("0", "block_jacobi"), ("0", "jacobi"), ("1", "jacobi"), ("1", "none")]:
        os.environ["RAFEM_CLUSTER"] = eng
        for tol in (1e-10, 1e-12):
            cfg = SolverConfig(backend="pcg", precondition=prec, tolerance=tol)
            best = 1e9
            for _ in range(3):
                x, st = solve(a, s.rhs, x0=x0, config=cfg)
                best = min(best, st.device_ms * 1e3 / max(st.iterations, 1))
            res = np.linalg.norm(s.rhs - O.matvec(a.row_ptr, a.col_idx, a.vals, x)) / np.linalg.norm(s.rhs)
            sols[(eng, prec, tol)] = x
            ref = sols.get(("0", "jacobi", tol))
            dx = np.max(np.abs(x - ref)) / np.max(np.abs(ref)) if ref is not None else float("nan")
            print(f"{dims} cluster={eng} {prec:12s} tol={tol:g} it={st.iterations} restarts={st.restarts} "
                  f"{best:.2f} us/it dev_ms={st.device_ms:.3f} true_res={res:.2e} reported={st.final_relative_residual:.2e} "
                  f"conv={st.converged} dx_vs_grid={dx:.1e} hist={len(st.residual_history)}", flush=True)
