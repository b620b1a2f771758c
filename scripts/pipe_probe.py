"""Pipelined vs single-reduction PCG at paper scale (standalone solves)."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
from oracle import rafem_oracle as O
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
for dims in [(20, 20, 21), (15, 15, 16)]:
    mesh = generate_box_mesh(*dims)
    n = mesh.node_count
    rng = np.random.default_rng(2409)
    t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
    s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
    a = s.matrix
    x0 = np.empty(2 * n); x0[0::2], x0[1::2] = v, t
    for pipe, prec in [("1", "block_jacobi"), ("1", "jacobi"), ("0", "jacobi")]:
        os.environ["RAFEM_PIPE"] = pipe
        for tol in (1e-10, 1e-12):
            cfg = SolverConfig(backend="pcg", precondition=prec, tolerance=tol)
            best = 1e9
            for _ in range(3):
                x, st = solve(a, s.rhs, x0=x0, config=cfg)
                best = min(best, st.device_ms * 1e3 / st.iterations)
            res = np.linalg.norm(s.rhs - O.matvec(a.row_ptr, a.col_idx, a.vals, x)) / np.linalg.norm(s.rhs)
            print(f"{dims} pipe={pipe} {prec:12s} tol={tol:g} it={st.iterations} restarts={st.restarts} {best:.2f} us/it "
                  f"true_res={res:.2e} reported={st.final_relative_residual:.2e} conv={st.converged}", flush=True)
