"""Per-phase timing of the persistent solvers on paper-scale systems."""
import ctypes as C, os, sys, numpy as np
sys.path.insert(0, ".")
from paper_2409_13036_b200 import _native as nat
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
L, ctx = nat.lib(), nat.context()
modes = sys.argv[1].split(",") if len(sys.argv) > 1 else ["grid"]
teams = sys.argv[2].split(",") if len(sys.argv) > 2 else [""]
for dims in [(20, 20, 21), (15, 15, 16)]:
    mesh = generate_box_mesh(*dims)
    n = mesh.node_count
    rng = np.random.default_rng(2409)
    t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
    s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
    x0 = np.empty(2 * n); x0[0::2], x0[1::2] = v, t
    for mode in modes:
        os.environ["RAFEM_SOLVER_MODE"] = mode
        for team in teams:
            if team: os.environ["RAFEM_TEAM"] = team
            elif "RAFEM_TEAM" in os.environ: del os.environ["RAFEM_TEAM"]
            for backend in ("pcg", "gmres"):
                L.rafem_set_trace(ctx, 1)
                cfg = SolverConfig(backend=backend, precondition="jacobi")
                x, st = solve(s.matrix, s.rhs, x0=x0, config=cfg)
                x, st = solve(s.matrix, s.rhs, x0=x0, config=cfg)
                md, nct = C.c_int32(), C.c_int32()
                L.rafem_last_solve_mode(ctx, C.byref(md), C.byref(nct))
                tr = np.zeros(8 * 4096, dtype=np.int64)
                L.rafem_get_trace(ctx, tr.ctypes.data, tr.size)
                tr = tr.reshape(-1, 8)
                k = min(st.iterations, 4095)
                line = (f"{dims} {mode:7s} team={team or 'auto':4s} {backend:5s} ctas={nct.value:3d} it={st.iterations} "
                        f"dev={st.device_ms*1e3:.0f}us -> {st.device_ms*1e3/max(st.iterations,1):.2f} us/it")
                rows = tr[5:k - 1]
                if backend == "pcg" and len(rows) > 2 and rows[0, 0] > 0:
                    sp = ((rows[:, 1] - rows[:, 0]).mean()) / 1.965e3
                    rd = ((rows[:, 4] - rows[:, 1]).mean()) / 1.965e3
                    per = (rows[1:, 0] - rows[:-1, 0]).mean() / 1.965e3
                    line += f" | spmv {sp:.2f} reduce {rd:.2f} | iter {per:.2f} us"
                print(line, flush=True)
    L.rafem_set_trace(ctx, 0)
