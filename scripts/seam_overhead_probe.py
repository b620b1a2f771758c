"""Fixed host-side cost of the plug-in seam's calls on the mesh-B analog:
assemble_global, the rhs download, and a device solve that converges at its
start (x0 = the solution), each timed over many calls (wall clock)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve

mesh = generate_box_mesh(20, 20, 21)
n = mesh.node_count
rng = np.random.default_rng(2409)
t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
mat, cfg = MaterialParams.default(), SimConfig()
for backend in ("pcg", "gmres"):
    scfg = SolverConfig(backend=backend, precondition="jacobi", tolerance=1e-10)
    s = assemble_global(mesh, mat, cfg, t, v, t, 0.5)
    b = s.rhs.copy()
    x, st = solve(s.matrix, b, x0=None, config=scfg)
    R = 200
    t0 = time.perf_counter()
    for _ in range(R):
        s = assemble_global(mesh, mat, cfg, t, v, t, 0.5)
    t1 = time.perf_counter()
    for _ in range(R):
        s._h._rhs = None
        b = s.rhs.copy()
    t2 = time.perf_counter()
    for _ in range(R):
        x2, st2 = solve(s.matrix, b, x0=x, config=scfg)
    t3 = time.perf_counter()
    from paper_2409_13036_b200 import krylov as K, _native as nat
    p = K._params(scfg, nat.METHOD_PCG if backend == "pcg" else nat.METHOD_GMRES)
    xo = np.empty(2 * n); stc = nat.SolveStatsC(); hb, cb = K._history_buffers(1000)
    ds = s.matrix.device_system
    t4 = time.perf_counter()
    for _ in range(R):
        ds.solve(b, x, p, xo, stc, hb, cb)
    t5 = time.perf_counter()
    pz = K._params(SolverConfig(backend=backend, precondition="none", tolerance=1e-10),
                   nat.METHOD_PCG if backend == "pcg" else nat.METHOD_GMRES)
    for _ in range(R):
        ds.solve(None, x, pz, xo, stc, hb, cb)
    t6 = time.perf_counter()
    print(f"  native rafem_system_solve {1e6*(t5-t4)/R:.1f} us; without b upload / Jacobi {1e6*(t6-t5)/R:.1f} us "
          f"(device {1e3*stc.device_ms:.1f} us, its {stc.iterations})")
    print(f"{backend}: assemble_global {1e6*(t1-t0)/R:.1f} us, rhs download {1e6*(t2-t1)/R:.1f} us, "
          f"solve at the solution {1e6*(t3-t2)/R:.1f} us (its {st2.iterations}, device {1e3*st2.device_ms:.1f} us)")

if len(sys.argv) > 1 and sys.argv[1] == "profile":
    import cProfile, pstats
    scfg = SolverConfig(backend="pcg", precondition="jacobi", tolerance=1e-10)
    def loop():
        for _ in range(300):
            s = assemble_global(mesh, mat, cfg, t, v, t, 0.5)
            b = s.rhs.copy()
            solve(s.matrix, b, x0=x, config=scfg)
    pr = cProfile.Profile()
    pr.enable(); loop(); pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
