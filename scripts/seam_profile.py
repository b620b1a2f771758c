"""cProfile of the plug-in seam path (run_simulation -> assemble_global -> solve)."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh, run_simulation
mesh = generate_box_mesh(20, 20, 21)
cfg = SimConfig(total_time=900.0, solver=SolverConfig(backend="pcg", precondition="block_jacobi"))
run_simulation(mesh, MaterialParams.default(), cfg)
t0 = time.perf_counter(); s = run_simulation(mesh, MaterialParams.default(), cfg); print("wall", time.perf_counter() - t0)
pr = cProfile.Profile(); pr.enable(); run_simulation(mesh, MaterialParams.default(), cfg); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
