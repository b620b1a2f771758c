"""cProfile of the reference's own run_simulation (baseline/_ref) with the
plug-in seam installed (device assemble_global + device PCG)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, ".")
REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
sys.path.insert(0, REF)
import rafem.fem as F
from rafem.mesh import generate_box_mesh as ref_box
from rafem.solver import SolverConfig as RefSolverConfig
from paper_2409_13036_b200 import plugin
solver = sys.argv[1] if len(sys.argv) > 1 else "pcg"
plugin.install("rafem.fem", solver=solver if solver == "pcg" else None,
               precondition="block_jacobi" if solver == "pcg" else None)
mesh, mat = ref_box(20, 20, 21), F.MaterialParams.default()
cfg = F.SimConfig(total_time=900.0, solver=RefSolverConfig(backend="gmres", precondition="jacobi"))
F.run_simulation(mesh, mat, cfg)
t0 = time.perf_counter(); s = F.run_simulation(mesh, mat, cfg); w = time.perf_counter() - t0
print("wall", w, "steps/s", s.accepted_steps / w)
pr = cProfile.Profile(); pr.enable(); F.run_simulation(mesh, mat, cfg); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
