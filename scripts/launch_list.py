"""Native run of the mesh-B analog for ncu captures (full 900 s unless a step cap is given)."""
import sys
sys.path.insert(0, ".")
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
from paper_2409_13036_b200.timeloop import DeviceRun
backend = sys.argv[1] if len(sys.argv) > 1 else "pcg"
r = DeviceRun(generate_box_mesh(20, 20, 21), MaterialParams.default())
cfg = SimConfig(total_time=900.0, solver=SolverConfig(backend=backend, precondition=__import__("os").environ.get("PREC", "jacobi")))
r.run(cfg, record_fields=False, max_steps=int(sys.argv[2]) if len(sys.argv) > 2 else None)
