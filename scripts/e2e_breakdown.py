"""Where the end-to-end (host mesh -> host fields) time of one 900 s mesh-B
run goes: DeviceRun construction (mesh upload, symbolic phase, system),
the streamed simulation, and the kernel's own time."""
import sys, time
sys.path.insert(0, ".")
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
from paper_2409_13036_b200.timeloop import DeviceRun
mesh, mat = generate_box_mesh(20, 20, 21), MaterialParams.default()
cfg = SimConfig(total_time=900.0, solver=SolverConfig(backend="pcg", precondition="block_jacobi"))
for rep in range(4):
    t0 = time.perf_counter()
    run = DeviceRun(mesh, mat, cached=False)
    t1 = time.perf_counter()
    recs = []
    summ = run.run_streamed(cfg, recs.append)
    t2 = time.perf_counter()
    print(f"construct {1e3*(t1-t0):.2f} ms, run_streamed {1e3*(t2-t1):.2f} ms (kernel {summ.wall_ms:.2f} ms), "
          f"total {1e3*(t2-t0):.2f} ms, {len(recs)} records", flush=True)
