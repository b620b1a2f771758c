"""Break down the e2e whole-simulation path (mesh upload, symbolic, run, records)."""
import sys, time
sys.path.insert(0, ".")
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
from paper_2409_13036_b200.assembly import DeviceMesh, SystemHandle
from paper_2409_13036_b200.timeloop import DeviceRun
mesh = generate_box_mesh(20, 20, 21)
mat = MaterialParams.default()
cfg = SimConfig(total_time=900.0, solver=SolverConfig(backend="pcg", precondition="block_jacobi"))
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    t0 = time.perf_counter(); dm = DeviceMesh(mesh, mat); t1 = time.perf_counter()
    run = DeviceRun.from_device_mesh(dm, mat); t2 = time.perf_counter()
    recs = []; s = run.run_streamed(cfg, recs.append); t3 = time.perf_counter()
    print(f"mesh {1e3*(t1-t0):.1f} ms, system {1e3*(t2-t1):.1f} ms, streamed run {1e3*(t3-t2):.1f} ms "
          f"(kernel wall {s.wall_ms:.1f})", flush=True)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    t0 = time.perf_counter(); r = DeviceRun(mesh, mat, cached=False); t1 = time.perf_counter()
    recs = []; s = r.run_streamed(cfg, recs.append); t2 = time.perf_counter()
    print(f"DeviceRun(cached=False) {1e3*(t1-t0):.1f} ms, streamed run {1e3*(t2-t1):.1f} ms", flush=True)
