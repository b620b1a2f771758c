"""Time of the per-mesh setup on the e2e path (rafem_mesh_create: uploads +
symbolic phase + geometry) and of the first simulation's extra setup."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
from paper_2409_13036_b200.assembly import DeviceMesh
from paper_2409_13036_b200.timeloop import DeviceRun
from paper_2409_13036_b200 import _native as nat
mesh = generate_box_mesh(20, 20, 21)
mat = MaterialParams.default()
nat.context()
for k in range(6):
    t0 = time.perf_counter(); dm = DeviceMesh(mesh, mat); t1 = time.perf_counter()
    print(f"DeviceMesh create {1e3 * (t1 - t0):.3f} ms")
    del dm
cfg = SimConfig(total_time=900.0, solver=SolverConfig(backend="pcg", precondition="block_jacobi"))
for k in range(4):
    t0 = time.perf_counter()
    s = DeviceRun(mesh, mat, cached=False).run_streamed(cfg, lambda r: None)
    t1 = time.perf_counter()
    print(f"e2e run {1e3 * (t1 - t0):.2f} ms  device-side wall {s.wall_ms:.2f} ms")
