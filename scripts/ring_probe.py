"""Record-streaming overhead of the fused simulation: kernel wall time of
the 900 s mesh-B run without records, with batch records, and streamed
through rings of 8 / 32 / 128 slots."""
import sys, time
sys.path.insert(0, ".")
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
from paper_2409_13036_b200.timeloop import DeviceRun
mesh = generate_box_mesh(20, 20, 21)
cfg = SimConfig(total_time=900.0, solver=SolverConfig(backend="pcg", precondition="block_jacobi"))
run = DeviceRun(mesh, MaterialParams.default())
for _ in range(2):
    run.run(cfg, record_fields=False)
for label, f in [("no records", lambda: run.run(cfg, record_fields=False)[1]),
                 ("batch records", lambda: run.run(cfg, record_fields=True)[1]),
                 ("stream 8", lambda: run.run_streamed(cfg, [].append, ring_slots=8)),
                 ("stream 32", lambda: run.run_streamed(cfg, [].append, ring_slots=32)),
                 ("stream 128", lambda: run.run_streamed(cfg, [].append, ring_slots=128))]:
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter(); s = f(); w = time.perf_counter() - t0
        best = min(best, s.wall_ms)
    print(f"{label:14s} kernel wall {best:6.2f} ms  (call {1e3*w:6.2f} ms)", flush=True)
