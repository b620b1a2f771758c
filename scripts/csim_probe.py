"""Cluster-resident simulation (cluster.cu) vs the 148-CTA fused simulation
kernel on the mesh-B analog, 900 s: ms per run, trajectory, fields."""
import os, subprocess, sys
sys.path.insert(0, ".")
code = r'''
import sys, time, numpy as np
sys.path.insert(0, ".")
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
from paper_2409_13036_b200.timeloop import DeviceRun
dims = tuple(int(a) for a in sys.argv[1:4]); prec = sys.argv[4]; T = float(sys.argv[5])
mesh = generate_box_mesh(*dims)
cfg = SimConfig(total_time=T, solver=SolverConfig(backend="pcg", precondition=prec))
run = DeviceRun(mesh, MaterialParams.default())
best = 1e9
for k in range(4):
    t0 = time.perf_counter()
    recs, s = run.run(cfg, record_fields=(k == 0))
    if k == 0:
        x = np.concatenate([np.stack([r.V, r.T], 1).ravel() for r in recs])
        np.save(sys.argv[6], x)
    best = min(best, s.wall_ms)
print(f"{run.last_mode} steps={s.accepted_steps} passes={s.passes} inner={s.total_solver_iterations} "
      f"ms={best:.2f} asm={s.assemble_ms:.2f} solve={s.solve_ms:.2f} us/it={s.solve_ms*1e3/max(s.total_solver_iterations,1):.2f}")
'''
import numpy as np
for dims, T in ((["20", "20", "21"], "900"), (["15", "15", "16"], "40")):
    for prec in ("jacobi", "block_jacobi"):
        outs = {}
        for name, extra in (("grid", {"RAFEM_SIM_CLUSTER": "0"}), ("cluster", {"RAFEM_SIM_CLUSTER": "1"})):
            env = dict(os.environ, **extra)
            f = f"/tmp/x_{name}.npy"
            o = subprocess.run([sys.executable, "-c", code] + dims + [prec, T, f], env=env, capture_output=True, text=True)
            print(dims, prec, name, o.stdout.strip() or o.stderr.strip()[-400:], flush=True)
            outs[name] = np.load(f) if os.path.exists(f) else None
            if os.path.exists(f): os.remove(f)
        a, b = outs["grid"], outs["cluster"]
        if a is not None and b is not None and a.shape == b.shape:
            print("   max field diff / peak:", float(np.max(np.abs(a - b)) / np.max(np.abs(a))), flush=True)
        elif a is not None and b is not None:
            print("   record shapes differ", a.shape, b.shape)
