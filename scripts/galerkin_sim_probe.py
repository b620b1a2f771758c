"""Fused simulation with the Galerkin solver start (default) vs without
(RAFEM_GALERKIN_K=0): ms per 900 s mesh-B run, iterations, trajectory and
fields; argv: optional list of window sizes."""
import os, subprocess, sys
sys.path.insert(0, ".")
code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
from paper_2409_13036_b200.timeloop import DeviceRun
dims = tuple(int(a) for a in sys.argv[1:4]); T = float(sys.argv[4])
mesh = generate_box_mesh(*dims)
cfg = SimConfig(total_time=T, solver=SolverConfig(backend="pcg", precondition="block_jacobi"))
run = DeviceRun(mesh, MaterialParams.default())
best = 1e9
for k in range(5):
    recs, s = run.run(cfg, record_fields=(k == 0))
    if k == 0:
        np.save(sys.argv[5], np.concatenate([np.stack([r.V, r.T], 1).ravel() for r in recs]))
        traj = [(r.time, r.dt, r.corrector_iters) for r in recs]
    best = min(best, s.wall_ms)
import json
json.dump(traj, open(sys.argv[5] + ".json", "w"))
print(f"{run.last_mode} steps={s.accepted_steps} passes={s.passes} inner={s.total_solver_iterations} "
      f"wall_ms={best:.2f} asm={s.assemble_ms:.2f} solve={s.solve_ms:.2f} us/it={s.solve_ms*1e3/max(s.total_solver_iterations,1):.2f}")
'''
import json
import numpy as np
for dims, T in ((["20", "20", "21"], "900"), (["15", "15", "16"], "40")):
    outs = {}
    ks = sys.argv[1].split(",") if len(sys.argv) > 1 else ["12"]
    for name, extra in [("no-galerkin", {"RAFEM_GALERKIN_K": "0"})] + [(f"galerkin-{k}", {"RAFEM_GALERKIN_K": k}) for k in ks]:
        env = dict(os.environ, **extra)
        f = f"/tmp/bj_{name}.npy"
        o = subprocess.run([sys.executable, "-c", code] + dims + [T, f], env=env, capture_output=True, text=True)
        print(dims, name, o.stdout.strip() or o.stderr.strip()[-500:], flush=True)
        if os.path.exists(f):
            outs[name] = (np.load(f), json.load(open(f + ".json")))
    for name in outs:
        if name == "no-galerkin" or "no-galerkin" not in outs:
            continue
        (a, ta), (b, tb) = outs["no-galerkin"], outs[name]
        print("   ", name, "same trajectory:", ta == tb, " max field diff / peak:",
              float(np.max(np.abs(a - b)) / np.max(np.abs(a))) if a.shape == b.shape else "shapes differ", flush=True)
