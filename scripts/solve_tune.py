"""Cold / hot PCG solves at C3 (and optionally C4) in both grid variants."""
import os
import sys
import time
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
from paper_2409_13036_b200 import _native as nat

dims = tuple(int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (80, 80, 79)
mesh = generate_box_mesh(*dims)
n = mesh.node_count
t = np.full(n, 37.0)
s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, np.zeros(n), t, 0.5)
S = s.device.mesh.slots
x0 = np.empty(2 * n); x0[0::2], x0[1::2] = 0.0, 37.0
cfg = SolverConfig(backend="pcg", precondition="jacobi", tolerance=1e-10)
B = 20 * S + 4 * (n + 1) + 12 * 16 * n
print(f"{dims}: {2*n} dofs, {S} slots, pcg bytes/iter {B/1e6:.1f} MB", flush=True)
for env in [{}, {"RAFEM_NO_CLASSES": "1"}, {"RAFEM_NO_STREAM_PCG": "1"}]:
    os.environ.update(env)
    for rep in range(2):
        x, st = solve(s.matrix, s.rhs, x0=x0, config=cfg)
    mode = nat.last_solve_mode()
    for k in env:
        del os.environ[k]
    us = 1e3 * st.device_ms / max(1, st.iterations)
    print(f"{str(env):32s} mode {mode} it {st.iterations} res {st.final_relative_residual:.3e} "
          f"{st.device_ms:.2f} ms  {us:.2f} us/it  {B/us/1e3:.0f} GB/s(alg 12x16N)", flush=True)
# kernel-per-phase PCG (csrc/shard.cu), one shard
from paper_2409_13036_b200.shard import ShardedSystem
import time as _t
t0 = _t.time()
for nc in ("0", "1"):
    os.environ["RAFEM_NO_CLASSES"] = nc
    sh = ShardedSystem(mesh, MaterialParams.default(), batch=int(os.environ.get("KP_BATCH", "32")))
    sh.assemble(t, np.zeros(n), t, 0.5, SimConfig())
    print(f"kp setup {_t.time()-t0:.1f}s", flush=True)
    for rep in range(2):
        w0 = _t.perf_counter()
        x, st = sh.solve(x0=x0, config=cfg)
        w = _t.perf_counter() - w0
    us = 1e3 * st.device_ms / max(1, st.iterations)
    print(f"{'kp classes=' + ('off' if nc == '1' else 'on'):32s} it {st.iterations} res {st.final_relative_residual:.3e} "
          f"{st.device_ms:.2f} ms (wall {1e3*w:.1f} ms)  {us:.2f} us/it  {B/us/1e3:.0f} GB/s(alg 12x16N)", flush=True)
    del sh
