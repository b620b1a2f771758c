"""C5 (64M dofs) kernel-per-phase PCG with and without the per-tile L2
prefetch of the SpMV source rows (RAFEM_KP_XPF): us per iteration of a
capped cold solve from the device box mesh (argv: xpf flag, iterations)."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import SimConfig, SolverConfig
from paper_2409_13036_b200.assembly import DeviceMesh
from paper_2409_13036_b200.shard import ShardedSystem
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40
dm = DeviceMesh.from_box(318, 318, 318)
n = dm.node_count
t = np.full(n, 37.0)
x0 = np.empty(2 * n); x0[0::2], x0[1::2] = 0.0, 37.0
for xpf in ("0", "1", "0", "1"):
    os.environ["RAFEM_KP_XPF"] = xpf  # read when the solver state is created
    sh = ShardedSystem.from_device_mesh(dm, batch=16)
    sh.assemble(t, np.zeros(n), t, 0.5, SimConfig())
    x, st = sh.solve(x0=x0, config=SolverConfig(backend="pcg", precondition="jacobi", max_total_iters=iters))
    print(f"xpf={xpf} its={st.iterations} {1e3 * st.device_ms / max(st.iterations, 1):.1f} us/it", flush=True)
    del sh, x
