"""Per-pass phase breakdown of the fused simulation kernel (mesh-B analog, 900 s)."""
import ctypes as C, sys
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import _native as nat
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
from paper_2409_13036_b200.timeloop import DeviceRun
L, ctx = nat.lib(), nat.context()
dims = tuple(int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (20, 20, 21)
run = DeviceRun(generate_box_mesh(*dims), MaterialParams.default())
import os
cfg = SimConfig(total_time=900.0, solver=SolverConfig(backend="pcg", precondition=os.environ.get("PREC", "jacobi")))
run.run(cfg, record_fields=False)
for rep in range(2):
    L.rafem_set_trace(ctx, 1)
    recs, out = run.run(cfg, record_fields=False)
    L.rafem_set_trace(ctx, 0)
    tr = np.zeros(8 * 4096, dtype=np.int64)
    L.rafem_get_trace(ctx, tr.ctypes.data, tr.size)
    tr = tr.reshape(-1, 8)[: int(out.passes)]
    d = np.diff(tr[:, :7], axis=1) / 1e3  # us
    its = tr[:, 7]
    names = ["top barrier", "element+max", "fill+diag reduce", "constrain+bnorm reduce", "pcg", "delta reduce"]
    tot = (tr[-1, 6] - tr[0, 0]) / 1e6
    print(f"{dims}: passes {out.passes}, pcg its {out.total_solver_iterations}, kernel {tot:.2f} ms "
          f"(summary wall {out.wall_ms:.2f} ms)")
    for i, nme in enumerate(names):
        print(f"  {nme:24s} mean {d[:, i].mean():7.2f} us  total {d[:, i].sum() / 1e3:7.2f} ms")
    print(f"  pcg per iteration       {d[:, 4].sum() / max(its.sum(), 1):7.2f} us over {its.sum()} its")
    gap = (tr[1:, 0] - tr[:-1, 6]) / 1e3
    print(f"  between passes          mean {gap.mean():7.2f} us  total {gap.sum() / 1e3:7.2f} ms")
