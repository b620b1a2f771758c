import sys
sys.path.insert(0, ".")
import numpy as np, os
from paper_2409_13036_b200 import _native as nat
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
from paper_2409_13036_b200.timeloop import DeviceRun
L, ctx = nat.lib(), nat.context()
run = DeviceRun(generate_box_mesh(20, 20, 21), MaterialParams.default())
cfg = SimConfig(total_time=900.0, solver=SolverConfig(backend="pcg", precondition="block_jacobi"))
run.run(cfg, record_fields=False)
L.rafem_set_trace(ctx, 1)
recs, out = run.run(cfg, record_fields=False)
L.rafem_set_trace(ctx, 0)
tr = np.zeros(8 * 4096, dtype=np.int64)
L.rafem_get_trace(ctx, tr.ctypes.data, tr.size)
tr = tr.reshape(-1, 8)[: int(out.passes)].astype(float)
# per-pass stamps (globaltimer ns): 0 pass start, 1 after the first-pass
# barrier, 2 element phase done, 3 fill + constraints done, 4 solve start,
# 5 PCG done, 6 delta done; slot 7 = PCG iterations
print("passes", out.passes, "PCG iterations", int(tr[:, 7].sum()))
ph = ["barrier (first pass)", "element phase", "fill + constraints", "to solve start", "solve (Galerkin + PCG)",
      "delta"]
for k, nm in enumerate(ph):
    print(f"  {nm:24s} {np.mean(tr[:, k + 1] - tr[:, k]) / 1e3:7.2f} us/pass")
print(f"  {'pass total':24s} {np.mean(np.diff(tr[:, 0])) / 1e3:7.2f} us/pass, {tr[:, 7].mean():.2f} PCG its/pass")
d = np.zeros(8 * 4096, dtype=np.int64)
L.rafem_get_trace(ctx, d.ctypes.data, d.size)
g = d[8 * 4000: 8 * 4000 + 10].astype(float) / 1.965e3
names = ["products", "stage D", "dots", "barrier", "fold", "barrier", "read totals",
         "Cholesky + solves", "x0, r0 update"]
print("last Galerkin start, CTA 0 (us):")
for k, nm in enumerate(names):
    print(f"  {nm:22s} {g[k + 1] - g[k]:6.2f}")
print(f"  {'total':22s} {g[9] - g[0]:6.2f}")
per = d[8 * 4002: 8 * 4002 + 148].astype(float) / 1.965e3
print("per-CTA start -> dots done (us): min %.2f median %.2f max %.2f (cta %d)" % (per.min(), np.median(per), per.max(), per.argmax()))
print("slowest CTAs:", np.argsort(per)[-8:], np.sort(per)[-8:].round(2))
