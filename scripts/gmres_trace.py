"""Per-phase timing of the persistent GMRES inner step (paper scale): the
one-reduce Arnoldi step (default) or, with RAFEM_GMRES_CGS2=1, the
three-synchronisation CGS2 step."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import _native as nat
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
L, ctx = nat.lib(), nat.context()
mesh = generate_box_mesh(20, 20, 21)
n = mesh.node_count
rng = np.random.default_rng(2409)
t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
x0 = np.empty(2 * n); x0[0::2], x0[1::2] = v, t
cfg = SolverConfig(backend="gmres", precondition="jacobi")
solve(s.matrix, s.rhs, x0=x0, config=cfg)
L.rafem_set_trace(ctx, 1)
x, st = solve(s.matrix, s.rhs, x0=x0, config=cfg)
L.rafem_set_trace(ctx, 0)
tr = np.zeros(8 * 4096, dtype=np.int64)
L.rafem_get_trace(ctx, tr.ctypes.data, tr.size)
cgs2 = os.environ.get("RAFEM_GMRES_CGS2") == "1"
if cgs2:
    names = ["basis row + spmv", "multidot1", "sync_gather1", "update1+multidot2", "sync_gather2", "update2+barrier"]
else:
    names = ["spmv", "pair dots", "barrier 1", "gather + alpha", "sweep + arrive", "Givens | H column | wait"]
ns = len(names) + 1
tr = tr.reshape(-1, 8)[5:min(st.iterations, 4000) - 1]
if not cgs2:
    print("explicit-norm steps:", int((tr[:, 7] > 0).sum()), "of", len(tr))
ok = (tr[:, :ns] > 0).all(axis=1)
tr = tr[ok]
d = np.diff(tr[:, :ns], axis=1) / 1.965e3
print(f"gmres ({'cgs2' if cgs2 else 'one-reduce'}): {st.iterations} its, {st.device_ms*1e3/st.iterations:.2f} us/it")
for i, nme in enumerate(names):
    print(f"  {nme:40s} {d[:, i].mean():6.2f} us")
print(f"  step (0->0)                              {np.diff(tr[:, 0]).mean() / 1.965e3:6.2f} us")
