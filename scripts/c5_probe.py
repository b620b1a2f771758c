"""configs[4] on ONE B200: the 64M-dof box built on the device (no host mesh),
assembled, and a capped kernel-per-phase PCG solve (HBM-sized, ~100 GB)."""
import sys, time
sys.path.insert(0, ".")
import ctypes as C
import numpy as np
from paper_2409_13036_b200 import MaterialParams, SolverConfig
from paper_2409_13036_b200 import _native as nat
from paper_2409_13036_b200.assembly import DeviceMesh, SystemHandle
from paper_2409_13036_b200.krylov import _params
dims = tuple(int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (318, 318, 318)
iters = int(sys.argv[4]) if len(sys.argv) >= 5 else 30
t0 = time.time()
dm = DeviceMesh.from_box(*dims)
t1 = time.time()
N, S = dm.node_count, dm.slots
print(f"{dims}: {2*N} dofs, {dm.tet_count} tets, {S} slots; device mesh + symbolic {t1-t0:.2f} s", flush=True)
h = SystemHandle(dm)
t = np.full(N, 37.0); v = np.zeros(N)
p = nat.AssembleParams(); p.dt = 0.5; p.applied_voltage = 25.0; p.boundary_temp = 37.0
p.apply_constraints = 1; p.equilibrate = 1
sc, bad = C.c_double(), C.c_int64()
for rep in range(3):
    a0 = time.time()
    nat.check(nat.lib().rafem_assemble(h.handle, nat.ptr(t), nat.ptr(v), nat.ptr(t), C.byref(p), C.byref(sc), C.byref(bad)), "assemble")
    print(f"assembly {1e3*(time.time()-a0):.1f} ms (incl. 3 x {8*N/1e6:.0f} MB H2D), scale {sc.value}", flush=True)
x0 = np.empty(2 * N); x0[0::2], x0[1::2] = 0.0, 37.0
x = np.empty(2 * N)
st = nat.SolveStatsC()
hist = np.empty(iters + 1); cyc = np.empty(iters + 1, dtype=np.int64)
prm = _params(SolverConfig(backend="pcg", precondition="jacobi", max_total_iters=iters), nat.METHOD_PCG)
for rep in range(2):
    rc = nat.lib().rafem_system_solve(h.handle, None, nat.ptr(x0), C.byref(prm), nat.ptr(x), C.byref(st),
                                      nat.ptr(hist), hist.size, nat.ptr(cyc), cyc.size)
    nat.check(rc, "solve")
mode = nat.last_solve_mode()
B = 20 * S + 4 * (N + 1) + 14 * 16 * N
us = 1e3 * st.device_ms / max(st.iterations, 1)
print(f"solve mode {mode}: {st.iterations} its, {st.device_ms:.1f} ms, {us:.1f} us/it, "
      f"{B/us/1e3:.0f} GB/s algorithmic ({B/1e9:.2f} GB/iteration)", flush=True)
free, total = C.c_size_t(), C.c_size_t()
import torch
f, tt = torch.cuda.mem_get_info()
print(f"device memory used {(tt - f)/1e9:.1f} GB of {tt/1e9:.1f}", flush=True)
