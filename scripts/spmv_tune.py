"""Tune / verify the streaming SpMV configurations on a device-assembled box.

    python scripts/spmv_tune.py [nx ny nz]     (default 80 80 79 = C3)
"""
import ctypes as C
import os
import sys
import time
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import MaterialParams, SimConfig, assemble_global, generate_box_mesh
from paper_2409_13036_b200 import _native as nat

dims = tuple(int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (80, 80, 79)
t0 = time.time()
mesh = generate_box_mesh(*dims)
n = mesh.node_count
rng = np.random.default_rng(2409)
t = 37.0 + rng.uniform(0, 30, n)
s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, rng.uniform(0, 25, n), t, 0.5)
h = s.device
S, N = h.mesh.slots, n
print(f"mesh {dims}: {2*N} dofs, {S} slots, setup {time.time()-t0:.1f}s", flush=True)
B = 20 * S + 4 * (N + 1) + 32 * N
x = rng.standard_normal(2 * N)
os.environ["RAFEM_NO_TMA_SPMV"] = "1"
y_ref = np.empty(2 * N)
nat.check(nat.lib().rafem_system_spmv(h.handle, x.ctypes.data, y_ref.ctypes.data), "spmv")
ms = C.c_double()
nat.check(nat.lib().rafem_system_spmv_bench(h.handle, 30, int(os.environ.get("FLUSH", "1")), C.byref(ms)), "bench")
print(f"thread-per-row      {1e3*ms.value:8.2f} us  {B/ms.value/1e6:8.1f} GB/s")
del os.environ["RAFEM_NO_TMA_SPMV"]
cfgs = os.environ.get("CFGS", "legacy 256,2,1 256,2,1/nocls 256,3,1 384,2,1 512,2,1 192,3,1 "
                      "128,3,1,2 96,4,1,2 128,2,1,3 64,4,1,3 192,2,1,2 128,4,1 128,2,1,2").split()
for cfg in cfgs:
    os.environ["RAFEM_NO_CLASSES"] = "1" if cfg.endswith("/nocls") else "0"
    cfg = cfg.split("/")[0]
    if cfg == "legacy":
        os.environ["RAFEM_SPMV_CFG"] = "1,1,1"  # no such config -> two-stage kernel
    else:
        os.environ["RAFEM_SPMV_CFG"] = cfg
    y = np.empty(2 * N)
    nat.check(nat.lib().rafem_system_spmv(h.handle, x.ctypes.data, y.ctypes.data), "spmv")
    best = 1e9
    for _ in range(3):
        nat.check(nat.lib().rafem_system_spmv_bench(h.handle, 30, int(os.environ.get("FLUSH", "1")), C.byref(ms)), "bench")
        best = min(best, ms.value)
    print(f"{cfg:18s}  {1e3*best:8.2f} us  {B/best/1e6:8.1f} GB/s  bitexact={np.array_equal(y, y_ref)}", flush=True)
