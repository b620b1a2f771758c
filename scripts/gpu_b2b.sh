#!/bin/bash
# back-to-back SpMV at 1M / 16M dofs with and without PDL, plus ncu DRAM bytes of one launch in the chain
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python - > gpurun_out/b2b.txt 2>&1 <<'PY'
import ctypes as C, os, sys
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import MaterialParams, SimConfig, assemble_global, generate_box_mesh, spmv
from paper_2409_13036_b200 import _native as nat
for dims in ((80, 80, 79), (200, 200, 200)):
    mesh = generate_box_mesh(*dims); n = mesh.node_count
    t = np.full(n, 37.0)
    s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, np.zeros(n), t, 0.5)
    h = s.device; S = h.mesh.slots
    B = 16 * S + n + 4 * (n + 1) + 32 * n
    x = np.random.default_rng(1).standard_normal(2 * n)
    y0 = spmv(s.matrix, x)
    for env in ({}, {"RAFEM_NO_PDL": "1"}):
        os.environ.update(env)
        ms = C.c_double()
        for reps in (1000, 1000):
            nat.check(nat.lib().rafem_system_spmv_bench(h.handle, reps, 0, C.byref(ms)), "b2b")
        for k in env: del os.environ[k]
        print(dims, env or "PDL", f"{1e3*ms.value:.2f} us/launch {B/ms.value/1e6:.0f} GB/s", flush=True)
    ms = C.c_double()
    nat.check(nat.lib().rafem_system_spmv_bench(h.handle, 20, 1, C.byref(ms)), "cold")
    print(dims, "cold", f"{1e3*ms.value:.2f} us/launch {B/ms.value/1e6:.0f} GB/s", flush=True)
    assert np.array_equal(spmv(s.matrix, x), y0)
PY
