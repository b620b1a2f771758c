#!/bin/bash
# DRAM bytes of SpMV launches inside a back-to-back chain (caches not flushed by ncu)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
cat > /tmp/b2b_one.py <<'PY'
import ctypes as C, sys
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import MaterialParams, SimConfig, assemble_global, generate_box_mesh
from paper_2409_13036_b200 import _native as nat
mesh = generate_box_mesh(80, 80, 79); n = mesh.node_count
t = np.full(n, 37.0)
s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, np.zeros(n), t, 0.5)
ms = C.c_double()
nat.check(nat.lib().rafem_system_spmv_bench(s.device.handle, 40, 0, C.byref(ms)), "b2b")
PY
timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:spmv_tma -s 20 -c 5 --csv python /tmp/b2b_one.py > gpurun_out/b2b_ncu.csv 2> gpurun_out/b2b_ncu.err
