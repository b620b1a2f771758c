"""C3 (1,011,200 dofs) device assembly + a few SpMV launches, for ncu captures."""
import ctypes as C
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2409_13036_b200 import MaterialParams, SimConfig, assemble_global, generate_box_mesh
from paper_2409_13036_b200 import _native as nat
mesh = generate_box_mesh(80, 80, 79)
t = np.full(mesh.node_count, 37.0)
s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, np.zeros(mesh.node_count), t, 0.5)
ms = C.c_double()
nat.check(nat.lib().rafem_system_spmv_bench(s.device.handle, 10, 0, C.byref(ms)), "spmv bench")
print("spmv ms", ms.value)
