"""configs[2] cold PCG solve (1M dofs) through each engine: the TMA-streaming
persistent kernel (default below 1 GB) and the kernel-per-phase engine."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
mesh = generate_box_mesh(80, 80, 79); n = mesh.node_count
t = np.full(n, 37.0)
s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, np.zeros(n), t, 0.5)
x0 = np.empty(2 * n); x0[0::2], x0[1::2] = 0.0, 37.0
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
cfg = SolverConfig(backend="pcg", precondition="jacobi")
for label, env in (("stream", {"RAFEM_KP": "0"}), ("kernel-per-phase", {"RAFEM_KP": "1"})):
    os.environ.update(env)
    try:
        solve(s.matrix, s.rhs, x0=x0, config=cfg)
        best = 1e9
        for _ in range(3):
            flush.fill_(1.0); torch.cuda.synchronize()
            x, st = solve(s.matrix, s.rhs, x0=x0, config=cfg)
            best = min(best, st.device_ms)
        print(f"{label:18s} its {st.iterations} {1e3 * best / st.iterations:7.2f} us/it  res {st.final_relative_residual:.2e}",
              flush=True)
    finally:
        for k in env: del os.environ[k]
