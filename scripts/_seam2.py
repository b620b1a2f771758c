import os, sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "baseline/_ref")
import torch, torch.distributed as dist
rank = int(os.environ.get("RANK", "0")); world = int(os.environ.get("WORLD_SIZE", "1"))
dist.init_process_group("gloo")
torch.cuda.set_device(0)
import rafem.fem as F
from rafem.mesh import generate_box_mesh as ref_box
from rafem.solver import SolverConfig as RS
from paper_2409_13036_b200 import plugin
rmesh, rmat = ref_box(20, 20, 21), F.MaterialParams.default()
for solver in ("pcg", None, None):
    plugin.install("rafem.fem", solver=solver, precondition="block_jacobi" if solver else None)
    cfg = F.SimConfig(total_time=900.0, solver=RS(backend="gmres", precondition="jacobi"))
    try:
        s = F.run_simulation(rmesh, rmat, cfg)
        print(rank, solver, "ok", s.accepted_steps, flush=True)
    except Exception as e:
        print(rank, solver, "FAIL", repr(e)[:200], flush=True)
    plugin.uninstall("rafem.fem")
    dist.barrier()
dist.destroy_process_group()
