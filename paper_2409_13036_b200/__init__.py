"""B200-native RAFEM hot path (arXiv 2409.13036): device assembly + Krylov solve.

Public surface mirrors the reference package ``rafem`` for the hot path:

* sparse:   CooMatrix, CsrMatrix, coo_to_csr, spmv            (rafem/sparse.py)
* solver:   SolverConfig, SolveStats, solve, gmres, pcg, errors (rafem/solver.py)
* assembly: assemble_global, MaterialParams, RegionMaterial, SimConfig,
            AssembledSystem, PhysicsRangeError                  (rafem/fem.py)
* callers:  run_simulation, corrector_step, predictor, ...     (rafem/fem.py)
* mesh:     TetMesh, generate_box_mesh                           (rafem/mesh.py)
* plugin:   install() rebinds rafem.fem.assemble_global / rafem.fem.solve

Compute runs in librafem_b200.so (hand-written sm_100a CUDA); there is no
CPU fallback.
"""

from .assembly import (AssembledSystem, MaterialParams, PhysicsRangeError, RegionMaterial,
                       SimConfig, assemble_global, set_exact_geometry)
from .boxmesh import TetMesh, generate_box_mesh
from .csr import CooMatrix, CsrMatrix, DeviceCsrMatrix, coo_to_csr, spmv
from .krylov import (GmresBreakdownError, KrylovBreakdownError, SolveStats, SolverConfig,
                     SolverError, SolverSession, gmres, pcg, solve)
from .timeloop import (StepFailureError, StepRecord, corrector_step, initial_state,
                       interleave_fields, predictor, run_simulation, simulate_device, split_fields)

__version__ = "0.1.0"
