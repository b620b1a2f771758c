"""Helper (test infrastructure): full runs of the REFERENCE's own
rafem.fem.run_simulation (staged in baseline/_ref) with plugin.install()
routing its corrector's assemble_global / solve to the B200 path.
Writes every accepted step to an .npz for tests/test_gpu_reference_seam.py.

    python tests/seam_runs.py OUT.npz NX NY NZ TOTAL_TIME [pcg|gmres] [TOL]
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(1, ROOT)


def main():
    out, nx, ny, nz, total = sys.argv[1], *map(int, sys.argv[2:5]), float(sys.argv[5])
    solver = sys.argv[6] if len(sys.argv) > 6 else "gmres"
    tol = float(sys.argv[7]) if len(sys.argv) > 7 else 1e-10
    import rafem
    import rafem.fem as F
    from rafem.mesh import generate_box_mesh
    from rafem.solver import SolverConfig
    from paper_2409_13036_b200 import plugin
    assert os.path.realpath(rafem.__file__).startswith(os.path.realpath(os.path.join(ROOT, "baseline", "_ref")))
    plugin.install("rafem.fem", solver=None if solver == "gmres" else solver)
    recs = []
    cfg = F.SimConfig(total_time=total, solver=SolverConfig(backend="gmres", precondition="jacobi", tolerance=tol))
    s = F.run_simulation(generate_box_mesh(nx, ny, nz), F.MaterialParams.default(), cfg, sink=recs.append)
    c = plugin.counters
    np.savez(out, time=[r.time for r in recs], dt=[r.dt for r in recs],
             corrector_iters=[r.corrector_iters for r in recs], T=np.array([r.T for r in recs]),
             V=np.array([r.V for r in recs]),
             summary=[s.accepted_steps, s.total_corrector_iters, s.total_solver_iterations],
             seam=[c.assemble, c.solve_device, c.solve_passthrough])


if __name__ == "__main__":
    main()
