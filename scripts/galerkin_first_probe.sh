for cfg in "0 12" "16 12" "16 16" "0 10"; do set -- $cfg; echo "dbg=$1 k=$2"; RAFEM_GAL_DBG=$1 RAFEM_GALERKIN_K=$2 timeout 100 python -c "
import sys; sys.path.insert(0,'.')
from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
from paper_2409_13036_b200.timeloop import DeviceRun
run = DeviceRun(generate_box_mesh(20,20,21), MaterialParams.default())
cfg = SimConfig(total_time=900.0, solver=SolverConfig(backend='pcg', precondition='block_jacobi'))
best=1e9
for k in range(5):
    r,s = run.run(cfg, record_fields=False); best=min(best, s.wall_ms)
print('its', s.total_solver_iterations, 'wall', round(best,2), 'solve', round(s.solve_ms,2))
"; done
