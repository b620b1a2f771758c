#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python scripts/asm_probe.py 80 80 79 5 > gpurun_out/asm_probe.log 2>&1
timeout 600 python scripts/asm_probe.py 200 200 200 5 >> gpurun_out/asm_probe.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_assembly_sim.py tests/test_gpu_scale.py tests/test_gpu_sparse_solver.py -q --timeout 1400 -rs -s > gpurun_out/pytest_r2c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2c.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fused_fill|element_kernel|fill_slots|constrain" -c 4 -o gpurun_out/prof_asm_c4 -f python scripts/asm_probe.py 200 200 200 1 > gpurun_out/ncu_asm.log 2>&1
