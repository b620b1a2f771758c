#!/bin/bash
# fused-simulation A/B while iterating: phase trace (new / RAFEM_NO_VX0), GPU tests, bench without the C4 leg
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
PREC=block_jacobi timeout 300 python scripts/sim_trace.py > gpurun_out/sim_trace_new.txt 2>&1
RAFEM_NO_VX0=1 PREC=block_jacobi timeout 300 python scripts/sim_trace.py > gpurun_out/sim_trace_old.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-c4 > gpurun_out/bench.log 2>&1
