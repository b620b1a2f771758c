#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py -q -x --timeout 600 -rs -k "ipc" > gpurun_out/pytest_ipc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ipc.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-c5 > gpurun_out/bench_expl.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_expl.log
