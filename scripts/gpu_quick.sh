#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py -x -q --timeout 600 > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-c3 > gpurun_out/bench_quick.log 2>&1; echo "rc=$?" >> gpurun_out/bench_quick.log
