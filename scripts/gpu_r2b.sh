#!/bin/bash
# Round-2: new shard-loop + at-scale parity tests, bench with the C4 / C5 legs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
free -g > gpurun_out/host_mem.txt
timeout 1500 python -m pytest tests/test_gpu_shard.py tests/test_gpu_scale.py -q -x --timeout 1400 -rs -s > gpurun_out/pytest_r2b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2b.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_r2b.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_r2b.log
