#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python scripts/spmv_tune.py > gpurun_out/spmv_tune.txt 2>&1
timeout 600 python scripts/spmv_tune.py 200 200 200 >> gpurun_out/spmv_tune.txt 2>&1
