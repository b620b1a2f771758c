#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python scripts/spmv_xpf_probe.py 80 80 79 > gpurun_out/spmv_xpf.log 2>&1
timeout 600 python scripts/spmv_xpf_probe.py 200 200 200 >> gpurun_out/spmv_xpf.log 2>&1
