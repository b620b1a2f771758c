#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 120 ./scripts/microbench > gpurun_out/microbench.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pcg_cluster -s 20 -c 1 -o gpurun_out/prof_pcg_cluster \
   python bench.py --steps 1 --warmup 0 --no-e2e --no-c3 --no-cpu > gpurun_out/ncu_pcg.log 2>&1
