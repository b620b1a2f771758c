#!/bin/bash
# Round-2 cluster-engine evidence: solver tests, GMRES probe, ncu of the cluster PCG.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sparse_solver.py -q -x > gpurun_out/pt_solver.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_solver.log
timeout 300 python scripts/cgmres_probe.py > gpurun_out/cgmres.txt 2>&1
timeout 300 ncu --set full --import-source on -k regex:cpcg -c 1 -s 1 -o gpurun_out/prof_cpcg python scripts/cluster_one.py > gpurun_out/ncu_cpcg.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cpcg.csv python scripts/cluster_one.py > /dev/null 2>&1
echo done > gpurun_out/r2c_done.txt
