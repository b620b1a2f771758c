cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_gpu_assembly_sim.py -q -x -k "exact or golden or two_regions" > gpurun_out/pt_exact.log 2>&1; echo "rc=$?" >> gpurun_out/pt_exact.log
timeout 300 ncu --set full --import-source on -k regex:cpcg -c 1 -s 1 -o gpurun_out/prof_cpcg python scripts/cluster_one.py > gpurun_out/ncu_cpcg.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cpcg.csv python scripts/cluster_one.py > /dev/null 2>&1
