#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_pcg.csv python scripts/launch_list.py pcg > gpurun_out/ncu_ll.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fill_kernel -s 3 -c 1 -o gpurun_out/prof_fill python scripts/launch_list.py pcg >> gpurun_out/ncu_ll.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pcg_grid -s 3 -c 1 -o gpurun_out/prof_pcg_grid python scripts/launch_list.py pcg >> gpurun_out/ncu_ll.log 2>&1
