#!/bin/bash
# Round-2 ncu captures of the dominant kernels, summarised ON the box
# (scripts/ncu_summary.py) so only the text summaries come back (the
# .ncu-rep files exceed gpurun's 64 MiB return limit).  TAG: profile prefix.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${TAG:-r2f}
mkdir -p gpurun_out/prof_txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-c4 --no-c3 --no-c5 > gpurun_out/ncu_ll.log 2>&1
PREC=block_jacobi timeout 900 ncu --set full --import-source on --clock-control none -k regex:simulate -c 1 -o /tmp/prof_simulate -f python scripts/launch_list.py pcg >> gpurun_out/ncu_ll.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gmres_grid -s 1 -c 1 -o /tmp/prof_gmres -f python scripts/gmres_trace.py >> gpurun_out/ncu_ll.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:spmv_tma -s 5 -c 1 -o /tmp/prof_spmv_c3 -f python scripts/c3_spmv.py >> gpurun_out/ncu_ll.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fused_fill|element_scalars|constrain" -c 3 -o /tmp/prof_asm_c4 -f python scripts/asm_probe.py 200 200 200 1 >> gpurun_out/ncu_ll.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"kp_spmv|kp_update" -s 10 -c 2 -o /tmp/prof_kp_c4 -f python scripts/kp_probe.py >> gpurun_out/ncu_ll.log 2>&1
python scripts/ncu_summary.py $TAG gpurun_out/launches_bench.csv /tmp/prof_simulate.ncu-rep /tmp/prof_gmres.ncu-rep /tmp/prof_spmv_c3.ncu-rep /tmp/prof_asm_c4.ncu-rep /tmp/prof_kp_c4.ncu-rep >> gpurun_out/ncu_ll.log 2>&1
cp profiles/${TAG}_* profiles/traffic.json gpurun_out/prof_txt/ 2>/dev/null
ncu -i /tmp/prof_simulate.ncu-rep --page source --csv --print-source sass > /tmp/sim_src.csv 2>/dev/null
ncu -i /tmp/prof_simulate.ncu-rep --page source --csv > gpurun_out/prof_txt/simulate_source_cuda.csv 2>/dev/null
ncu -i /tmp/prof_gmres.ncu-rep --page source --csv > gpurun_out/prof_txt/gmres_source_cuda.csv 2>/dev/null
gzip -f gpurun_out/prof_txt/*_source_cuda.csv
rm -f gpurun_out/launches_bench.csv
echo done > gpurun_out/ncu_done.txt
