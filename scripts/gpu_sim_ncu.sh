#!/bin/bash
# One ncu --set full capture of the fused simulation kernel (mesh-B,
# block-Jacobi), its SASS source page as CSV (for scripts/sass_line_stalls.py
# against `nvdisasm -gi` of the same build) and the summary; text only.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/prof_txt
PREC=block_jacobi timeout 600 ncu --set full --import-source on --clock-control none -k regex:simulate -c 1 -o /tmp/prof_simulate -f python scripts/launch_list.py pcg > gpurun_out/ncu_sim.log 2>&1
ncu -i /tmp/prof_simulate.ncu-rep --page source --csv > gpurun_out/prof_txt/sim_sass.csv 2>>gpurun_out/ncu_sim.log
gzip -f gpurun_out/prof_txt/sim_sass.csv
python scripts/ncu_summary.py ${TAG:-tmp} /tmp/prof_simulate.ncu-rep >> gpurun_out/ncu_sim.log 2>&1
cp profiles/${TAG:-tmp}_prof_simulate.txt gpurun_out/prof_txt/ 2>/dev/null
