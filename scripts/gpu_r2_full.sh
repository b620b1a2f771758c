#!/bin/bash
# Round-2 full GPU pass: smoke, every GPU test, bench (both arms), launch
# list, ncu --set full captures of the dominant kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 3000 python -m pytest tests -q -m gpu --timeout 1800 -rs ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_ref.log
if [ -z "$SKIP_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-c4 --no-c3 --no-c5 > gpurun_out/ncu_ll.log 2>&1
PREC=block_jacobi timeout 900 ncu --set full --import-source on --clock-control none -k regex:simulate -c 1 -o gpurun_out/prof_simulate -f python scripts/launch_list.py pcg >> gpurun_out/ncu_ll.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:spmv_tma -s 5 -c 1 -o gpurun_out/prof_spmv_c3 -f python scripts/c3_spmv.py >> gpurun_out/ncu_ll.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"kp_spmv|kp_update" -s 10 -c 2 -o gpurun_out/prof_kp_c4 -f python scripts/kp_probe.py >> gpurun_out/ncu_ll.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fused_fill|element_scalars|constrain" -c 3 -o gpurun_out/prof_asm_c4 -f python scripts/asm_probe.py 200 200 200 1 >> gpurun_out/ncu_ll.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gmres_grid -s 1 -c 1 -o gpurun_out/prof_gmres -f python scripts/gmres_trace.py >> gpurun_out/ncu_ll.log 2>&1
fi
echo done > gpurun_out/round_done.txt
