#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python scripts/asm_probe.py 200 200 200 5 > gpurun_out/asm_probe.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fused_fill|element_scalars|constrain" -c 3 -o gpurun_out/prof_fused_fill -f python scripts/asm_probe.py 200 200 200 1 > gpurun_out/ncu_asm.log 2>&1
