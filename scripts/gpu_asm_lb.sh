#!/bin/bash
# A/B of the fused half-warp fill's occupancy: the committed launch bounds,
# then __launch_bounds__(256, 5), rebuilt on the box (scratch copy only).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python scripts/asm_probe.py 200 200 200 5 > gpurun_out/asm_lb.log 2>&1
sed -i 's/__global__ void __launch_bounds__(256) fused_fill_half_kernel/__global__ void __launch_bounds__(256, 5) fused_fill_half_kernel/' paper_2409_13036_b200/csrc/assembly.cu
python -c "from paper_2409_13036_b200 import build as b; b.build()" >> gpurun_out/asm_lb.log 2>&1
grep -A2 fused_fill_half paper_2409_13036_b200/_build/assembly.o.ptxas.txt >> gpurun_out/asm_lb.log
echo "--- (256, 5)" >> gpurun_out/asm_lb.log
timeout 300 python scripts/asm_probe.py 200 200 200 5 >> gpurun_out/asm_lb.log 2>&1
