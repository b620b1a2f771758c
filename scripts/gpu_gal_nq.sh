#!/bin/bash
# Galerkin products: sources per sweep (GAL_NQ) x slots per lane in flight
# (GAL_SL), rebuilt on the box for each setting (scratch copy only).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/gal_nq.log
: > $out
for cfg in "6 4" "3 7" "5 5" "2 14"; do
  set -- $cfg
  sed -i "s/^#define GAL_NQ .*/#define GAL_NQ $1  \/\/ Galerkin products: sources per sweep/; s/^#define GAL_SL .*/#define GAL_SL $2  \/\/ Galerkin products: slots per lane in flight/" paper_2409_13036_b200/csrc/simulate_dev.cuh
  python -c "from paper_2409_13036_b200 import build as b; b.build()" > /dev/null 2>&1
  echo "=== NQ=$1 SL=$2" >> $out
  grep -A2 "simulate_kernel" paper_2409_13036_b200/_build/krylov.o.ptxas.txt | grep spill | head -2 >> $out
  timeout 120 python scripts/galerkin_trace.py 2>&1 | grep -E "products|pass total|total  " >> $out
  timeout 200 python scripts/galerkin_sim_probe.py 14 2>&1 | grep "20., .20., .21.. galerkin" >> $out
done
