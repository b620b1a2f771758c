#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pcg_stream -c 1 -o gpurun_out/prof_pcg_stream_c4 -f python scripts/stream_pcg_probe.py 200 200 200 20 > gpurun_out/ncu_stream.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pcg_stream -c 1 -o gpurun_out/prof_pcg_stream_c3 -f python scripts/stream_pcg_probe.py 80 80 79 100 >> gpurun_out/ncu_stream.log 2>&1
