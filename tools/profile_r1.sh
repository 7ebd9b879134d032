#!/bin/bash
# Round-1 profiling recipe (run under gpurun on one B200).
set -x
mkdir -p gpurun_out
# 1) launch list of our kernels during a short 8x7B bench (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ffn_pass|route_kernel|combine" \
  -s 30 -c 300 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/launches_r1.log 2>&1
# 2) full capture of the top kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ffn_pass_kernel" -s 40 -c 2 \
  -o gpurun_out/ffn_r1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ffn_r1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"route_kernel" -s 40 -c 1 \
  -o gpurun_out/router_r1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/router_r1.log 2>&1
ls -la gpurun_out
