#!/bin/bash
# ncu capture of the fused FFN kernel + router on the budget-256 decode (mostly resident experts)
mkdir -p gpurun_out
tag=${1:-r1b}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ffn_kernel" -s 60 -c 3 \
  -o gpurun_out/ffn_$tag python bench.py --steps 1 --warmup 1 --budget 256 --no-cpu-baseline > gpurun_out/ffn_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"route_kernel" -s 40 -c 2 \
  -o gpurun_out/router_$tag python bench.py --steps 1 --warmup 1 --budget 256 --no-cpu-baseline > gpurun_out/router_$tag.log 2>&1
ls -la gpurun_out | grep $tag
