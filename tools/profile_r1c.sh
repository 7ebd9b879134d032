#!/bin/bash
# ncu evidence for K2 row-owner kernel + K1 (round 1, after the redesign); one GPU.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ffn_rows_kernel" -s 200 -c 2 \
  -o gpurun_out/k2_b64_r1c python bench.py --steps 1 --warmup 1 --budget 64 --no-cpu-baseline --host-alias 40 \
  > gpurun_out/k2_b64_r1c.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ffn_rows_kernel" -s 60 -c 2 \
  -o gpurun_out/k2_b256_r1c python bench.py --steps 1 --warmup 1 --budget 256 --no-cpu-baseline --host-alias 40 \
  > gpurun_out/k2_b256_r1c.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ffn_rows|route_kernel|combine" \
  -s 100 -c 400 --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  --host-alias 40 > gpurun_out/launches_r1c.log 2>&1
ls -la gpurun_out | grep r1c
