#!/bin/bash
# ncu evidence, round 1 session 3 (tile-merged launches, K1 window routing): launch list of the
# default bench (budget 64, batch 1), a full capture of K2 launches inside that decode and of the K1
# window launch.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"ffn_rows|route|combine" -s 20 -c 400 --csv --log-file gpurun_out/launches_r1n.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-resident-check > gpurun_out/launches_r1n.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ffn_rows_kernel" -s 150 -c 6 \
  -o gpurun_out/k2_merged_r1n python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-resident-check \
  > gpurun_out/k2_merged_r1n.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"route" -c 2 \
  -o gpurun_out/k1_window_r1n python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-resident-check \
  > gpurun_out/k1_window_r1n.log 2>&1
ls -la gpurun_out | grep r1n
