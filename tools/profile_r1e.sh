#!/bin/bash
# ncu evidence, round 1 session 3 (final code): K2 (batch-1 row-owner) on the budget-64 bench, K3 (grouped
# tcgen05) in isolation at the Mixtral-8x7B shape, and the launch list of the default bench.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ffn_rows_kernel" -s 300 -c 3 \
  -o gpurun_out/k2_b64_r1e python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-resident-check --host-alias 40 \
  > gpurun_out/k2_b64_r1e.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"grouped_kernel" -s 4 -c 2 \
  -o gpurun_out/k3_r1e tools/bin/grouped_check bench-only > gpurun_out/k3_r1e.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"ffn_rows|route_kernel|combine|grouped|gather" -s 100 -c 500 --csv --log-file gpurun_out/launches_r1e.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-resident-check --host-alias 40 > gpurun_out/launches_r1e.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -k regex:"grouped|gather|gcombine|route_kernel" -s 60 -c 300 --csv --log-file gpurun_out/launches_b16_r1e.csv \
  python bench.py --batch 16 --budget 256 --steps 1 --warmup 1 --no-cpu-baseline --no-resident-check --host-alias 40 \
  > gpurun_out/launches_b16_r1e.log 2>&1
ls -la gpurun_out | grep r1e
