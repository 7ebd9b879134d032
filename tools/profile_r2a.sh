#!/bin/bash
# ncu evidence, round 2 (K2 TMA ring, one FFN launch per layer): launch list of the default bench
# (8x7B batch 1, budget 64) with DRAM bytes per launch, and one full capture of K2 launches inside
# that decode.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"ffn_|route|combine" -s 20 -c 300 --csv --log-file gpurun_out/launches_r2a.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-resident-check > gpurun_out/launches_r2a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ffn_ring_kernel" -s 40 -c 4 \
  -o gpurun_out/k2_ring_r2a python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-resident-check \
  > gpurun_out/k2_ring_r2a.log 2>&1
ls -la gpurun_out | grep r2a
