#!/bin/bash
# ncu evidence, round 2 final (XBH store): launch list of the default bench (8x7B batch 1, budget 64)
# with DRAM bytes per launch — K2, the XBH decode + escape patch, combine, router — and one full
# capture each of K2 and of the XBH decode kernel inside that decode.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"ffn_|route|combine|decode_kernel|patch_kernel" -c 600 --csv --log-file gpurun_out/launches_r2h.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-resident-check > gpurun_out/launches_r2h.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ffn_ring_kernel|decode_kernel" -s 40 -c 4 \
  -o gpurun_out/r2h_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-resident-check \
  > gpurun_out/r2h_full.log 2>&1
ls -la gpurun_out | grep r2h
