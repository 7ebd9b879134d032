#!/bin/bash
# ncu evidence, round 2 final: launch lists of the default bench (8x7B batch 1, budget 64, XBH store)
# — FFN / router / combine, and the coded-tile decode kernels separately (they outnumber the FFN
# launches) — plus full captures of K2 (ffn_ring_kernel), the XBH decode kernel, and K3
# (grouped_kernel, batch 16) inside their decodes.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"ffn_|route|combine" -c 200 --csv \
  --log-file gpurun_out/launches_r2j_ffn.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-resident-check \
  > gpurun_out/launches_r2j_ffn.log 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:"decode_kernel|patch_kernel" -c 200 --csv \
  --log-file gpurun_out/launches_r2j_decode.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-resident-check \
  > gpurun_out/launches_r2j_decode.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ffn_ring_kernel" -s 8 -c 3 \
  -o gpurun_out/r2j_k2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-resident-check \
  > gpurun_out/r2j_k2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_kernel" -s 40 -c 2 \
  -o gpurun_out/r2j_xbh python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-resident-check \
  > gpurun_out/r2j_xbh.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"grouped_kernel" -s 16 -c 4 \
  -o gpurun_out/r2j_k3 python bench.py --batch 16 --steps 1 --warmup 1 --no-cpu-baseline --no-resident-check \
  > gpurun_out/r2j_k3.log 2>&1
ls -la gpurun_out | grep r2j
