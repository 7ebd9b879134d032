#!/bin/bash
# ncu of the final XBH tile decoder inside the default decode (launch list + 2 full captures).
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"decode_kernel|patch_kernel" -c 200 --csv \
  --log-file gpurun_out/launches_r2m_decode.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-resident-check \
  > gpurun_out/launches_r2m_decode.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_kernel" -s 40 -c 2 \
  -o gpurun_out/r2m_xbh python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-resident-check \
  > gpurun_out/r2m_xbh.log 2>&1
ls -la gpurun_out | grep r2m
