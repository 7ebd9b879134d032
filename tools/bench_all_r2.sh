#!/bin/bash
# Round-2 bench set on one B200 (XBH store by default): headline, free-running, batched, 8x22B
# rehearsal, and the bf16 / XB12 stores for the A/B.  Output: gpurun_out/${TAG}_*.jsonl
TAG=${TAG:-r2k}
mkdir -p gpurun_out
run() { local name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/${TAG}_$name.jsonl 2> gpurun_out/${TAG}_$name.err; echo "$name rc=$?"; }
run default
run free_running --free-running --no-cpu-baseline
run b16 --batch 16 --no-cpu-baseline
run b64 --batch 64 --no-cpu-baseline
run xb12 --store-format xb12 --no-cpu-baseline --no-resident-check
run bf16 --store-format bf16 --no-cpu-baseline --no-resident-check
run 8x22b_l16 --config mixtral-8x22b --layers 16 --steps 3 --no-cpu-baseline
python bench.py --impl reference > gpurun_out/${TAG}_reference.jsonl 2>&1
