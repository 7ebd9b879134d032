#!/bin/bash
# Build + run K2 streaming variants (run under gpurun).
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/bin
for cfg in "8 64 4 0 0"; do
  set -- $cfg
  nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -DADAPMOE_FFN_WARPS=$1 -DADAPMOE_FFN_STAGE_KB=$2 \
       -DADAPMOE_FFN_BATCH=$3 -DADAPMOE_FFN_SPLIT=$4 -DADAPMOE_FFN_L2AHEAD=$5 -o tools/bin/ffn_w$1_s$2_b$3_x$4_p$5 tools/ffn_microbench.cu 2>/dev/null &
done
wait
for f in tools/bin/ffn_w*; do echo "== $f"; timeout 120 $f | grep -v ldg; done; timeout 60 tools/bin/ffn_w8_s64_b4_x0_p0 | grep ldg

FFN_V3=1 timeout 120 tools/bin/ffn_w8_s64_b4_x0_p0
