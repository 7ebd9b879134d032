#!/bin/bash
# Build + run K2 streaming variants of the product kernel (run under gpurun).
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/bin
for b in 8 16; do
  nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -DADAPMOE_FFN_P2_BATCH=$b \
       -o tools/bin/ffn_p2b$b tools/ffn_microbench.cu 2>/dev/null &
done
wait
for b in 8 16; do echo "== phase-2 batch $b"; timeout 120 tools/bin/ffn_p2b$b | grep -E "product|ldg"; done
