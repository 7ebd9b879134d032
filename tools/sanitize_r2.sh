#!/bin/bash
# compute-sanitizer over the round-2 coded expert stores: XB12 / XBH encoders (store build), the
# copy engine's staging ring + decode stream, and decodes over coded stores (tiny goldens, real
# weights with raw-tile fallback, copy_tiles at Mixtral width).
mkdir -p gpurun_out
CS=compute-sanitizer
T="tests/test_coded_store_gpu.py"
SEL="$T::test_store_records_match_reference_encoder $T::test_expert_set_real_weights_encode_and_raw_fallback $T::test_decode_over_coded_store_is_bit_identical"
timeout 2400 $CS --tool memcheck --error-exitcode 9 python -m pytest -q -x -m gpu -k "256 or real or tiny" $SEL \
  > gpurun_out/san_r2_memcheck.log 2>&1
echo "memcheck rc=$?"
timeout 1800 $CS --tool racecheck --error-exitcode 9 python -m pytest -q -x -m gpu -k "256-896-4-xbh or tiny-xbh" $SEL \
  > gpurun_out/san_r2_racecheck.log 2>&1
echo "racecheck rc=$?"
timeout 1800 $CS --tool synccheck --error-exitcode 9 python -m pytest -q -x -m gpu -k "256-896-4-xbh or tiny-xbh" $SEL \
  > gpurun_out/san_r2_synccheck.log 2>&1
echo "synccheck rc=$?"
for f in gpurun_out/san_r2_*.log; do echo "== $f"; tail -n 3 "$f"; done
