#!/bin/bash
# compute-sanitizer after the routing-ahead decode (round 1, session 3): memcheck over the batch-1,
# batched and slot-reuse decode tests, racecheck + synccheck over the batch-1 decode.
mkdir -p gpurun_out
CS=compute-sanitizer
timeout 1200 $CS --tool memcheck --error-exitcode 9 python -m pytest -q -x -m gpu \
  "tests/test_decode_gpu.py::test_decode_trace_tiny[tiny]" "tests/test_decode_gpu.py::test_slot_reuse_ordering_every_output" \
  "tests/test_batch.py::test_batched_decode_tiny[4-caps0]" "tests/test_free_running_gpu.py" \
  > gpurun_out/san_m_memcheck.log 2>&1
echo "decode memcheck rc=$?"
for tool in racecheck synccheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 python -m pytest -q -x -m gpu \
    "tests/test_decode_gpu.py::test_decode_trace_tiny[tiny_budget0]" > gpurun_out/san_m_$tool.log 2>&1
  echo "decode $tool rc=$?"
done
for f in gpurun_out/san_m_*.log; do echo "== $f"; tail -n 2 "$f"; done
