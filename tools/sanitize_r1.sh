#!/bin/bash
# compute-sanitizer over the product kernels (one GPU): memcheck + racecheck + synccheck on the
# grouped tcgen05 kernels (standalone check), memcheck on the batch-1 and batched decode paths and
# the router / trainer through the parity tests.
mkdir -p gpurun_out
CS=compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 600 $CS --tool $tool --error-exitcode 9 tools/bin/grouped_check check-small > gpurun_out/san_k3_$tool.log 2>&1
  echo "k3 $tool rc=$?"
done
timeout 900 $CS --tool memcheck --error-exitcode 9 python -m pytest -q -x -m gpu \
  "tests/test_decode_gpu.py::test_decode_trace_tiny[tiny]" "tests/test_batch.py::test_batched_decode_tiny[4-caps0]" \
  "tests/test_router_gpu.py" "tests/test_trainer_gpu.py::test_gpu_trainer_rejects_empty_training_set" \
  > gpurun_out/san_decode_memcheck.log 2>&1
echo "decode memcheck rc=$?"
timeout 900 $CS --tool racecheck --error-exitcode 9 python -m pytest -q -x -m gpu \
  "tests/test_decode_gpu.py::test_decode_trace_tiny[tiny]" > gpurun_out/san_decode_racecheck.log 2>&1
echo "decode racecheck rc=$?"
for f in gpurun_out/san_*.log; do echo "== $f"; tail -n 2 "$f"; done
