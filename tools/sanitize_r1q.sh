#!/bin/bash
# compute-sanitizer over the paths added in round 1 session 3: stream-level router, real-weight
# store, tile-grouped launches, the combine with the fused next-layer RMSNorm (free-running).
mkdir -p gpurun_out
CS=compute-sanitizer
timeout 1500 $CS --tool memcheck --error-exitcode 9 python -m pytest -q -x -m gpu \
  "tests/test_router_gpu.py::test_router_forward_matches_route_trace" \
  "tests/test_decode_gpu.py::test_expert_set_checkpoint_layout" "tests/test_decode_gpu.py::test_tile_merge_every_output" \
  "tests/test_free_running_gpu.py" > gpurun_out/san_q_memcheck.log 2>&1
echo "memcheck rc=$?"
timeout 900 $CS --tool racecheck --error-exitcode 9 python -m pytest -q -x -m gpu \
  "tests/test_free_running_gpu.py" > gpurun_out/san_q_racecheck.log 2>&1
echo "racecheck rc=$?"
timeout 900 $CS --tool synccheck --error-exitcode 9 python -m pytest -q -x -m gpu \
  "tests/test_free_running_gpu.py" > gpurun_out/san_q_synccheck.log 2>&1
echo "synccheck rc=$?"
for f in gpurun_out/san_q_*.log; do echo "== $f"; tail -n 2 "$f"; done
