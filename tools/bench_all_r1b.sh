#!/bin/bash
# Round-1 bench sweep (session 3) on one B200 (results: gpurun_out/r1_final4.jsonl, one JSON line per run).
out=gpurun_out/r1_final4.jsonl
: > $out
run() {
  echo "== bench.py $*" >&2
  timeout 900 python bench.py "$@" > gpurun_out/_b.json 2> gpurun_out/_b.err
  rc=$?
  if [ $rc -eq 0 ]; then tail -n 1 gpurun_out/_b.json >> $out; else echo "rc=$rc"; tail -n 5 gpurun_out/_b.err; fi
}
run --impl reference
run
run --free-running
run --batch 16 --steps 4
run --batch 64 --steps 4
run --config mixtral-8x22b --steps 4
wc -l $out
timeout 900 python bench.py --pipeline > gpurun_out/r1_final4_pipeline.jsonl 2> gpurun_out/_p.err
timeout 1500 python tools/sweep.py --targets 0,0.12,0.24,0.36,0.48 --out gpurun_out/r1_final4_sweep.jsonl > gpurun_out/_s.log 2>&1
wc -l gpurun_out/r1_final4_pipeline.jsonl gpurun_out/r1_final4_sweep.jsonl
