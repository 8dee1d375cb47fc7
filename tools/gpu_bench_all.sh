#!/bin/bash
# Round-2 bench lines of every config / schedule (under gpurun): gpurun_out/r2_lines.jsonl
set -u
O=gpurun_out; mkdir -p $O
: > $O/r2_lines.jsonl
run() {
  timeout 900 python bench.py "$@" > $O/b.json 2> $O/b.err
  rc=$?
  if [ $rc -eq 0 ]; then tail -1 $O/b.json >> $O/r2_lines.jsonl; else echo "{\"failed\": \"$*\", \"rc\": $rc}" >> $O/r2_lines.jsonl; fi
}
run --steps 5 --warmup 3
for c in "C3 --tk 1" "C3 --tk 2" "C4 --tk 1" "C4 --tk 2" "C5 --tk 2" "C2 --tk 1" "C2 --tk 2" "C2 --tk 4" "C1"; do
  run --config $c --steps 5 --warmup 3 --no-cpu-baseline
done
