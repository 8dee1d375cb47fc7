#!/bin/bash
# T = 1 vs T_k = 2 across space orders on 512^3 (wave, 200 steps) and heat: gpurun_out/study.jsonl
set -u
O=gpurun_out; mkdir -p $O; : > $O/study.jsonl
for so in 2 4 6 8 10 12 14 16; do
  for tk in 1 2; do
    timeout 300 python bench.py --config C3 --so $so --nt 200 --tk $tk --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> $O/study.jsonl
  done
done
for tk in 1 2 4; do
  timeout 300 python bench.py --config C2 --grid 512x512x512 --nt 100 --tk $tk --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> $O/study.jsonl
done
