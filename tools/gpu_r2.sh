#!/bin/bash
# Round-2 GPU session helper (under gpurun):
#   bash tools/gpu_r2.sh "<pytest args or none>" "<bench args>" "<bench args>" ...
# Each bench line goes to gpurun_out/r2_bench_<i>.json (+ .err); pytest to gpurun_out/r2_pytest.log.
set -u
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/r2_smi.txt 2>&1
python -m paper_1707_02347_b200.build > $O/r2_build.log 2>&1 || { echo "build failed"; exit 1; }
sel=$1; shift
if [[ "$sel" != none ]]; then
  timeout 1500 python -m pytest tests -q -x $sel > $O/r2_pytest.log 2>&1; echo "pytest exit $?" >> $O/r2_pytest.log
  tail -3 $O/r2_pytest.log
fi
i=0
for c in "$@"; do
  i=$((i+1))
  timeout 900 python bench.py $c > $O/r2_bench_$i.json 2> $O/r2_bench_$i.err
  echo "exit $? :: $c" >> $O/r2_bench_$i.json
  tail -c 600 $O/r2_bench_$i.json
done
