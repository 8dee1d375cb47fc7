#!/bin/bash
# Quick GPU check under gpurun: a pytest selection, then bench lines for the given configs.
#   gpurun --timeout 1200 -- 'bash tools/gpu_quick.sh "<pytest -k expr or none>" "C5 --tk 1" "C3 --tk 2" ...'
set -u
O=gpurun_out
mkdir -p $O
sel=$1; shift
if [[ "$sel" != none ]]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$sel" > $O/q_pytest.log 2>&1; echo "pytest exit $?" >> $O/q_pytest.log
fi
i=0
for c in "$@"; do
  i=$((i+1))
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/q_bench_$i.json 2> $O/q_bench_$i.err
  echo "$c" >> $O/q_bench_$i.json
done
echo done > $O/q_done.txt
