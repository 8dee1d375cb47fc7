#!/bin/bash
# C1 / stencil_run_from check under gpurun: the new tests, host-vs-device loop, bench lines.
set -u
O=gpurun_out
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -k "run_from or graph or resident or abi" > $O/c1_pytest.log 2>&1; echo "pytest exit $?" >> $O/c1_pytest.log
timeout 300 python tools/c1_host.py > $O/c1_host.txt 2>&1
for st in 5 200 2000; do
  timeout 300 python bench.py --config C1 --steps $st --warmup 5 --no-cpu-baseline >> $O/c1_bench.jsonl 2>> $O/c1_bench.err
done
timeout 300 python bench.py --config C1 --steps 200 --warmup 5 --graph --no-cpu-baseline >> $O/c1_bench.jsonl 2>> $O/c1_bench.err
echo done > $O/c1_done.txt
