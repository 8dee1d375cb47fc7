#!/bin/bash
# Pipelined-e2e check under gpurun: tests, then bench lines pipelined vs serial.
set -u
O=gpurun_out
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -k "pipelined or run_from or graph" > $O/e2e_pytest.log 2>&1; echo "pytest exit $?" >> $O/e2e_pytest.log
for c in "C1 --steps 200" "C1 --steps 200 --e2e serial" "C3 --steps 3" "C3 --steps 3 --e2e-serial" "C2 --steps 20" "C5 --steps 3" "C5 --steps 3 --e2e-serial"; do
  timeout 600 python bench.py --config $c --warmup 3 --no-cpu-baseline >> $O/e2e_bench.jsonl 2>> $O/e2e_bench.err
done
echo done > $O/e2e_done.txt
