#!/bin/bash
# Round-2 closing run #3 (bench value pass without timed events, C1 graph replay): GPU suite, smoke,
# every bench line the DESIGN table quotes, the reference arm.
set -u
O=gpurun_out/final3; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in "C5 --tk 1" "C5 --tk 2" "C3 --tk 1" "C3 --tk 2" "C4 --tk 1" "C2 --tk auto" "C2 --tk 1" "C1 --tk auto"; do
  set -- $c
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$1_tk$3.json 2> $O/bench_$1_tk$3.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
echo done > $O/done.txt
