#!/bin/bash
# Round-2 closing run #4 (stencil_run_from bench step, pipelined e2e, heat uploads u^n only): GPU
# suite, smoke, every bench line the DESIGN table quotes, the reference arm, ncu of the changed
# resident kernel (C1) and its launch list.
set -u
O=gpurun_out/final4; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in "C5 --tk 1" "C5 --tk 2" "C3 --tk 1" "C3 --tk 2" "C4 --tk 1" "C2 --tk auto" "C2 --tk 1" "C1 --tk auto"; do
  set -- $c
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$1_tk$3.json 2> $O/bench_$1_tk$3.err
done
timeout 600 python bench.py --config C1 --steps 2000 --warmup 5 --no-cpu-baseline > $O/bench_C1_2000.json 2> $O/bench_C1_2000.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_C1.csv \
  python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_launch_C1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:resident2d -s 10 -c 1 -o $O/ncu_full_C1 \
  python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_full_C1.log 2>&1
echo done > $O/done.txt
