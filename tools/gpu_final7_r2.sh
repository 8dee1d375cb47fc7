#!/bin/bash
# Round-2 closing run #7 (a-box skip also in the dynamic-ring sweep1: C3 and r = 3, 4, 7; new
# undamped-tile tests): C3 line first, then the GPU suite, smoke, default bench, launch list.
set -u
O=gpurun_out/final7; mkdir -p $O
timeout 600 python bench.py --config C3 --tk 1 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C3_tk1.json 2> $O/bench_C3_tk1.err
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --config C3 --tk 2 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C3_tk2.json 2> $O/bench_C3_tk2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_C5.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch_C5.log 2>&1
CMD="python tools/prof_run.py --config C3 --tk 1 --nt 4"
timeout 300 $CMD > $O/plain_C3.log 2>&1 &&
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep1_kernel -s 2 -c 1 -o $O/prof_C3_tk1 -f $CMD > $O/ncu_C3.log 2>&1
python tools/ncu_summary.py $O/prof_C3_tk1.ncu-rep > $O/ncu_full_C3_tk1.txt 2>&1
rm -f $O/prof_C3_tk1.ncu-rep
echo done > $O/done.txt
