#!/bin/bash
# Round-2 closing run #6 (planar medium + a-box skip in sweep1s; IPC mapping cache): GPU suite,
# smoke, the driver's bench command, C3/C4 lines, reference arm, launch list of the default bench.
set -u
O=gpurun_out/final6; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_driver_cmd.json 2> $O/bench_driver_cmd.err
for c in "C3 --tk 1" "C4 --tk 1"; do
  set -- $c
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$1_tk$3.json 2> $O/bench_$1_tk$3.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_C5.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch_C5.log 2>&1
echo done > $O/done.txt
