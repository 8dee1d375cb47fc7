#!/bin/bash
# One GPU session under gpurun: parity tests, bench (C5 default + C3), ncu launch list of the bench
# command, and one `ncu --set full` capture each of the untiled (C5) and time-tiled (C3) sweep.
#   gpurun --timeout 2400 -- 'bash tools/gpu_session.sh [tests|bench|ncu|all]'
# Every step writes its log under gpurun_out/; a failing step does not stop the later ones
# except that ncu runs only after its own command exited 0 without ncu.
set -u
what=${1:-all}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
ls -la paper_1707_02347_b200/libstencil.so oracle/liboracle.so > $O/build.log 2>&1

if [[ $what == all || $what == tests ]]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
fi
if [[ $what == all || $what == bench ]]; then
  timeout 900 python bench.py --steps 3 --warmup 3 > $O/bench_C5.json 2> $O/bench_C5.err
  for c in "C3 --tk 1" "C3 --tk 2" "C4 --tk 1" "C2 --tk 1" "C2 --tk 2" "C2 --tk 4" "C1 --tk 1"; do
    set -- $c
    timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$1_tk$3.json 2> $O/bench_$1_tk$3.err
  done
  timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
fi
if [[ $what == all || $what == ncu ]]; then
  # launch list of the bench command (short nt: same launch mix per step)
  CMD="python bench.py --steps 2 --warmup 3 --nt 40 --no-cpu-baseline"
  timeout 300 $CMD > $O/plain_launch.log 2>&1 &&
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $O/launches_C5.csv $CMD > $O/ncu_launch.log 2>&1
  # top kernel, untiled C5 (SO12, T=1)
  CMD="python tools/prof_run.py --config C5 --tk 1 --nt 4"
  timeout 300 $CMD > $O/plain_prof_c5.log 2>&1 &&
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep -s 2 -c 1 \
      -o $O/prof_C5_tk1 -f $CMD > $O/ncu_c5.log 2>&1
  # untiled C4 (SO16, T=1)
  CMD="python tools/prof_run.py --config C4 --tk 1 --nt 4"
  timeout 300 $CMD > $O/plain_prof_c4.log 2>&1 &&
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep -s 2 -c 1 \
      -o $O/prof_C4_tk1 -f $CMD > $O/ncu_c4.log 2>&1
  # time-tiled C3 (SO8, T_k=2)
  CMD="python tools/prof_run.py --config C3 --tk 2 --nt 6"
  timeout 300 $CMD > $O/plain_prof_c3.log 2>&1 &&
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep2 -s 1 -c 1 \
      -o $O/prof_C3_tk2 -f $CMD > $O/ncu_c3.log 2>&1
fi
echo done > $O/session_done.txt
