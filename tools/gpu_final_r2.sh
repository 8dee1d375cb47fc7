#!/bin/bash
# Round-2 closing measurements (under gpurun): GPU suite + smoke, bench lines, launch list, ncu --set full
# of the headline untiled kernel (C5), the C3 untiled kernel and the heat time-tiled kernel (C2).
#   gpurun --timeout 3600 -- 'bash tools/gpu_final_r2.sh [tests] [bench] [ncu]'
set -u
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
for what in "$@"; do
if [[ $what == tests ]]; then
  timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
fi
if [[ $what == bench ]]; then
  timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_C5.json 2> $O/bench_C5.err
  for c in "C3 --tk 1" "C3 --tk 2" "C4 --tk 1" "C2 --tk auto" "C2 --tk 1" "C2 --tk 4" "C1 --tk auto"; do
    set -- $c
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$1_tk$3.json 2> $O/bench_$1_tk$3.err
  done
  for tk in 1 2 3 4; do
    timeout 300 python bench.py --config C2 --grid 512x512x512 --nt 96 --tk $tk --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_heat512_tk$tk.json 2> $O/bench_heat512_tk$tk.err
  done
  timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
fi
if [[ $what == ncu ]]; then
  CMD="python bench.py --steps 2 --warmup 3 --nt 40 --no-cpu-baseline"
  timeout 300 $CMD > $O/plain_launch.log 2>&1 &&
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $O/launches_C5.csv $CMD > $O/ncu_launch.log 2>&1
  for spec in "C5 1 4 sweep1s" "C3 1 4 sweep1_" "C2 3 6 sweeph"; do
    set -- $spec
    CMD="python tools/prof_run.py --config $1 --tk $2 --nt $3"
    timeout 300 $CMD > $O/plain_prof_$1.log 2>&1 &&
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 \
        -o $O/prof_$1_tk$2 -f $CMD > $O/ncu_$1.log 2>&1
    ncu -i $O/prof_$1_tk$2.ncu-rep --page source --csv --print-source sass > $O/src_$1.csv 2>/dev/null
    python tools/ncu_summary.py $O/prof_$1_tk$2.ncu-rep > $O/ncu_full_$1_tk$2.txt 2>&1
    python tools/ncu_stalls.py $O/src_$1.csv 25 > $O/stalls_$1_tk$2.txt 2>&1
    rm -f $O/src_$1.csv
  done
fi
done
echo done > $O/done.txt
