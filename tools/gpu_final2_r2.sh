#!/bin/bash
# Round-2 closing run #2 (after the G5 region-shape change): GPU suite + smoke, C2/heat/C5 bench
# lines, ncu --set full of the C2 heat instance the planner picks.
set -u
O=gpurun_out/final2; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_C5.json 2> $O/bench_C5.err
for c in "C2 --tk auto" "C2 --tk 1" "C2 --tk 2" "C2 --tk 3"; do
  set -- $c
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$1_tk$3.json 2> $O/bench_$1_tk$3.err
done
for tk in 1 2 3 4; do
  timeout 300 python bench.py --config C2 --grid 512x512x512 --nt 96 --tk $tk --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_heat512_tk$tk.json 2> $O/bench_heat512_tk$tk.err
done
CMD="python tools/prof_run.py --config C2 --tk 4 --nt 8"
timeout 300 $CMD > $O/plain_prof_C2.log 2>&1 &&
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweeph -s 1 -c 1 -o $O/prof_C2_tk4 -f $CMD > $O/ncu_C2.log 2>&1
ncu -i $O/prof_C2_tk4.ncu-rep --page source --csv --print-source sass > $O/src.csv 2>/dev/null
python tools/ncu_summary.py $O/prof_C2_tk4.ncu-rep > $O/ncu_full_C2_tk4.txt 2>&1
python tools/ncu_stalls.py $O/src.csv 25 > $O/stalls_C2_tk4.txt 2>&1
rm -f $O/src.csv
echo done > $O/done.txt
