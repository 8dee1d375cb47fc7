#!/bin/bash
O=gpurun_out/c4prof; mkdir -p $O
CMD="python tools/prof_run.py --config C4 --tk 1 --nt 3"
timeout 300 $CMD > $O/plain.log 2>&1 &&
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep1s -s 1 -c 1 -o $O/prof_C4_tk1 -f $CMD > $O/ncu.log 2>&1
ncu -i $O/prof_C4_tk1.ncu-rep --page source --csv --print-source sass > $O/src.csv 2>/dev/null
python tools/ncu_summary.py $O/prof_C4_tk1.ncu-rep > $O/ncu_full_C4_tk1.txt 2>&1
python tools/ncu_stalls.py $O/src.csv 25 > $O/stalls_C4_tk1.txt 2>&1
rm -f $O/src.csv
ncu -i $O/prof_C4_tk1.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
