#!/bin/bash
# ncu --set full of the sweep1s kernels with the a-box skip (C5 and C4), mid-run launch.
O=gpurun_out/askip_prof; mkdir -p $O
for C in C5 C4; do
  CMD="python tools/prof_run.py --config $C --tk 1 --nt 4"
  timeout 300 $CMD > $O/plain_$C.log 2>&1 &&
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep1s -s 2 -c 1 -o $O/prof_${C}_tk1 -f $CMD > $O/ncu_$C.log 2>&1
  ncu -i $O/prof_${C}_tk1.ncu-rep --page source --csv --print-source sass > $O/src.csv 2>/dev/null
  python tools/ncu_summary.py $O/prof_${C}_tk1.ncu-rep > $O/ncu_full_${C}_tk1.txt 2>&1
  python tools/ncu_stalls.py $O/src.csv 25 > $O/stalls_${C}_tk1.txt 2>&1
  rm -f $O/src.csv $O/prof_${C}_tk1.ncu-rep
done
echo done > $O/done.txt
