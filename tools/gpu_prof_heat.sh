#!/bin/bash
# ncu --set full of the heat time-tiled kernel (one launch) at 512^3; gpurun -- 'bash tools/gpu_prof_heat.sh TK'
O=gpurun_out; mkdir -p $O
for tk in "$@"; do
  python tools/prof_run.py --config C2 --grid 512x512x512 --tk $tk --nt $((tk*2)) > $O/ph_$tk.log 2>&1 || { echo fail; cat $O/ph_$tk.log; }
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweeph -s 1 -c 1 -o $O/heat_tk$tk -f \
    python tools/prof_run.py --config C2 --grid 512x512x512 --tk $tk --nt $((tk*2)) > $O/ncu_heat_tk$tk.log 2>&1
  ncu -i $O/heat_tk$tk.ncu-rep --page source --csv --print-source sass > $O/heat_tk${tk}_src.csv 2>/dev/null
  python tools/ncu_stalls.py $O/heat_tk${tk}_src.csv 30 > $O/heat_tk${tk}_stalls.txt 2>&1
  python tools/ncu_summary.py $O/heat_tk$tk.ncu-rep > $O/heat_tk${tk}_summary.txt 2>&1
done
