#!/bin/bash
# A/B of experiment libraries: bash tools/ab_libs.sh "<bench args>" lib1 lib2 ...  (lib "default" = in-tree)
set -u
O=gpurun_out; mkdir -p $O
args=$1; shift
for L in "$@"; do
  if [[ "$L" == default ]]; then unset ST_LIB; else export ST_LIB=paper_1707_02347_b200/_varlib/libstencil_$L.so; fi
  r=$(timeout 600 python bench.py $args --no-cpu-baseline 2>$O/ab_err_$L.txt | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print(f\"{d['value']:8.1f} GPts/s  per_launch {r['per_launch_ms']:.4f} ms  clk {d['clocks']['sm_mhz']}\")" 2>&1)
  echo "$L :: $args :: $r"
done
