#!/bin/bash
# Bench each experimental library variant on C5 / C3 / C4 (short nt), print GPts/s and roofline frac.
for v in "$@"; do
  for c in "C5 --nt 400" "C3 --nt 200" "C4 --nt 200"; do
    set -- $c
    ST_LIB=paper_1707_02347_b200/_varlib/libstencil_$v.so python bench.py --config $c --tk 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/v_${v}_$1.json 2>gpurun_out/v_${v}_$1.err
    python -c "import json,sys;d=json.load(open('gpurun_out/v_${v}_$1.json'));print('$v','$1',d['value'],d['roofline']['frac'],d['clocks']['sm_mhz'])" 2>/dev/null || echo "$v $1 FAILED"
  done
done
