#!/bin/bash
# Bench each experimental library variant (tools/build_variants.py) on short runs of C5/C3/C4/C2
# and run a parity subset against it:  bash tools/gpu_variants.sh base rot ...
O=gpurun_out; mkdir -p $O
for v in "$@"; do
  export ST_LIB=paper_1707_02347_b200/_varlib/libstencil_$v.so
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ragged or tiny or composition" > $O/v_${v}_pytest.log 2>&1; echo "exit $?" >> $O/v_${v}_pytest.log
  for c in ${CFGS:-"C3 --tk 2 --nt 200" "C2 --tk 2" "C2 --tk 4"}; do
    set -- $c
    timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/v_${v}_$1_$3.json 2>$O/v_${v}_$1_$3.err
    python -c "import json;d=json.load(open('$O/v_${v}_$1_$3.json'));print('$v','$1','tk$3',d['value'],d['roofline']['frac'],d['clocks']['sm_mhz'])" >> $O/v_summary.txt 2>/dev/null || echo "$v $1 tk$3 FAILED" >> $O/v_summary.txt
  done
done
