#!/bin/bash
# Bench each experimental library variant (tools/build_variants.py) and run a parity subset:
#   CFGS="C3_--tk_2_--nt_200 C2_--tk_2" bash tools/gpu_variants.sh base rot ...
# (underscores in a CFGS item stand for spaces)
O=gpurun_out; mkdir -p $O
CFGS=${CFGS:-"C3_--tk_2_--nt_200 C2_--tk_2 C2_--tk_4"}
for v in "$@"; do
  export ST_LIB=paper_1707_02347_b200/_varlib/libstencil_$v.so
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ragged or tiny or composition" > $O/v_${v}_pytest.log 2>&1; echo "exit $?" >> $O/v_${v}_pytest.log
  for c in $CFGS; do
    args=${c//_/ }; lab=$(echo "$args" | tr -d ' -')
    timeout 300 python bench.py --config $args --steps 3 --warmup 3 --no-cpu-baseline > $O/v_${v}_$lab.json 2>$O/v_${v}_$lab.err
    python -c "import json;d=json.load(open('$O/v_${v}_$lab.json'));print('$v','$lab',d['value'],d['roofline']['frac'],d['clocks']['sm_mhz'])" >> $O/v_summary.txt 2>/dev/null || echo "$v $lab FAILED" >> $O/v_summary.txt
  done
done
