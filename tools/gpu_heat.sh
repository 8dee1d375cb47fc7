#!/bin/bash
# Heat time tiling on the register-resident kernel (sweeph): parity tests, then T=1 vs T_k bench
# lines on 512^3 (96 steps) and C2.  gpurun -- 'bash tools/gpu_heat.sh [pytest -k expr|none]'
O=gpurun_out; mkdir -p $O; : > $O/heat.txt
sel=${1:-none}
if [[ "$sel" != none ]]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$sel" > $O/heat_pytest.log 2>&1; echo "pytest exit $?" >> $O/heat_pytest.log
  tail -3 $O/heat_pytest.log >> $O/heat.txt
fi
run() {  # label, bench args...
  local lab=$1; shift
  timeout 300 python bench.py "$@" --steps 3 --warmup 3 --no-cpu-baseline > $O/h_$lab.json 2> $O/h_$lab.err
  python -c "import json;d=json.load(open('$O/h_$lab.json'));r=d['roofline'];print('$lab',d['value'],'GPts/s frac',r['frac'],'kernel',r['kernel'],'ms/launch',r['per_launch_ms'],'clk',d['clocks']['sm_mhz'])" >> $O/heat.txt 2>/dev/null || { echo "$lab FAILED" >> $O/heat.txt; tail -3 $O/h_$lab.err >> $O/heat.txt; }
}
for tk in 1 2 3 4; do run heat512_tk$tk --config C2 --grid 512x512x512 --tk $tk --nt 96; done
for tk in 1 2 3 4; do run heatC2_tk$tk --config C2 --tk $tk; done
cat $O/heat.txt
