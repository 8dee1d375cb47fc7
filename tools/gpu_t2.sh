#!/bin/bash
# Time-tiled kernel iteration: parity subset, benches, optional ncu of the C3 T_k=2 sweep.
set -u
MODE=${1:-}
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ragged or tiny or composition or C1 or C2" > $O/t2_pytest.log 2>&1; echo "exit $?" >> $O/t2_pytest.log
for c in "C3 --tk 2" "C2 --tk 2" "C2 --tk 4"; do
  set -- $c
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/t2_bench_$1_$3.json 2> $O/t2_bench_$1_$3.err
done
if [[ $MODE == ncu ]]; then
  CMD="python tools/prof_run.py --config C3 --tk 2 --nt 6"
  timeout 300 $CMD > $O/t2_plain.log 2>&1 &&
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep -s 1 -c 1 \
      -o $O/prof_C3_tk2_s2 -f $CMD > $O/t2_ncu.log 2>&1
fi
echo done > $O/t2_done.txt
