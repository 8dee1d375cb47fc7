#!/bin/bash
# Resident 2-D kernel variants (strip height, threads per CTA): parity subset + C1 bench lines.
O=gpurun_out/resv; mkdir -p $O
for v in strip3 strip4 thr768; do
  if [[ $v == base ]]; then unset ST_LIB; else export ST_LIB=paper_1707_02347_b200/_varlib/libstencil_$v.so; fi
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "resident or run_from or graph or pipelined or C1" > $O/${v}_pytest.log 2>&1; echo "exit $?" >> $O/${v}_pytest.log
  for st in 2000 2000; do
    timeout 300 python bench.py --config C1 --steps $st --warmup 20 --no-cpu-baseline >> $O/${v}_c1.jsonl 2>>$O/${v}_c1.err
  done
  python -c "
import json
for l in open('$O/${v}_c1.jsonl'):
    d=json.loads(l); print('$v', d['value'], d['clocks']['sm_mhz'])" >> $O/summary.txt 2>&1
done
echo done > $O/done.txt
