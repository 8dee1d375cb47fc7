#!/bin/bash
# TMA E ring in the static-ring untiled kernel: parity subset, then same-box A/B vs cp.async staging.
O=gpurun_out; mkdir -p $O; : > $O/c5ab.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "orders or C5 or C4 or snapshots or slabs or fullnt or composition or exchange" > $O/c5ab_pytest.log 2>&1; echo "pytest exit $?" >> $O/c5ab_pytest.log
tail -3 $O/c5ab_pytest.log >> $O/c5ab.txt
for i in 1 2; do
  bash tools/ab_libs.sh "--config C5 --tk 1 --steps 3 --warmup 3" default s1s_cp >> $O/c5ab.txt
done
bash tools/ab_libs.sh "--config C4 --tk 1 --steps 2 --warmup 3" default s1s_cp >> $O/c5ab.txt
cat $O/c5ab.txt
