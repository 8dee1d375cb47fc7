#!/bin/bash
# TMA E ring in the dynamic-ring untiled kernel (sweep1): parity subset, same-box A/B vs cp.async.
O=gpurun_out; mkdir -p $O; : > $O/c3ab.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "orders or tiny or composition or slabs or snapshots or replica or C3 or exchange or split" > $O/c3ab_pytest.log 2>&1; echo "pytest exit $?" >> $O/c3ab_pytest.log
tail -3 $O/c3ab_pytest.log >> $O/c3ab.txt
for i in 1 2; do
  bash tools/ab_libs.sh "--config C3 --tk 1 --steps 3 --warmup 3" default s1_cp >> $O/c3ab.txt
done
bash tools/ab_libs.sh "--config C3 --so 2 --tk 1 --nt 200 --steps 3 --warmup 3" default s1_cp >> $O/c3ab.txt
cat $O/c3ab.txt
