#!/bin/bash
O=gpurun_out; mkdir -p $O; : > $O/c4ab.txt
ST_LIB=paper_1707_02347_b200/_varlib/libstencil_c4_12x2d.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "orders_ragged and 16" > $O/c4ab_pytest.log 2>&1; echo "pytest exit $?" >> $O/c4ab_pytest.log
tail -2 $O/c4ab_pytest.log >> $O/c4ab.txt
for i in 1 2; do
  bash tools/ab_libs.sh "--config C4 --tk 1 --steps 2 --warmup 3" default c4_12x2d c4_16x1d >> $O/c4ab.txt
done
cat $O/c4ab.txt
