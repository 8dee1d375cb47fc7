#!/bin/bash
# Heat time-tiled kernel region shapes: parity of the variant, then same-box A/B.
#   gpurun -- 'bash tools/gpu_heat_ab.sh VARIANT'
O=gpurun_out; mkdir -p $O; V=$1; : > $O/heat_ab.txt
ST_LIB=paper_1707_02347_b200/_varlib/libstencil_$V.so timeout 900 python -m pytest tests/test_gpu_heat_tiled.py -x -q > $O/heat_ab_pytest.log 2>&1; echo "pytest exit $?" >> $O/heat_ab_pytest.log
tail -2 $O/heat_ab_pytest.log >> $O/heat_ab.txt
for tk in 2 3 4; do
  bash tools/ab_libs.sh "--config C2 --tk $tk --steps 5 --warmup 3" default $V >> $O/heat_ab.txt
  bash tools/ab_libs.sh "--config C2 --grid 512x512x512 --nt 96 --tk $tk --steps 3 --warmup 3" default $V >> $O/heat_ab.txt
done
cat $O/heat_ab.txt
