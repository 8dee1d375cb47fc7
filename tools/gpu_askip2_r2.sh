#!/bin/bash
set -u
O=gpurun_out/askip2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "order or full_grid or snap" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err
timeout 600 python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
echo done > $O/done.txt
