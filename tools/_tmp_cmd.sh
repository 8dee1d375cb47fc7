python tools/_cmp_runs.py C5 600 > gpurun_out/cmp.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fix_bench_C5.json 2>&1
timeout 600 python bench.py --config C3 --tk 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fix_bench_C3.json 2>&1
timeout 600 python bench.py --config C4 --tk 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fix_bench_C4.json 2>&1
