set -u
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 600 python bench.py --config C4 --tk 1 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_C4_tk1.json 2> $O/bench_C4_tk1.err
CMD="python tools/prof_run.py --config C4 --tk 1 --nt 4"
timeout 300 $CMD > $O/plain_prof_c4.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep -s 2 -c 1 -o $O/prof_C4_tk1 -f $CMD > $O/ncu_c4.log 2>&1
echo done > $O/final5_done.txt
