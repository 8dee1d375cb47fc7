O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ragged or tiny or composition or replica or snapshots or full_grid" > $O/m_pytest.log 2>&1; echo "exit $?" >> $O/m_pytest.log
for c in C5 C3 C4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/m_bench_$c.json 2>&1; done
python tools/_cmp_runs.py C5 600 > $O/cmp.log 2>&1
