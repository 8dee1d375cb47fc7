O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ragged or tiny or composition or replica_scaled" > $O/t3_pytest.log 2>&1; echo "exit $?" >> $O/t3_pytest.log
bash tools/gpu_study.sh
