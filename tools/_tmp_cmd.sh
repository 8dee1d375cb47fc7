timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/full_pytest.log 2>&1; echo "exit $?" >> gpurun_out/full_pytest.log
