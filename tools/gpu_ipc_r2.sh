#!/bin/bash
# The fused halo push across processes (CUDA IPC, ranks taking turns on cuda:0) + the fused-push
# tests of the one-process emulation, after the shared IPC-mapping change in stencil_ipc_open.
set -u
O=gpurun_out/ipc; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_slabs.py -m gpu -q -k "fused" > $O/pytest_ipc.log 2>&1; echo "pytest exit $?" >> $O/pytest_ipc.log
echo done > $O/done.txt
