#!/bin/bash
# K1 iteration loop: parity tests of the encode path, then the microbench.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/k1_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/k1_pytest.log
timeout 240 python scripts/microbench.py ${MB_ARGS} > gpurun_out/micro.json 2> gpurun_out/micro.err; echo "micro rc=$?"; tail -3 gpurun_out/micro.err
