set -x
timeout 600 python -m pytest tests/test_gpu_k1_resident.py -x -q -m gpu > gpurun_out/k1r.log 2>&1; tail -30 gpurun_out/k1r.log
timeout 600 python -m pytest tests/test_gpu_extensions.py tests/test_gpu_config1.py -x -q -m gpu > gpurun_out/ext.log 2>&1; tail -30 gpurun_out/ext.log
timeout 300 python scripts/k1_ab.py > gpurun_out/k1_ab.txt 2>&1; cat gpurun_out/k1_ab.txt
