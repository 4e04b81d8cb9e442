set -x
timeout 900 python -m pytest tests/test_gpu_topk_resident.py tests/test_gpu_topk.py -x -q -p no:cacheprovider > gpurun_out/tk_res.log 2>&1; tail -15 gpurun_out/tk_res.log
timeout 600 python scripts/exp/topk_time.py > gpurun_out/tk_time3.txt 2>&1; cat gpurun_out/tk_time3.txt
