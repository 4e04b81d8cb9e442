export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_topk_resident.py -x -q -p no:cacheprovider > gpurun_out/tk_res.log 2>&1; tail -3 gpurun_out/tk_res.log
timeout 600 python scripts/exp/topk_time.py > gpurun_out/tk_time5.txt 2>&1; cat gpurun_out/tk_time5.txt
