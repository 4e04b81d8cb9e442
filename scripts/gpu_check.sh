set -x
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_lowrank.py -x -q 2>&1 | tail -15
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/codec_trace2.csv python scripts/codec_trace.py > /dev/null 2>&1; echo ncu=$?
