timeout 900 python -m pytest tests/test_gpu_fused_decode.py -x -q -p no:cacheprovider 2>&1 | tail -15
