timeout 900 python -m pytest tests/test_gpu_rng.py tests/test_gpu_lowrank.py -x -q -p no:cacheprovider 2>&1 | tail -2
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_rng.py -x -q -p no:cacheprovider 2>&1 | tail -1; done
timeout 600 python scripts/exp/topk_time.py 2>&1 | grep -v timeline | head -14
