timeout 1200 python -m pytest tests/test_gpu_topk.py tests/test_gpu_topk_resident.py tests/test_gpu_exchange_sim.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 600 python scripts/exp/topk_sim_ab.py 2>/dev/null | tail -1
