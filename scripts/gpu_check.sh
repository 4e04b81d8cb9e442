timeout 900 python -m pytest tests/test_gpu_lowrank.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "lowrank or really" 2>&1 | tail -30
