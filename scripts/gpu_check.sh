set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "fused or full_flux or edge" 2>&1 | tail -3
timeout 300 python scripts/microbench.py --rows 4096 --cols 3072
timeout 300 python scripts/microbench.py --rows 512 --cols 3072
