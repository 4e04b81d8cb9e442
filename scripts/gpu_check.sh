set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "fused or full_flux or golden or edge" 2>&1 | tail -5
for s in "4096 3072" "1024 3072" "512 3072"; do set -- $s; timeout 300 python scripts/microbench.py --rows $1 --cols $2; done
