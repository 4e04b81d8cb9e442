set -x
timeout 900 python -m pytest tests/test_gpu_nm.py -x -q 2>&1 | tail -5
timeout 600 python scripts/microbench.py --rows 4096 --cols 3072 --layers 8 > gpurun_out/mb_full.json 2> gpurun_out/mb_full.err; tail -3 gpurun_out/mb_full.err
