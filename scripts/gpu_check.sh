timeout 300 python scripts/microbench.py --rows 4096 --cols 3072
