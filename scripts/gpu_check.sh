set -x
timeout 300 python scripts/microbench.py --rows 4096 --cols 3072
timeout 300 python scripts/microbench.py --rows 512 --cols 3072
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_fused" -s 20 -c 1 -o gpurun_out/prof4 python scripts/microbench.py --rows 4096 --cols 3072 --reps 4 --layers 4 > /dev/null 2>&1; echo ncu=$?
