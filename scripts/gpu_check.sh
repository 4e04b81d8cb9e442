set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_fused" -s 2 -c 1 -o gpurun_out/prof5 python scripts/microbench.py --rows 4096 --cols 3072 --reps 4 --layers 4 > /dev/null 2>&1; echo ncu=$?
