set -x
timeout 600 python scripts/microbench.py --rows 4096 --cols 3072 --layers 8 > gpurun_out/mb_full.json 2> gpurun_out/mb_full.err; tail -3 gpurun_out/mb_full.err
timeout 600 python scripts/microbench.py --rows 1024 --cols 3072 --layers 16 > gpurun_out/mb_p4.json 2> gpurun_out/mb_p4.err; tail -3 gpurun_out/mb_p4.err
cat gpurun_out/mb_full.json gpurun_out/mb_p4.json
