set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -25
timeout 600 python bench.py --no-cpu > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -3 gpurun_out/bench2.err; cat gpurun_out/bench2.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 2 --warmup 1 --layers 8 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_fused|k_decode_vec" -s 20 -c 2 -o gpurun_out/prof2 python bench.py --steps 2 --warmup 1 --layers 8 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu2=$?
