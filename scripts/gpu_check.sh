set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench6.json 2> gpurun_out/bench6.err; tail -5 gpurun_out/bench6.err; cat gpurun_out/bench6.json
timeout 600 python bench.py --no-graph --no-e2e --no-cpu > gpurun_out/bench6_nograph.json 2>&1; tail -2 gpurun_out/bench6_nograph.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"cc::|fused|k_" -c 60 --csv --log-file gpurun_out/launches6.csv python bench.py --steps 2 --warmup 1 --layers 8 --no-e2e --no-cpu --no-graph > /dev/null 2>&1; echo ncu1=$?
