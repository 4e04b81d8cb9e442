set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30
timeout 600 python bench.py --no-cpu > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -3 gpurun_out/bench3.err; cat gpurun_out/bench3.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches3.csv python bench.py --steps 2 --warmup 1 --layers 8 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_fused" -s 10 -c 1 -o gpurun_out/prof3 python bench.py --steps 2 --warmup 1 --layers 8 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu2=$?
