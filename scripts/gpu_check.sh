set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench5.json 2> gpurun_out/bench5.err; tail -3 gpurun_out/bench5.err; cat gpurun_out/bench5.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref5.json 2>&1; cat gpurun_out/ref5.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches5.csv python bench.py --steps 2 --warmup 1 --layers 8 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_fused|k_decode_vec" -s 16 -c 2 -o gpurun_out/prof6 python bench.py --steps 2 --warmup 1 --layers 8 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu2=$?
