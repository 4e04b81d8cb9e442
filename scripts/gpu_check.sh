set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -3 gpurun_out/bench1.err; cat gpurun_out/bench1.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref1.json 2>&1; cat gpurun_out/ref1.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches1.csv python bench.py --steps 2 --warmup 1 --layers 8 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_quant_vec|k_scale_vec|k_decode_vec" -s 30 -c 3 -o gpurun_out/prof1 python bench.py --steps 2 --warmup 1 --layers 8 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu2=$?
ls -la gpurun_out
