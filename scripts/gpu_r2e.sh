timeout 900 python -m pytest tests/test_gpu_capi_exchange.py -x -q -m gpu > gpurun_out/capi.log 2>&1; tail -30 gpurun_out/capi.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err; tail -3 gpurun_out/bench_b.err; cat gpurun_out/bench_b.json
