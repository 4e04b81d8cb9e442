set -x
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -m gpu > gpurun_out/mp.log 2>&1; tail -15 gpurun_out/mp.log
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.log 2>&1; tail -15 gpurun_out/gpu_all.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-sim > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; tail -5 gpurun_out/bench_a.err; cat gpurun_out/bench_a.json
