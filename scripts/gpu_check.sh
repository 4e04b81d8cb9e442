set -x
timeout 600 python bench.py > gpurun_out/bench7.json 2> gpurun_out/bench7.err; tail -5 gpurun_out/bench7.err; cat gpurun_out/bench7.json
