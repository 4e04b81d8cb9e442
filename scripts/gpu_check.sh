set -x
timeout 600 python bench.py --no-cpu > gpurun_out/b_ov.json 2> gpurun_out/b_ov.err; tail -2 gpurun_out/b_ov.err
timeout 600 python bench.py --no-cpu --no-overlap > gpurun_out/b_noov.json 2> gpurun_out/b_noov.err; tail -2 gpurun_out/b_noov.err
