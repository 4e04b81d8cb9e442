#!/bin/bash
mkdir -p gpurun_out
./scripts/exp/stream_bench > gpurun_out/stream_bench.txt 2>&1
timeout 600 python scripts/microbench.py > gpurun_out/micro.json 2> gpurun_out/micro.err
tail -3 gpurun_out/micro.err
