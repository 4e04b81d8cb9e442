set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json
for v in 0 1; do CC_K1_L2PF=$v timeout 300 python scripts/k1_ab.py --rows 2048,4096 --layers 16 > gpurun_out/k1ab_pf$v.txt 2>&1; echo "pf=$v"; cut -c1-200 gpurun_out/k1ab_pf$v.txt; done
CC_K1_L2PF=0 timeout 600 python bench.py --no-sim --no-cpu --no-e2e > gpurun_out/bench_pf0.json 2>&1; tail -c 600 gpurun_out/bench_pf0.json
