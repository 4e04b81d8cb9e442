#!/bin/bash
# Round-3 evidence refresh: GPU suite, smoke, bench line, reference arm, bench launch
# list, ncu full sections of the resident K1 at the P = 1 / 8 shapes, K1 timelines.
#   bash scripts/gpu_evidence3.sh r3
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
TAG=${1:-r3}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'k1_|k_decode|k_warmup|k_raw' -s 456 -c 228 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-sim > gpurun_out/${TAG}_launches_bench.log 2>&1; echo "launches rc=$?"
for R in 4096 512; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_resident -s 12 -c 1 \
  -o gpurun_out/${TAG}_k1r_${R} -f python scripts/profile_path.py --rows $R --layers 16 > gpurun_out/${TAG}_ncu_k1r_${R}.log 2>&1; echo "k1 $R rc=$?"
done
timeout 300 python scripts/k1_ab.py --rows 512,1024,2048,4096 --layers 16 > gpurun_out/${TAG}_k1_timelines.txt 2>&1; echo "k1_ab rc=$?"
