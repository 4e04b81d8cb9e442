#!/bin/bash
# ncu evidence for profiles/: full sections of one K1 and one K2 launch, plus the
# launch list (device time + DRAM bytes per launch) of a short bench run.
mkdir -p gpurun_out
TAG=${1:-r1}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_fused -s 12 -c 1 \
  -o gpurun_out/${TAG}_k1 -f python scripts/profile_path.py > gpurun_out/${TAG}_ncu_k1.log 2>&1; echo "k1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode -s 12 -c 1 \
  -o gpurun_out/${TAG}_k2 -f python scripts/profile_path.py > gpurun_out/${TAG}_ncu_k2.log 2>&1; echo "k2 rc=$?"
# our kernels only (-k), after the raw warmup step and 3 warmup steps of 57 layers (K1 + K2 each)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'k1_fused|k_decode|k_warmup|k_raw' -s 456 -c 228 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_launches_bench.log 2>&1; echo "launches rc=$?"
