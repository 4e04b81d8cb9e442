#!/bin/bash
# Round-2 evidence for the kernels added this round: ncu full sections of the resident
# top-k, the cluster CholQR2, the device Gaussian draw, the fused low-rank apply, and
# launch lists of the per-rank top-k / patch P=8 steps.   bash scripts/gpu_evidence2.sh r2
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
TAG=${1:-r2}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k4_resident -s 8 -c 1 \
  -o gpurun_out/${TAG}_k4 -f python scripts/profile_codecs.py --codec topk --rows 512 --keep 0.01 --reps 12 > gpurun_out/${TAG}_ncu_k4.log 2>&1; echo "k4 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_orth_cl|k_gauss|k_outer_apply' -s 12 -c 5 \
  -o gpurun_out/${TAG}_lrk -f python scripts/profile_codecs.py --codec lowrank --rows 1024 --rank 8 --reps 3 --device-key > gpurun_out/${TAG}_ncu_lrk.log 2>&1; echo "lr rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_sim_topk8.csv python scripts/exp/sim_one.py topk 8 0.01 > /dev/null 2>&1; echo "sim topk rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_sim_q8.csv python scripts/exp/sim_one.py quant2bit 8 > /dev/null 2>&1; echo "sim q8 rc=$?"
