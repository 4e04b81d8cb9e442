#!/bin/bash
# Round evidence for profiles/: bench line, ncu launch list of the bench, full
# sections of K1 (resident) / K2, and launch lists + full sections of the top-k,
# N:M and low-rank encode paths.   bash scripts/gpu_evidence.sh r2
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
TAG=${1:-r2}
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/${TAG}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'k1_|k_decode|k_warmup|k_raw' -s 456 -c 228 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-sim > gpurun_out/${TAG}_launches_bench.log 2>&1; echo "launches rc=$?"
for R in 4096 1024 512; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_resident -s 12 -c 1 \
  -o gpurun_out/${TAG}_k1r_${R} -f python scripts/profile_path.py --rows $R > gpurun_out/${TAG}_ncu_k1r_${R}.log 2>&1; echo "k1 $R rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode -s 12 -c 1 \
  -o gpurun_out/${TAG}_k2 -f python scripts/profile_path.py > gpurun_out/${TAG}_ncu_k2.log 2>&1; echo "k2 rc=$?"
for C in "topk --rows 512 --keep 0.01" "topk --rows 4096 --keep 0.01" "nm_block --rows 4096" "lowrank --rows 1024 --rank 8"; do
  T=$(echo $C | tr ' .' '__' | tr -d '-')
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.sum --clock-control none \
    --csv --log-file gpurun_out/${TAG}_codec_${T}.csv python scripts/profile_codecs.py --codec $C --reps 3 > gpurun_out/${TAG}_codec_${T}.log 2>&1; echo "codec $T rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 2 -c 2 \
  -o gpurun_out/${TAG}_lr_tc -f python scripts/profile_codecs.py --codec lowrank --rows 1024 --rank 8 --reps 2 > gpurun_out/${TAG}_ncu_lr.log 2>&1; echo "lr full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_nm -s 3 -c 1 \
  -o gpurun_out/${TAG}_nm -f python scripts/profile_codecs.py --codec nm_block --rows 4096 --reps 2 > gpurun_out/${TAG}_ncu_nm.log 2>&1; echo "nm full rc=$?"
