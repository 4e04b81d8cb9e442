export PATH=/usr/local/cuda/bin:$PATH
for v in 4 2 1; do
CC_TC_CTAS_PER_SM=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tc_$v.csv python scripts/profile_codecs.py --codec lowrank --rows 1024 --rank 8 --reps 2 --device-key > /dev/null 2>&1
python scripts/ncu_summary.py launches gpurun_out/tc_$v.csv gpurun_out/tc_$v.txt; echo "== $v"; grep -E "tc_gemm|tc_reduce" gpurun_out/tc_$v.txt | cut -c1-120
CC_TC_CTAS_PER_SM=$v python -c "
import bench
print(bench.sim_rank_measure('patch', 4, 'lowrank', 8, 4096, 3072, steps=5, warmup=3, spec_kw={'rank': 8, 'iterations': 2}))
"
done
