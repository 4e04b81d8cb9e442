export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_lowrank.py tests/test_gpu_rng.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lr6_launches.csv python scripts/profile_codecs.py --codec lowrank --rows 1024 --rank 8 --reps 3 --device-key > gpurun_out/lr6_launches.log 2>&1; echo ncu done
timeout 600 python -c "
import bench
print(bench.sim_rank_measure('patch', 4, 'lowrank', 8, 4096, 3072, steps=5, warmup=3, spec_kw={'rank': 8, 'iterations': 2}))
"
