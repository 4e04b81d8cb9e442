export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_lowrank.py -x -q -p no:cacheprovider > gpurun_out/lr.log 2>&1; tail -3 gpurun_out/lr.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lr4_launches.csv python scripts/profile_codecs.py --codec lowrank --rows 1024 --rank 8 --reps 3 > gpurun_out/lr4_launches.log 2>&1; echo ncu done
