export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python -m pytest tests/test_gpu_rng.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lr5_launches.csv python scripts/profile_codecs.py --codec lowrank --rows 1024 --rank 8 --reps 3 --device-key > gpurun_out/lr5_launches.log 2>&1; echo ncu done
