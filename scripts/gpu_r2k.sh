export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k4_resident -s 40 -c 1 -o gpurun_out/tk5 -f python scripts/profile_codecs.py --codec topk --rows 512 --keep 0.01 --reps 50 > gpurun_out/ncu_tk5.log 2>&1; tail -2 gpurun_out/ncu_tk5.log
timeout 900 python -m pytest tests/test_gpu_lowrank.py tests/test_gpu_rng.py -x -q -p no:cacheprovider > gpurun_out/lr.log 2>&1; tail -5 gpurun_out/lr.log
timeout 300 python scripts/profile_codecs.py --codec lowrank --rows 1024 --rank 8 --reps 20 --time > gpurun_out/lr_time.txt 2>&1; cat gpurun_out/lr_time.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lr2_launches.csv python scripts/profile_codecs.py --codec lowrank --rows 1024 --rank 8 --reps 3 > gpurun_out/lr2_launches.log 2>&1; echo done
