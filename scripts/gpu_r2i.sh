export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python scripts/exp/topk_time.py > gpurun_out/tk_time4.txt 2>&1; cat gpurun_out/tk_time4.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k4_resident -s 40 -c 1 -o gpurun_out/tk4 -f python scripts/profile_codecs.py --codec topk --rows 512 --keep 0.01 --reps 50 > gpurun_out/ncu_tk4.log 2>&1; tail -2 gpurun_out/ncu_tk4.log
