export PATH=/usr/local/cuda/bin:$PATH
timeout 300 ncu --set full --import-source on -k regex:k1_resident -s 8 -c 1 -o gpurun_out/k1r4096 python scripts/profile_path.py --rows 4096 > gpurun_out/ncu_k1r4096.log 2>&1; tail -3 gpurun_out/ncu_k1r4096.log
timeout 300 ncu --set full --import-source on -k regex:k1_resident -s 8 -c 1 -o gpurun_out/k1r1024 python scripts/profile_path.py --rows 1024 > gpurun_out/ncu_k1r1024.log 2>&1; tail -3 gpurun_out/ncu_k1r1024.log
