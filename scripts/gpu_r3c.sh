mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_resident -s 12 -c 1 \
  -o gpurun_out/r3_k1r_4096 -f python scripts/profile_path.py > gpurun_out/r3_ncu_k1.log 2>&1; echo "k1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_resident -s 12 -c 1 \
  -o gpurun_out/r3_k1r_512 -f python scripts/profile_path.py --rows 512 --layers 16 > gpurun_out/r3_ncu_k1_512.log 2>&1; echo "k1 512 rc=$?"
