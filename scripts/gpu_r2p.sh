export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python bench.py --no-sim --no-cpu --no-e2e > gpurun_out/bench_p.json 2> gpurun_out/bench_p.err; tail -2 gpurun_out/bench_p.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_p.json').read().strip().splitlines()[-1])
print('value',d['value'],'ms',d['ms_per_step']); print(d['kernels']); print(d['roofline'])
"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum --clock-control none -k regex:'k1_resident|k_decode' -s 40 -c 4 --csv --log-file gpurun_out/k1_traffic.csv python scripts/profile_path.py --rows 4096 > gpurun_out/k1_traffic.log 2>&1; cat gpurun_out/k1_traffic.csv | tail -20
