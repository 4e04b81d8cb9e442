export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_lowrank.py -x -q -p no:cacheprovider > gpurun_out/lr.log 2>&1; tail -3 gpurun_out/lr.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lr3_launches.csv python scripts/profile_codecs.py --codec lowrank --rows 1024 --rank 8 --reps 3 > gpurun_out/lr3_launches.log 2>&1; echo ncu done
timeout 900 python bench.py > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err; tail -2 gpurun_out/bench_l.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_l.json').read().strip().splitlines()[-1])
print('value',d['value'],'k1',d['kernels']['k1_encode_ms'],'k2',d['kernels']['k2_decode_ms'])
for k,v in (d.get('per_rank_sim') or {}).items(): print(k, v)
"
