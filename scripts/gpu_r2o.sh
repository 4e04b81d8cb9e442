export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python bench.py > gpurun_out/bench_o.json 2> gpurun_out/bench_o.err; tail -2 gpurun_out/bench_o.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_o.json').read().strip().splitlines()[-1])
print('value',d['value'],'k1',d['kernels']['k1_encode_ms'],'k2',d['kernels']['k2_decode_ms'], 'e2e', d['e2e']['value'], 'cpu', d['cpu_baseline']['value'])
for k,v in (d.get('per_rank_sim') or {}).items(): print(k, v)
"
