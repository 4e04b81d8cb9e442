set -x
timeout 2400 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/gpu_all2.log 2>&1; tail -5 gpurun_out/gpu_all2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; tail -2 gpurun_out/smoke2.log
timeout 900 python bench.py > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err; tail -2 gpurun_out/bench_s.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_s.json').read().strip().splitlines()[-1])
print('value',round(d['value'],1),'ms',round(d['ms_per_step'],3),'k1',round(d['kernels']['k1_encode_ms']*1e3,2),'k2',round(d['kernels']['k2_decode_ms']*1e3,2),'frac',round(d['roofline']['frac'],3),'e2e',round(d['e2e']['value'],1),'cpu',d['cpu_baseline']['value'], 'launches', d['gpu_launches'], d['clocks'])
for k,v in (d.get('per_rank_sim') or {}).items(): print(k, v)
"
