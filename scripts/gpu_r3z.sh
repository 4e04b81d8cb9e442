timeout 600 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/b_u.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b_u.json').read().strip().splitlines()[-1]);print('U8 bench', round(d['value'],1), 'layer us', round(d['ms_per_step']/57*1e3,2), 'k2', round(d['kernels']['k2_decode_ms']*1e3,1), {k:v['ms_per_layer'] for k,v in d['per_rank_sim'].items()})"
