for c in 0 1 2 4; do
CC_K2_CTAS_PER_SM=$c timeout 600 python bench.py --no-sim --no-cpu --no-e2e --steps 10 > gpurun_out/b_c.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b_c.json').read().strip().splitlines()[-1]);print('cap $c bench', round(d['value'],1), 'layer us', round(d['ms_per_step']/57*1e3,2), 'k2', round(d['kernels']['k2_decode_ms']*1e3,1))"
CC_K2_CTAS_PER_SM=$c timeout 600 python scripts/exp/k2cap_ab.py 2>/dev/null | tail -1
done
