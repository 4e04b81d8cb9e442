for G in 148 144 142 140 138 136 134; do
CC_K1_RESIDENT_GRID=$G timeout 600 python bench.py --no-sim --no-cpu --no-e2e --steps 10 > gpurun_out/b_g.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b_g.json').read().strip().splitlines()[-1]);print('G $G bench', round(d['value'],1), 'layer us', round(d['ms_per_step']/57*1e3,2), 'k1', round(d['kernels']['k1_encode_ms']*1e3,1))"
done
for G in 136 128; do CC_K1_RESIDENT_GRID=$G timeout 600 python scripts/exp/k2cap_ab.py 2>/dev/null | tail -1; done
