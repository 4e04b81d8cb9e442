for cfg in "0 0 0" "0 0 1" "8 1 0" "8 1 1" "8 0 1"; do set -- $cfg
for gr in "" "--no-graph"; do
CC_K1_SHARE_SMEM1_KB=$1 CC_K2_SMALL=$2 CC_K1_PRIO=$3 timeout 600 python bench.py --no-sim --no-cpu --no-e2e --steps 6 $gr > gpurun_out/b_p.json 2>gpurun_out/b_p.err; python -c "
import json;d=json.loads(open('gpurun_out/b_p.json').read().strip().splitlines()[-1]);print('share $1 small $2 prio $3 $gr', round(d['value'],1), 'layer us', round(d['ms_per_step']/57*1e3,2))" || tail -3 gpurun_out/b_p.err
done; done
