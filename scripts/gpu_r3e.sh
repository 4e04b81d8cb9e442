for cfg in "0 0" "0 1" "2 1" "8 1" "8 0"; do set -- $cfg
CC_K1_SHARE_SMEM1_KB=$1 CC_K2_SMALL=$2 timeout 600 python bench.py --no-sim --no-cpu --no-e2e --steps 10 > gpurun_out/b_sh$1_$2.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b_sh$1_$2.json').read().strip().splitlines()[-1]);print('share $1 small $2', round(d['value'],1), 'k1', round(d['kernels']['k1_encode_ms']*1e3,1), 'k2', round(d['kernels']['k2_decode_ms']*1e3,1), 'layer us', round(d['ms_per_step']/57*1e3,2))"
done
