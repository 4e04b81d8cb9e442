timeout 900 python -m pytest tests/test_gpu_fused_decode.py -x -q -p no:cacheprovider 2>&1 | tail -1
CC_K1_DEC_HANDOFF=0 timeout 900 python -m pytest tests/test_gpu_fused_decode.py -x -q -p no:cacheprovider 2>&1 | tail -1
for cfg in "0 1" "1 1" "1 0" "0 1"; do set -- $cfg
CC_K1_DEC_HANDOFF=$2 timeout 600 python bench.py --no-sim --no-cpu --no-e2e --steps 10 --fuse-decode $1 > gpurun_out/b_f.json 2>gpurun_out/b_f.err; python -c "
import json;d=json.loads(open('gpurun_out/b_f.json').read().strip().splitlines()[-1]);print('fuse $1 handoff $2', round(d['value'],1), 'layer us', round(d['ms_per_step']/57*1e3,2), 'k1ev', round(d['kernels']['k1_in_step_events_ms']*1e3,1))" || tail -3 gpurun_out/b_f.err
done
