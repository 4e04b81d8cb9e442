timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exchange_sim.py tests/test_gpu_config1.py -x -q -p no:cacheprovider 2>&1 | tail -2
for t in 0 1; do
CC_K2_TMA=$t timeout 600 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/b_t.json 2>gpurun_out/b_t.err; python -c "
import json;d=json.loads(open('gpurun_out/b_t.json').read().strip().splitlines()[-1]);print('tma $t bench', round(d['value'],1), 'layer us', round(d['ms_per_step']/57*1e3,2), 'k1', round(d['kernels']['k1_encode_ms']*1e3,1), 'k2', round(d['kernels']['k2_decode_ms']*1e3,1), d['consistency'], {k:v['ms_per_layer'] for k,v in d['per_rank_sim'].items()})" || tail -3 gpurun_out/b_t.err
done
