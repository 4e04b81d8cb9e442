for l in 0 1 0 1; do
CC_BENCH_DECODE_LATE=$l timeout 600 python bench.py --no-sim --no-cpu --no-e2e --steps 10 > gpurun_out/b_l.json 2>gpurun_out/b_l.err; python -c "
import json;d=json.loads(open('gpurun_out/b_l.json').read().strip().splitlines()[-1]);print('late $l bench', round(d['value'],1), 'layer us', round(d['ms_per_step']/57*1e3,2), d['consistency'])" || tail -3 gpurun_out/b_l.err
done
