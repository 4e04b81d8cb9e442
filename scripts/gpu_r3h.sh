for f in 0 1; do
timeout 600 python bench.py --no-sim --no-cpu --no-e2e --steps 10 --fuse-decode $f > gpurun_out/b_f$f.json 2>gpurun_out/b_f$f.err; python -c "
import json;d=json.loads(open('gpurun_out/b_f$f.json').read().strip().splitlines()[-1]);print('fuse $f', round(d['value'],1), 'layer us', round(d['ms_per_step']/57*1e3,2), 'k1ev', round(d['kernels']['k1_in_step_events_ms']*1e3,1), d['consistency'], d['gpu_launches'])" || tail -3 gpurun_out/b_f$f.err
done
