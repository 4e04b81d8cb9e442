for v in 1 2; do
CC_K1_RESIDENT_NQ=$v timeout 600 python bench.py --no-sim --no-cpu --no-e2e --overlap > gpurun_out/bench_q$v.json 2> gpurun_out/bench_q$v.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_q$v.json').read().strip().splitlines()[-1])
print('nq $v overlap value',round(d['value'],1),'ms',round(d['ms_per_step'],3), 'k1', round(d['kernels']['k1_encode_ms']*1e3,1))
"
done
CC_K1_RESIDENT_NQ=2 timeout 600 python bench.py --no-sim --no-cpu --no-e2e > gpurun_out/bench_q3.json 2> gpurun_out/bench_q3.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_q3.json').read().strip().splitlines()[-1])
print('nq 2 no-overlap value',round(d['value'],1),'ms',round(d['ms_per_step'],3), 'k1', round(d['kernels']['k1_encode_ms']*1e3,1))
"
timeout 600 python -m pytest tests/test_gpu_k1_resident.py tests/test_gpu_config1.py -x -q -p no:cacheprovider 2>&1 | tail -2
