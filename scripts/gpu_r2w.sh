for v in 0 1; do
CC_K2_SMALL=$v timeout 600 python bench.py --no-sim --no-cpu --no-e2e --overlap > gpurun_out/bench_w$v.json 2> gpurun_out/bench_w$v.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_w$v.json').read().strip().splitlines()[-1])
print('k2small $v overlap value',round(d['value'],1),'ms',round(d['ms_per_step'],3))
"
CC_K2_SMALL=$v timeout 600 python scripts/exp/nq_ab.py 2>&1 | grep "nq 2" | head -1
done
CC_K2_SMALL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -1
