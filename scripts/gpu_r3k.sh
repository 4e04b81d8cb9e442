timeout 900 python -m pytest tests/test_gpu_k1_resident.py tests/test_gpu_parity.py tests/test_gpu_config1.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 600 python bench.py --no-sim --no-cpu --no-e2e --steps 4 --no-graph > gpurun_out/b_ng.json 2>gpurun_out/b_ng.err; tail -c 300 gpurun_out/b_ng.json; tail -2 gpurun_out/b_ng.err
timeout 300 python scripts/k1_ab.py --rows 512,1024,2048,4096 --layers 16 > gpurun_out/k1ab_r3k.txt 2>&1; cut -c1-160 gpurun_out/k1ab_r3k.txt
timeout 600 python bench.py > gpurun_out/bench_r3k.json 2>gpurun_out/bench_r3k.err; python -c "
import json;d=json.loads(open('gpurun_out/bench_r3k.json').read().strip().splitlines()[-1]);print('bench', d['value'], d['kernels']['k1_encode_ms'], d['roofline']['frac'], {k:v['ms_per_layer'] for k,v in d['per_rank_sim'].items()})"
