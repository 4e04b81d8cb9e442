timeout 900 python -m pytest tests/test_gpu_k1_resident.py tests/test_gpu_parity.py tests/test_gpu_config1.py -x -q -p no:cacheprovider 2>&1 | tail -2
for nq in 0 2; do CC_K1_RESIDENT_NQ=$nq timeout 300 python scripts/k1_ab.py --rows 512,1024,2048,4096 --layers 16 > gpurun_out/k1ab_nq$nq.txt 2>&1; echo "nq=$nq"; python - <<PY
import json
for l in open('gpurun_out/k1ab_nq$nq.txt'):
    if l.startswith('{'):
        d=json.loads(l); print(d['rows'], d['resident']['us'], {k:v for k,v in d.get('resident_timeline_us',{}).items() if k in ('first_data','A_done','sync1','sync2','B_done','end')})
PY
done
timeout 600 python bench.py --no-sim --no-cpu --no-e2e > gpurun_out/bench_r3d.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/bench_r3d.json').read().strip().splitlines()[-1]);print('bench', d['value'], d['kernels']['k1_encode_ms'], d['roofline']['frac'])"
