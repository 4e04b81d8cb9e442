for v in 0 2 1; do CC_K1_L2PF=$v timeout 300 python scripts/k1_ab.py --rows 2048,4096 --layers 16 > gpurun_out/k1ab_pf$v.txt 2>&1; echo "pf=$v"; python - <<PY
import json
for l in open('gpurun_out/k1ab_pf$v.txt'):
    if l.startswith('{'):
        d=json.loads(l); print(d['rows'], d['resident']['us'], {k:v for k,v in d.get('resident_timeline_us',{}).items() if k in ('A_done','sync1','sync2','B_done','end')})
PY
done
for v in 0 2; do CC_K1_L2PF=$v timeout 600 python bench.py --no-sim --no-cpu --no-e2e > gpurun_out/bench_pf$v.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/bench_pf$v.json').read().strip().splitlines()[-1]);print('pf $v', d['value'], d['kernels']['k1_encode_ms'])"; done
