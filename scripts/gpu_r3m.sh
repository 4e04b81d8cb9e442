for G in 148 120 96 74; do echo "G=$G"; CC_K1_RESIDENT_GRID=$G timeout 300 python scripts/k1_ab.py --rows 512,1024,2048 --layers 16 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); t=d.get('resident_timeline_us',{}); print(d['rows'], d['resident']['us'], d['resident']['resident_ran'], {k:t[k] for k in ('first_data','A_done','sync1','sync2','B_done','end') if k in t})
"; CC_K1_RESIDENT_GRID=$G timeout 600 python scripts/exp/k2cap_ab.py 2>/dev/null | tail -1; done
