for n in 24 32; do for c in 24 32 48; do CC_K2_TMA=1 CC_K2_TMA_CTAS=$c timeout 300 python scripts/exp/green_ab.py $n 2>&1 | tail -1 | sed "s/^/ctas=$c /"; done; done
CC_K2_TMA=1 CC_K2_TMA_CTAS=32 CC_K1_RESIDENT_GRID=-1 timeout 300 python scripts/exp/green_ab.py 32 2>&1 | tail -1 | sed "s/^/k1full /"
