for n in 0 8 16 24; do timeout 300 python scripts/exp/green_ab.py $n 2>&1 | tail -3; done
for n in 16 24; do CC_K1_RESIDENT_GRID=-1 timeout 300 python scripts/exp/green_ab.py $n 2>&1 | tail -1; done
