for n in 16 24 32; do G=$((148-n)); CC_K1_RESIDENT_GRID=$G timeout 300 python scripts/exp/green_ab.py $n split 2>&1 | tail -3 | sed "s/^/G=$G /"; done
