for G in -1 140 132 128; do CC_K1_RESIDENT_GRID=$G timeout 300 python scripts/exp/prio_ab.py 1 2>&1 | tail -1 | sed "s/^/G=$G /"; done
