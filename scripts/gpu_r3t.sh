for nq in 0 1 2; do CC_K1_RESIDENT_NQ=$nq timeout 600 python scripts/exp/k2cap_ab.py 2>/dev/null | tail -1 | sed "s/^/nq=$nq /"; done
for G in 112 104; do CC_K1_RESIDENT_GRID=$G timeout 600 python scripts/exp/k2cap_ab.py 2>/dev/null | tail -1 | sed "s/^/G=$G /"; done
