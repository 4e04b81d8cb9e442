for p in 0 1 0 1; do timeout 300 python scripts/exp/prio_ab.py $p 2>&1 | tail -2; done
