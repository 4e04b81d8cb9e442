for r in 0 8 16 28 40 0; do CC_TOPK_RESIDENT_RESERVE=$r timeout 600 python scripts/exp/topk_sim_ab.py 2>/dev/null | tail -1; done
