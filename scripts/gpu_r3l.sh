for c in 0 2 1 3 0; do CC_K2_CTAS_PER_SM=$c timeout 600 python scripts/exp/k2cap_ab.py 2>/dev/null | tail -1; done
