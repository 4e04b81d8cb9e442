for kb in 0 48 96; do echo "share $kb KB"; CC_K1_SHARE_SMEM_KB=$kb timeout 600 python scripts/exp/nq_ab.py 2>&1 | grep "nq 2" | head -1; done
