# round 2, call bq: L2 eviction hints with the final kernel (loads evict_first / stores evict_first)
set -u
out=gpurun_out
CFGS=C5,C2,C3,C4,P1,P2 ROUNDS=5 timeout 1500 python tools/ab_multi.py "" "ADHA_L2_HINTS=1" "ADHA_L2_HINTS=2" "ADHA_L2_HINTS=3" > $out/bq_hints.log 2>&1; echo "ab=$?"
