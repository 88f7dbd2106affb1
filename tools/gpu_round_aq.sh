# round 2, call aq: which part of "40 KB x 3 stages" helps C5/C2 -- the third stage or T = 512
# (a power of two: dst SoA chunks of 2/4 KB); last-round balancing on/off
set -u
out=gpurun_out
CFGS=C5,C2,C3,C4,P1,P2 ROUNDS=5 timeout 1500 python tools/ab_multi.py "" \
  "ADHA_STAGE_BYTES=40960,ADHA_BALANCE=0" "ADHA_STAGE_BYTES=40960" \
  "ADHA_STAGE_BYTES=49152,ADHA_BALANCE=0" "ADHA_STAGE_BYTES=40960,ADHA_STAGES=2,ADHA_BALANCE=0" \
  "ADHA_STAGE_BYTES=20480,ADHA_STAGES=6,ADHA_BALANCE=0" "ADHA_STAGE_BYTES=32768,ADHA_BALANCE=0" > $out/aq_stage_ab.log 2>&1; echo "ab=$?"
