# round 2, call ap: stage size x input stages on C5 (and C2) with the final kernel
set -u
out=gpurun_out
CFGS=C5,C2 ROUNDS=5 timeout 1500 python tools/ab_multi.py "" \
  "ADHA_STAGE_BYTES=40960,ADHA_STAGES=2" "ADHA_STAGE_BYTES=40960,ADHA_STAGES=3" \
  "ADHA_STAGE_BYTES=36864,ADHA_STAGES=3" "ADHA_STAGE_BYTES=32768,ADHA_STAGES=4" \
  "ADHA_STAGE_BYTES=45056,ADHA_STAGES=2" "ADHA_STAGE_BYTES=49152,ADHA_STAGES=2,ADHA_L2_HINTS=1" \
  "ADHA_STAGE_BYTES=49152,ADHA_STAGES=2,ADHA_L2_HINTS=2" > $out/ap_stage_ab.log 2>&1; echo "ab=$?"
