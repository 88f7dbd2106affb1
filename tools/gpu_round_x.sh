# round 2, call x: stage size / stage count of the remap kernel vs the pure-copy optimum found
# in call w (TMA load + LDS/STG copy: 32 KB x 2 stages 6746 GB/s > copy_ 6650)
set -u
out=gpurun_out
CFGS=C5,C2,C3,C4 ROUNDS=5 timeout 1200 python tools/ab_multi.py "" \
  "ADHA_STAGE_BYTES=32768,ADHA_STAGES=2" "ADHA_STAGE_BYTES=32768,ADHA_STAGES=3" \
  "ADHA_STAGE_BYTES=16384,ADHA_STAGES=3" "ADHA_STAGE_BYTES=16384,ADHA_STAGES=4" \
  "ADHA_STAGE_BYTES=24576,ADHA_STAGES=3" "ADHA_STAGE_BYTES=40960,ADHA_STAGES=2" \
  "ADHA_STAGE_BYTES=32768,ADHA_STAGES=2,ADHA_OUT_BUFFERS=1" > $out/x_stage_ab.log 2>&1; echo "ab=$?"
