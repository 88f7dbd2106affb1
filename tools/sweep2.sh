#!/bin/bash
# sweep2.sh CFG "sb:stages:outbufs ..." [reps] -- GB/s per setting (each repeated), plan as chosen
cfg=$1; combos=$2; reps=${3:-2}
for combo in $combos; do
  IFS=: read sb st ob <<< "$combo"
  vals=""
  for r in $(seq 1 $reps); do
    out=$(ADHA_STAGE_BYTES=$sb ADHA_STAGES=$st ADHA_OUT_BUFFERS=$ob timeout 120 python bench.py --config $cfg --no-cpu-baseline --no-e2e --no-copy-ref --soak-s 0.3 --steps 30 2>&1 | tail -1)
    v=$(python -c "import json,sys; d=json.loads(sys.argv[1]); k=d['config']['kernel']; print('%.0f' % d['value'], 'T=%d/s_in=%d/s_out=%d' % (k['T'], k['s_in'], k['s_out']))" "$out" 2>/dev/null || echo ERR)
    vals="$vals | $v"
  done
  echo "$cfg $combo $vals"
done
