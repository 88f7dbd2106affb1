#!/bin/bash
# L2 eviction-hint variants (ADHA_L2_HINTS bit0 loads, bit1 stores), 2 runs each
for c in ${CFGS:-C2 C3 C4 P2}; do
  for h in 0 1 2 3; do
    vals=""
    for r in 1 2; do
      out=$(ADHA_L2_HINTS=$h timeout 120 python bench.py --config $c --no-cpu-baseline --no-e2e --no-copy-ref --soak-s 0.3 --steps 30 2>&1 | tail -1)
      vals="$vals $(python -c "import json,sys; print('%.0f' % json.loads(sys.argv[1])['value'])" "$out" 2>/dev/null || echo ERR)"
    done
    echo "$c hints=$h $vals"
  done
done
