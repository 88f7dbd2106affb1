#!/bin/bash
for c in ${CFGS:-C2 C3 C4 P2}; do
  for o in interleaved blocked; do
    vals=""
    for r in 1 2; do
      out=$(ADHA_TILE_ORDER=$o timeout 120 python bench.py --config $c --no-cpu-baseline --no-e2e --no-copy-ref --soak-s 0.3 --steps 30 2>&1 | tail -1)
      vals="$vals $(python -c "import json,sys; print('%.0f' % json.loads(sys.argv[1])['value'])" "$out" 2>/dev/null || echo ERR)"
    done
    echo "$c $o $vals"
  done
done
