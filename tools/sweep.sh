#!/bin/bash
# Tile/stage sweep of the remap kernel on one config: prints setting, GB/s, roofline frac.
cfg=${1:-C2}; shift
sbs=${SBS:-"16384 32768 49152"}
sts=${STS:-"2 4"}
for sb in $sbs; do
  for st in $sts; do
    out=$(ADHA_STAGE_BYTES=$sb ADHA_STAGES=$st timeout 120 python bench.py --config $cfg --no-cpu-baseline --no-e2e --no-copy-ref --soak-s 0.3 --steps 30 "$@" 2>&1 | tail -1)
    python - "$cfg" "$sb" "$st" "$out" <<'PY'
import json, sys
try:
    d = json.loads(sys.argv[4]); k = d["config"]["kernel"]
    print(sys.argv[1], sys.argv[2], sys.argv[3], "T=%d s_in=%d" % (k["T"], k["s_in"]), "%.0f GB/s" % d["value"], "frac %.3f" % d["roofline"]["frac"])
except Exception as e:
    print(sys.argv[1], sys.argv[2], sys.argv[3], "ERR", sys.argv[4][-300:])
PY
  done
done
