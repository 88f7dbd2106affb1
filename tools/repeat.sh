#!/bin/bash
# Repeatability: run one config R times; print GB/s and per-launch min/max.
cfg=${1:-C2}; R=${2:-5}; shift 2
for i in $(seq 1 $R); do
  out=$(timeout 120 python bench.py --config $cfg --no-cpu-baseline --no-e2e --soak-s 0.3 --steps 30 "$@" 2>&1 | tail -1)
  python - "$cfg" "$out" <<'PY'
import json, sys
try:
    d = json.loads(sys.argv[2]); r = d["roofline"]
    print(sys.argv[1], "%.0f GB/s" % d["value"], "frac %.3f" % r["frac"], "launch avg %.4f ms" % r["avg_launch_ms"], "copy %.0f" % (d["same_run_copy_gbs_per_gpu"] or 0), d["clocks"])
except Exception as e:
    print("ERR", sys.argv[2][-300:])
PY
done
